// alskit drop-in (B200) umbrella header: the reference's in-scope API (proj/include/alskit/
// alskit.hpp:8-16 minus the host-only config/driver layers; dataio.hpp only its binary cache)
// over libalskit_cuda.so.
#pragma once

#include "alskit/common.hpp"
#include "alskit/dataio.hpp"
#include "alskit/factor.hpp"
#include "alskit/parallel.hpp"
#include "alskit/solver.hpp"
#include "alskit/sparse.hpp"
