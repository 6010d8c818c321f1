// Measurement switches: profiling counters, dry runs and A/B variants are
// read from the environment only in a measurement build (ALSK_MEASURE=1 python
// paper_1603_03820_b200/build.py, which compiles with -DALSK_MEASURE). The product library
// ignores them and always runs the default, result-preserving configuration.
#pragma once

#include <cstdlib>

namespace alsk {
inline const char* measure_env(const char* name) {
#ifdef ALSK_MEASURE
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}
}  // namespace alsk
