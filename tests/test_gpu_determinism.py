"""Run-to-run bit-identity of the warp-specialised kernels (tensor-core Hermitian, TMEM
Cholesky, transposes). compute-sanitizer's racecheck cannot follow the mbarrier phases that
order their producer/consumer rings (profiles/r02_evidence/sanitizer_racecheck.log reports
hazards only between the staging-ring writers and readers of tc_update, which the full/empty
barrier pairs separate); a real race would show up here as run-to-run differences under
varying timing (rows of very different lengths, several launches, other work in between)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("f", [16, 100, 119])
def test_tensor_core_half_sweep_is_deterministic(A, gpu, f):
    m, n = 2000, 900
    rng = np.random.default_rng(f)
    lengths = rng.choice([0, 1, 7, 33, 250, 900], size=m, p=[0.05, 0.1, 0.3, 0.3, 0.2, 0.05])
    rows = np.repeat(np.arange(m), lengths)
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lengths])
    rp = np.zeros(m + 1, np.int64)
    np.cumsum(lengths, out=rp[1:])
    r = A.CsrMatrix(m, n, 0, rp, cols.astype(np.int32), rng.standard_normal(len(cols)).astype(np.float32))
    th = A.random_factor(n, f, 5)
    cfg = A.SolverConfig(f=f, lambda_=0.05, accumulate_double=False)
    with A.use_fp32_engine("tensor"):
        outs = []
        for it in range(4):
            x = A.update_x(r, th, cfg)
            outs.append(x.entries.copy())
            if it == 1:
                A.csr_to_csc(r)  # unrelated work between launches
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    c1 = A.csr_to_csc(r)
    c2 = A.csr_to_csc(r)
    assert np.array_equal(c1.row_idx, c2.row_idx) and np.array_equal(c1.values.view(np.uint32), c2.values.view(np.uint32))
