#!/bin/bash
# Tensor-core engine: its parity tests, the full GPU suite, per-half timings, a short bench.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/tc.log 2>&1; echo "tc exit $?" >> gpurun_out/status.txt
timeout 600 python scripts/diag_step.py 2 3 > gpurun_out/diag.txt 2>&1; echo "diag exit $?" >> gpurun_out/status.txt
if [[ "${FULL:-0}" == 1 ]]; then
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/status.txt
fi
