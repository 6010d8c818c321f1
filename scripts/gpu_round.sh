#!/bin/bash
# One gpurun call: GPU tests, smoke, our bench arm and the reference arm (the driver's order
# is reference first; both share the binary cache under /tmp). Outputs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
STEPS=${STEPS:-test,bench,ref}
if [[ $STEPS == *test* ]]; then
  timeout 1500 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> gpurun_out/status.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/status.txt
fi
if [[ $STEPS == *ref* ]]; then
  timeout 1500 python bench.py --impl reference ${BENCH_ARGS:-} > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref exit $?" >> gpurun_out/status.txt
fi
if [[ $STEPS == *bench* ]]; then
  timeout 1500 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/status.txt
fi
