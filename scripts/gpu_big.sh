#!/bin/bash
# Transpose tests and probe, then the big named shapes on one GPU (Hugewiki, SparkALS).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/mem.txt
timeout 900 python -m pytest tests/test_gpu_transpose.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_tr.log 2>&1; echo "pytest exit $?" >> gpurun_out/status.txt
for c in netflix hugewiki; do
  timeout 600 python scripts/probe_transpose.py $c 5 > gpurun_out/tr_$c.json 2> gpurun_out/tr_$c.err; echo "probe $c exit $?" >> gpurun_out/status.txt
done
ALSK_TRANSPOSE_RADIX=1 timeout 600 python scripts/probe_transpose.py netflix 5 > gpurun_out/tr_netflix_radix.json 2>&1
for c in ${CONFIGS:-hugewiki sparkals}; do
  timeout 1800 python bench.py --config $c --steps 3 --warmup 1 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c exit $?" >> gpurun_out/status.txt
done
