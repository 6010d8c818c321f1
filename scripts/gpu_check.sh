#!/bin/bash
# One gpurun call: GPU tests, smoke, the bench, the ncu launch list and full ncu captures of
# the tensor-core Hermitian kernel and the batched Cholesky. Everything lands in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
STEP=${STEP:-all}
if [[ $STEP == all || $STEP == test ]]; then
  timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> gpurun_out/status.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/status.txt
fi
if [[ $STEP == all || $STEP == bench ]]; then
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/status.txt
fi
if [[ $STEP == all || $STEP == ncu ]]; then
  timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
  echo "ncu launches exit $?" >> gpurun_out/status.txt
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"tc_update|tc_solve" -c 2 \
     -o gpurun_out/prof_tc python scripts/prof_step.py netflix 1 > gpurun_out/ncu_full.log 2>&1
  echo "ncu full exit $?" >> gpurun_out/status.txt
fi
