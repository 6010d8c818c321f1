#!/bin/bash
# Round-2 evidence in one gpurun call: GPU tests, smoke, the bench (FP32 and the FP64-exact
# drop-in default), the ncu launch list of the benched step, ncu --set full of the benched
# tensor-core Hermitian (X and Theta halves) and the warp Cholesky, the transpose launch list
# and timings, compute-sanitizer logs.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
S=${STEPS:-test,bench,fp64,ncu,san}
if [[ $S == *test* ]]; then
  timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> gpurun_out/status.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/status.txt
fi
if [[ $S == *bench* ]]; then
  timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/status.txt
fi
if [[ $S == *fp64* ]]; then
  timeout 1200 python bench.py --precision fp64 --steps 3 --warmup 1 --no-cpu > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err; echo "bench fp64 exit $?" >> gpurun_out/status.txt
fi
if [[ $S == *ncu* ]]; then
  timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
  echo "ncu launches exit $?" >> gpurun_out/status.txt
  timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"tc_update|warp_solve" -c 3 \
     -o gpurun_out/prof_tc python scripts/prof_step.py netflix 1 > gpurun_out/ncu_full.log 2>&1
  echo "ncu full exit $?" >> gpurun_out/status.txt
  timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:tr_ --csv --log-file gpurun_out/tr_launches.csv python scripts/probe_transpose.py netflix 1 > /dev/null 2>&1
  timeout 600 python scripts/probe_transpose.py netflix 5 > gpurun_out/tr_netflix.json 2>&1
  timeout 900 python scripts/probe_transpose.py hugewiki 3 > gpurun_out/tr_hugewiki.json 2>&1
  echo "transpose exit $?" >> gpurun_out/status.txt
fi
if [[ $S == *san* ]]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1200 $CS --tool $tool --print-limit 50 python scripts/sanitize_small.py > gpurun_out/sanitizer_$tool.log 2>&1
    echo "sanitizer $tool exit $?" >> gpurun_out/status.txt
  done
fi
