#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python - > gpurun_out/probe.txt 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
from paper_1603_03820_b200 import _native as N
print("ffma peak", N.LIB.alsk_fp32_peak_probe())
for v in (0,1,2,3,4):
    print("variant", v, [round(N.LIB.alsk_herm_loop_probe(c, v),1) for c in (1,2,3,4,5)])
PY
