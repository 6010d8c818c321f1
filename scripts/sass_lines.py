"""Join an ncu SASS source page (csv) with nvdisasm line info of the same kernel: samples
and executed instructions per CUDA source line. usage:
python scripts/sass_lines.py <ncu_sass.csv> <cubin> <kernel-substring> [top]"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

csv_path, cubin, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
# split by function
cur, line, funcs = None, None, defaultdict(list)
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), line, m.group(2).strip()))
fn = [f for f in funcs if kname in f]
assert len(fn) == 1, fn
ins = funcs[fn[0]]
rows = list(csv.reader(open(csv_path)))
h = rows[1]
data = [r for r in rows[2:] if len(r) > 5]
isamp, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
assert len(data) == len(ins), (len(data), len(ins))
by = defaultdict(lambda: [0.0, 0.0])
ts = te = 0.0
for (addr, src, op), r in zip(ins, data):
    s = float(r[isamp] or 0)
    e = float((r[iex] or "0").replace(",", ""))
    by[src][0] += s
    by[src][1] += e
    ts += s
    te += e
for src, (s, e) in sorted(by.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{src:28s} samples {100 * s / ts:5.1f}%  inst {100 * e / te:5.1f}%")
