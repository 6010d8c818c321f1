"""bench.py's launch contract on CPU: --gpus N without torchrun re-launches itself with N
ranks (torch.distributed.run, 127.0.0.1 rendezvous), and the reference arm runs the
unmodified reference (oracle/_ref) without loading libalskit_cuda.so."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _json_line(out: str) -> dict:
    for line in reversed(out.splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise AssertionError(out[-2000:])


@pytest.mark.timeout(300)
def test_gpus_2_spawns_two_ranks():
    env = {k: v for k, v in __import__("os").environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, env=env, timeout=280)
    assert res.returncode == 0, res.stderr[-2000:]
    line = _json_line(res.stdout)
    assert line["n_gpus"] == 2 and sorted(r["rank"] for r in line["ranks"]) == [0, 1]
    assert len({r["pid"] for r in line["ranks"]}) == 2


@pytest.mark.timeout(300)
def test_reference_arm_loads_only_the_reference(ref, tmp_path):
    """ML-1M shape, one full iteration: the process maps oracle/_ref/libalskit_ref.so and
    never the product library."""
    code = (
        "import sys, runpy, json\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--config', 'ml1m', '--steps', '1', '--warmup', '0',"
        f" '--cache-dir', {str(tmp_path)!r}]\n"
        f"runpy.run_path({str(ROOT / 'bench.py')!r}, run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'maps_ref': 'libalskit_ref.so' in maps, 'maps_product': 'libalskit_cuda.so' in maps}))\n")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    bench_line, maps = lines[-2], lines[-1]
    assert bench_line["impl"] == "reference" and bench_line["steps"] == 1 and bench_line["value"] > 0
    assert bench_line["config"]["nnz_train"] == 900189
    assert maps == {"maps_ref": True, "maps_product": False}


def test_library_has_no_unresolved_internal_symbols():
    """Every internal (alsk::) function the library calls is defined in it."""
    lib = ROOT / "paper_1603_03820_b200" / "libalskit_cuda.so"
    res = subprocess.run(["nm", "-D", "--undefined-only", str(lib)], capture_output=True, text=True)
    assert res.returncode == 0
    bad = [l for l in res.stdout.splitlines() if "alsk" in l]
    assert not bad, bad
