"""Build libalskit_cuda.so in-tree (nvcc for sm_100a, g++ for host C++).

The shared library is the product: hand-written sm_100a kernels plus the C ABI declared in
include/alskit_cuda.h. It is built in-tree so it travels to the GPU box with the repo
snapshot. Incremental: an object is rebuilt only when its source (or a header) is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libalskit_cuda.so"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}",
]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-pthread", f"-I{INCLUDE}", f"-I{CSRC}"]
# ALSK_MEASURE=1 builds the measurement library (profiling counters, dry runs, A/B variants
# read from the environment; csrc/measure.cuh). The product build ignores those switches.
# It is built next to the product library (libalskit_cuda_measure.so, objects in
# _build_measure) and loaded with ALSK_MEASURE_LIB=1.
if os.environ.get("ALSK_MEASURE") == "1":
    NVCC_FLAGS.append("-DALSK_MEASURE")
    CXX_FLAGS.append("-DALSK_MEASURE")
    BUILD = PKG / "_build_measure"
    LIB = PKG / "libalskit_cuda_measure.so"


def _headers_mtime() -> float:
    hs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    if src.suffix == ".cu":
        cmd = [NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", *CXX_FLAGS, "-I/usr/local/cuda/include", "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = BUILD / (src.name + ".log")
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {src.name}\n{res.stderr[-4000:]}")
    if verbose:
        print(f"[build] {src.name}", file=sys.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    hm = _headers_mtime()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed\n{res.stderr[-4000:]}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"[build] linked {LIB}", file=sys.stderr)
    return LIB


CPP_TESTS = [ROOT / "tests" / "cpp" / "dropin_test.cpp", ROOT / "tests" / "cpp" / "train_run_cli.cpp"]


def build_cpp_tests(verbose: bool = False) -> list[Path]:
    """Compile the C++ drop-in API tests (include/alskit/*.hpp over libalskit_cuda.so)."""
    lib = build(verbose)
    outs = []
    for src in CPP_TESTS:
        exe = src.with_suffix("")
        if exe.exists() and exe.stat().st_mtime >= max(src.stat().st_mtime, lib.stat().st_mtime,
                                                         max(h.stat().st_mtime for h in (INCLUDE / "alskit").glob("*.hpp"))):
            outs.append(exe)
            continue
        cmd = ["g++", "-std=c++20", "-O2", f"-I{INCLUDE}", str(src), f"-L{PKG}", "-lalskit_cuda",
               "-Wl,-rpath,$ORIGIN/../../paper_1603_03820_b200", "-o", str(exe)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"C++ drop-in test build failed\n{res.stderr[-4000:]}")
        outs.append(exe)
    return outs


if __name__ == "__main__":
    print(build(verbose=True))
