"""The reference's C++ API (include/alskit/*.hpp drop-in headers over the C ABI): the test
binary is built by __graft_entry__.build(); on a GPU it must pass the reference's unit-test
expectations (tests/cpp/dropin_test.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "tests" / "cpp" / "dropin_test"


def test_dropin_binary_builds_and_links():
    from paper_1603_03820_b200 import build as B
    B.build_cpp_tests()
    out = subprocess.run(["ldd", str(EXE)], capture_output=True, text=True).stdout
    assert "libalskit_cuda.so" in out and "not found" not in out


@pytest.mark.gpu
def test_dropin_cpp_api_on_device(gpu):
    if not EXE.exists():
        from paper_1603_03820_b200 import build as B
        B.build_cpp_tests()
    res = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "OK (0 failures)" in res.stdout
