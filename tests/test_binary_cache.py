"""Binary ratings cache (dataio.hpp:116-163), after the reference's
own BinaryCache tests (test_dataio.cpp:112-146):

* save -> load is bit-exact, and the bytes on disk equal the reference writer's;
* a file the reference wrote loads bit-identically here, and vice versa;
* truncation, bad magic, a bad version, a corrupt header and CSR invariant violations are
  IoErrors, with the reference's texts (checked against oracle/_ref side by side);
* (gpu) the device loader fills HBM with the same arrays and the same errors.
"""
from __future__ import annotations

import struct

import numpy as np
import pytest

from oracle import binding


def random_matrix(A, seed, m, n, nnz):
    return A.synth_csr(m, n, nnz, seed)


def ref_csr(r):
    return binding.csr_struct(r.rows, r.cols, r.row_ptr, r.col_idx, r.values, r.col_offset)


def same(a, b):
    assert (a.rows, a.cols) == (b.rows, b.cols)
    assert np.array_equal(a.row_ptr, b.row_ptr)
    assert np.array_equal(a.col_idx, b.col_idx)
    assert a.values.tobytes() == b.values.tobytes()


def test_round_trip_is_bit_exact(A, tmp_path):
    a = random_matrix(A, 17, 11, 23, 140)
    p = tmp_path / "r.cache"
    A.save_binary_cache(a, p)
    same(a, A.load_binary_cache(p))
    assert A.cache_header(p) == (11, 23, 140)


@pytest.mark.parametrize("shape", [(0, 0, 0), (5, 7, 0), (1, 1, 1), (300, 40, 5000)])
def test_round_trip_edge_shapes(A, tmp_path, shape):
    m, n, z = shape
    a = A.CsrMatrix(m, n, 0, np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32)) \
        if z == 0 else random_matrix(A, 5, m, n, z)
    p = tmp_path / "e.cache"
    A.save_binary_cache(a, p)
    assert p.stat().st_size == 40 + 8 * (m + 1) + 8 * z
    same(a, A.load_binary_cache(p))


def test_files_match_the_reference_writer(A, ref, tmp_path):
    a = random_matrix(A, 9, 120, 33, 900)
    mine, theirs = tmp_path / "mine.cache", tmp_path / "ref.cache"
    A.save_binary_cache(a, mine)
    assert ref.save_cache(ref_csr(a), str(theirs)) == 0
    assert mine.read_bytes() == theirs.read_bytes()
    same(a, A.load_binary_cache(theirs))
    st, rows, cols, rp, ci, vv = ref.load_cache(str(mine), a.rows, a.nnz())
    assert st == 0 and (rows, cols) == (a.rows, a.cols)
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(ci, a.col_idx)
    assert vv.tobytes() == a.values.tobytes()


def _corrupt_files(A, tmp_path):
    """(name, path) pairs covering every error the reference's loader raises."""
    a = A.CsrMatrix(3, 5, 0, np.array([0, 2, 3, 5], np.int64), np.array([1, 4, 0, 2, 3], np.int32),
                    np.arange(1, 6, dtype=np.float32))
    good = tmp_path / "good.cache"
    A.save_binary_cache(a, good)
    raw = bytearray(good.read_bytes())
    out = []

    def put(name, data):
        p = tmp_path / f"{name}.cache"
        p.write_bytes(bytes(data))
        out.append((name, p))

    put("truncated", raw[:-5])
    put("junk", b"this is not a cache file at all, but long enough to read")
    put("short_header", raw[:20])
    bad = bytearray(raw); bad[8:16] = struct.pack("<Q", 2); put("version", bad)
    bad = bytearray(raw); bad[16:24] = struct.pack("<Q", 1 << 41); put("header_bounds", bad)
    put("trailing", raw + b"\0" * 8)
    rp_at = lambda u: 40 + 8 * u  # noqa: E731
    ci_at = lambda k: 40 + 8 * 4 + 4 * k  # noqa: E731
    bad = bytearray(raw); bad[rp_at(0):rp_at(0) + 8] = struct.pack("<q", 1); put("rp_start", bad)
    bad = bytearray(raw); bad[rp_at(3):rp_at(3) + 8] = struct.pack("<q", 4); put("rp_end", bad)
    bad = bytearray(raw); bad[rp_at(2):rp_at(2) + 8] = struct.pack("<q", 1); put("rp_decrease", bad)
    bad = bytearray(raw); bad[ci_at(2):ci_at(2) + 4] = struct.pack("<i", 5); put("col_range", bad)
    bad = bytearray(raw); bad[ci_at(4):ci_at(4) + 4] = struct.pack("<i", -1); put("col_negative", bad)
    bad = bytearray(raw); bad[ci_at(1):ci_at(1) + 4] = struct.pack("<i", 1); put("col_order", bad)
    bad = bytearray(raw); bad[24:32] = struct.pack("<Q", 1 << 31); put("cols_32bit", bad)
    return out


EXPECTED = {
    "truncated": "cache size does not match its header",
    "junk": "not a ratings cache (bad magic)",
    "short_header": "truncated while reading rows",
    "version": "unsupported cache version",
    "header_bounds": "corrupt cache header",
    "trailing": "cache size does not match its header",
    "rp_start": "corrupt cache (row_ptr must start at 0 and end at nnz)",
    "rp_end": "corrupt cache (row_ptr must start at 0 and end at nnz)",
    "rp_decrease": "corrupt cache (row_ptr must be non-decreasing)",
    "col_range": "corrupt cache (column index 5 out of range in row 1)",
    "col_negative": "corrupt cache (column index -1 out of range in row 2)",
    "col_order": "corrupt cache (column indices must be strictly increasing within row 0)",
    "cols_32bit": "corrupt cache (column count 2147483648 exceeds the 32-bit index range)",
}


def test_loader_never_writes_past_the_callers_buffers(A, tmp_path):
    """The header is re-read by the load: a file that grew since the caller sized its buffers
    (a replaced cache) is an IoError instead of an overrun."""
    import ctypes as C
    from paper_1603_03820_b200 import _native as N
    big = random_matrix(A, 3, 40, 30, 300)
    p = tmp_path / "r.cache"
    A.save_binary_cache(big, p)
    rp = np.zeros(11, np.int64)
    ci = np.zeros(100, np.int32)
    va = np.zeros(100, np.float32)
    st = N.LIB.alsk_load_cache(str(p).encode(), 10, 100, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
    assert st == 4 and "file changed since its header was read" in N.LIB.alsk_last_error().decode()
    assert not rp.any() and not ci.any()


def test_errors_are_io_errors_naming_the_file(A, tmp_path):
    for name, p in _corrupt_files(A, tmp_path):
        with pytest.raises(A.IoError) as e:
            A.load_binary_cache(p)
        assert str(e.value) == f"{p}: {EXPECTED[name]}", name
    with pytest.raises(A.IoError, match="cannot open /nonexistent/r.cache"):
        A.load_binary_cache("/nonexistent/r.cache")
    with pytest.raises(A.IoError, match="cannot open /nonexistent/dir/r.cache for writing"):
        A.save_binary_cache(random_matrix(A, 1, 3, 3, 2), "/nonexistent/dir/r.cache")


def test_error_texts_match_the_reference(A, ref, tmp_path):
    for name, p in _corrupt_files(A, tmp_path):
        st, *_ = ref.load_cache(str(p), 16, 16)
        assert st == 4, name  # IoError
        with pytest.raises(A.IoError) as e:
            A.load_binary_cache(p)
        assert str(e.value) == ref.last_error(), name


@pytest.mark.gpu
def test_device_loader_matches_the_host_loader(A, gpu, tmp_path):
    import torch
    from paper_1603_03820_b200.session import DeviceCsr
    # > 64 MB of col_idx so the pinned double buffer cycles several times, with rows that
    # straddle the chunk boundaries
    a = random_matrix(A, 3, 200_000, 50_000, 40_000_000)
    p = tmp_path / "big.cache"
    A.save_binary_cache(a, p)
    d = DeviceCsr.from_cache(p, torch.device("cuda"))
    torch.cuda.synchronize()
    assert (d.rows, d.cols, d.nnz) == (a.rows, a.cols, a.nnz())
    assert np.array_equal(d.row_ptr.cpu().numpy(), a.row_ptr)
    assert np.array_equal(d.col_idx.cpu().numpy(), a.col_idx)
    assert d.values.cpu().numpy().tobytes() == a.values.tobytes()


@pytest.mark.gpu
def test_device_loader_errors(A, gpu, tmp_path):
    import torch
    from paper_1603_03820_b200.session import DeviceCsr
    for name, p in _corrupt_files(A, tmp_path):
        with pytest.raises(A.IoError) as e:
            DeviceCsr.from_cache(p, torch.device("cuda"))
        assert str(e.value) == f"{p}: {EXPECTED[name]}", name
