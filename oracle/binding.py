"""ORACLE binding — TEST INFRASTRUCTURE ONLY.

ctypes access to oracle/liboracle.so (our CPU restatement of the reference path) and
oracle/_ref/libalskit_ref.so (the unmodified reference compiled from /root/reference).
Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libalskit_ref.so"

TRIPLET_DTYPE = np.dtype([("row", "<i8"), ("col", "<i8"), ("value", "<f4")], align=True)


class CsrT(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("col_offset", C.c_int64),
                ("nnz", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("values", C.c_void_p)]


def build(ref_include: str | None = None) -> None:
    """Compile liboracle.so and, when the reference headers exist, _ref/libalskit_ref.so."""
    cmd = ["make", "-s", "-C", str(HERE)]
    if ref_include:
        cmd.append(f"REF_INCLUDE={ref_include}")
    subprocess.run(cmd, check=True)


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def csr_struct(rows, cols, row_ptr, col_idx, values, col_offset=0) -> CsrT:
    c = CsrT(rows, cols, col_offset, values.size, row_ptr.ctypes.data, col_idx.ctypes.data,
             values.ctypes.data)
    c._keep = (row_ptr, col_idx, values)  # keep the arrays alive with the struct
    return c


class _Lib:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(path)
        self.lib = C.CDLL(str(path))
        self.lib.__getattr__(f"{self.prefix}last_error").restype = C.c_char_p

    def last_error(self) -> str:
        return getattr(self.lib, f"{self.prefix}last_error")().decode()

    def call(self, name, *args, restype=C.c_int):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = restype
        return fn(*args)


class Oracle(_Lib):
    """Our restatement (liboracle.so)."""
    prefix = "orc_"

    def __init__(self):
        super().__init__(ORACLE_SO)

    def hermitian(self, csr: CsrT, theta, theta_rows, f, lam, acc_double, rb, re, check_shape=1):
        A = np.zeros((re - rb) * f * f, np.float32)
        B = np.zeros((re - rb) * f, np.float32)
        st = self.call("hermitian", C.byref(csr), _p(theta), C.c_int64(theta_rows), f, C.c_double(lam),
                       int(acc_double), C.c_int64(rb), C.c_int64(re), check_shape, _p(A), _p(B))
        return st, A, B

    def batch_solve(self, A, B, count, f, zero_row=0):
        X = np.zeros(count * f, np.float32)
        st = self.call("batch_solve", _p(A), _p(B), C.c_int64(count), f, zero_row, _p(X))
        return st, X

    def update_x(self, csr: CsrT, theta, theta_rows, f, lam, acc_double=1, batch_rows=4096):
        X = np.zeros(csr.rows * f, np.float32)
        st = self.call("update_x", C.byref(csr), _p(theta), C.c_int64(theta_rows), f, C.c_double(lam),
                       int(acc_double), C.c_int64(batch_rows), _p(X))
        return st, X

    def loss(self, csr: CsrT, x, x_rows, theta, theta_rows, f, lam):
        out = C.c_double()
        st = self.call("loss", C.byref(csr), _p(x), C.c_int64(x_rows), _p(theta), C.c_int64(theta_rows),
                       f, C.c_double(lam), C.byref(out))
        return st, out.value

    def rmse(self, test, x, x_rows, theta, theta_rows, f):
        out = C.c_double()
        st = self.call("rmse", _p(test), C.c_int64(test.size), _p(x), C.c_int64(x_rows), _p(theta),
                       C.c_int64(theta_rows), f, C.byref(out))
        return st, out.value

    def csr_to_csc(self, csr: CsrT):
        cp = np.zeros(csr.cols + 1, np.int64)
        ri = np.zeros(csr.nnz, np.int32)
        vv = np.zeros(csr.nnz, np.float32)
        st = self.call("csr_to_csc", C.byref(csr), _p(cp), _p(ri), _p(vv))
        return st, cp, ri, vv

    def csr_from_triplets(self, m, n, t):
        rp = np.zeros(m + 1, np.int64)
        ci = np.zeros(t.size, np.int32)
        vv = np.zeros(t.size, np.float32)
        st = self.call("csr_from_triplets", C.c_int64(m), C.c_int64(n), _p(t), C.c_int64(t.size),
                       _p(rp), _p(ci), _p(vv))
        return st, rp, ci, vv

    def random_factor(self, rows, f, seed):
        out = np.zeros(rows * f, np.float32)
        self.call("random_factor", C.c_int64(rows), f, C.c_uint64(seed), _p(out), restype=None)
        return out

    def mix_seed(self, seed, salt):
        return int(self.call("mix_seed", C.c_uint64(seed), C.c_uint64(salt), restype=C.c_uint64))

    def random_triplets(self, seed, m, n, nnz):
        out = np.zeros(nnz, TRIPLET_DTYPE)
        self.call("random_triplets", C.c_uint64(seed), C.c_int64(m), C.c_int64(n), C.c_int64(nnz),
                  _p(out), restype=None)
        return out

    def split_train_test(self, csr: CsrT, holdout, seed):
        k = C.c_int64()
        st = self.call("split_train_test", C.byref(csr), C.c_double(holdout), C.c_uint64(seed),
                       C.byref(k), None, None, None, None)
        if st:
            return st, None
        trp = np.zeros(csr.rows + 1, np.int64)
        tci = np.zeros(csr.nnz - k.value, np.int32)
        tv = np.zeros(csr.nnz - k.value, np.float32)
        test = np.zeros(k.value, TRIPLET_DTYPE)
        st = self.call("split_train_test", C.byref(csr), C.c_double(holdout), C.c_uint64(seed),
                       C.byref(k), _p(trp), _p(tci), _p(tv), _p(test))
        return st, (trp, tci, tv, test)

    def grid_partition(self, csr: CsrT, p, q):
        rc = np.zeros(q + 1, np.int64)
        cc = np.zeros(p + 1, np.int64)
        bn = np.zeros(p * q, np.int64)
        st = self.call("grid_partition_counts", C.byref(csr), p, q, _p(rc), _p(cc), _p(bn))
        if st:
            return st, None
        blocks = []
        for j in range(q):
            lr = int(rc[j + 1] - rc[j])
            for i in range(p):
                blocks.append((np.zeros(lr + 1, np.int64), np.zeros(bn[j * p + i], np.int32),
                               np.zeros(bn[j * p + i], np.float32)))
        arr = lambda k: (C.c_void_p * (p * q))(*[_p(b[k]) for b in blocks])  # noqa: E731
        st = self.call("grid_partition_fill", C.byref(csr), p, q, arr(0), arr(1), arr(2))
        return st, (rc, cc, blocks)

    def slice_cuts(self, count, p):
        out = np.zeros(p + 1, np.int64)
        self.call("slice_cuts", C.c_int64(count), p, _p(out), restype=None)
        return out

    def parallel_reduce(self, parts_a, parts_b, count, f):
        p = len(parts_a)
        cuts = self.slice_cuts(count, p)
        oa = [np.zeros((cuts[i + 1] - cuts[i]) * f * f, np.float32) for i in range(p)]
        ob = [np.zeros((cuts[i + 1] - cuts[i]) * f, np.float32) for i in range(p)]
        ptrs = lambda xs: (C.c_void_p * p)(*[_p(x) for x in xs])  # noqa: E731
        st = self.call("parallel_reduce", ptrs(parts_a), ptrs(parts_b), p, C.c_int64(count), f,
                       ptrs(oa), ptrs(ob))
        return st, oa, ob


class Reference(_Lib):
    """The unmodified reference (oracle/_ref/libalskit_ref.so)."""
    prefix = "ref_"

    def __init__(self):
        super().__init__(REF_SO)

    def hardware_threads(self) -> int:
        return int(self.call("hardware_threads"))

    def save_cache(self, csr, path: str) -> int:
        return self.call("save_cache", C.byref(csr), str(path).encode())

    def write_checkpoint(self, dir: str, iteration, which, rows, f, digest, entries) -> int:
        e = np.ascontiguousarray(entries, np.float32)
        return self.call("write_checkpoint", str(dir).encode(), C.c_int(iteration), C.c_int(which), C.c_int64(rows),
                         C.c_int(f), C.c_uint64(digest), _p(e))

    def read_checkpoint(self, path: str, cap: int):
        it, wh, f = C.c_int(), C.c_int(), C.c_int()
        rows, dg = C.c_int64(), C.c_uint64()
        e = np.zeros(max(cap, 1), np.float32)
        st = self.call("read_checkpoint", str(path).encode(), C.byref(it), C.byref(wh), C.byref(rows), C.byref(f),
                       C.byref(dg), _p(e), C.c_int64(cap))
        return st, it.value, wh.value, rows.value, f.value, dg.value, e[: rows.value * f.value]

    def restore_latest(self, dir: str):
        it, wh, found = C.c_int(), C.c_int(), C.c_int()
        st = self.call("restore_latest_iteration", str(dir).encode(), C.byref(it), C.byref(wh), C.byref(found))
        return st, (it.value, wh.value) if found.value else None

    def load_cache(self, path: str, cap_rows: int, cap_nnz: int):
        rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        rp = np.zeros(cap_rows + 1, np.int64)
        ci = np.zeros(max(cap_nnz, 1), np.int32)
        vv = np.zeros(max(cap_nnz, 1), np.float32)
        st = self.call("load_cache", str(path).encode(), C.byref(rows), C.byref(cols), C.byref(nnz), _p(rp), _p(ci),
                       _p(vv), C.c_int64(cap_rows), C.c_int64(cap_nnz))
        return st, rows.value, cols.value, rp[: rows.value + 1], ci[: nnz.value], vv[: nnz.value]

    def hermitian_mo(self, csr, theta, theta_rows, f, lam, acc_double, rb, re, bin=16):
        A = np.zeros((re - rb) * f * f, np.float32)
        B = np.zeros((re - rb) * f, np.float32)
        st = self.call("hermitian_mo", C.byref(csr), _p(theta), C.c_int64(theta_rows), f, C.c_double(lam),
                       int(acc_double), bin, C.c_int64(rb), C.c_int64(re), _p(A), _p(B))
        return st, A, B

    def batch_solve(self, A, B, count, f, zero_row=0):
        X = np.zeros(count * f, np.float32)
        st = self.call("batch_solve", _p(A), _p(B), C.c_int64(count), f, zero_row, _p(X))
        return st, X

    def update_x(self, csr, theta, theta_rows, f, lam, acc_double=1, batch_rows=4096, threads=1):
        X = np.zeros(csr.rows * f, np.float32)
        st = self.call("update_x", C.byref(csr), _p(theta), C.c_int64(theta_rows), f, C.c_double(lam),
                       int(acc_double), C.c_int64(batch_rows), threads, _p(X))
        return st, X

    def loss(self, csr, x, x_rows, theta, theta_rows, f, lam):
        out = C.c_double()
        st = self.call("loss", C.byref(csr), _p(x), C.c_int64(x_rows), _p(theta), C.c_int64(theta_rows),
                       f, C.c_double(lam), C.byref(out))
        return st, out.value

    def rmse(self, test, x, x_rows, theta, theta_rows, f):
        out = C.c_double()
        st = self.call("rmse", _p(test), C.c_int64(test.size), _p(x), C.c_int64(x_rows), _p(theta),
                       C.c_int64(theta_rows), f, C.byref(out))
        return st, out.value

    def csr_to_csc(self, csr):
        cp = np.zeros(csr.cols + 1, np.int64)
        ri = np.zeros(csr.nnz, np.int32)
        vv = np.zeros(csr.nnz, np.float32)
        st = self.call("csr_to_csc", C.byref(csr), _p(cp), _p(ri), _p(vv))
        return st, cp, ri, vv

    def csr_from_triplets(self, m, n, t):
        rp = np.zeros(m + 1, np.int64)
        ci = np.zeros(t.size, np.int32)
        vv = np.zeros(t.size, np.float32)
        st = self.call("csr_from_triplets", C.c_int64(m), C.c_int64(n), _p(t), C.c_int64(t.size),
                       _p(rp), _p(ci), _p(vv))
        return st, rp, ci, vv

    def random_factor(self, rows, f, seed):
        out = np.zeros(rows * f, np.float32)
        self.call("random_factor", C.c_int64(rows), f, C.c_uint64(seed), _p(out), restype=None)
        return out

    def mix_seed(self, seed, salt):
        return int(self.call("mix_seed", C.c_uint64(seed), C.c_uint64(salt), restype=C.c_uint64))

    def split_train_test(self, csr, holdout, seed):
        k = C.c_int64()
        st = self.call("split_train_test", C.byref(csr), C.c_double(holdout), C.c_uint64(seed),
                       C.byref(k), None, None, None, None)
        if st:
            return st, None
        trp = np.zeros(csr.rows + 1, np.int64)
        tci = np.zeros(csr.nnz - k.value, np.int32)
        tv = np.zeros(csr.nnz - k.value, np.float32)
        test = np.zeros(k.value, TRIPLET_DTYPE)
        st = self.call("split_train_test", C.byref(csr), C.c_double(holdout), C.c_uint64(seed),
                       C.byref(k), _p(trp), _p(tci), _p(tv), _p(test))
        return st, (trp, tci, tv, test)

    def grid_partition(self, csr, p, q):
        rc = np.zeros(q + 1, np.int64)
        cc = np.zeros(p + 1, np.int64)
        bn = np.zeros(p * q, np.int64)
        st = self.call("grid_partition_counts", C.byref(csr), p, q, _p(rc), _p(cc), _p(bn))
        if st:
            return st, None
        blocks = []
        for j in range(q):
            lr = int(rc[j + 1] - rc[j])
            for i in range(p):
                blocks.append((np.zeros(lr + 1, np.int64), np.zeros(bn[j * p + i], np.int32),
                               np.zeros(bn[j * p + i], np.float32)))
        arr = lambda k: (C.c_void_p * (p * q))(*[_p(b[k]) for b in blocks])  # noqa: E731
        st = self.call("grid_partition_fill", C.byref(csr), p, q, arr(0), arr(1), arr(2))
        return st, (rc, cc, blocks)

    def parallel_reduce(self, parts_a, parts_b, count, f, group_of=None, two_phase=False):
        p = len(parts_a)
        base, rem = divmod(count, p)
        sizes = [base + (1 if i < rem else 0) for i in range(p)]
        oa = [np.zeros(s * f * f, np.float32) for s in sizes]
        ob = [np.zeros(s * f, np.float32) for s in sizes]
        ptrs = lambda xs: (C.c_void_p * p)(*[_p(x) for x in xs])  # noqa: E731
        g = None if group_of is None else np.ascontiguousarray(group_of, np.int32)
        st = self.call("parallel_reduce", ptrs(parts_a), ptrs(parts_b), p, C.c_int64(count), f,
                       _p(g), int(two_phase), ptrs(oa), ptrs(ob))
        return st, oa, ob

    def su_als_update_x(self, csr, theta, theta_rows, f, p, q, lam, acc_double=1, two_phase=0):
        X = np.zeros(csr.rows * f, np.float32)
        st = self.call("su_als_update_x", C.byref(csr), _p(theta), C.c_int64(theta_rows), f, p, q,
                       C.c_double(lam), int(acc_double), int(two_phase), _p(X))
        return st, X

    def plan_partition(self, m, n, nnz, f, workers, capacity, headroom=0):
        p, q, fp = C.c_int(), C.c_int(), C.c_int64()
        st = self.call("plan_partition", C.c_int64(m), C.c_int64(n), C.c_int64(nnz), f, workers,
                       C.c_int64(capacity), C.c_int64(headroom), C.byref(p), C.byref(q), C.byref(fp))
        return st, p.value, q.value, fp.value


    # ---- bench.py's reference arm (ref_bench_*: the reference's own train_run iteration) ----
    def bench_write_cache(self, m, n, nnz, seed, path) -> int:
        return self.call("bench_write_cache", C.c_int64(m), C.c_int64(n), C.c_int64(nnz), C.c_uint64(seed),
                         str(path).encode())

    def bench_prepare(self, path, holdout, seed, f, lam):
        tn, tc = C.c_int64(), C.c_int64()
        setup = (C.c_double * 4)()
        st = self.call("bench_prepare", str(path).encode(), C.c_double(holdout), C.c_uint64(seed), f,
                       C.c_double(lam), C.byref(tn), C.byref(tc), setup)
        return st, tn.value, tc.value, list(setup)

    def bench_iteration(self):
        xs, ts = C.c_double(), C.c_double()
        st = self.call("bench_iteration", C.byref(xs), C.byref(ts))
        return st, xs.value, ts.value

    def bench_sample(self, kx, kt):
        xs, ts, nx, nt = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        st = self.call("bench_sample", C.c_int64(kx), C.c_int64(kt), C.byref(xs), C.byref(ts), C.byref(nx),
                       C.byref(nt))
        return st, xs.value, ts.value, nx.value, nt.value

    def bench_eval(self):
        lo, rm, ls, rs = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        st = self.call("bench_eval", C.byref(lo), C.byref(rm), C.byref(ls), C.byref(rs))
        return st, lo.value, rm.value, ls.value, rs.value

    def bench_factors(self, m, n, f):
        x = np.zeros(m * f, np.float32)
        t = np.zeros(n * f, np.float32)
        st = self.call("bench_factors", _p(x), _p(t))
        return st, x, t

    def bench_release(self) -> None:
        self.call("bench_release", restype=None)


def oracle() -> Oracle:
    return Oracle()


def reference() -> Reference | None:
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None
