#!/usr/bin/env python
"""bench.py — seconds per ALS iteration (X half-sweep + Theta half-sweep) on the
Netflix-shape synthetic workload (480,189 x 17,770, 99M ratings, 10% holdout, f=100,
lambda=0.05), BASELINE.json's metric.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config netflix]

N>1 runs under torchrun, one rank per GPU: rows of X (then Theta) are model-partitioned
over the ranks with the other factor replicated, and the solved slices are all-gathered
over NCCL after each half. Timing: CUDA events on the launching stream
between barriers + synchronize, max over ranks. Inputs (CSR 713 MB, CSC 713 MB) exceed L2,
so no explicit flush is needed.

Extra keys: roofline (the tensor-core Hermitian kernel vs the measured dense tensor peak
taken as TF32 = bf16/2 from MEASURED_PEAKS.json, with the FP32-FFMA-equivalent fraction the
north star quotes beside it, and the batched-Cholesky phase), cpu_baseline
(the UNMODIFIED reference compiled into oracle/_ref, timed on this host's cores on a bounded
row sample, extrapolated by nonzeros), e2e (the same metric through the host-buffer C ABI:
alsk_update_x / alsk_update_theta on pinned host buffers, H2D + D2H inside the timed region;
at N > 1 GPUs each rank's input slices from pinned memory around the model-parallel step).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (m, n, nnz_total, f, lambda)
    "ml1m": (6040, 3706, 1000209, 10, 0.05),
    "netflix": (480189, 17770, 99_000_000, 100, 0.05),
    "yahoo": (1000990, 624961, 252_800_000, 100, 1.4),
}
SHAPE_ID = {"ml1m": 0, "netflix": 1, "yahoo": 2}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="netflix", choices=list(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-dist", action="store_true", help="the multi-GPU end-to-end leg even at one GPU")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_data(cfg_name):
    """Deterministic synthetic ratings + the reference driver's split (driver.hpp:113)."""
    from paper_1603_03820_b200 import alskit as A
    m, n, nnz, f, lam = CONFIGS[cfg_name]
    R = A.synth_csr(m, n, nnz, A.mix_seed(42, 100 + SHAPE_ID[cfg_name]))
    sp = A.split_train_test(R, 0.1, A.mix_seed(42, 2))
    return sp.train, sp.test


# ------------------------------------------------------------------ clocks ---------
class Clocks:
    def __init__(self, out: Path):
        self.out = out
        self.proc = None

    def __enter__(self):
        try:
            self.f = open(self.out, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.f.close()

    def summary(self, device_index=0):
        try:
            rows = [l.split(",") for l in self.out.read_text().splitlines() if l.strip()]
        except OSError:
            return None
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 8 and r[0].strip() == str(device_index)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------------ reference arm --
def cpu_reference_sample(train, test, cfg_name, target_s=12.0):
    """Time the UNMODIFIED reference (oracle/_ref) update_x on all host threads, on a row
    sample of each half, extrapolated to a full iteration by nonzero count. Only the
    cpu_baseline leg / --impl reference may run this."""
    from oracle import binding
    from paper_1603_03820_b200 import alskit as A
    ref = binding.reference()
    if ref is None:
        return None
    m, n, nnz, f, lam = CONFIGS[cfg_name]
    threads = ref.hardware_threads()
    csc = A.csr_to_csc(train) if A.device_available() else None
    if csc is None:
        st, cp, ri, vv = binding.oracle().csr_to_csc(binding.csr_struct(m, n, train.row_ptr, train.col_idx, train.values))
        rt = (cp, ri, vv)
    else:
        rt = (csc.col_ptr, csc.row_idx, csc.values)
    x0 = A.random_factor(m, f, 42).entries
    t0 = A.random_factor(n, f, A.mix_seed(42, 1)).entries

    def sample(row_ptr, col_idx, values, rows, cols, theta, theta_rows, k):
        rp = (row_ptr[: k + 1]).copy()
        nz = int(rp[-1])
        c = binding.csr_struct(k, cols, rp, col_idx[:nz].copy(), values[:nz].copy())
        t = time.perf_counter()
        st, _ = ref.update_x(c, theta, theta_rows, f, lam, acc_double=1, batch_rows=4096, threads=0)
        dt = time.perf_counter() - t
        assert st == 0, ref.last_error()
        return dt, nz

    # size the samples from a small probe so each half costs ~target_s/2
    total_x = int(train.row_ptr[-1])
    kx = max(64, min(m, 2000))
    dx, nzx = sample(train.row_ptr, train.col_idx, train.values, m, n, t0, n, kx)
    kx = int(min(m, max(kx, kx * (target_s / 2) / max(dx, 1e-3))))
    dx, nzx = sample(train.row_ptr, train.col_idx, train.values, m, n, t0, n, kx)
    kt = max(4, min(n, 40))
    dt_, nzt = sample(rt[0], rt[1], rt[2], n, m, x0, m, kt)
    kt = int(min(n, max(kt, kt * (target_s / 2) / max(dt_, 1e-3))))
    dt_, nzt = sample(rt[0], rt[1], rt[2], n, m, x0, m, kt)
    per_iter = dx * total_x / nzx + dt_ * total_x / nzt
    return {"value": per_iter, "unit": "s/ALS-iter", "cores": threads, "kind": "reference",
            "sample": f"reference update_x (accumulate_double, threads=0) on the first {kx} rows "
                      f"({nzx} nnz) of the X-half and {kt} items ({nzt} nnz) of the Theta-half, "
                      f"{dx:.2f}s + {dt_:.2f}s, extrapolated by nnz to {total_x} train ratings per half"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    train, test = make_data(args.config)
    m, n, nnz, f, lam = CONFIGS[args.config]
    vals = []
    base = None
    for i in range(args.warmup + args.steps):
        b = cpu_reference_sample(train, test, args.config, target_s=8.0)
        if b is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
            return
        if i >= args.warmup:
            vals.append(b["value"])
        base = b
    v = float(np.median(vals))
    base["value"] = v
    print(json.dumps({
        "impl": "reference", "metric": f"s/ALS-iter ({args.config}-shape f={f})", "value": v, "unit": "s/ALS-iter",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64-accumulate",
        "data": "synthetic (planted rank-10 + U[-0.5,0.5) noise; SURVEY \u00a78(d) generator)",
        "config": {"workload": args.config, "m": m, "n": n, "nnz_total": nnz, "nnz_train": int(train.row_ptr[-1]),
                   "f": f, "lambda": lam, "holdout": 0.1, "parallelism": "host threads (reference thread pool)"},
        "cpu_baseline": base, "e2e": {"value": v, "unit": "s/ALS-iter", "h2d_bytes_per_step": 0,
                                      "d2h_bytes_per_step": 0}}))


# ------------------------------------------------------------------ our arm --------
def fp32_peak_probe():
    """Measured FFMA throughput of this device (TFLOP/s), from libalskit_cuda's probe kernel."""
    from paper_1603_03820_b200 import _native as N
    fn = getattr(N.LIB, "alsk_fp32_peak_probe", None)
    if fn is None:
        return None
    fn.restype = C.c_double
    fn.argtypes = []
    return float(fn())


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1603_03820_b200 import _native as N
    from paper_1603_03820_b200 import alskit as A
    from paper_1603_03820_b200.session import DeviceCsr, PREC_FP32

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    m, n, nnz, f, lam = CONFIGS[args.config]
    train, test = make_data(args.config)
    nz_train = int(train.row_ptr[-1])
    R = DeviceCsr.from_host(train, dev)
    RT = R.transpose()
    from paper_1603_03820_b200.distributed import ModelParallelALS
    als = ModelParallelALS(R, RT, m, n, f, lam, PREC_FP32,
                           torch.from_numpy(A.random_factor(m, f, 42).entries).to(dev),
                           torch.from_numpy(A.random_factor(n, f, A.mix_seed(42, 1)).entries).to(dev))
    step = als.step

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = A.kernel_launch_count()
    clocks = Clocks(ROOT / "gpurun_out" / f"clocks_rank{rank}.csv") if (ROOT / "gpurun_out").exists() else Clocks(Path(f"/tmp/clocks_rank{rank}.csv"))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        N.LIB.alsk_profile_begin()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        kms, kl = C.c_double(), C.c_uint64()
        hm, hn, sm_, sn = C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()
        N.LIB.alsk_profile_phases(C.byref(hm), C.byref(hn), C.byref(sm_), C.byref(sn))
        N.LIB.alsk_profile_end(C.byref(kms), C.byref(kl))
    ms = e0.elapsed_time(e1) / args.steps
    launches = A.kernel_launch_count() - launches0
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    # objective / RMSE after the run (reported, not timed)
    rmse = None
    if rank == 0 and test is not None:
        out = C.c_double()
        tt = np.ascontiguousarray(test)
        rows = torch.from_numpy(tt["row"].copy()).to(dev)
        cols = torch.from_numpy(tt["col"].copy()).to(dev)
        vals = torch.from_numpy(tt["value"].copy()).to(dev)
        X, T = als.factors()
        A._check(N.LIB.alsk_dev_rmse(rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), len(tt), X.data_ptr(), m,
                                     T.data_ptr(), n, f, C.byref(out), torch.cuda.current_stream().cuda_stream))
        rmse = out.value

    result = None
    if rank == 0:
        flops_half = nz_train * (f * (f + 1) + 2 * f)  # Nz (f(f+1) + 2f) per half-sweep
        ffma_peak = fp32_peak_probe()
        nominal_ffma = 148 * 128 * 2 * 1.965e9 / 1e12
        peaks = {}
        try:
            peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        except (OSError, ValueError):
            pass
        bf16 = peaks.get("bf16_tflops")
        tf32_peak = bf16 / 2 if bf16 else 2250.0 / 2 * 1.0  # dense TF32 = half the dense bf16 rate
        traffic = None
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():
            try:
                traffic = json.loads(tf.read_text()).get(args.config)
            except (OSError, ValueError):
                traffic = None
        if hn.value > 0:
            # tensor-core engine: Hermitian launches and batched-Cholesky launches timed apart
            herm_flops = 2 * args.steps * flops_half / world
            herm_ms_launch = hm.value / hn.value
            flops_launch = herm_flops / hn.value
            achieved = flops_launch / (herm_ms_launch * 1e-3) / 1e12
            solve_flops = args.steps * (m + n) * (f ** 3 / 3 + 2 * f * f) / world
            pk_row = 4 * (((f * (f + 1) // 2 + f) + 3) // 4 * 4)
            herm_bytes = args.steps * (2 * nz_train * (4 * f + 8) + 8 * (m + n + 2) + (m + n) * pk_row) / world
            roof = {"bound": "tensor", "kernel": "tc_update_kernel (tcgen05 tf32x2 Hermitian + bias, packed rows)",
                    "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s", "frac": achieved / tf32_peak,
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (dense TF32)" if bf16 else
                    "nominal dense TF32 (MEASURED_PEAKS.json absent)",
                    "traffic": traffic, "flops_per_launch": flops_launch, "kernel_ms_avg": herm_ms_launch,
                    "launches": int(hn.value), "kernel_share_of_step": (hm.value / args.steps) / ms,
                    "fp32_ffma_equiv": {"peak": ffma_peak or nominal_ffma, "frac": achieved / (ffma_peak or nominal_ffma),
                                        "peak_source": "measured FFMA probe (alsk_fp32_peak_probe)"},
                    # a split-precision tensor-core kernel is also reported
                    # against the TF32 peak / 3 (three tf32 products per FP32-accurate product)
                    "tf32x3_equiv": {"peak": tf32_peak / 3, "frac": achieved / (tf32_peak / 3)},
                    # the same launches against HBM: algorithmic bytes = per rating the column
                    # index, the value and the gathered factor row (4f), per row the row pointer
                    # and the packed A/B row written for the solve
                    "gather": {"bytes_per_launch": herm_bytes / hn.value,
                               "achieved": herm_bytes / (hm.value * 1e-3) / 1e9, "peak": peaks.get("hbm_gbs"),
                               "unit": "GB/s",
                               "frac": (herm_bytes / (hm.value * 1e-3) / 1e9) / peaks["hbm_gbs"]
                               if peaks.get("hbm_gbs") else None,
                               "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
                    "solve": {"kernel": "tc_solve_kernel (TMEM-resident Cholesky, tensor-core rank-8 updates)",
                              "ms_per_step": sm_.value / args.steps, "launches": int(sn.value),
                              "achieved_tflops": solve_flops / (sm_.value * 1e-3) / 1e12 if sm_.value else None,
                              "share_of_step": (sm_.value / args.steps) / ms}}
        else:
            # FFMA engine (f outside the tensor-core range): one fused kernel per half
            kernel_ms = kms.value / max(kl.value, 1)
            nbk = (f + 1 + 7) // 8
            kname = (f"small_update_kernel<{f}> (thread or warp per row: hermitian+bias+cholesky+solve in registers)"
                     if f <= 15 else f"fused_update_kernel<{nbk}> (hermitian+bias+cholesky+solve)")
            if f <= 32:
                # small f is HBM-bound; algorithmic gather bytes per half
                bytes_half = (nz_train * (4 + 4 + 4 * f) + 8 * (max(m, n) + 1)) / world
                achieved = bytes_half / (kernel_ms * 1e-3) / 1e9
                hbm = peaks.get("hbm_gbs")
                roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                        "frac": achieved / hbm if hbm else None, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                        "traffic": None, "bytes_per_launch": bytes_half, "kernel_ms_avg": kernel_ms,
                        "kernel_share_of_step": (kms.value / args.steps) / ms}
            else:
                achieved = flops_half / world / (kernel_ms * 1e-3) / 1e12
                peak = ffma_peak or nominal_ffma
                roof = {"bound": "fp32-fma", "kernel": kname,
                        "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                        "peak_source": "measured FFMA probe (alsk_fp32_peak_probe)", "traffic": traffic,
                        "flops_per_launch": flops_half / world, "kernel_ms_avg": kernel_ms,
                        "kernel_share_of_step": (kms.value / args.steps) / ms}
        result = {
            "metric": f"s/ALS-iter ({args.config}-shape f={f})",
            "value": ms / 1e3, "unit": "s/ALS-iter", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (planted rank-10 + U[-0.5,0.5) noise; SURVEY §8(d) generator)",
            "config": {"workload": args.config, "m": m, "n": n, "nnz_total": nnz, "nnz_train": nz_train, "f": f,
                       "lambda": lam, "holdout": 0.1, "parallelism": f"model-parallel rows x{world} + NCCL all-gather"
                       if world > 1 else "single GPU", "l2": f"inputs > L2 (CSR+CSC {2 * (8 * (m + n) / 2 + 8 * nz_train) / 1e9:.1f} GB), no flush",
                       "engine": A.fp32_engine()},
            "roofline": roof,
            "gpu_launches": int(launches),
            "test_rmse_after_run": rmse,
        }
        cs = clocks.summary(local)
        if cs:
            result["clocks"] = cs
    if world > 1:
        dist.barrier()
    if not args.no_e2e and (world > 1 or args.e2e_dist):
        e2e = run_e2e_dist(args, train, R, RT, als, rank, world, dev)
        if rank == 0:
            result["e2e"] = e2e
    return result, train, test


def run_e2e_dist(args, train, R, RT, als, rank, world, dev):
    """End to end at N GPUs: every step each rank copies its share of the inputs from pinned
    host memory (the CSR rows of its X slice, the CSC columns of its Theta slice, and the
    starting Theta), runs the model-parallel iteration (NCCL all-gathers included) and copies
    its solved X and Theta slices back. Max over ranks of the wall time per step."""
    import torch
    import torch.distributed as dist
    from paper_1603_03820_b200 import alskit as A
    m, n, nnz, f, lam = CONFIGS[args.config]
    (rb, re), (cb, ce) = als.xs[rank], als.ts[rank]
    csc = A.csr_to_csc(train)
    k0, k1 = int(train.row_ptr[rb]), int(train.row_ptr[re])
    c0, c1 = int(csc.col_ptr[cb]), int(csc.col_ptr[ce])
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    ci_h, vv_h = pin(train.col_idx[k0:k1]), pin(train.values[k0:k1])
    ri_h, cv_h = pin(csc.row_idx[c0:c1]), pin(csc.values[c0:c1])
    t_h = pin(A.random_factor(n, f, A.mix_seed(42, 1)).entries)
    x_out = torch.empty((re - rb) * f, dtype=torch.float32).pin_memory()
    t_out = torch.empty((ce - cb) * f, dtype=torch.float32).pin_memory()

    side = torch.cuda.Stream(device=dev)  # the CSC slice uploads run under the X half-sweep

    def step():
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            RT.col_idx[c0:c1].copy_(ri_h, non_blocking=True)
            RT.values[c0:c1].copy_(cv_h, non_blocking=True)
        R.col_idx[k0:k1].copy_(ci_h, non_blocking=True)
        R.values[k0:k1].copy_(vv_h, non_blocking=True)
        als.T[: n * f].copy_(t_h, non_blocking=True)
        als.half_x()
        main.wait_stream(side)
        als.half_theta()
        x_out.copy_(als.X[rb * f: re * f], non_blocking=True)
        t_out.copy_(als.T[cb * f: ce * f], non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(max(1, args.warmup // 2)):
        step()
    steps = max(2, args.steps // 2)
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    for _ in range(steps):
        step()
    sec = torch.tensor([(time.perf_counter() - t) / steps, 0.0, 0.0], dtype=torch.float64, device=dev)
    sec[1] = (k1 - k0) * 8 + (c1 - c0) * 8 + n * f * 4
    sec[2] = ((re - rb) + (ce - cb)) * f * 4
    if world > 1:
        mx = sec[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sec, op=dist.ReduceOp.SUM)
        sec[0] = mx[0]
    return {"value": float(sec[0]), "unit": "s/ALS-iter", "h2d_bytes_per_step": int(sec[1]),
            "d2h_bytes_per_step": int(sec[2]),
            "path": f"model-parallel iteration on {world} GPU(s) from pinned host buffers (each rank: its CSR rows, "
                    "CSC columns and the starting Theta H2D, its X and Theta slices D2H), wall clock, max over ranks",
            "steps": steps}


def run_e2e(args, train, test):
    """Same metric through the host-buffer C ABI (reference-facing call): pinned host CSR, CSC
    and factors; every step copies the inputs H2D and the solved factors D2H."""
    import torch
    from paper_1603_03820_b200 import _native as N
    from paper_1603_03820_b200 import alskit as A
    m, n, nnz, f, lam = CONFIGS[args.config]
    csc = A.csr_to_csc(train)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    rp, ci, vv = pin(train.row_ptr), pin(train.col_idx), pin(train.values)
    cp, ri, cv = pin(csc.col_ptr), pin(csc.row_idx), pin(csc.values)
    X = pin(A.random_factor(m, f, 42).entries)
    T = pin(A.random_factor(n, f, A.mix_seed(42, 1)).entries)
    nz = int(train.row_ptr[-1])
    csr = N.CsrT(m, n, 0, nz, rp.data_ptr(), ci.data_ptr(), vv.data_ptr())
    cfg = N.SolverConfigT(f, lam, 16, 4096, 0, 0, 42)

    def step():
        A._check(N.LIB.alsk_update_x(C.byref(csr), T.data_ptr(), n, f, C.byref(cfg), X.data_ptr()))
        A._check(N.LIB.alsk_update_theta(m, n, nz, cp.data_ptr(), ri.data_ptr(), cv.data_ptr(), X.data_ptr(), m, f,
                                         C.byref(cfg), T.data_ptr()))

    for _ in range(max(1, args.warmup // 2)):
        step()
    steps = max(2, args.steps // 2)
    t = time.perf_counter()
    for _ in range(steps):
        step()
    sec = (time.perf_counter() - t) / steps
    h2d = (rp.numel() * 8 + ci.numel() * 4 + vv.numel() * 4 + T.numel() * 4) + \
          (cp.numel() * 8 + ri.numel() * 4 + cv.numel() * 4 + X.numel() * 4)
    d2h = X.numel() * 4 + T.numel() * 4
    return {"value": sec, "unit": "s/ALS-iter", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "path": "alsk_update_x + alsk_update_theta (host buffers, pinned), wall clock per step", "steps": steps}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    out = run_ours(args)
    rank, world, _ = dist_env()
    if rank != 0:
        return
    result, train, test = out
    if not args.no_e2e and world == 1 and "e2e" not in result:
        result["e2e"] = run_e2e(args, train, test)
    if not args.no_cpu and world == 1:
        result["cpu_baseline"] = cpu_reference_sample(train, test, args.config)
    print(json.dumps(result))


if __name__ == "__main__":
    main()
