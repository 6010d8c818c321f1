#!/usr/bin/env python
"""bench.py — seconds per ALS iteration (X half-sweep + Theta half-sweep), BASELINE.json's
metric, on the Netflix-shape synthetic workload by default (480,189 x 17,770, 99M ratings,
10% holdout, f=100, lambda=0.05); --config picks another named shape (ml1m, yahoo,
hugewiki, sparkals).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config netflix]

--gpus N > 1 without torchrun in the environment re-launches itself under
`torch.distributed.run` with N ranks (127.0.0.1 rendezvous), one process per GPU. Multi-GPU
runs use libalskit_cuda's C++ session (alsk_mp_*) with NCCL inside the library:
model-parallel rows of X then Theta with in-place all-gathers (netflix, yahoo, hugewiki), or
the hybrid split with a data-parallel Theta half and a partial-Hermitian reduce-scatter
(sparkals). Every rank builds only its own share of the data in HBM from the row-seeded
generator; the holdout split runs once (rank 0) and travels as a bitmask.

Timing: W warm-up iterations, then K iterations between a barrier + synchronize on each
side, CUDA events on the launching stream, max over ranks. Inputs (CSR + CSC of the train
matrix, >= 1.4 GB at Netflix) exceed L2, so no flush is needed.

Extra keys: roofline (the dominant kernel against its measured peak; for N > 1 also the
collectives' bytes and bus bandwidth against NVLink), cpu_baseline (the unmodified
reference, oracle/_ref, run in a separate process on a bounded sample that keeps every
host thread busy), e2e (the same metric through the host-buffer C ABI, H2D + D2H inside the
timed region).

--impl reference runs the reference's own train_run iteration (oracle/_ref: update_x on the
train CSR, then on its transpose; threads = hardware_concurrency) on the same input bytes,
read from a shared binary cache with the reference's load_binary_cache. That process never
loads libalskit_cuda.so.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name: (m, n, nnz_total, f, lambda)  — SURVEY.md §8(d); lambdas from PAPER.md Table 4
CONFIGS = {
    "ml1m": (6040, 3706, 1000209, 10, 0.05),
    "netflix": (480189, 17770, 99_000_000, 100, 0.05),
    "yahoo": (1000990, 624961, 252_800_000, 100, 1.4),
    "hugewiki": (50082604, 39781, 3_100_000_000, 100, 0.05),
    "sparkals": (660_000_000, 2_400_000, 3_500_000_000, 10, 0.05),
}
SHAPE_ID = {"ml1m": 0, "netflix": 1, "yahoo": 2, "hugewiki": 3, "sparkals": 4}
# shapes whose whole matrix the CPU reference can hold and iterate in a bench run
REF_FULL = {"ml1m", "netflix", "yahoo"}
RUN_SEED = 42
MASK64 = (1 << 64) - 1


def mix_seed(seed: int, salt: int) -> int:
    """splitmix64 finaliser (reference common.hpp:70-75)."""
    z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def data_seed(cfg: str) -> int:
    return mix_seed(RUN_SEED, 100 + SHAPE_ID[cfg])


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="netflix", choices=list(CONFIGS))
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"],
                    help="fp32: the FP32 path (tensor cores where 16 <= f <= 119); fp64: the reference-order "
                         "FP64-exact kernels (SolverConfig.accumulate_double, the drop-in's default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cache-dir", default=os.environ.get("ALSK_BENCH_CACHE", "/tmp/alsk_bench_cache"))
    ap.add_argument("--cpu-sample", action="store_true",
                    help="(reference arm) the bounded cpu_baseline sample instead of full iterations")
    ap.add_argument("--ref-max-iters", type=int, default=3, help="(reference arm) cap on timed full iterations")
    ap.add_argument("--dry-run", action="store_true", help="rendezvous only: every rank reports in, no GPU work")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args) -> int:
    """Re-launch this script under torch.distributed.run with --gpus ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def cache_path(args) -> Path:
    return Path(args.cache_dir) / f"{args.config}_{data_seed(args.config):016x}.cache"


def cpu_info() -> dict:
    model = None
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "hardware_concurrency": os.cpu_count(),
            "sched_getaffinity": len(os.sched_getaffinity(0))}


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
def _ref():
    from oracle import binding  # the reference arm loads oracle/_ref only
    ref = binding.reference()
    if ref is None:
        raise RuntimeError("oracle/_ref not built (needs /root/reference at build time)")
    return ref


def ref_prepare(args, ref) -> tuple[dict, int, int]:
    """Shared binary cache (written once with the reference's save_binary_cache from the
    shared generator) -> the reference's load / split / transpose / init."""
    m, n, nnz, f, lam = CONFIGS[args.config]
    path = cache_path(args)
    setup = {}
    if not path.exists():
        path.parent.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".tmp{os.getpid()}")
        t = time.perf_counter()
        st = ref.bench_write_cache(m, n, nnz, data_seed(args.config), tmp)
        assert st == 0, ref.last_error()
        os.replace(tmp, path)
        setup["write_cache_s"] = time.perf_counter() - t
    st, nz_train, n_test, secs = ref.bench_prepare(path, 0.1, RUN_SEED, f, lam)
    assert st == 0, ref.last_error()
    setup.update({"load_binary_cache_s": secs[0], "split_train_test_s": secs[1], "transpose_s": secs[2],
                  "random_factor_s": secs[3], "cache": str(path)})
    return setup, nz_train, n_test


def ref_sample(args, ref, nz_train: int) -> dict:
    """Bounded sample that keeps every reference thread busy: whole update_x batches
    (batch_rows = 4096, parallel_for chunks of 32 rows, solver.hpp:107, 330-345) of each
    half, extrapolated to a full iteration by nonzero count."""
    kx, kt = 32 * 4096, 4096
    st, dx, dt, nzx, nzt = ref.bench_sample(kx, kt)
    assert st == 0, ref.last_error()
    per_iter = dx * nz_train / nzx + dt * nz_train / nzt
    threads = ref.hardware_threads()
    return {"value": per_iter, "unit": "s/ALS-iter", "cores": threads, "kind": "reference",
            "sample": f"reference update_x (accumulate_double, threads=0 -> {threads}) on the first {kx} rows "
                      f"({nzx} nnz) of the X half and the first {kt} items ({nzt} nnz) of the Theta half: "
                      f"{dx:.2f} s + {dt:.2f} s, extrapolated by nnz to {nz_train} train ratings per half",
            **cpu_info()}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    m, n, nnz, f, lam = CONFIGS[args.config]
    base_line = {"impl": "reference", "metric": f"s/ALS-iter ({args.config}-shape f={f})", "unit": "s/ALS-iter",
                 "n_gpus": args.gpus, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
                 "dtype": "f64-accumulate", "data": "synthetic (planted rank-10 + U[-0.5,0.5) noise; SURVEY §8(d) "
                 "generator), shared binary cache"}
    if args.config not in REF_FULL:
        print(json.dumps({**base_line, "unavailable": f"the CPU reference cannot hold and iterate the "
                          f"{args.config} shape ({nnz} ratings) within a bench run; see DESIGN.md"}))
        return
    ref = _ref()
    setup, nz_train, n_test = ref_prepare(args, ref)
    if args.cpu_sample:
        print(json.dumps(ref_sample(args, ref, nz_train)))
        return
    warm = min(args.warmup, 1)
    steps = max(1, min(args.steps, args.ref_max_iters))
    for _ in range(warm):
        st, _, _ = ref.bench_iteration()
        assert st == 0, ref.last_error()
    halves = []
    for _ in range(steps):
        st, xs, ts = ref.bench_iteration()
        assert st == 0, ref.last_error()
        halves.append((xs, ts))
    it = [x + t for x, t in halves]
    v = float(np.median(it))
    st, loss, rmse, loss_s, rmse_s = ref.bench_eval()
    threads = ref.hardware_threads()
    print(json.dumps({
        **base_line, "value": v, "steps": steps, "warmup": warm, "steps_requested": args.steps,
        "warmup_requested": args.warmup, "ms_per_step": v * 1e3,
        "config": {"workload": args.config, "m": m, "n": n, "nnz_total": nnz, "nnz_train": nz_train, "f": f,
                   "lambda": lam, "holdout": 0.1, "parallelism": f"host threads (reference thread pool, {threads})"},
        "iterations_s": [{"x_half": x, "theta_half": t} for x, t in halves],
        "eval": {"train_J": loss, "test_rmse": rmse, "loss_s": loss_s, "rmse_s": rmse_s,
                 "note": "serial in the reference; timed apart, not part of the iteration"},
        "setup": setup,
        "cpu_baseline": {"value": v, "unit": "s/ALS-iter", "cores": threads, "kind": "reference",
                         "sample": f"{steps} full iteration(s) of train_run's loop (driver.hpp:256-258) after "
                                   f"{warm} warm-up, median", **cpu_info()},
        "e2e": {"value": v, "unit": "s/ALS-iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
    ref.bench_release()


def cpu_baseline_subprocess(args) -> dict | None:
    """The reference's bounded sample, in its own process (which never loads libalskit_cuda)."""
    cmd = [sys.executable, str(Path(__file__).resolve()), "--impl", "reference", "--cpu-sample", "--config",
           args.config, "--cache-dir", args.cache_dir]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    for line in reversed(res.stdout.splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return {"unavailable": (res.stderr or res.stdout)[-300:]}


# ------------------------------------------------------------------ our arm --------
def dry_run(args):
    import torch.distributed as dist
    import torch
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    seen = [None] * world
    me = {"rank": rank, "local_rank": local, "pid": os.getpid()}
    if world > 1:
        dist.all_gather_object(seen, me)
    else:
        seen = [me]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "requested": args.gpus, "ranks": seen}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    del torch


def fp32_peak_probe():
    from paper_1603_03820_b200 import _native as N
    fn = getattr(N.LIB, "alsk_fp32_peak_probe", None)
    return float(fn()) if fn is not None else None


def phase(N, k):
    ms, n = C.c_double(), C.c_uint64()
    N.LIB.alsk_profile_phase(k, C.byref(ms), C.byref(n))
    return ms.value, n.value


def build_inputs(args, rank, world, dev):
    """This rank's train CSR slices and test triplets (datagen.build_rank_data), or at one
    GPU the shared binary cache when the reference arm left one (same bytes)."""
    import torch
    import torch.distributed as dist
    from paper_1603_03820_b200 import datagen as G
    from paper_1603_03820_b200.session import DeviceCsr
    m, n, nnz, f, lam = CONFIGS[args.config]
    mode = "hybrid" if (args.config == "sparkals" and world > 1) else "model"
    path = cache_path(args)
    t0 = time.perf_counter()
    if world == 1 and path.exists():
        R = DeviceCsr.from_cache(path, dev)
        x, test = R.split_train_test(0.1, G.split_seed())
        del R
        t = x.transpose()
        src = f"binary cache {path} (the reference arm's input bytes), device split"
        rd = G.RankData(args.config, m, n, f, lam, 0, 1, mode, (0, m), (0, n), x, t, test, nnz, x.nnz)
    else:
        if rank == 0:
            mask = G.holdout_mask(nnz, 0.1, G.split_seed())
        else:
            mask = np.zeros(max(1, (nnz + 31) // 32), np.uint32)
        if world > 1:
            tm = torch.from_numpy(mask.view(np.int32))
            dist.broadcast(tm, src=0)
        rd = G.build_rank_data(args.config, rank, world, dev, mask, mode=mode)
        del mask
        src = "row-seeded device generator per rank (bit-identical to the shared cache) + holdout bitmask " \
              "from rank 0"
    torch.cuda.synchronize()
    return rd, mode, src, time.perf_counter() - t0


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1603_03820_b200 import _native as N
    from paper_1603_03820_b200 import alskit as A
    from paper_1603_03820_b200.distributed import HYBRID, MODEL, MultiGpuALS, NativeComm
    from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo")  # plumbing (id exchange, barriers, max of timings)
    comm = NativeComm.from_process_group(local) if world > 1 else None
    m, n, nnz, f, lam = CONFIGS[args.config]
    prec = PREC_FP64_EXACT if args.precision == "fp64" else PREC_FP32
    rd, mode_name, data_src, setup_s = build_inputs(args, rank, world, dev)
    mode = HYBRID if mode_name == "hybrid" else MODEL
    theta0 = torch.from_numpy(A.random_factor(n, f, A.mix_seed(RUN_SEED, 1)).entries).to(dev)
    # X needs no initial value: the first X half overwrites it (train_run, driver.hpp:256)
    als = MultiGpuALS(comm, mode, m, n, f, lam, prec, rd.x, rd.t, None, theta0)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        als.step()
    als.check()
    barrier()
    launches0 = A.kernel_launch_count()
    clocks = Clocks((ROOT / "gpurun_out" if (ROOT / "gpurun_out").exists() else Path("/tmp")) /
                    f"clocks_rank{rank}.csv")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        N.LIB.alsk_profile_begin()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            als.step()
        e1.record(stream)
        torch.cuda.synchronize()
        als.check()
        herm = phase(N, 0)
        solve = phase(N, 1)
        fused = phase(N, 2)
        coll = phase(N, 3)
        N.LIB.alsk_profile_end(C.byref(C.c_double()), C.byref(C.c_uint64()))
    ms_local = e0.elapsed_time(e1) / args.steps
    launches = A.kernel_launch_count() - launches0
    coll_bytes, coll_calls = als.collective_stats()
    per_rank = np.array([ms_local, herm[0], solve[0], fused[0], coll[0], rd.x.nnz, rd.t.nnz, launches], np.float64)
    if world > 1:
        import torch as _t
        allr = [_t.zeros(len(per_rank), dtype=_t.float64) for _ in range(world)]
        dist.all_gather(allr, _t.from_numpy(per_rank))
        table = np.stack([a.numpy() for a in allr])
    else:
        table = per_rank[None, :]
    ms = float(table[:, 0].max())  # max over ranks

    # test RMSE after the run (reported, not timed): per-rank squared-error sums combined
    rmse = None
    if rd.test.shape[0] > 0 or world > 1:
        sse, cnt = 0.0, 0
        if rd.test.shape[0] > 0:
            tt = rd.test.view(torch.int64)  # rows of TRIPLET_DTYPE: row i64, col i64, value f32 (+pad)
            rows = tt[:, 0].contiguous()
            cols = tt[:, 1].contiguous()
            vals = rd.test[:, 16:20].contiguous().view(torch.float32).reshape(-1)
            xp, xb, tp = als.pointers()
            out = C.c_double()
            if xb:  # hybrid: the X slab starts at global row xb
                xp -= xb * f * 4
            A._check(N.LIB.alsk_dev_rmse(rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), rows.numel(), xp,
                                         rd.xs[1], tp, n, f, C.byref(out), stream.cuda_stream))
            sse, cnt = out.value ** 2 * rows.numel(), rows.numel()
        if world > 1:
            import torch as _t
            v = _t.tensor([sse, float(cnt)], dtype=_t.float64)
            dist.all_reduce(v)
            sse, cnt = float(v[0]), int(v[1])
        rmse = (sse / cnt) ** 0.5 if cnt else None

    result = None
    if rank == 0:
        nz_x, nz_t = float(table[0, 5]), float(table[0, 6])
        nz_train_total = float(table[:, 5].sum())
        peaks = {}
        try:
            peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        except (OSError, ValueError):
            pass
        roof = roofline(args, f, m, n, nz_x, nz_t, world, herm, solve, fused, coll, coll_bytes, coll_calls, ms, peaks)
        result = {
            "metric": f"s/ALS-iter ({args.config}-shape f={f})",
            "value": ms / 1e3, "unit": "s/ALS-iter", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if prec == PREC_FP32 else "f64-accumulate",
            "data": "synthetic (planted rank-10 + U[-0.5,0.5) noise; SURVEY §8(d) generator)",
            "config": {"workload": args.config, "m": m, "n": n, "nnz_total": nnz, "nnz_train": int(nz_train_total),
                       "f": f, "lambda": lam, "holdout": 0.1,
                       "parallelism": ("single GPU" if world == 1 else
                                       f"{'hybrid: model-parallel X + data-parallel Theta (NCCL reduce-scatter)' if mode == HYBRID else 'model-parallel rows'}"
                                       f" x{world} + NCCL all-gather (libalskit_cuda alsk_mp)"),
                       "precision": args.precision, "input": data_src, "setup_s": round(setup_s, 2),
                       "l2": "inputs > L2 (train CSR + CSC), no flush",
                       "engine": A.fp32_engine()},
            "roofline": roof,
            "gpu_launches": int(table[:, 7].sum()),
            "test_rmse_after_run": rmse,
            "per_rank_ms": [round(float(v), 3) for v in table[:, 0]],
        }
        cs = clocks.summary(local)
        if cs:
            result["clocks"] = cs
    barrier()
    if not args.no_e2e and args.config in REF_FULL:
        e2e = run_e2e(args, rd, als, comm, rank, world, dev, prec)
        if rank == 0:
            result["e2e"] = e2e
    als.close()
    return result


def roofline(args, f, m, n, nz_x, nz_t, world, herm, solve, fused, coll, coll_bytes, coll_calls, ms, peaks):
    """The dominant kernel against its measured peak (SURVEY.md §8(d) units), plus the
    collectives at N > 1. Figures are rank 0's (its launches, its nonzeros)."""
    steps = args.steps
    flops_per_nz = f * (f + 1) + 2 * f  # lower triangle as FMA = 2 flop, + B
    bf16 = peaks.get("bf16_tflops")
    hbm = peaks.get("hbm_gbs")
    ffma = fp32_peak_probe() or 148 * 128 * 2 * 1.965e9 / 1e12
    herm_ms, herm_n = herm
    if args.precision == "fp64":
        # reference-order FP64 kernels (materialised A/B + exact solve): the Hermitian against
        # the FP64 FMA peak (148 SMs x 64 DFMA x 2 flop x 1.965 GHz; no measured figure)
        flops = steps * (nz_x + nz_t) * flops_per_nz
        fp64 = 148 * 64 * 2 * 1.965e9 / 1e12
        achieved = flops / (herm_ms * 1e-3) / 1e12 if herm_ms else None
        roof = {"bound": "fp64", "kernel": "herm_mat_kernel<double> (reference-order FP64 Hermitian + bias)",
                "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
                "frac": achieved / fp64 if achieved else None,
                "peak_source": "nominal FP64 FMA peak at the max SM clock (MEASURED_PEAKS.json has none)",
                "traffic": None, "flops_per_launch": flops / max(herm_n, 1), "kernel_ms_avg": herm_ms / max(herm_n, 1),
                "launches": int(herm_n), "kernel_share_of_step": (herm_ms / steps) / ms,
                "solve": {"kernel": "solve_exact_kernel (reference-order FP64 Cholesky)",
                          "ms_per_step": solve[0] / steps, "share_of_step": (solve[0] / steps) / ms}}
    elif herm_n > 0 and f > 15:
        # tensor-core engine: Hermitian (tc_update_kernel) and batched Cholesky timed apart
        flops = steps * (nz_x + nz_t) * flops_per_nz
        achieved = flops / (herm_ms * 1e-3) / 1e12
        tf32 = bf16 / 2 if bf16 else 2250.0 / 2
        rows = (m + n) / world
        solve_flops = steps * rows * (f ** 3 / 3 + 2 * f * f)
        pk_row = 4 * (8 * (((f + 7) // 8) * (f + 1) - 4 * ((f + 7) // 8) * ((f + 7) // 8 - 1)))
        hbytes = steps * ((nz_x + nz_t) * (4 * f + 8) + 8 * (rows + 2) + rows * pk_row)
        roof = {"bound": "tensor", "kernel": "tc_update_kernel (tcgen05 tf32x2 Hermitian + bias, packed rows)",
                "achieved": achieved, "peak": tf32, "unit": "TFLOP/s", "frac": achieved / tf32,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (dense TF32)" if bf16 else "nominal dense TF32",
                "traffic": traffic_for(args.config, f),
                "flops_per_launch": flops / herm_n, "kernel_ms_avg": herm_ms / herm_n, "launches": int(herm_n),
                "kernel_share_of_step": (herm_ms / steps) / ms,
                "fp32_ffma_equiv": {"peak": ffma, "frac": achieved / ffma,
                                    "peak_source": "measured FFMA probe (alsk_fp32_peak_probe)"},
                "tf32x3_equiv": {"peak": tf32 / 3, "frac": achieved / (tf32 / 3)},
                "gather": {"bytes_per_launch": hbytes / herm_n, "achieved": hbytes / (herm_ms * 1e-3) / 1e9,
                           "peak": hbm, "unit": "GB/s",
                           "frac": hbytes / (herm_ms * 1e-3) / 1e9 / hbm if hbm else None},
                "solve": {"kernel": "warp_solve_kernel (one system per warp in shared memory, mma.sync tf32x2 "
                                    "Schur updates)",
                          "ms_per_step": solve[0] / steps, "launches": int(solve[1]),
                          "achieved_tflops": solve_flops / (solve[0] * 1e-3) / 1e12 if solve[0] else None,
                          "packed_rows_gbs": steps * rows * pk_row / (solve[0] * 1e-3) / 1e9 if solve[0] else None,
                          "share_of_step": (solve[0] / steps) / ms}}
    else:
        # register/FFMA engines (f <= 15 here): HBM-bound gather, SURVEY.md §8(d)
        kms, kn = (fused if fused[1] else herm)
        rows = (m + n) / world
        bytes_ = steps * ((nz_x + nz_t) * (8 + 4 * f) + 8 * (rows + 2))
        kname = (f"small_update_kernel<{f}> (thread or warp per row; Hermitian + bias + Cholesky in registers)"
                 if f <= 15 else "fused_update_kernel (FFMA)")
        achieved = bytes_ / (kms * 1e-3) / 1e9 if kms else None
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm if (hbm and achieved) else None, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "traffic": traffic_for(args.config, f), "bytes_per_launch": bytes_ / max(kn, 1),
                "kernel_ms_avg": kms / max(kn, 1), "launches": int(kn),
                "kernel_share_of_step": (kms / steps) / ms if kms else None}
    if world > 1:
        nvl = peaks.get("nvlink_gbs") or 900.0
        gb_s = coll_bytes / (coll[0] * 1e-3) / 1e9 if coll[0] else None
        roof["collectives"] = {
            "kind": "ncclAllGather (in place)" + (" + ncclReduceScatter" if args.config == "sparkals" else ""),
            "bytes_per_rank_per_step": coll_bytes / steps, "calls_per_step": coll_calls / steps,
            "ms_per_step": coll[0] / steps, "busbw_gbs": gb_s, "peak": nvl,
            "frac": gb_s / nvl if gb_s else None,
            "peak_source": "MEASURED_PEAKS.json nvlink_gbs" if peaks.get("nvlink_gbs") else
            "nominal NVLink 5 per direction (900 GB/s)",
            "share_of_step": (coll[0] / steps) / ms,
            "bytes_formula": "(P-1)/P * rows * f * 4 per all-gather (SURVEY §8(d))"}
    return roof


def traffic_for(config, f):
    tf = ROOT / "profiles" / "traffic.json"
    try:
        t = json.loads(tf.read_text())
        return t.get(config)
    except (OSError, ValueError):
        return None


def run_e2e(args, rd, als, comm, rank, world, dev, prec):
    """The same metric end to end. One GPU: the reference-facing host-buffer C ABI
    (alsk_update_x + alsk_update_theta on pinned host CSR/CSC/factors). N GPUs: every rank
    copies its CSR slices and the starting Theta from pinned host memory, runs the
    multi-GPU iteration, and copies its solved X and Theta slices back. Wall clock, max over
    ranks."""
    import torch
    import torch.distributed as dist
    from paper_1603_03820_b200 import _native as N
    from paper_1603_03820_b200 import alskit as A
    m, n, nnz, f, lam = CONFIGS[args.config]
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    theta_h = pin(torch.from_numpy(A.random_factor(n, f, A.mix_seed(RUN_SEED, 1)).entries))
    if world == 1:
        x, t = rd.x, rd.t
        rp, ci, vv = pin(x.row_ptr[: x.rows + 1]), pin(x.col_idx[: x.nnz]), pin(x.values[: x.nnz])
        cp, ri, cv = pin(t.row_ptr[: t.rows + 1]), pin(t.col_idx[: t.nnz]), pin(t.values[: t.nnz])
        X = torch.zeros(m * f, dtype=torch.float32).pin_memory()
        T = theta_h.clone().pin_memory()
        csr = N.CsrT(m, n, 0, x.nnz, rp.data_ptr(), ci.data_ptr(), vv.data_ptr())
        cfg = N.SolverConfigT(f, lam, 16, 4096, 1 if args.precision == "fp64" else 0, 0, RUN_SEED)

        def step():
            T.copy_(theta_h)
            A._check(N.LIB.alsk_update_x(C.byref(csr), T.data_ptr(), n, f, C.byref(cfg), X.data_ptr()))
            A._check(N.LIB.alsk_update_theta(m, n, x.nnz, cp.data_ptr(), ri.data_ptr(), cv.data_ptr(), X.data_ptr(),
                                             m, f, C.byref(cfg), T.data_ptr()))
        h2d = rp.nbytes + ci.nbytes + vv.nbytes + cp.nbytes + ri.nbytes + cv.nbytes + theta_h.nbytes + X.nbytes
        d2h = X.nbytes + T.nbytes
        path = "alsk_update_x + alsk_update_theta (host buffers, pinned), wall clock per step"
    else:
        x, t = rd.x, rd.t
        xi, xv = pin(x.col_idx[: x.nnz]), pin(x.values[: x.nnz])
        ti, tv = pin(t.col_idx[: t.nnz]), pin(t.values[: t.nnz])
        xp, xb, tp = als.pointers()
        (rb, re), (cb, ce) = als.xs, als.ts
        x_out = torch.empty((re - rb) * f, dtype=torch.float32).pin_memory()
        t_out = torch.empty((ce - cb) * f, dtype=torch.float32).pin_memory()
        stream = torch.cuda.current_stream()

        def step():
            x.col_idx[: x.nnz].copy_(xi, non_blocking=True)
            x.values[: x.nnz].copy_(xv, non_blocking=True)
            t.col_idx[: t.nnz].copy_(ti, non_blocking=True)
            t.values[: t.nnz].copy_(tv, non_blocking=True)
            A._check(N.LIB.alsk_host_to_dev(tp, theta_h.data_ptr(), theta_h.nbytes, stream.cuda_stream))
            als.step()
            xoff = 0 if xb else rb * f * 4
            A._check(N.LIB.alsk_dev_to_host(x_out.data_ptr(), xp + xoff, x_out.nbytes, stream.cuda_stream))
            A._check(N.LIB.alsk_dev_to_host(t_out.data_ptr(), tp + cb * f * 4, t_out.nbytes, stream.cuda_stream))
            als.check()
        h2d = xi.nbytes + xv.nbytes + ti.nbytes + tv.nbytes + theta_h.nbytes
        d2h = x_out.nbytes + t_out.nbytes
        path = (f"multi-GPU iteration on {world} GPUs from pinned host buffers (each rank: its CSR slices and the "
                "starting Theta H2D, its X and Theta slices D2H), wall clock, max over ranks")
    for _ in range(max(1, args.warmup // 2)):
        step()
    steps = max(2, args.steps // 2)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    v = torch.tensor([sec, float(h2d), float(d2h)], dtype=torch.float64)
    if world > 1:
        mx = v[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(v)
        v[0] = mx[0]
    return {"value": float(v[0]), "unit": "s/ALS-iter", "h2d_bytes_per_step": int(v[1]),
            "d2h_bytes_per_step": int(v[2]), "path": path, "steps": steps}


def main():
    args = parse()
    rank, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn(args))
    if world != args.gpus and not (args.impl == "reference" and args.cpu_sample):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        dry_run(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    result = run_ours(args)
    if rank != 0:
        return
    if not args.no_cpu and world == 1:
        result["cpu_baseline"] = cpu_baseline_subprocess(args)
    print(json.dumps(result))


if __name__ == "__main__":
    main()
