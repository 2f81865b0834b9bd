"""Benchmark: CAKF + CAKS time-steps/s on the ERA5-shaped synthetic workload (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl cakf|reference]

One bench "step" = one full pass of the hot path: T predict /
update / truncate steps of the filter followed by the T-step smoother sweep, on the same
device-resident synthetic inputs.  value = time-steps processed per second over the timed
region (whole job: summed over ranks, max-over-ranks device time).  The trace (25.6 GB at
cfg3) is far larger than the 126 MB L2, so inputs are larger than L2 between iterations.

--impl reference times the CPU oracle (oracle/mfree.py, as it stands) on a bounded sample
of the same workload and extrapolates to time-steps/s (sample described in the JSON).
N > 1 (torchrun): one problem, the two Gram products sharded over the ranks (K1 by
symmetric tile-block units + NCCL all-reduce, K2 by output-row slices + NCCL all-gather),
the rest replicated; strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")
METRIC = "filter+smoother time-steps/sec at D=231,360 on 1/2/4/8 B200; % roofline"

# ALU roofline of the kernel-evaluation pair: every pair needs one sqrt
# and one exp2 on the MUFU (16 ops/clk/SM on B200) => 8 pairs/clk/SM.
SMS = 148
MUFU_PER_SM_CLK = 16
MUFU_PER_PAIR = 2
FP32_FLOP_PER_SM_CLK = 256  # 128 FFMA lanes x 2
# K2 computes each fp32 product from an exact 3-way bf16 split with 6 bf16 MMAs
BF16_PRODUCTS_PER_FP32_MAC = 6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--impl", default="cakf", choices=["cakf", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cull", action="store_true", help="disable exact-zero culling (results are bit-identical)")
    ap.add_argument("--no-dense", action="store_true", help="skip the reference timing with culling off")
    ap.add_argument("--no-interp", action="store_true", help="skip the temporal-interpolation query timing")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--serving", type=int, default=2,
                    help="also time P independent problems per GPU on P streams (reported as 'serving'; <2: skip)")
    ap.add_argument("--T", type=int, default=None, help="override T (debug only; invalidates the metric)")
    return ap.parse_args()


def peaks():
    try:
        with open(MEASURED) as f:
            mp = json.load(f)
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1]))
                    mx.append(float(p[2]))
                except ValueError:
                    continue
                for n, v in zip(names, p[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle baseline
def host_info():
    """lscpu model, physical cores, threads the oracle's BLAS / thread pools use, host RAM."""
    import platform
    info = {"cpu_model": platform.processor() or "unknown", "physical_cores": None, "logical_cpus": os.cpu_count(),
            "ram_gib": None}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        import psutil
        info["physical_cores"] = psutil.cpu_count(logical=False)
        info["ram_gib"] = round(psutil.virtual_memory().total / 2 ** 30, 1)
    except Exception:
        pass
    try:
        import threadpoolctl
        info["blas_threads"] = max([p.get("num_threads", 1) for p in threadpoolctl.threadpool_info()] + [1])
    except Exception:
        info["blas_threads"] = None
    return info


def oracle_rates(wl, rows=(2048, 96, 640), lr_rows=16384):
    """Per-operation rates of the matrix-free oracle O8 (oracle/mfree.py, as it stands) on bounded samples
    of workload `wl`: seconds per kernel evaluation of a K_TT s matvec, of a K_XX B product with the
    smoother's 2(1+r) right-hand sides and of a K(X, X_T) [v V] product (1 + max_iter columns); seconds per
    flop of its dense low-rank algebra (numpy matmuls of the step's shapes on a row slab)."""
    from oracle import mfree
    Xn = wl.coords
    idx = wl.obs_idx[0]
    Xt = Xn[idx]
    N, NX = len(idx), len(Xn)
    r = max(wl.max_rank, 0)
    C_post, C_sm = 1 + wl.max_iter, 2 * (1 + r)
    rng = np.random.default_rng(0)
    a, b, c = (min(x, y) for x, y in zip(rows, (N, NX, NX)))
    s = rng.standard_normal(N)
    t0 = time.perf_counter()
    mfree.gram_apply(Xt, Xt, s, wl.nu_x, wl.ell_x, chunk=1024, rows=(0, a))
    t1 = time.perf_counter()
    mfree.gram_apply(Xn, Xn, rng.standard_normal((NX, C_sm)), wl.nu_x, wl.ell_x, chunk=96, rows=(0, b))
    t2 = time.perf_counter()
    mfree.gram_apply(Xn, Xt, rng.standard_normal((N, C_post)), wl.nu_x, wl.ell_x, chunk=640, rows=(0, c))
    t3 = time.perf_counter()
    # low-rank algebra (M^T X, M (M^T X): the smoother's D x r x (1+r) products) on a row slab
    L = min(lr_rows, wl.D)
    M = rng.standard_normal((L, r + wl.max_iter))
    X = rng.standard_normal((L, 1 + r))
    t4 = time.perf_counter()
    T = M.T @ X
    _ = M @ T
    t5 = time.perf_counter()
    lr_flop = 4.0 * L * (r + wl.max_iter) * (1 + r)
    return {"s_per_eval_matvec": (t1 - t0) / (a * N), "s_per_eval_smooth": (t2 - t1) / (b * NX),
            "s_per_eval_post": (t3 - t2) / (c * N), "s_per_flop_lowrank": (t5 - t4) / lr_flop,
            "sample_s": t5 - t0,
            "sample": (f"O8 gram_apply rows [0,{a}) of K_TT s ({a}x{N}), rows [0,{b}) of K_XX x {C_sm} RHS, rows "
                       f"[0,{c}) of K(X,X_T) x {C_post} RHS; numpy M^T X, M (M^T X) on a {L}-row slab")}


def oracle_step_seconds(wl, rt):
    """Cost model of one O8 time step (filter update + truncation + smoother step) from the measured rates:
    per step the oracle runs 3 G applications per CG iteration (G s, G d for CGS2, G d), one K(X, X_T) [v V]
    product, the truncation's M^T M / M Q, and in the smoother K_XX on the 2 derivative blocks of the
    (1+r) carriers plus ~3 D x r x (1+r) low-rank products."""
    N, NX, D = wl.n_obs(1), wl.n_space, wl.D
    r = max(wl.max_rank, 0)
    n = wl.max_iter
    c = r + n
    t_loop = n * 3 * N * N * rt["s_per_eval_matvec"]
    t_post = NX * N * rt["s_per_eval_post"] + 4.0 * D * r * (1 + n) * rt["s_per_flop_lowrank"]
    t_trunc = (2.0 * D * c * c + 2.0 * D * c * r) * rt["s_per_flop_lowrank"]
    t_smooth = wl.d_time * NX * NX * rt["s_per_eval_smooth"] + 3 * 4.0 * D * r * (1 + r) * rt["s_per_flop_lowrank"] \
        + (2.0 * D * c * c + 4.0 * D * c * r) * rt["s_per_flop_lowrank"]
    parts = {"filter_loop": t_loop, "post_loop": t_post, "truncation": t_trunc, "smoother_step": t_smooth}
    return sum(parts.values()), parts


def cpu_baseline(wl):
    """The oracle O8 on the host: (1) a full CAKF + CAKS run at cfg2 (D = 14,640) for T = 2, measured end to
    end; (2) per-step rates of O8 on bounded samples of `wl` (the bench's workload), (3) the cost model of
    oracle_step_seconds at `wl` -> time-steps/s, labelled extrapolated, with the same model evaluated at
    cfg2 beside the cfg2 measurement as its calibration."""
    from oracle import mfree
    from synth import make_workload
    # calibration: a complete O8 run (as it stands: kernel rows regenerated per product) at cfg2 with 4 actions
    # per step and rank cap 4 (truncation active from step 2), T = 2, against the same cost model
    w2 = make_workload("cfg2", T=2, max_iter=4, max_rank=4)
    t0 = time.perf_counter()
    mfree.run_mf(w2, dtype_round=np.float32)
    cfg2_s = time.perf_counter() - t0
    rt2 = oracle_rates(w2, rows=(2048, 512, 2048), lr_rows=w2.D)
    step2_s, _ = oracle_step_seconds(w2, rt2)
    rt = oracle_rates(wl, rows=(1536, 64, 512))
    step_s, parts = oracle_step_seconds(wl, rt)
    hi = host_info()
    return {"value": 1.0 / step_s, "unit": "time-steps/s", "cores": hi.get("blas_threads") or hi["logical_cpus"],
            "kind": "oracle", "extrapolated": True,
            "sample": (f"{rt['sample']}; per-step cost model (filter 3 x {wl.max_iter} K_TT matvecs, post-loop, "
                       f"truncation, smoother step) extrapolated to one {wl.name} time step"),
            "s_per_time_step_model": step_s, "model_parts_s": {k: round(v, 2) for k, v in parts.items()},
            "calibration": {"workload": "cfg2 (D=14,640), 4 CG actions/step, rank cap 4, T=2 filter+smoother, "
                            "oracle/mfree.run_mf as it stands", "measured_wall_s": round(cfg2_s, 2),
                            "measured_time_steps_per_s": 2.0 / cfg2_s, "model_s_per_step": round(step2_s, 3),
                            "model_over_measured": round(step2_s * 2.0 / cfg2_s, 3)},
            "host": hi, "sample_sec": round(rt["sample_s"] + cfg2_s, 2)}


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores.  Each bench step is one bounded sample of
    the workload (the rates of oracle_rates); value = the extrapolated time-steps/s of the cost model,
    ms_per_step = the measured wall time of one sample step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import make_workload
    wl = make_workload(args.config)
    for _ in range(args.warmup):
        oracle_rates(wl, rows=(256, 16, 64), lr_rows=2048)
    walls, vals = [], []
    rt = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rt = oracle_rates(wl)
        walls.append(time.perf_counter() - t0)
        vals.append(1.0 / oracle_step_seconds(wl, rt)[0])
    value = statistics.median(vals)
    hi = host_info()
    ms_step = statistics.median(walls) * 1e3
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "time-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "D": wl.D, "N_X": wl.n_space, "N": wl.n_obs(1), "T": wl.T,
                   "policy": wl.policy, "max_iter": wl.max_iter, "max_rank": wl.max_rank},
        "extrapolated": True,
        "note": ("each bench step runs a bounded sample of the oracle (ms_per_step is its measured wall time); value "
                 "is the oracle's time-steps/s on the full workload from the per-step cost model "
                 "(bench.py oracle_step_seconds)"),
        "cpu_baseline": {"value": value, "unit": "time-steps/s", "cores": hi.get("blas_threads") or hi["logical_cpus"],
                         "kind": "oracle", "extrapolated": True, "sample": rt["sample"], "host": hi},
        "e2e": {"value": value, "unit": "time-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------------ roofline helpers
def nonzero_pair_frac(wl, rows=256, seed=0):
    """Fraction of kernel pairs whose fp32 value is not exactly zero: a = |x - y| sqrt(3)/ell <= 126/log2(e)
    (ex2.approx.ftz underflows beyond), on `rows` random rows against all columns (host numpy): K1's
    training x training pairs and K2's all x training pairs."""
    rng = np.random.default_rng(seed)
    sc = np.sqrt(2.0 * wl.nu_x) / wl.ell_x
    X = (wl.coords * sc).astype(np.float32).astype(np.float64)
    idx = np.asarray(wl.obs_idx[0])
    Xt = X[idx]
    cut = 126.0 / np.log2(np.e)
    ri = rng.choice(len(Xt), min(rows, len(Xt)), replace=False)
    d2 = ((Xt[ri, None, :] - Xt[None, :, :]) ** 2).sum(-1)
    k1 = float(np.mean(d2 <= cut * cut))
    rx = rng.choice(len(X), min(rows, len(X)), replace=False)
    d2 = ((X[rx, None, :] - Xt[None, :, :]) ** 2).sum(-1)
    k2 = float(np.mean(d2 <= cut * cut))
    return {"k1": k1, "k2_post": k2, "sample": f"{len(ri)} random training rows x {len(Xt)} (K1), {len(rx)} random "
            f"grid rows x {len(Xt)} (K2 post), host fp64 distances of the fp32-rounded prescaled coordinates"}


def pass_roofline(wl, prof, live, nz, hbm_gbs, pass_ms):
    """Whole-pass lower bound (per phase max(evals c / ALU peak, MMA flop / tensor peak, bytes / HBM)):
    K1 on its truly nonzero unique pairs at the live MUFU pair rate; the post-loop K2 on its nonzero kernel
    evaluations (2 MUFU each); every other phase on its algorithmic HBM bytes (each operand read once, each
    output written once, fp32); the eigensolver's bytes are negligible (latency-bound, bound 0)."""
    N, NX, D, T = wl.n_obs(1), wl.n_space, wl.D, wl.T
    n, r = wl.max_iter, max(wl.max_rank, 0)
    B = 4.0
    pair_rate = live["mufu_ops_per_s"] / MUFU_PER_PAIR
    k1_s = T * n * nz["k1"] * N * (N + 1) / 2 / pair_rate
    k2_s = T * nz["k2_post"] * NX * N / pair_rate
    stage_bytes = lowrank_bytes = trunc_bytes = 0.0
    cols = 0
    for k in range(1, T + 1):
        rin = cols
        c = rin + n
        # inner loop: V, Z read twice (CGS2) per iteration, HM^- twice (u = HM^T s, HM u), ~12 N-vectors
        stage_bytes += sum(4 * N * (i - 1) * B + 2 * N * rin * B + 12 * N * B for i in range(1, n + 1))
        # post-loop low-rank: (HM)^T [v V] reads HM, [v V]; M^- U reads M^-, writes D x (1+n)
        lowrank_bytes += (N * rin + N * (1 + n) + D * rin + D * (1 + n)) * B
        cols = min(r, c) if r >= 0 else c
        if r >= 0 and c > r:
            trunc_bytes += (D * c + D * c + D * r) * B          # Gram read, M Q_r read + write
        # smoother step k-1: M^-T x, M^- (M^-T x) (reads M^- twice, X twice, y read+write), B_k t, V t, KV t
        q = min(r, n + rin) if r >= 0 else n + rin
        C = 1 + q
        lowrank_bytes += (2 * D * rin + 2 * D * C + 2 * D * C + D * n + N * n + NX * (1 + n) + N * C + NX * C) * B
        if r >= 0 and n + q > r:
            trunc_bytes += (D * (n + q) + 2 * D * (n + q) + 2 * D * r) * B
    hbm_s = (stage_bytes + lowrank_bytes + trunc_bytes) / (hbm_gbs * 1e9)
    bound_ms = (k1_s + k2_s + hbm_s) * 1e3
    return {"bound_ms": round(bound_ms, 2), "measured_ms": round(pass_ms, 2), "frac": bound_ms / pass_ms,
            "phases_bound_ms": {"k1_nonzero_pairs_mufu": round(k1_s * 1e3, 2), "k2_post_nonzero_evals_mufu":
                                round(k2_s * 1e3, 2), "stages_hbm": round(stage_bytes / hbm_gbs / 1e6, 2),
                                "lowrank_hbm": round(lowrank_bytes / hbm_gbs / 1e6, 2),
                                "truncation_hbm": round(trunc_bytes / hbm_gbs / 1e6, 2), "eigensolver": 0.0},
            "phases_measured_ms": {kk: round(v[0], 2) for kk, v in prof.items()},
            "peaks": f"MUFU {live['mufu_ops_per_s'] / 1e12:.2f} T ops/s live; HBM {hbm_gbs:.0f} GB/s (MEASURED_PEAKS)"}


# ------------------------------------------------------------------ GPU arm
def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: re-run this script under torch.distributed.run with N ranks on
    this node (rendezvous on 127.0.0.1); rank 0's JSON line is relayed."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, text=True)
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            print(line)
    return r.returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2405_08971_b200 import CAKF_SMOOTH, binding, runner
    from synth import make_workload

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kw = {} if args.T is None else {"T": args.T}
    wl = make_workload(args.config, **kw)
    trans, _ = runner.transitions(wl)
    # a dedicated (non-default) stream, made current: the library then runs on it (a null stream would make the
    # library create its own, which the events below would not bracket: they would time the host enqueue)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nccl_id = None
    if world > 1:
        obj = [binding.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    h = runner.make_handle(wl, args.dtype, stream=stream.cuda_stream, rank=rank, world=world, nccl_id=nccl_id,
                           cull_zero=not args.no_cull)
    inputs = runner.stage_inputs(wl, args.dtype)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        runner.run(h, trans, inputs, smooth=True)
    barrier()
    # ---------------- timed region (device-resident inputs; no per-launch profiling events)
    launches0 = binding.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = []
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):   # filter and smoother bracketed separately (two extra events)
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            runner.run(h, trans, inputs, smooth=False)
            ea.record(stream)
            h.smooth()
            eb.record(stream)
            evs.append((ea, eb))
        ev1.record(stream)
        barrier()
    launches = binding.kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    smoother_ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    filter_ms = ms / args.steps - smoother_ms
    total_timesteps = args.steps * wl.T            # one problem sharded over all ranks (strong scaling)
    value = total_timesteps / (ms / 1e3)
    clocks = clk.summary()

    # ---------------- end to end through the C-ABI with pinned HOST buffers
    npdt = np.float32 if args.dtype == "f32" else np.float64
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    host_in = []
    h2d = 0
    for (idx, y, nv, order) in runner.host_inputs(wl, args.dtype):
        ti = torch.from_numpy(idx).pin_memory()
        ty = torch.from_numpy(y).pin_memory()
        tn = torch.from_numpy(nv).pin_memory()
        to = None if order is None else torch.from_numpy(order).pin_memory()
        host_in.append((ti, ty, tn, to))
        h2d += idx.nbytes + y.nbytes + nv.nbytes + (0 if order is None else order.nbytes)
    outm = [torch.empty(wl.D, dtype=tdt).pin_memory() for _ in range(wl.T + 1)]
    outv = [torch.empty(wl.D, dtype=tdt).pin_memory() for _ in range(wl.T + 1)]
    d2h = 2 * (wl.T + 1) * wl.D * np.dtype(npdt).itemsize
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        runner.run(h, trans, host_in, smooth=True)
        for k in range(wl.T + 1):
            h.get(k, CAKF_SMOOTH, outm[k], outv[k])
    e1.record(stream)
    barrier()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e = {"value": args.e2e_steps * wl.T / max(ms_e2e / 1e3, 1e-9), "unit": "time-steps/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---------------- one separate pass with per-launch CUDA events: the phase split and the launch times
    # of the roofline kernels (profiling stays out of the timed region above)
    h.profile(True)
    h.profile_read(reset=True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    runner.run(h, trans, inputs, smooth=True)
    p1.record(stream)
    barrier()
    prof = h.profile_read(reset=True)
    h.profile(False)
    ms_profiled = p0.elapsed_time(p1)
    live = binding.alu_peaks(stream.cuda_stream)

    # ---------------- roofline of the dominant kernel (live CUDA-event timings, live MUFU peak)
    mp, src = peaks()
    clock_hz = float(mp.get("sm_max_mhz", 1965.0)) * 1e6
    N = wl.n_obs(1)
    nz = nonzero_pair_frac(wl)
    # exact-zero culling: the kernels evaluate only tiles with a nonzero fp32 value; the roofline
    # is taken on the evaluated work, the dense-equivalent rate is reported beside it
    cull = h.cull_stats()
    smooth_k2 = os.environ.get("CAKF_SMOOTH_K2") == "1"   # direct smoother K2 (default: propagated products)
    cat_ms = {c: prof[c][0] for c in (("k1_matvec", "k2_post", "k2_smooth") if smooth_k2 else ("k1_matvec", "k2_post"))}
    if not smooth_k2:
        cull.pop("k2_smooth", None)
    dom = max(cat_ms, key=cat_ms.get)
    tot, nl = prof[dom]
    avg_s = tot / max(nl, 1) / 1e3
    traffic = None
    try:
        with open(TRAFFIC) as f:
            traffic = json.load(f).get(dom)
    except Exception:
        pass
    if dom == "k1_matvec":
        # symmetric kernel: the algorithmic minimum is the N(N+1)/2 unique pairs
        dense = float(N) * (float(N) + 1.0) / 2.0
        pairs = dense * cull["k1_matvec"]
        achieved = pairs / avg_s / 1e9
        peak = live["mufu_ops_per_s"] / MUFU_PER_PAIR / 1e9
        nonzero = dense * nz["k1"]
        roof = {"bound": "alu", "kernel": "k1_matvec (symmetric fused Matern-3/2 eval x vector)",
                "achieved": achieved, "peak": peak, "unit": "Gpair/s", "frac": achieved / peak, "traffic": traffic,
                "algorithmic_per_launch": f"{pairs:.4g} evaluated unique pairs = {cull['k1_matvec']:.4f} x N(N+1)/2",
                "evaluated_frac": cull["k1_matvec"], "nonzero_frac": nz["k1"],
                "frac_on_nonzero_pairs": nonzero / avg_s / 1e9 / peak,
                "frac_on_dense_pairs": dense / avg_s / 1e9 / peak,
                "dense_equivalent_achieved": dense / avg_s / 1e9,
                "avg_launch_ms": avg_s * 1e3, "launches": nl,
                "peak_source": (f"measured live in this run (cakf_alu_peaks): {live['mufu_ops_per_s'] / 1e12:.3f} "
                                f"T MUFU ops/s (sqrt/ex2 mix) / {MUFU_PER_PAIR} MUFU per pair; spec: {SMS} x "
                                f"{MUFU_PER_SM_CLK}/clk x "
                                f"{clock_hz / 1e6:.0f} MHz / 2 = {SMS * MUFU_PER_SM_CLK / 2 * clock_hz / 1e9:.0f} Gpair/s"),
                "nonzero_sample": nz["sample"]}
    else:
        M = wl.n_space
        Kd = N if dom == "k2_post" else wl.n_space
        C = (1 + wl.max_iter) if dom == "k2_post" else wl.d_time * (1 + max(wl.max_rank, 0))
        dense = 2.0 * M * Kd * C
        flops = dense * cull[dom]
        achieved = flops / avg_s / 1e12
        bf16 = float(mp.get("bf16_tflops_sustained", mp.get("bf16_tflops", 1590.0)))
        peak = bf16 / BF16_PRODUCTS_PER_FP32_MAC
        roof = {"bound": "tensor", "kernel": f"{dom} (fused kernel-eval GEMM on tcgen05, 3xBF16 split)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "algorithmic_per_launch": f"{flops:.4g} evaluated fp32-equivalent flop = {cull[dom]:.4f} x 2 M K C",
                "evaluated_frac": cull[dom], "dense_equivalent_achieved": dense / avg_s / 1e12,
                "avg_launch_ms": avg_s * 1e3, "launches": nl,
                "peak_source": f"measured bf16 dense {bf16:.0f} TFLOP/s (sustained, {src}) / "
                               f"{BF16_PRODUCTS_PER_FP32_MAC} bf16 MMAs per fp32-accurate MAC"}
    step_ms = ms / args.steps
    breakdown = {c: round(prof[c][0], 3) for c in prof}   # one profiled pass
    if not smooth_k2:   # the smoother's (I (x) K) x is propagated from the post-loop products
        breakdown["smooth_kx"] = breakdown.pop("k2_smooth")
    out = {
        "metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": args.config, "D": wl.D, "N_X": wl.n_space, "N": N, "T": wl.T,
                   "policy": wl.policy, "max_iter": wl.max_iter, "max_rank": wl.max_rank,
                   "cull_zero": not args.no_cull, "evaluated_frac": {k: round(v, 4) for k, v in cull.items()},
                   "step": "one full CAKF (T predict/update/truncate) + CAKS (T smoother steps) pass",
                   "smoother": ("direct K2 per smoother step (CAKF_SMOOTH_K2=1)" if smooth_k2 else
                                "kernel products propagated exactly from the stored post-loop K(X,T_k)[v V]"),
                   "parallelism": (f"row-sharded Gram products x{world} (NCCL all-reduce / all-gather)"
                                   if world > 1 else "single GPU"),
                   "l2": "inputs larger than L2 (trace 25.6 GB vs 126 MB L2)"},
        "clocks": clocks,
        "gpu_launches": int(launches),
        "e2e": e2e,
        "roofline": roof,
        "pass_roofline": pass_roofline(wl, prof, live, nz, float(mp.get("hbm_gbs", 6551.4)), ms / args.steps),
        "alu_peaks_live": live,
        "phase_ms_per_step": breakdown,
        "phase_split_source": f"one separate profiled pass ({ms_profiled:.1f} ms with per-launch events)",
        "filter_ms_per_step": round(filter_ms, 3), "smoother_ms_per_step": round(smoother_ms, 3),
        "filter_time_steps_per_s": wl.T / (filter_ms / 1e3), "smoother_time_steps_per_s": wl.T / (smoother_ms / 1e3),
    }
    h.destroy()
    if not args.no_cull and not args.no_dense and args.dtype == "f32":
        # the same pass with exact-zero culling off (bit-identical results): the dense-work rate and
        # K1's roofline fraction on the full N(N+1)/2 pairs, reported separately
        hd = runner.make_handle(wl, args.dtype, stream=stream.cuda_stream, rank=rank, world=world, nccl_id=nccl_id,
                                cull_zero=False)
        runner.run(hd, trans, inputs, smooth=True)
        barrier()
        hd.profile(True)
        hd.profile_read(reset=True)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        runner.run(hd, trans, inputs, smooth=True)
        d1.record(stream)
        barrier()
        dprof = hd.profile_read(reset=True)
        dms = d0.elapsed_time(d1)
        if world > 1:
            t = torch.tensor([dms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dms = float(t.item())
        k1_ms, k1_n = dprof["k1_matvec"]
        pairs = float(N) * (float(N) + 1.0) / 2.0
        k1_rate = pairs / (k1_ms / max(k1_n, 1) / 1e3) / 1e9
        out["dense"] = {"value": wl.T / (dms / 1e3), "unit": "time-steps/s", "ms_per_step": dms, "steps": 1,
                        "warmup": 1, "cull_zero": False,
                        "k1_roofline": {"achieved": k1_rate, "peak": roof.get("peak") if dom == "k1_matvec" else None,
                                        "unit": "Gpair/s", "frac": (k1_rate / roof["peak"]) if dom == "k1_matvec" else None,
                                        "algorithmic_per_launch": f"{pairs:.4g} unique pairs N(N+1)/2"},
                        "phase_ms_per_step": {c: round(dprof[c][0], 3) for c in dprof}}
        hd.destroy()
    if world == 1 and not args.no_interp:
        # temporal interpolation (Cor. A.10): one pass with the smoother carriers
        # kept, then filter / smoother queries at mid-interval times, device-timed per query
        from paper_2405_08971_b200 import CAKF_FILTER
        hi = runner.make_handle(wl, args.dtype, stream=stream.cuda_stream, cull_zero=not args.no_cull,
                                keep_carriers=True)
        runner.run(hi, trans, inputs, smooth=True)
        barrier()
        q = {}
        for which, name in ((CAKF_FILTER, "filter"), (CAKF_SMOOTH, "smoother")):
            times_ms = []
            for k in sorted({max(1, min(wl.T - 1, x)) for x in (wl.T // 4, wl.T // 2, (3 * wl.T) // 4)}):
                dt = float(wl.dts[min(k, wl.T - 1)])
                A1, Q1, _ = binding.matern_transition(wl.nu_t, wl.ell_t, wl.sigma, 0.5 * dt)
                A2 = binding.matern_transition(wl.nu_t, wl.ell_t, wl.sigma, 0.5 * dt)[0]
                q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                q0.record(stream)
                hi.interpolate(k, A1, Q1, A2, which)      # synchronises (device -> host copy of the result)
                q1.record(stream)
                q1.synchronize()
                times_ms.append(q0.elapsed_time(q1))
            q[name] = round(statistics.median(times_ms), 3)
        out["interpolation_ms_per_query"] = dict(q, note="cakf_interpolate at t = (t_k + t_k+1)/2, k = T/4, T/2, "
                                                 "3T/4; includes the D2H copy of mean and variance")
        # posterior sampler (alg:cakf-caks-sampler): S joint samples of all T+1
        # states; the draws are standard normal here (timing only: the cost does not depend on them)
        S = 4
        rng = np.random.default_rng(0)
        npdt = np.float32 if args.dtype == "f32" else np.float64
        x0 = torch.from_numpy(rng.standard_normal((S, wl.D)).astype(npdt)).cuda().T.contiguous().T
        qd = torch.from_numpy(rng.standard_normal((wl.T, S, wl.D)).astype(npdt)).cuda()
        ed = torch.from_numpy(rng.standard_normal(sum(len(i) for i in wl.obs_idx) * S).astype(npdt)).cuda()
        outd = torch.empty(((wl.T + 1) * S * wl.D,), dtype=qd.dtype, device="cuda")
        smp = {}
        for which, name in ((CAKF_FILTER, "filter"), (CAKF_SMOOTH, "smoother")):
            # one untimed call first: the handle's grow-only sampler workspace is allocated on the first
            # call (a stream-ordered pool allocation whose cost varies run to run), not in later ones
            binding._check(hi.lib.cakf_sample(hi.h, S, x0.data_ptr(), qd.data_ptr(), ed.data_ptr(), which,
                                              outd.data_ptr()))
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            binding._check(hi.lib.cakf_sample(hi.h, S, x0.data_ptr(), qd.data_ptr(), ed.data_ptr(), which,
                                              outd.data_ptr()))
            s1.record(stream)
            s1.synchronize()
            smp[name] = round(s0.elapsed_time(s1), 3)
        out["sampler_ms_per_call"] = dict(smp, samples=S, note="cakf_sample: S joint samples of the T+1 states "
                                          "(device buffers; standard-normal draws for timing; after one untimed "
                                          "call that allocates the workspace)")
        hi.destroy()
    if world == 1 and args.serving > 1:
        # serving mode: P independent problems per GPU, one handle + stream + host thread each, so one
        # problem's latency-bound phases (truncation eigensolver, CG stage reductions) are filled by
        # another's K1 (scripts/concurrent_bench.py; tests/test_gpu_concurrent.py)
        import threading
        P = args.serving
        sts = [torch.cuda.Stream() for _ in range(P)]
        hs = [runner.make_handle(wl, args.dtype, stream=s.cuda_stream, cull_zero=not args.no_cull) for s in sts]

        def drive(p, n):
            for _ in range(n):
                runner.run(hs[p], trans, inputs, smooth=True)

        def run_all(n):
            ths = [threading.Thread(target=drive, args=(p, n)) for p in range(P)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()

        run_all(1)
        barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for s in sts:
            s.wait_event(c0)
        run_all(args.steps)
        for s in sts:
            ev = torch.cuda.Event()
            ev.record(s)
            stream.wait_event(ev)
        c1.record(stream)
        barrier()
        cms = c0.elapsed_time(c1)
        out["serving"] = {"problems_per_gpu": P, "value": P * args.steps * wl.T / (cms / 1e3), "unit": "time-steps/s",
                          "ms_per_pass_per_problem": cms / args.steps, "steps": args.steps, "warmup": 1,
                          "note": "independent problems (same workload, device-resident inputs), one stream + host "
                                  "thread each, CUDA events bracketing all streams; no profiling events"}
        for x in hs:
            x.destroy()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
