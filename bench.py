#!/usr/bin/env python
"""SOR-SVD benchmark (BASELINE.json metric: SOR-SVD wall time & effective
GFLOP/s = 2*m*n*ell*passes / time, vs roofline, on 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Default workload: C3 fp64 (BASELINE.json configs[2], the 1/2/4/8-GPU config the
metric is quoted on; strong-scaled: the same 200000 x 20000 A split by rows).
`--gpus N` with no torchrun environment re-launches this script under
torch.distributed.run with N ranks (one per GPU); under torchrun WORLD_SIZE
must equal N.

One JSON line on rank 0. "ours": A and Omega resident in HBM, K timed calls of
sor_svd_power through the C ABI (CUDA events, L2 flushed between steps, max
over ranks); e2e: the same call through the public host-buffer API (H2D of A,
Omega draw + upload, D2H of U, sigma, V inside the timed region). "reference":
the compiled reference (oracle/_ref = the unmodified reference headers on
OpenBLAS) on all host cores, same config and metric.
Multi-GPU (torchrun): A is row-sharded; configs marked weak keep m rows per
rank, strong configs split the fixed m.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SOR-SVD effective GFLOP/s (2*m*n*ell*passes / wall time)"

CONFIGS = {
    # BASELINE.json configs[0]
    "c1": dict(m=1000, n=1000, k=20, q=0, scaling="weak",
               desc="C1 fp64 m=n=1000 k=ell=20 q=0, A = X Y^T + N(0,1e-4)"),
    # BASELINE.json configs[1]
    "c2": dict(m=4000, n=4000, k=100, q=1, scaling="weak",
               desc="C2 fp64 m=n=4000 k=ell=100 q=1, A = U diag(j^-2) V^T (Haar U, V)"),
    # BASELINE.json configs[2], fp64 variant (default workload)
    "c3": dict(m=200000, n=20000, k=256, q=1, scaling="strong",
               desc="C3 fp64 m=200000 n=20000 k=ell=256 q=1, A = X diag(10^(-j/64)) Y^T + N(0,1e-6)"),
    # BASELINE.json configs[2], fp32 variant: A stored in FP32, passes in FP64 arithmetic (default fp32_mode)
    "c3f32": dict(m=200000, n=20000, k=256, q=1, scaling="strong", dtype="f32", mode="fp64",
                  desc="C3 fp32 m=200000 n=20000 k=ell=256 q=1, same A rounded to fp32 (FP64 DMMA passes)"),
    # the same on the TF32 tensor cores (fp32_mode="tf32")
    "c3tf32": dict(m=200000, n=20000, k=256, q=1, scaling="strong", dtype="f32", mode="tf32",
                   desc="C3 fp32 m=200000 n=20000 k=ell=256 q=1 (TF32 tcgen05 passes), same A rounded to fp32"),
    # BASELINE.json configs[3]: inexact-ALM RPCA, SOR-SVD (k = 10, q = 1) per iteration; one step = one solve
    "c4": dict(m=25344, n=300, k=10, q=1, scaling="strong", kind="rpca",
               desc="C4 RPCA fp64 25344x300 (176x144 frames), D = X Y^T (rank 5) + 10% sparse U[-50,50], "
                    "lambda = 1/sqrt(m), tol 1e-7, max 100 iterations, SOR-SVD k=10 q=1 per iteration"),
    # BASELINE.json configs[4]: 68.7 GB FP32 matrix, FP64 arithmetic
    "c5": dict(m=131072, n=131072, k=512, q=2, scaling="strong", dtype="f32", mode="fp64",
               desc="C5 fp32 m=n=131072 k=ell=512 q=2, A = X diag(1/j) Y^T + N(0,1e-8) (FP64 DMMA passes)"),
    "c5tf32": dict(m=131072, n=131072, k=512, q=2, scaling="strong", dtype="f32", mode="tf32",
                   desc="C5 fp32 m=n=131072 k=ell=512 q=2 (TF32 tcgen05 passes; leading sigmas only)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------- data -----
def make_matrix(cfg_name, m_local, n, rank, world, device, row0=0):
    import torch
    g = torch.Generator(device=device)
    f64 = torch.float64
    if cfg_name == "c1":
        g.manual_seed(1000 + rank)
        x = torch.randn(m_local, 20, generator=g, device=device, dtype=f64)
        g.manual_seed(2000)
        y = torch.randn(n, 20, generator=g, device=device, dtype=f64)
        g.manual_seed(3000 + rank)
        return x @ y.T + 1e-2 * torch.randn(m_local, n, generator=g, device=device, dtype=f64)
    if cfg_name == "c2":
        g.manual_seed(1000 + rank)
        u, _ = torch.linalg.qr(torch.randn(m_local, m_local, generator=g, device=device, dtype=f64))
        g.manual_seed(2000)
        v, _ = torch.linalg.qr(torch.randn(n, n, generator=g, device=device, dtype=f64))
        r = min(m_local, n)
        s = 1.0 / torch.arange(1, r + 1, device=device, dtype=f64) ** 2
        return (u[:, :r] * s) @ v[:, :r].T
    if cfg_name == "c4":
        g.manual_seed(1000 + rank)
        x = torch.randn(m_local, 5, generator=g, device=device, dtype=f64)
        g.manual_seed(2000)
        y = torch.randn(n, 5, generator=g, device=device, dtype=f64)
        d = x @ y.T
        g.manual_seed(3000 + rank)
        nnz = int(round(0.1 * m_local * n))
        idx = torch.randperm(m_local * n, generator=g, device=device)[:nnz]
        vals = -50.0 + 100.0 * torch.rand(nnz, generator=g, device=device, dtype=f64)
        d.view(-1)[idx] += vals
        return d
    if cfg_name in ("c5", "c5tf32", "c3", "c3f32", "c3tf32"):
        # the global A is the same for every rank count (strong scaling): X's rows and the
        # noise come from fixed 4096-row chunks seeded by the chunk's global index, and each
        # rank materialises the chunks that overlap its row block [row0, row0 + m_local)
        c5 = cfg_name.startswith("c5")
        mg, r = (CONFIGS["c5"]["m"], 512) if c5 else (CONFIGS["c3"]["m"], 256)
        noise = 1e-4 if c5 else 1e-3
        s = (1.0 / torch.arange(1, r + 1, device=device, dtype=f64) if c5
             else 10.0 ** (-torch.arange(1, r + 1, device=device, dtype=f64) / 64.0))
        g.manual_seed(2000)
        y = torch.randn(n, r, generator=g, device=device, dtype=f64) / math.sqrt(n)
        ys = (y * s).T.contiguous()
        out_dt = f64 if cfg_name == "c3" else torch.float32
        a = torch.empty(m_local, n, device=device, dtype=out_dt)
        step = 4096
        for c0 in range((row0 // step) * step, row0 + m_local, step):
            c1 = min(c0 + step, mg)
            g.manual_seed(1_000_000 + c0 // step)
            x = torch.randn(c1 - c0, r, generator=g, device=device, dtype=f64) / math.sqrt(mg)
            blk = x @ ys
            blk += noise * torch.randn(c1 - c0, n, generator=g, device=device, dtype=f64)
            lo, hi = max(c0, row0), min(c1, row0 + m_local)
            a[lo - row0:hi - row0] = blk[lo - c0:hi - c0].to(out_dt)
            del blk, x
        return a
    raise ValueError(cfg_name)


# ------------------------------------------------------------- clocks -----
class ClockSampler:
    """SM clock and throttle reasons sampled with NVML every ~2 ms on a
    background thread; only samples taken while `recording` is set (the timed
    region) are reported. Started before the warm-up so that NVML's own
    start-up cost never lands inside the timed steps."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.recording = False
        self.stop_flag = False
        self.ok = False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self.stop_flag:
            if self.recording:
                try:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    try:
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    except Exception:
                        rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                    self.samples.append((sm, rs))
                except Exception:
                    pass
            time.sleep(0.002)

    def stop(self):
        self.stop_flag = True
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.t.join(timeout=2)
        sm = [a for a, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "NVML, ~2 ms polling during the timed steps"}


# ------------------------------------------------------- CPU reference ----
def _prefer_avx512_blas():
    """OpenBLAS 0.3.15 (the reference's BLAS here) falls back to its generic
    Prescott kernels on this CPU model; select its AVX-512 kernels when the
    host has them, so the reference runs at its best (must precede loading)."""
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return
    if "avx512f" in flags:
        os.environ.setdefault("OPENBLAS_CORETYPE", "SKYLAKEX")


def cpu_reference(a_host, k, ell, q, seed, steps, min_seconds=0.0, threads=None):
    """Times the compiled reference (oracle/_ref: unmodified reference headers on
    OpenBLAS) on host cores. Returns (per-call seconds list, cores, kind)."""
    _prefer_avx512_blas()
    from oracle import sorsvd_oracle as O
    cores = threads or os.cpu_count() or 1
    O.Ref.set_threads(cores)
    kind = "reference"
    times = []
    t_start = time.perf_counter()
    i = 0
    while i < steps or (time.perf_counter() - t_start) < min_seconds:
        t0 = time.perf_counter()
        O.Ref.sor_svd_power(a_host, k, O.SketchConfig(ell, q, seed + i))
        times.append(time.perf_counter() - t0)
        i += 1
        if i >= 200:
            break
    return times, cores, kind


def cpu_sample(cfg_name, a_dev, cfg):
    """Bounded sample of the workload for the CPU leg (about 10-30 s)."""
    if cfg_name == "c3":
        rows = 20000  # 1/10 of the rows, same n, k, q: ~1/10 of the work
        return a_dev[:rows].cpu().numpy(), f"row-block sample {rows}x{cfg['n']} of the C3 matrix (same n, k, q)"
    return a_dev.cpu().numpy(), f"full {cfg_name.upper()} instance"


# ---------------------------------------------------------------- C4 -----
def _rpca_flops(m, n, ell, q, iterations):
    """SOR-SVD flops of a solve: 2*m*n*ell*(2q+3) per iteration (the metric's numerator)."""
    return 2.0 * m * n * ell * (2 * q + 3) * iterations


def run_rpca(args, cfg, D, ctx, dist, rank, world, local_rank, device, stream, m_global, workload):
    """Config 4: one step = one inexact-ALM solve on the device-resident D (mu0
    estimated on the device), L2 flushed between steps; e2e = the host-buffer
    API (H2D of D, D2H of L and S inside the timed region)."""
    import numpy as np
    import torch
    import paper_1804_00462_b200 as P
    from paper_1804_00462_b200 import dist as Dm
    m, n = D.shape
    ell, q = cfg["k"], cfg["q"]
    rcfg = P.RpcaConfig(lam=1.0 / math.sqrt(max(m_global, n)), mu0=0.0, ell=ell, q=q, seed=9, max_iter=100)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    clocks = ClockSampler(local_rank)
    clocks.start()
    for _ in range(max(args.warmup, 0)):
        r = P.rpca_alm(D, rcfg, ctx=ctx, m_global=m_global)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks.recording = True
    t_wall = time.perf_counter()
    iters = []
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        r = P.rpca_alm(D, rcfg, ctx=ctx, m_global=m_global)
        ev[i][1].record(stream)
        iters.append(r.iterations)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    clocks.recording = False
    clk = clocks.stop()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms_per_step = Dm.max_over_ranks(dist, sum(ms_steps), device) / args.steps
    it = iters[-1]
    flops = _rpca_flops(m_global, n, ell, q, it)
    value = flops / (ms_per_step * 1e-3) / 1e9
    # HBM roofline of an iteration: 2q+3 passes over D (8 B/entry each) + the fused
    # update (read D, Y; write S, Y, W: 40 B/entry); the dominant traffic
    mp = {}
    mp_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp_path):
        try:
            mp = json.load(open(mp_path))
        except Exception:
            mp = {}
    hbm_peak = mp.get("hbm_gbs", 6650.0)
    bytes_iter = 8.0 * m * n * (2 * q + 3) + 40.0 * m * n
    achieved = bytes_iter * it / (ms_per_step * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": None, "kernel": "whole RPCA iteration (2q+3 A-passes + fused rpca_update_kernel)",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)", "bytes_per_iteration": bytes_iter,
            "ms_per_iteration": ms_per_step / it}
    # e2e: host buffers through the public API
    e2e = None
    if not args.no_e2e:
        dh = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
        dh.copy_(D)
        d_np = dh.numpy()
        P.rpca_alm(d_np, rcfg, ctx=ctx, m_global=m_global)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            P.rpca_alm(d_np, rcfg, ctx=ctx, m_global=m_global)
        el = Dm.max_over_ranks(dist, time.perf_counter() - t0, device) / args.steps
        e2e = {"value": flops / el / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(8 * m * n),
               "d2h_bytes_per_step": int(2 * 8 * m * n), "ms_per_step": el * 1e3,
               "path": "sorsvd_rpca_alm (host D in, host L and S out)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        _prefer_avx512_blas()
        from oracle import sorsvd_oracle as O
        O.Ref.set_threads(os.cpu_count() or 1)
        d_cpu = D.cpu().numpy()
        t0 = time.perf_counter()
        rr = O.Ref.rpca_alm(d_cpu, O.RpcaConfig(lam=rcfg.lam, mu0=r.mu0, ell=ell, q=q, seed=9, max_iter=100))
        sec = time.perf_counter() - t0
        cpu = {"value": _rpca_flops(m, n, ell, q, rr.iterations) / sec / 1e9, "unit": "GFLOP/s",
               "cores": os.cpu_count(), "kind": "reference",
               "sample": f"full C4 solve ({rr.iterations} iterations, same mu0), {sec:.1f}s",
               "ms_per_call": sec * 1e3, "iterations": rr.iterations}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(workload, iterations=it, rank_l=r.rank_l, nnz_s=r.nnz_s, rel_error=r.rel_error),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(r.stats.get("launches", 0)),
                "clocks": clk, "wall_s_timed_region": t_wall, "ms_steps": [round(x, 4) for x in ms_steps]}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_rpca_reference(args, cfg, workload, O):
    """--impl reference for C4: the compiled reference's sor_svd_power inside the
    SPEC.md:386-398 loop (oracle/_ref) on all host cores, same distribution."""
    import numpy as np
    O.Ref.set_threads(os.cpu_count() or 1)
    D, _, _ = O.gen_c4(4, m=cfg["m"], n=cfg["n"])
    rc = O.RpcaConfig(lam=1.0 / math.sqrt(max(D.shape)), mu0=0.0, ell=cfg["k"], q=cfg["q"], seed=9, max_iter=100)
    times, its = [], 0
    for i in range(max(args.steps, 1)):
        t0 = time.perf_counter()
        rr = O.Ref.rpca_alm(D, rc)
        times.append(time.perf_counter() - t0)
        its = rr.iterations
    sec = sum(times) / len(times)
    val = _rpca_flops(D.shape[0], D.shape[1], cfg["k"], cfg["q"], its) / sec / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": 1,
            "steps": len(times), "warmup": 0, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload, iterations=its),
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                             "sample": "full C4 solve"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ launcher --
def relaunch(n):
    """`--gpus N` outside torchrun: one rank per GPU under torch.distributed.run
    (rendezvous on 127.0.0.1), same arguments; returns the launcher's exit code."""
    import socket
    import subprocess
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    # NCCL's init lines (one per rank) on stderr, so the rank count is visible in the log
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log("bench.py: launching " + " ".join(cmd[1:]))
    return subprocess.call(cmd, env=env)


def plan_only(args, cfg, workload, rank, world, local_rank, m_local, row0):
    """The multi-rank plumbing without device work: process group (NCCL on
    GPUs, gloo otherwise), the row partition and the max-over-ranks reduction;
    rank 0 prints the plan as one JSON line."""
    import torch
    from paper_1804_00462_b200 import dist as Dm
    dist = None
    cuda = torch.cuda.is_available()
    dev = torch.device("cuda", local_rank) if cuda else None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if cuda else "gloo")
    rows = [[row0, m_local]]
    if dist:
        t = torch.tensor([row0, m_local], dtype=torch.int64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        rows = [[int(x[0]), int(x[1])] for x in allt]
    slowest = Dm.max_over_ranks(dist, float(rank), dev)
    if rank == 0:
        print(json.dumps({"plan": True, "n_gpus": world, "config": workload, "rank_rows": rows,
                          "max_over_ranks_check": slowest}), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--plan-only", action="store_true",
                    help="launch the ranks, partition the rows, exchange ids and time nothing (CPU-testable)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
        return 2
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    k = ell = cfg["k"]
    q = cfg["q"]
    passes = 2 * q + 3
    from paper_1804_00462_b200.dist import row_partition
    row0 = 0
    if cfg["scaling"] == "weak":
        m_local, m_global = cfg["m"], cfg["m"] * world
        row0 = rank * m_local
    else:
        m_global = cfg["m"]
        row0, m_local = row_partition(m_global, world, rank)
    n = cfg["n"]
    workload = dict(workload=cfg["desc"], m=m_global, n=n, k=k, ell=ell, q=q, passes=passes,
                    rows_per_rank=m_local, parallelism=f"row-sharded x{world}" if world > 1 else "single GPU",
                    l2="flushed between timed steps (256 MiB write)")

    if args.plan_only:
        return plan_only(args, cfg, workload, rank, world, local_rank, m_local, row0)

    if args.impl == "reference":
        if rank != 0:
            return 0
        _prefer_avx512_blas()
        import numpy as np
        from oracle import sorsvd_oracle as O
        # same synthetic distribution, generated on the host with the oracle RNG
        if args.config == "c1":
            a = O.gen_c1(1)
            sample = "full C1 instance"
        elif args.config == "c2":
            a = O.gen_c2(2, n=n, m=cfg["m"])
            sample = "full C2 instance"
        elif args.config == "c4":
            return run_rpca_reference(args, cfg, workload, O)
        elif args.config.startswith("c5"):
            a = O.gen_lowrank_decay(16384, 16384, 512, lambda j: 1.0 / j, 4e-4, 5).astype(np.float32).astype(np.float64)
            sample = ("16384x16384 instance of the C5 distribution (k=512, q=2, noise scaled to keep ||E|| ~ 0.07); "
                      "the metric is per-flop, extrapolated linearly in m*n*k*passes")
            n = 16384
        else:
            a = O.gen_lowrank_decay(20000, n, 256, lambda j: 10.0 ** (-j / 64.0), 1e-3, 3)
            sample = "row-block sample 20000x20000 of the C3 distribution (same n, k, q)"
        if args.warmup:
            cpu_reference(a, k, ell, q, 7, min(args.warmup, 3))
        times, cores, kind = cpu_reference(a, k, ell, q, 7, args.steps)
        sec = sum(times) / len(times)
        mm = a.shape[0]
        val = 2.0 * mm * n * ell * passes / sec / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": world,
                "steps": len(times), "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
                "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload,
                "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores, "kind": kind, "sample": sample,
                                 "blas": O.ref_lib().ref_blas_config().decode()},
                "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import numpy as np
    import torch
    import paper_1804_00462_b200 as P

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    from paper_1804_00462_b200 import dist as D
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    ctx = D.make_context(dist, local_rank, rank, world, device)
    log(f"[rank {rank}/{world}] cuda:{local_rank} library context up"
        + (" (NCCL communicator over NVLink)" if world > 1 else "") + f"; rows [{row0}, {row0 + m_local}) of {m_global}")
    stream = torch.cuda.current_stream(device)
    ctx.set_stream(stream.cuda_stream)

    def live_peaks():
        import ctypes
        pk, hb = ctypes.c_double(), ctypes.c_double()
        P._check(P._capi.lib().sorsvd_measure_peaks(ctx.handle, ctypes.byref(pk), ctypes.byref(hb)), ctx.handle)
        return pk.value, hb.value
    # FP64 DMMA burst peak, first taken on the idle GPU: after the sustained timed steps the same
    # microbenchmark runs at the power-capped clock and can read below what a long DMMA pass achieves
    peaks_idle = live_peaks()

    t_gen = time.perf_counter()
    A = make_matrix(args.config, m_local, n, rank, world, device, row0=row0)
    torch.cuda.synchronize()
    log(f"[rank {rank}] generated {m_local}x{n} fp64 in {time.perf_counter() - t_gen:.1f}s")
    if cfg.get("kind") == "rpca":
        return run_rpca(args, cfg, A, ctx, dist, rank, world, local_rank, device, stream, m_global, workload)
    omega = torch.from_numpy(P.gaussian_matrix(n, ell, 7)).to(device)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    scfg = P.SketchConfig(ell=ell, q=q, seed=7)

    fp32_mode = cfg.get("mode", "fp64")

    def call():
        return P.sor_svd_power(A, k, scfg, omega=omega, ctx=ctx, m_global=m_global, fp32_mode=fp32_mode)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    clocks.start()
    for _ in range(max(args.warmup, 0)):
        call()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    clocks.recording = True
    launches = 0
    t_wall = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        f = call()
        ev[i][1].record(stream)
        launches += int(f.stats["launches"])
    barrier()
    t_wall = time.perf_counter() - t_wall
    clocks.recording = False
    clk = clocks.stop()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms_total = D.max_over_ranks(dist, sum(ms_steps), device)
    ms_per_step = ms_total / args.steps
    flops_step = 2.0 * m_global * n * ell * passes
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # ---- per-stage device times of one extra call (no graph, STAGE_TIMES) ----
    fs = P.sor_svd_power(A, k, scfg, omega=omega, ctx=ctx, m_global=m_global, stage_times=True,
                         fp32_mode=fp32_mode)
    stages = {key: round(fs.stats[key], 4) for key in ("ms_total", "ms_passes", "ms_qr", "ms_project", "ms_svd",
                                                        "ms_basis")}
    stages["jacobi_sweeps"] = fs.stats["jacobi_sweeps"]
    pass_kind = int(fs.stats.get("pass_kind", 0))  # 0 FP64 DMMA, 1 Ozaki int8 (FP64), 2 TF32
    oz_planes = bool(fs.stats.get("oz_planes", 0))   # Ozaki: A cut into int8 digit planes once per call
    stages["pass_engine"] = ["fp64 DMMA", "fp64 via Ozaki int8 tensor cores", "tf32 tensor cores"][pass_kind]
    stages["note"] = "un-graphed call with per-stage CUDA events; passes = the 2q+2 sketch passes"

    # ---- roofline of the dominant kernel (the A-streaming pass) ----
    import ctypes
    f32 = cfg.get("dtype") == "f32"
    tf32 = f32 and fp32_mode == "tf32"
    esz = 4 if f32 else 8
    fp64_peak = max(peaks_idle[0], live_peaks()[0])  # idle-GPU burst vs after the timed steps: the higher
    mp = {}
    mp_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp_path):
        try:
            mp = json.load(open(mp_path))
        except Exception:
            mp = {}
    hbm_peak = mp.get("hbm_gbs", 6650.0)
    if tf32:
        # TF32 peak: a plain library GEMM (cuBLAS TF32, 8192^3) measured live, like the bf16 entry
        torch.backends.cuda.matmul.allow_tf32 = True
        xa = torch.randn(8192, 8192, device=device, dtype=torch.float32)
        xb = torch.randn(8192, 8192, device=device, dtype=torch.float32)
        for _ in range(3):
            xa @ xb
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record(stream)
            xa @ xb
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        tensor_peak = 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12
        peak_src = "live cuBLAS TF32 8192^3 GEMM (burst); MEASURED_PEAKS.json has no TF32 entry"
        del xa, xb
        Np = ((ell + 31) // 32) * 32 if ell <= 256 else ((ell + 255) // 256) * 256
        tdt = torch.float32
        pass_fn = P._capi.lib().sorsvd_pass_f32_device
        kname = "tc_gemm_tf32_kernel (tcgen05.mma kind::tf32, TMA, TMEM)"
    else:
        tensor_peak = fp64_peak
        peak_src = "live FP64 DMMA burst (sorsvd_measure_peaks, the higher of idle-GPU and post-run readings); MEASURED_PEAKS.json has no FP64 entry"
        Np = (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128  # npad()
        tdt = torch.float64
        pass_fn = P._capi.lib().sorsvd_pass_f32a_device if f32 else P._capi.lib().sorsvd_pass_device
        kname = ("gemm_f64_kernel<float A> (FP32 tile widened to FP64, DMMA m8n8k4)" if f32
                 else "gemm_f64_kernel (DMMA m8n8k4, cp.async ring)")
    X = torch.zeros(n, Np, dtype=tdt, device=device)
    X[:, :ell] = omega.to(tdt)
    T = torch.zeros(m_local, Np, dtype=tdt, device=device)
    ms_pass = ctypes.c_double()
    lpp = ctypes.c_int32()
    P._check(pass_fn(ctx.handle, 0, m_local, n, n, ell, A.data_ptr(), X.data_ptr(), T.data_ptr(), max(args.steps, 5),
                     ctypes.byref(ms_pass), ctypes.byref(lpp)), ctx.handle)
    T2 = torch.zeros(n, Np, dtype=tdt, device=device)
    ms_pass_t = ctypes.c_double()
    P._check(pass_fn(ctx.handle, 1, m_local, n, n, ell, A.data_ptr(), T.data_ptr(), T2.data_ptr(), max(args.steps, 5),
                     ctypes.byref(ms_pass_t), ctypes.byref(lpp)), ctx.handle)
    pass_flops = 2.0 * m_local * n * ell
    pass_bytes = float(esz) * m_local * n
    ai = pass_flops / pass_bytes
    ridge = tensor_peak * 1e12 / (hbm_peak * 1e9)
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get(args.config, {}).get(
                ("pass_nn_dram_bytes_ozaki_planes" if oz_planes else "pass_nn_dram_bytes_ozaki") if pass_kind == 1
                else "pass_nn_dram_bytes")
        except Exception:
            traffic = None
    if pass_kind == 1:
        # the library's pass engine here: ozaki_planes_gemm_kernel (A's digit planes cut once per
        # call, ozaki_planes_i8.cuh) or ozaki_gemm_kernel (A converted inside the pass), both
        # tcgen05 kind::i8. Its roofline is the
        # INT8 tensor rate: sorsvd_ozaki_products() int8 digit products per FP64 multiply-add (ozaki_i8.cuh), against
        # 2 x the measured BF16 burst (the INT8 dense rate is twice BF16 on B200; MEASURED_PEAKS.json
        # has no INT8 entry). The FP64-equivalent rate is reported beside it.
        oz = P._capi.lib().sorsvd_pass_ozaki_device
        ms_o, ms_sc = ctypes.c_double(), ctypes.c_double()
        dt_code = 1 if f32 else 0
        P._check(oz(ctx.handle, 0, m_local, n, n, ell, dt_code, A.data_ptr(), X.data_ptr(), T.data_ptr(),
                    max(args.steps, 5), ctypes.byref(ms_o), ctypes.byref(ms_sc)), ctx.handle)
        ms_ot = ctypes.c_double()
        P._check(oz(ctx.handle, 1, m_local, n, n, ell, dt_code, A.data_ptr(), T.data_ptr(), T2.data_ptr(),
                    max(args.steps, 5), ctypes.byref(ms_ot), ctypes.byref(ms_sc)), ctx.handle)
        n_prod = int(P._capi.lib().sorsvd_ozaki_products())
        int8_ops = float(n_prod) * pass_flops
        i8_peak = 2.0 * mp.get("bf16_tflops", 1590.0)
        achieved = int8_ops / (ms_o.value * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": i8_peak, "unit": "TOPS (int8)",
                "frac": achieved / i8_peak, "traffic": traffic,
                "kernel": ("ozaki_planes_gemm_kernel (tcgen05.mma kind::i8 on A's int8 digit planes, cut once per call "
                           f"and streamed by 3-D TMA; {n_prod} digit products / FP64 FMA), NN pass T1 = A*X" if oz_planes else
                           f"ozaki_gemm_kernel (tcgen05.mma kind::i8, TMA-staged A converted in the pass, {n_prod} digit "
                           "products / FP64 FMA), NN pass T1 = A*X"),
                "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (burst): INT8 dense = 2x BF16 on B200",
                "ms_per_launch": ms_o.value, "int8_ops_per_launch": int8_ops, "flops_per_launch": pass_flops,
                "fp64_equiv_tflops": pass_flops / (ms_o.value * 1e-3) / 1e12,
                "fp64_equiv_over_dmma_peak": pass_flops / (ms_o.value * 1e-3) / 1e12 / fp64_peak,
                "dmma_peak_tflops": fp64_peak, "ms_scales_per_call": ms_sc.value,
                "scales_per_call": ("row exponents + the 7 digit planes of A in one read (ozaki_rowplanes_kernel)"
                                    if oz_planes else "row / column exponents of A (ozaki_absmax_kernel)"),
                "tn_pass": {"ms": ms_ot.value, "achieved": int8_ops / (ms_ot.value * 1e-3) / 1e12},
                "dmma_pass_for_comparison": {"ms_nn": ms_pass.value, "ms_tn": ms_pass_t.value,
                                             "tflops_nn": pass_flops / (ms_pass.value * 1e-3) / 1e12},
                "hbm_gbs_measured": hbm_peak, "hbm_frac": pass_bytes / (ms_o.value * 1e-3) / 1e9 / hbm_peak}
    elif ai >= ridge:
        achieved = pass_flops / (ms_pass.value * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tensor_peak, "unit": "TFLOP/s",
                "frac": achieved / tensor_peak, "traffic": traffic, "kernel": kname + ", NN pass T1 = A*X",
                "peak_source": peak_src, "ms_per_launch": ms_pass.value, "flops_per_launch": pass_flops,
                **({"frac_of_half_measured_bf16": achieved / (0.5 * mp.get("bf16_tflops", 1590.0)),
                    "frac_of_nominal_tf32_1125": achieved / 1125.0,
                    "note_peaks": "TF32 dense is half the BF16 rate: also shown against 0.5 x MEASURED_PEAKS bf16_tflops "
                                  "and against the nominal 1125 TFLOP/s (the live cuBLAS TF32 GEMM reaches ~2/3 of nominal)"}
                   if tf32 else {}),
                "tn_pass": {"ms": ms_pass_t.value, "achieved": pass_flops / (ms_pass_t.value * 1e-3) / 1e12},
                "hbm_gbs_measured": hbm_peak, "hbm_frac": pass_bytes / (ms_pass.value * 1e-3) / 1e9 / hbm_peak}
    else:
        achieved = pass_bytes / (ms_pass.value * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "kernel": kname + ", NN pass T1 = A*X",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)", "ms_per_launch": ms_pass.value,
                "bytes_per_launch": pass_bytes,
                "tn_pass": {"ms": ms_pass_t.value, "achieved": pass_bytes / (ms_pass_t.value * 1e-3) / 1e9}}
    del X, T, T2

    # ---- e2e through the public host-buffer API ----
    e2e = None
    if not args.no_e2e:
        a_host = torch.empty((m_local, n), dtype=A.dtype, pin_memory=True)
        a_host.copy_(A)
        a_np = a_host.numpy()
        del A
        torch.cuda.empty_cache()
        hcfg = P.SketchConfig(ell=ell, q=q, seed=7)
        for _ in range(max(1, min(args.warmup, 2))):
            P.sor_svd_power(a_np, k, hcfg, ctx=ctx, m_global=m_global, fp32_mode=fp32_mode)
        barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            P.sor_svd_power(a_np, k, hcfg, ctx=ctx, m_global=m_global, fp32_mode=fp32_mode)
        el = D.max_over_ranks(dist, time.perf_counter() - t0, device)
        e2e = {"value": flops_step / (el / args.steps) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(m_local * n * esz + n * ell * 8),
               "d2h_bytes_per_step": int((m_local + n) * k * 8 + k * 8),
               "ms_per_step": el / args.steps * 1e3,
               "path": "sorsvd_sor_svd_power (host buffers, pinned A; Omega drawn from seed inside)"}
    else:
        a_np = None

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if a_np is None:
            a_np = A.cpu().numpy()
        if args.config in ("c3", "c3f32", "c3tf32"):
            a_cpu = np.ascontiguousarray(a_np[:20000], dtype=np.float64)
            sample = "row-block sample 20000x20000 of the C3 matrix (same n, k, q)"
        elif args.config.startswith("c5"):
            a_cpu = np.ascontiguousarray(a_np[:16384, :16384], dtype=np.float64)
            sample = ("16384x16384 block of the C5 matrix (k=512, q=2); per-flop rate, extrapolated linearly "
                      "in m*n*k*passes")
        else:
            a_cpu = a_np
            sample = f"full {args.config.upper()} instance"
        times, cores, kind = cpu_reference(a_cpu, k, ell, q, 7, 3, min_seconds=10.0)
        sec = statistics.median(times)
        cpu = {"value": 2.0 * a_cpu.shape[0] * a_cpu.shape[1] * ell * passes / sec / 1e9, "unit": "GFLOP/s",
               "cores": cores,
               "kind": kind, "sample": f"{sample}; median of {len(times)} calls ({sum(times):.1f}s)",
               "ms_per_call": sec * 1e3}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": cfg["scaling"], "vs_baseline": None,
                "dtype": (("f32/tf32" if tf32 else "f32 storage, f64 arithmetic") if f32 else "f64")
                + (" (passes: exact int8 digit products on the tensor cores, Ozaki)" if pass_kind == 1 else ""),
                "data": "synthetic", "config": workload, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk, "stages_ms": stages,
                "wall_s_timed_region": t_wall, "ms_steps": [round(x, 4) for x in ms_steps]}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
