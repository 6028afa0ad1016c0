"""Batched trials (bounds.hpp Monte-Carlo loop) vs one call per trial: device
time per trial on the C2 matrix (ell = 100, q = 1, FP64-bound passes) and on
the C4-shaped matrix (25344 x 300, ell = 10, HBM-bound passes). A resident,
L2 flushed before each timed call."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1804_00462_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for name, cfgname, k, q in (("C2", "c2", 100, 1), ("C4 shape", "c4", 10, 1)):
    c = bench.CONFIGS[cfgname]
    A = bench.make_matrix(cfgname, c["m"], c["n"], 0, 1, dev)
    cfg = P.SketchConfig(k, q, 1)
    single = timed(lambda: P.sor_svd_power(A, k, cfg))
    for T in (4, 8):
        oms = torch.from_numpy(np.stack([P.gaussian_matrix(c["n"], k, 1 + t) for t in range(T)])).to(dev)
        ms = timed(lambda: P.sor_svd_power_batch(A, k, cfg, T, omegas=oms))
        loop = timed(lambda: [P.sor_svd_power(A, k, P.SketchConfig(k, q, 1 + t), omega=oms[t]) for t in range(T)])
        print(json.dumps({"matrix": name, "m": c["m"], "n": c["n"], "ell": k, "q": q, "trials": T,
                          "ms_single_call": single, "ms_batch": ms, "ms_loop_of_calls": loop,
                          "ms_per_trial_batch": ms / T, "speedup_vs_loop": loop / ms}), flush=True)
