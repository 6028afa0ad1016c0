"""Time the core SVD (K5) at several k: cluster ring (k <= 256) vs the
rotation-log kernel (k > 256, or forced with the SORSVD_OPT_JACOBI context option)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402


def run(k, forced=False, reps=5, variant=None):
    ctx = P.Context(0)
    if forced:
        ctx.set_option(P.Context.OPT_JACOBI, P.Context.JACOBI_ROTLOG)
    if variant is not None:
        ctx.set_option(P.Context.OPT_JACOBI, variant)
    rng = np.random.default_rng(k)
    u0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    v0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    mm = torch.from_numpy((u0 / np.arange(1, k + 1)) @ v0.T).cuda()
    P.full_svd(mm, ctx=ctx)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, _, _, sw = P.full_svd(mm, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return {"k": k, "forced_big": forced, "variant": variant, "ms": float(np.median(ts)), "sweeps": sw}


out = ([run(k) for k in (20, 100, 160, 200, 256, 300, 384, 512)] + [run(k, True) for k in (100, 200, 256)]
       + [run(k, variant=P.Context.JACOBI_BARRIER) for k in (100,)])
for o in out:
    print(json.dumps(o))
