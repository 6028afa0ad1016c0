"""Time the core SVD (K5) at several k: cluster ring (k <= 256) vs the
rotation-log kernel (k > 256, or forced with SORSVD_JACOBI_BIG)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402


def run(k, forced=False, reps=5):
    if forced:
        os.environ["SORSVD_JACOBI_BIG"] = "1"
    else:
        os.environ.pop("SORSVD_JACOBI_BIG", None)
    rng = np.random.default_rng(k)
    u0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    v0, _ = np.linalg.qr(rng.standard_normal((k, k)))
    mm = torch.from_numpy((u0 / np.arange(1, k + 1)) @ v0.T).cuda()
    P.full_svd(mm)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, _, _, sw = P.full_svd(mm)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return {"k": k, "forced_big": forced, "ms": float(np.median(ts)), "sweeps": sw}


out = [run(k) for k in (100, 256, 300, 384, 512)] + [run(k, True) for k in (100, 256)]
for o in out:
    print(json.dumps(o))
