"""Time thin_qr (K3) paths: CholeskyQR2 (well conditioned), Householder TSQR
(ill conditioned, k <= 256), adaptive CholeskyQR (k > 256)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402


def case(m, k, cond_exp, reps=3):
    g = torch.Generator(device="cuda").manual_seed(m + k)
    x = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
    q, _ = torch.linalg.qr(x)
    v, _ = torch.linalg.qr(torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g))
    s = torch.logspace(0, -cond_exp, k, dtype=torch.float64, device="cuda")
    t = (q * s) @ v.T
    del x, q
    P.thin_qr(t)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        qq, rr = P.thin_qr(t)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    orth = float((qq.T @ qq - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max())
    return {"m": m, "k": k, "cond": 10.0 ** cond_exp, "ms": float(np.median(ts)), "orth": orth}


for args in [(131072, 256, 3), (131072, 256, 13), (131072, 128, 13), (131072, 512, 3), (131072, 512, 13),
             (20000, 256, 13), (4000, 100, 13)]:
    print(json.dumps(case(*args)))
