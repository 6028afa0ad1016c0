"""Time the C2-shaped Householder QR (4000 x 100, ill-conditioned) under the
current environment (SORSVD_* switches)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402

m, k = int(sys.argv[1]) if len(sys.argv) > 1 else 4000, int(sys.argv[2]) if len(sys.argv) > 2 else 100
g = torch.Generator(device="cuda").manual_seed(1)
q, _ = torch.linalg.qr(torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g))
v, _ = torch.linalg.qr(torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g))
t = (q * torch.logspace(0, -13, k, dtype=torch.float64, device="cuda")) @ v.T
P.thin_qr(t)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    qq, rr = P.thin_qr(t)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
orth = float((qq.T @ qq - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max())
res = float((qq @ rr - t).abs().max())
print(json.dumps({"env": {k_: v_ for k_, v_ in os.environ.items() if k_.startswith("SORSVD")}, "m": m, "k": k,
                  "ms": float(np.median(ts)), "orth": orth, "res": res}))
