"""Time the C3 call (device-resident A, Omega given) under context options:
  python tools/c3_variants.py "7=1" "7=0" "7=1,6=1"      # key=value lists (SORSVD_OPT_*), one variant each
Prints the median of 7 calls per variant (CUDA events on the context's stream = torch's current stream)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
import bench  # noqa: E402

c = bench.CONFIGS["c3"]
A = bench.make_matrix("c3", c["m"], c["n"], 0, 1, torch.device("cuda", 0))
om = torch.from_numpy(P.gaussian_matrix(c["n"], c["k"], 7)).cuda()
cfg = P.SketchConfig(c["k"], c["q"], 7)
ref = None
for spec in sys.argv[1:] or ["7=1"]:
    ctx = P.Context(0)
    for kv in spec.split(","):
        k, v = kv.split("=")
        ctx.set_option(int(k), int(v))
    ts = []
    for i in range(9):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f = P.sor_svd_power(A, c["k"], cfg, omega=om, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    s = f.sigma.cpu().numpy()
    same = None if ref is None else bool((s == ref).all())
    if ref is None:
        ref = s
    print(f"{spec:>12s}  median {ts[len(ts)//2]:.2f} ms  min {ts[0]:.2f}  max {ts[-1]:.2f}  sigma identical to first: {same}", flush=True)
    ctx.close()
