"""One SOR-SVD call on the C4 iteration shape (W 25344 x 300, ell = 10, q = 1): per-stage device times
(un-graphed) and the graphed call time, with the fused NN+TN sweeps on and off."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00462_b200 as P

torch.manual_seed(0)
W = torch.randn(25344, 5, dtype=torch.float64, device="cuda") @ torch.randn(5, 300, dtype=torch.float64, device="cuda")
W += 0.1 * torch.randn(25344, 300, dtype=torch.float64, device="cuda")
cfg = P.SketchConfig(10, 1, 3)
for fused in (1, 0):
    ctx = P.Context(0)
    ctx.set_option(P.Context.OPT_FUSED_PAIR, fused)
    for _ in range(3):
        f = P.sor_svd_power(W, 10, cfg, ctx=ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        f = P.sor_svd_power(W, 10, cfg, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    st = P.sor_svd_power(W, 10, cfg, ctx=ctx, stage_times=True).stats
    print(f"fused={fused}: graphed call {e0.elapsed_time(e1) / 50 * 1000:.1f} us; stages (us): " +
          ", ".join(f"{k[3:]} {v * 1000:.1f}" for k, v in st.items() if k.startswith("ms_") and v), "launches", st["launches"],
          "sigma1", float(f.sigma[0]))
