"""Host-buffer (e2e) call on bench.py's C3 matrix: wall time per call, the device span, and the bare
pinned H2D copy of A for comparison (the floor of the call)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1804_00462_b200 as P

c = bench.CONFIGS["c3"]
A = bench.make_matrix("c3", c["m"], c["n"], 0, 1, torch.device("cuda", 0))
pin = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
pin.copy_(A)
dst = A  # reuse as the copy target
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dst.copy_(pin, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print(f"bare H2D of A: {e0.elapsed_time(e1):.1f} ms = {A.numel() * 8 / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
del A, dst
torch.cuda.empty_cache()
a_np = pin.numpy()
cfg = P.SketchConfig(c["k"], c["q"], 7)
ctx = P.Context(0)
for planes in (1, 0):
    ctx.set_option(P.Context.OPT_OZAKI_PLANES, planes)
    for i in range(3):
        t0 = time.perf_counter()
        f = P.sor_svd_power(a_np, c["k"], cfg, ctx=ctx)
        wall = (time.perf_counter() - t0) * 1e3
        st = f.stats
        print(f"planes={planes} call {i}: wall {wall:.1f} ms, device span {st['ms_total']:.1f}, h2d {st['ms_h2d']:.1f}, "
              f"d2h {st['ms_d2h']:.1f}, oz_planes {st['oz_planes']}")
