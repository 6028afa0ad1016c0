import sys, os, time
sys.path.insert(0, '/root/repo')
import torch, bench, paper_1804_00462_b200 as P
A = bench.make_matrix("c2", 4000, 4000, 0, 1, torch.device("cuda", 0))
for kind in ("rsvd", "tsr", "sor"):
    for g in (True, False):
        for i in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            if kind == "rsvd": f = P.r_svd(A, 100, 1, 21, use_graph=g)
            elif kind == "tsr": f = P.tsr_svd(A, 100, 21, use_graph=g)
            else: f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 21), use_graph=g)
            torch.cuda.synchronize(); t1 = time.perf_counter()
        print(kind, "graph" if g else "nograph", "wall %.3f ms" % ((t1 - t0) * 1e3), "ms_total %.3f" % f.stats["ms_total"], "sweeps", f.stats["jacobi_sweeps"], "launches", f.stats["launches"])
