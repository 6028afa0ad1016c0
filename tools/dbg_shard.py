import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_multirank import _run_sharded
for (world, m, n, k, q) in [(4, 6000, 1100, 64, 1), (4, 6000, 1100, 64, 0), (2, 6000, 1100, 64, 1), (4, 6000, 500, 64, 1)]:
    A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + world + 1)
    base = O.sor_svd_power(A, k, O.SketchConfig(k, q, 13))
    res = {}
    for mode in ("dmma", "ozaki"):
        out, u = _run_sharded(P, torch, A, k, P.SketchConfig(k, q, 13), world, fp64_mode=mode)
        res[mode] = O.sigma_rel_err(out[0].sigma.cpu().numpy(), base.sigma).max()
    single = P.sor_svd_power(A, k, P.SketchConfig(k, q, 13), fp64_mode="ozaki")
    res["single_ozaki"] = O.sigma_rel_err(single.sigma, base.sigma).max()
    print(world, m, n, k, q, {a: "%.1e" % b for a, b in res.items()}, flush=True)
