"""Where the Ozaki (int8 digit planes) engine starts to beat the FP64 DMMA passes: graphed sor_svd_power
call time in both modes over a size sweep (q = 1, device-resident A, Omega given)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00462_b200 as P

torch.manual_seed(0)
for m, n, ell in [(4000, 4000, 100), (6000, 6000, 100), (8000, 8000, 128), (10000, 10000, 128), (16000, 8000, 64),
                  (12000, 12000, 256), (30000, 3000, 200), (20000, 20000, 64), (50000, 10000, 32)]:
    A = torch.randn(m, 40, dtype=torch.float64, device="cuda") @ torch.randn(40, n, dtype=torch.float64, device="cuda")
    A += 1e-3 * torch.randn(m, n, dtype=torch.float64, device="cuda")
    om = torch.from_numpy(P.gaussian_matrix(n, ell, 7)).cuda()
    sc = P.SketchConfig(ell, 1, 7)
    res = {"m": m, "n": n, "ell": ell, "log2_mnl": round(float(torch.log2(torch.tensor(float(m) * n * ell))), 2)}
    for mode in ("dmma", "ozaki"):
        for _ in range(2):
            P.sor_svd_power(A, ell, sc, omega=om, fp64_mode=mode)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f = P.sor_svd_power(A, ell, sc, omega=om, fp64_mode=mode)
        e1.record()
        torch.cuda.synchronize()
        res[mode + "_ms"] = round(e0.elapsed_time(e1) / 5, 3)
    res["ozaki_over_dmma"] = round(res["ozaki_ms"] / res["dmma_ms"], 3)
    print(json.dumps(res), flush=True)
    del A
    torch.cuda.empty_cache()
