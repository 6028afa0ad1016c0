"""Graphed sor_svd_power call time per config in fp64_mode dmma vs ozaki (device-resident A, Omega given)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1804_00462_b200 as P
cfgs = sys.argv[1:] or ["c1", "c2", "c3", "c5"]
for name in cfgs:
    cfg = bench.CONFIGS[name]
    A = bench.make_matrix(name, cfg["m"], cfg["n"], 0, 1, torch.device("cuda", 0))
    om = torch.from_numpy(P.gaussian_matrix(cfg["n"], cfg["k"], 7)).cuda()
    sc = P.SketchConfig(cfg["k"], cfg["q"], 7)
    res = {"config": name}
    sig = {}
    for mode in ("dmma", "ozaki"):
        P.sor_svd_power(A, cfg["k"], sc, omega=om, fp64_mode=mode)
        reps = 3 if name in ("c3", "c5") else 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            f = P.sor_svd_power(A, cfg["k"], sc, omega=om, fp64_mode=mode)
        e1.record()
        torch.cuda.synchronize()
        res[mode + "_ms"] = round(e0.elapsed_time(e1) / reps, 4)
        sig[mode] = f.sigma.cpu()
        st = P.sor_svd_power(A, cfg["k"], sc, omega=om, fp64_mode=mode, stage_times=True).stats
        res[mode + "_stages"] = {k: round(v, 3) for k, v in st.items() if k.startswith("ms_") and v}
    res["sigma_maxrel_dmma_vs_ozaki"] = float(((sig["dmma"] - sig["ozaki"]).abs() / sig["dmma"].abs()).max())
    print(json.dumps(res), flush=True)
    del A
    torch.cuda.empty_cache()
