timeout 600 python tools/oz_check.py > gpurun_out/oz_check.txt 2>&1
python tools/oz_pass.py 200000 20000 256 0 3 > gpurun_out/oz_dbg.txt 2>&1
python tools/oz_pass.py 200000 20000 256 1 3 >> gpurun_out/oz_dbg.txt 2>&1
python - >> gpurun_out/oz_dbg.txt 2>&1 <<'PY'
import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import bench, paper_1804_00462_b200 as P
cfg = bench.CONFIGS["c3"]
A = bench.make_matrix("c3", cfg["m"], cfg["n"], 0, 1, torch.device("cuda", 0))
om = torch.from_numpy(P.gaussian_matrix(cfg["n"], 256, 7)).cuda()
for mode in ("dmma", "ozaki", "ozaki"):
    f = P.sor_svd_power(A, 256, P.SketchConfig(256, 1, 7), omega=om, fp64_mode=mode, stage_times=True)
    print(mode, json.dumps({k: round(v, 3) for k, v in f.stats.items() if k.startswith("ms")}))
for mode in ("dmma", "ozaki"):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    P.sor_svd_power(A, 256, P.SketchConfig(256, 1, 7), omega=om, fp64_mode=mode)
    ev[0].record()
    for _ in range(3):
        f = P.sor_svd_power(A, 256, P.SketchConfig(256, 1, 7), omega=om, fp64_mode=mode)
    ev[1].record(); torch.cuda.synchronize()
    print(mode, "graphed call ms", ev[0].elapsed_time(ev[1]) / 3, f.sigma[:3].tolist())
PY
