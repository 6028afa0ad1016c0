"""One A-streaming pass (NN or TN) on a bench config's matrix, for ncu captures."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1804_00462_b200 as P
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--ta", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
dev = torch.device("cuda", 0)
A = bench.make_matrix(a.config, cfg["m"], cfg["n"], 0, 1, dev)
ell = cfg["k"]
f32 = cfg.get("dtype") == "f32"
tf32 = f32 and cfg.get("mode") == "tf32"  # FP32 A: TF32 tensor cores, else FP64 DMMA on the widened tile
if tf32:
    Np = ((ell + 31) // 32) * 32 if ell <= 256 else ((ell + 255) // 256) * 256
else:
    Np = (ell + 7) // 8 * 8 if ell <= 128 else (ell + 127) // 128 * 128
dt = torch.float32 if tf32 else torch.float64
X = torch.randn(cfg["m"] if a.ta else cfg["n"], Np, device=dev, dtype=dt)
T = torch.empty(cfg["n"] if a.ta else cfg["m"], Np, device=dev, dtype=dt)
ctx = P.default_context(0)
ms = ctypes.c_double(); l = ctypes.c_int32()
lib = P._capi.lib()
fn = lib.sorsvd_pass_f32_device if tf32 else (lib.sorsvd_pass_f32a_device if f32 else lib.sorsvd_pass_device)
P._check(fn(ctx.handle, a.ta, cfg["m"], cfg["n"], cfg["n"], ell, A.data_ptr(), X.data_ptr(), T.data_ptr(), a.reps,
            ctypes.byref(ms), ctypes.byref(l)), ctx.handle)
torch.cuda.synchronize()
print(f"{a.config} ta={a.ta} pass {ms.value:.4f} ms, launches/pass {l.value}")
