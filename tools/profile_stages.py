"""Per-stage device times of one sor_svd_power call (STAGE_TIMES flag) for a
bench config; also usable under ncu for a launch list."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1804_00462_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--graph", action="store_true")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda", 0)
A = bench.make_matrix(args.config, cfg["m"], cfg["n"], 0, 1, dev)
om = torch.from_numpy(P.gaussian_matrix(cfg["n"], cfg["k"], 7)).to(dev)
sc = P.SketchConfig(cfg["k"], cfg["q"], 7)
for r in range(args.reps):
    f = P.sor_svd_power(A, cfg["k"], sc, omega=om, stage_times=not args.graph)
    torch.cuda.synchronize()
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in f.stats.items()}))
