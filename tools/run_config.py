"""Run one call of a BASELINE config after a warm-up call (the target of the ncu
launch lists and kernel captures in tools/ncu_*.sh).

  python tools/run_config.py c2      # sor_svd_power on the C2 matrix (graph off: one launch per kernel)
  python tools/run_config.py c4      # one RPCA solve on the C4 matrix
  python tools/run_config.py c3      # sor_svd_power on bench.py's C3 matrix
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402


def main(cfg: str) -> None:
    if cfg == "c2":
        A = torch.from_numpy(O.gen_c2(2)).cuda()
        for _ in range(2):
            f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 21), use_graph=False)
        torch.cuda.synchronize()
        print(f.sigma[:3])
    elif cfg == "c4":
        D, _, _ = O.gen_c4(4)
        Dd = torch.from_numpy(D).cuda()
        rc = P.RpcaConfig(lam=1 / np.sqrt(25344), mu0=0.0, ell=10, q=1, seed=9, max_iter=100)
        for _ in range(2):
            r = P.rpca_alm(Dd, rc)
        torch.cuda.synchronize()
        print(r.iterations)
    elif cfg == "c3":  # bench.py's own C3 instance (device-generated)
        import bench
        c = bench.CONFIGS["c3"]
        A = bench.make_matrix("c3", c["m"], c["n"], 0, 1, torch.device("cuda", 0))
        om = torch.from_numpy(P.gaussian_matrix(c["n"], c["k"], 7)).cuda()
        for _ in range(2):
            f = P.sor_svd_power(A, c["k"], P.SketchConfig(c["k"], c["q"], 7), omega=om, use_graph=False)
        torch.cuda.synchronize()
        print(f.sigma[:3], f.stats)
    else:
        raise SystemExit(f"unknown config {cfg!r}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2")
