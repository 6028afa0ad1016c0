"""One C4 RPCA solve (after a warm-up) for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402

D, _, _ = O.gen_c4(4)
Dd = torch.from_numpy(D).cuda()
cfg = P.RpcaConfig(lam=1 / np.sqrt(25344), mu0=0.0, ell=10, q=1, seed=9, max_iter=100)
P.rpca_alm(Dd, cfg)
torch.cuda.synchronize()
r = P.rpca_alm(Dd, cfg)
torch.cuda.synchronize()
print(r.iterations)
