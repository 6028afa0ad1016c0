"""One C2 sor_svd_power call (graph disabled) for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402

A = torch.from_numpy(O.gen_c2(2)).cuda()
f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 21), use_graph=False)
f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 21), use_graph=False)
torch.cuda.synchronize()
print(f.sigma[:3])
