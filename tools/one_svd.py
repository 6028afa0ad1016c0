"""One core SVD at k (argv[1]) for ncu captures."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 512
rng = np.random.default_rng(k)
u0, _ = np.linalg.qr(rng.standard_normal((k, k)))
v0, _ = np.linalg.qr(rng.standard_normal((k, k)))
mm = torch.from_numpy((u0 / np.arange(1, k + 1)) @ v0.T).cuda()
print(P.full_svd(mm)[3])
torch.cuda.synchronize()
