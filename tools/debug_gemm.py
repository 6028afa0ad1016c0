import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
rng = np.random.default_rng(0)
A = rng.standard_normal((2000, 3000))
X = rng.standard_normal((3000, 100))
ext = (A.astype(np.longdouble) @ X.astype(np.longdouble))
npr = A @ X
g = P.matmul(torch.from_numpy(A).cuda(), torch.from_numpy(X).cuda()).cpu().numpy()
tc = (torch.from_numpy(A).cuda() @ torch.from_numpy(X).cuda()).cpu().numpy()
scale = np.abs(ext).mean()
for nm, c in (("numpy", npr), ("gpu-dmma", g), ("torch-cublas", tc)):
    e = (c.astype(np.longdouble) - ext).astype(np.float64)
    print(nm, "mean abs err/scale", np.abs(e).mean()/scale, "max", np.abs(e).max()/scale, "mean signed", e.mean()/scale)
# transposed
ext = (A.T.astype(np.longdouble) @ rng.standard_normal((2000,100)).astype(np.longdouble))
