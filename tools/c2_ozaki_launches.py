"""C2 with the Ozaki engine forced (un-graphed, two calls) for an ncu launch list: where the time goes below the crossover."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00462_b200 as P
from oracle import sorsvd_oracle as O
A = torch.from_numpy(O.gen_c2(2)).cuda()
for _ in range(2):
    f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 21), use_graph=False, fp64_mode=sys.argv[1] if len(sys.argv) > 1 else "ozaki")
torch.cuda.synchronize()
print(f.sigma[:3], f.stats["pass_kind"], f.stats["oz_planes"])
