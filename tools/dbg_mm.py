import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1804_00462_b200 as P
for (M, K, N, ta) in [(6000, 1100, 64, 0), (6000, 500, 64, 0), (1100, 6000, 64, 1), (6000, 1100, 24, 0),
                      (3000, 1100, 64, 0), (6000, 1100, 128, 0), (6000, 1100, 256, 0), (200000, 20000, 256, 0)]:
    g = torch.Generator(device="cuda"); g.manual_seed(M + K)
    a = torch.randn((K, M) if ta else (M, K), generator=g, device="cuda", dtype=torch.float64)
    b = torch.randn(K, N, generator=g, device="cuda", dtype=torch.float64)
    c = P.matmul(a, b, transpose_a=bool(ta))
    ref = (a.T if ta else a) @ b
    err = ((c - ref).abs().max() / ref.abs().max()).item()
    rows = ((c - ref).abs().amax(1) > 1e-10 * ref.abs().max()).nonzero().flatten()
    print(M, K, N, ta, "%.1e" % err, "bad rows", rows[:8].tolist(), len(rows), flush=True)
