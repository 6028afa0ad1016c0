"""Concurrent thin_qr on identical inputs from several host threads / contexts:
every result must be bit-identical (determinism under concurrency)."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402

nth = 8
ctxs = [P.Context(0) for _ in range(nth)]
for (m, k, cond) in [(400, 10, 3), (1000, 10, 3), (80, 10, 3), (400, 10, 12)]:
    u, _ = np.linalg.qr(O.gaussian_matrix(m, k, 5))
    v, _ = np.linalg.qr(O.gaussian_matrix(k, k, 6))
    T = torch.from_numpy((u * np.logspace(0, -cond, k)) @ v.T).cuda()
    bad = 0
    for rep in range(30):
        out = [None] * nth

        def work(r):
            out[r] = P.thin_qr(T.clone(), ctx=ctxs[r])
            torch.cuda.synchronize()

        th = [threading.Thread(target=work, args=(r,)) for r in range(nth)]
        [t.start() for t in th]
        [t.join() for t in th]
        q0 = out[0][0].cpu().numpy()
        d = [r for r in range(1, nth) if not np.array_equal(out[r][0].cpu().numpy(), q0)]
        if d:
            bad += 1
    print(f"thin_qr m={m} k={k} cond=1e{cond}: {bad} of 30 reps had differing Q", flush=True)
