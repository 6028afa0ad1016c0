"""Stress the emulated world-G sharded schedule: run the same problem N times
and report which ranks' replicated outputs (sigma, V) differ from rank 0."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402

world, m, n, k, q = 8, 8000, 400, 10, 1
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
A = O.gen_lowrank_decay(m, n, 40, lambda j: 2.0 ** (-j / 4), 1e-3, m + world)
blocks = np.array_split(np.arange(m), world)
bad = 0
for rep in range(reps):
    g = P.EmuGroup(world)
    ctxs = [P.Context(0, rank=r, emu_group=g) for r in range(world)]
    out = [None] * world

    def work(r):
        blk = torch.from_numpy(np.ascontiguousarray(A[blocks[r][0]:blocks[r][-1] + 1])).cuda()
        out[r] = P.sor_svd_power(blk, k, P.SketchConfig(k, q, 11), ctx=ctxs[r], m_global=m)
        torch.cuda.synchronize()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    s0, v0 = out[0].sigma.cpu().numpy(), out[0].v.cpu().numpy()
    diffs = [(r, float(np.abs(out[r].sigma.cpu().numpy() - s0).max()), float(np.abs(out[r].v.cpu().numpy() - v0).max()))
             for r in range(1, world)]
    d = [x for x in diffs if x[1] or x[2]]
    if d:
        bad += 1
        print("rep", rep, "differs:", d, flush=True)
    [c.close() for c in ctxs]
    g.close()
print("bad", bad, "of", reps, {k_: v_ for k_, v_ in os.environ.items() if k_.startswith("SORSVD")})
