"""Host-buffer API (e2e path) breakdown for C2: H2D / device / D2H per call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402

A = O.gen_c2(2)
pin = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
pin.copy_(torch.from_numpy(A))
a_np = pin.numpy()
cfg = P.SketchConfig(100, 1, 21)
for _ in range(3):
    P.sor_svd_power(a_np, 100, cfg)
for _ in range(5):
    t0 = time.perf_counter()
    f = P.sor_svd_power(a_np, 100, cfg)
    wall = (time.perf_counter() - t0) * 1e3
    st = f.stats
    print(f"wall {wall:.3f} ms  h2d {st['ms_h2d']:.3f}  device {st['ms_total']:.3f}  d2h {st['ms_d2h']:.3f}  "
          f"h2d GB/s {A.nbytes / st['ms_h2d'] / 1e6:.1f}")
