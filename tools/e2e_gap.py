"""Where the host-API (e2e) time goes beyond H2D + device + D2H on C2: the Python
wrapper vs the C call itself, and the host-drawn Omega vs a given one."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_00462_b200 as P  # noqa: E402
from paper_1804_00462_b200 import _capi as C  # noqa: E402
from oracle import sorsvd_oracle as O  # noqa: E402

A = O.gen_c2(2)
pin = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
pin.copy_(torch.from_numpy(A))
a_np = pin.numpy()
m, n, k = 4000, 4000, 100
cfg = P.SketchConfig(100, 1, 21)
ctx = P.default_context(0)
u = torch.empty((m, k), dtype=torch.float64, pin_memory=True).numpy()
s = torch.empty((k,), dtype=torch.float64, pin_memory=True).numpy()
v = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
om = P.gaussian_matrix(n, 100, 21)
om_pin = torch.empty(om.shape, dtype=torch.float64, pin_memory=True).numpy()
om_pin[:] = om


def direct(omega=None):
    d = P._desc(m, n, n, k, cfg, C.FLAG_OMEGA_GIVEN if omega is not None else 0)
    st = C.SorsvdStats()
    rc = C.lib().sorsvd_sor_svd_power(ctx.handle, ctypes.byref(d), a_np.ctypes.data_as(ctypes.c_void_p),
                                      omega.ctypes.data_as(C.c_dp) if omega is not None else None,
                                      u.ctypes.data_as(C.c_dp), s.ctypes.data_as(C.c_dp), v.ctypes.data_as(C.c_dp),
                                      ctypes.byref(st))
    assert rc == 0
    return st


for name, fn in (("python api", lambda: P.sor_svd_power(a_np, k, cfg).stats),
                 ("direct C, drawn omega", lambda: direct()),
                 ("direct C, given pageable omega", lambda: direct(om)),
                 ("direct C, given pinned omega", lambda: direct(om_pin))):
    for _ in range(3):
        fn()
    ws = []
    for _ in range(10):
        t0 = time.perf_counter()
        st = fn()
        ws.append((time.perf_counter() - t0) * 1e3)
    st = st if isinstance(st, dict) else {f: getattr(st, f) for f, _ in st._fields_}
    print(f"{name:32s} wall {np.median(ws):.3f} ms  h2d {st['ms_h2d']:.3f} device {st['ms_total']:.3f} d2h {st['ms_d2h']:.3f}",
          flush=True)
