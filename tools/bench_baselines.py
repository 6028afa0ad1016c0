"""Time the sketch.hpp baselines r_svd (:124) and tsr_svd (:139) on the C2
matrix (m = n = 4000, ell = 100, q = 1 for r_svd): device API with A resident
(CUDA events, L2 flushed between calls), the host-buffer API (e2e), and the
compiled reference on all host cores; parity of the leading sigmas against
the reference on the same matrix. One JSON line per method."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1804_00462_b200 as P  # noqa: E402

bench._prefer_avx512_blas()
from oracle import sorsvd_oracle as O  # noqa: E402

m = n = 4000
ell, q, seed = 100, 1, 21
dev = torch.device("cuda", 0)
A = bench.make_matrix("c2", m, n, 0, 1, dev)
Ah = A.cpu().numpy()
Ap = torch.from_numpy(Ah).pin_memory().numpy()
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
cores = os.cpu_count() or 1
O.Ref.set_threads(cores)


def run(kind, a, **kw):
    return P.r_svd(a, ell, q, seed, **kw) if kind == "rsvd" else P.tsr_svd(a, ell, seed, **kw)


for kind in ("rsvd", "tsr"):
    launched = 2 * q + 2 if kind == "rsvd" else 2  # sweeps over A actually issued
    for _ in range(3):
        run(kind, A)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        f = run(kind, A)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    te = []
    for _ in range(5):
        t0 = time.perf_counter()
        fh = run(kind, Ap)
        te.append((time.perf_counter() - t0) * 1e3)
    tc = []
    for i in range(3):
        t0 = time.perf_counter()
        r = O.Ref.r_svd(Ah, ell, q, seed) if kind == "rsvd" else O.Ref.tsr_svd(Ah, ell, seed)
        tc.append((time.perf_counter() - t0) * 1e3)
    es = O.sigma_rel_err(f.sigma.cpu().numpy(), r.sigma)
    flops = 2.0 * m * n * ell * launched
    print(json.dumps({
        "method": kind, "workload": f"C2 matrix m=n={m}, ell={ell}" + (f", q={q}" if kind == "rsvd" else ""),
        "passes_reference": int(f.passes), "sweeps_launched": launched,
        "ms_per_call": ms, "gflops": flops / (ms * 1e-3) / 1e9,
        "e2e_ms": float(np.median(te)), "cpu_ref_ms": float(np.median(tc)), "cpu_cores": cores,
        "speedup_e2e_vs_cpu": float(np.median(tc) / np.median(te)),
        "sigma_rel_err_leading40_vs_ref": float(es[:40].max()), "sigma_rel_err_all_vs_ref": float(es.max()),
        "note": "C2's tail sigmas (j^-2 spectrum, q = 1) are rounding-defined for every implementation",
    }), flush=True)
