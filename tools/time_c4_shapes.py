"""Per-shape device time of the C4 skinny GEMMs (W 25344x300, ell = 10 padded to 16):
the NN pass W*X, the TN pass W^T*T and the CholeskyQR Gram T^T*T. L2 flushed before each call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_00462_b200 as P

torch.manual_seed(0)
W = torch.randn(25344, 300, dtype=torch.float64, device="cuda")
X = torch.randn(300, 10, dtype=torch.float64, device="cuda")
T = torch.randn(25344, 10, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cases = {"NN W*X": lambda: P.matmul(W, X), "TN W^T*T": lambda: P.matmul(W, T, transpose_a=True),
         "Gram T^T*T": lambda: P.matmul(T, T, transpose_a=True)}
for name, f in cases.items():
    for _ in range(3):
        f()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort()
    print(f"{name}: median {ts[len(ts)//2]:.1f} us, min {ts[0]:.1f} us")
