#!/bin/bash
# ncu --set full of the non-pass kernels that dominate the calls (one launch each):
# the C2 Householder QR, the k = 100 p2p Jacobi ring, the C4 RPCA update, approx_error.
set -u
mkdir -p gpurun_out
cap() {  # regex tag cmd...
  local re=$1 tag=$2; shift 2
  ncu -f --set full --clock-control none -k regex:"$re" -c 1 -o /tmp/k_$tag "$@" > gpurun_out/ncuk_$tag.log 2>&1
  echo "$tag rc=$?"
  ncu -i /tmp/k_$tag.ncu-rep --page raw --csv > gpurun_out/ncuk_${tag}_raw.csv 2>/dev/null
}
cap cqr_kernel cqr python tools/time_qr.py 4000 100
cap jacobi_p2p jac100 python tools/time_jacobi.py 100
cap rpca_update rpca python tools/run_config.py c4
cap approx_err aerr python -c "
import sys; sys.path.insert(0, '.')
import torch, bench, paper_1804_00462_b200 as P
A = bench.make_matrix('c2', 4000, 4000, 0, 1, torch.device('cuda', 0))
f = P.sor_svd_power(A, 100, P.SketchConfig(100, 1, 3))
print(P.approx_error(A, f))"
