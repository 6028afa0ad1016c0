"""TEST INFRASTRUCTURE — CPU oracles for parity tests (see sorsvd_oracle.py).
Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference leg. The CUDA product never imports this package."""
