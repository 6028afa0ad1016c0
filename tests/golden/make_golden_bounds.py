"""Golden vectors for the bound harness (bounds.hpp) from the COMPILED REFERENCE
(oracle/_ref/libsorsvd_ref.so = the unmodified /root/reference headers).

    python tests/golden/make_golden_bounds.py     # needs /root/reference at build time only

Writes tests/golden/golden_bounds.npz: the formula evaluators (bounds.hpp:94-222) on
seeded spectra, omega_split (bounds.hpp:50-71) on a seeded basis, and two
bound_tightness_experiment runs (bounds.hpp:265-379) on a 120 x 80 matrix."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import sorsvd_oracle as O  # noqa: E402

Ref = O.Ref
OUT = os.path.dirname(os.path.abspath(__file__))

FORMULA_CASES = [  # (spectrum family, n, k, ell, p, q, ||Omega_2||, ||Omega_1^+||)
    ("poly1", 200, 10, 20, 5, 1, 30.0, 0.5), ("poly1", 200, 10, 20, 2, 0, 31.5, 0.21), ("poly2", 100, 5, 12, 4, 2, 12.0, 0.9),
    ("geo", 64, 8, 16, 8, 0, 9.0, 1.7), ("geo", 64, 3, 5, 2, 3, 7.5, 3.0), ("poly1", 30, 20, 30, 10, 1, 2.0, 0.4),
    ("lowrank", 50, 4, 10, 3, 1, 11.0, 0.6), ("poly1", 1000, 20, 38, 18, 2, 33.0, 0.8), ("poly1", 1000, 20, 38, 1, 0, 35.0, 0.3),
]


def spectrum(fam, n):
    j = np.arange(1, n + 1, dtype=np.float64)
    if fam == "poly1":
        return 1.0 / j
    if fam == "poly2":
        return 3.0 / j**2
    if fam == "geo":
        return 2.0 ** (-(j - 1) / 4.0)
    s = np.zeros(n)
    s[:6] = [5, 4, 3, 2, 1, 0.5]
    return s


def experiment_matrix():
    """120 x 80, singular values 1/j (j <= 80) on seeded orthonormal factors."""
    u, _ = np.linalg.qr(O.gaussian_matrix(120, 80, 901))
    v, _ = np.linalg.qr(O.gaussian_matrix(80, 80, 902))
    return (u * (1.0 / np.arange(1, 81))) @ v.T


def main():
    Ref.set_threads(1)
    g = {}
    for i, (fam, n, k, ell, p, q, n2, n1p) in enumerate(FORMULA_CASES):
        r = Ref.bound_formulas(spectrum(fam, n), k, ell, p, q, n2, n1p)
        g[f"f{i}_det_sv"], g[f"f{i}_avg_sv"] = r["det_sv"], r["avg_sv"]
        g[f"f{i}_scal"] = np.array([r["det_f"], r["det_2"], r["avg_f"], r["avg_2"], r["best_f"], r["best_2"]])
    a = experiment_matrix()
    g["exp_A"] = a
    _, s, v = Ref.full_svd(a)
    g["exp_sigma"], g["exp_V"] = s, v
    om = O.gaussian_matrix(80, 12, 77)
    g["split_norms"] = np.array(Ref.omega_split(v, om, 6, 12, 3, 1), dtype=np.float64)
    for name, (q, kind, trials, seed) in {"expdet": (1, 0, 6, 4100), "expavg": (0, 1, 8, 4200)}.items():
        r = Ref.bound_experiment(a, 6, 12, 3, q, trials, seed, kind)
        for key in ("sv_lower_bounds", "realized_sigmas", "bound_satisfied", "trial_vals", "trial_flags"):
            g[f"{name}_{key}"] = np.asarray(r[key])
        g[f"{name}_scal"] = np.array([r["lowrank_bound_frobenius"], r["lowrank_bound_spectral"],
                                      r["realized_error_frobenius"], r["realized_error_spectral"]])
        with open(os.path.join(OUT, f"golden_bounds_{name}.csv"), "w") as fh:
            fh.write(r["csv"])
    np.savez_compressed(os.path.join(OUT, "golden_bounds.npz"), **g)
    with open(os.path.join(OUT, "golden_bounds_meta.json"), "w") as fh:
        json.dump({"formula_cases": FORMULA_CASES, "experiment": {"m": 120, "n": 80, "k": 6, "ell": 12, "p": 3,
                   "expdet": {"q": 1, "kind": "deterministic", "trials": 6, "seed": 4100},
                   "expavg": {"q": 0, "kind": "average", "trials": 8, "seed": 4200}},
                   "split": {"n": 80, "ell": 12, "p": 3, "k": 6, "q": 1, "omega_seed": 77}}, fh, indent=1)
    print("wrote golden_bounds.npz", {k: v.shape for k, v in g.items() if k.startswith("exp")})


if __name__ == "__main__":
    main()
