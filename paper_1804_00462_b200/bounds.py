"""The bound-verification harness of the reference (bounds.hpp) over the GPU hot path.

Same names and semantics as ``/root/reference/proj/include/sorsvd/bounds.hpp``:
``BoundParams`` (:20-33), ``OmegaSplit`` / ``omega_split`` (:38-71), the
evaluators ``det_sv_lower_bound`` (:94-115), ``det_lowrank_bound`` (:121-150),
``avg_nu1`` / ``avg_nu2`` (:154-162), ``avg_sv_lower_bound`` (:168-188),
``avg_lowrank_bound`` (:192-209), ``avg_lowrank_bound_best_p`` (:212-222),
``BoundTrial`` / ``BoundReport`` (:227-256), ``bound_tightness_experiment``
(:265-379) and ``bound_report_csv`` (:383-404).

What runs where:
  * the Monte-Carlo loop's ``sor_svd_power`` calls (bounds.hpp:288) run as
    batched trials on the device (every pass over A serves a whole batch of
    trials: ``sor_svd_power_batch``);
  * ``approx_error`` in both norms (bounds.hpp:289-290) runs on the device
    (fused Frobenius pass; spectral: the difference formed on the device and
    its sigma_1 from the Gram / Rayleigh-Ritz estimate);
  * ``omega_split``'s two projections V_1^T Omega, V_2^T Omega are device
    GEMMs, sigma(Omega_1) the device Jacobi SVD, ||Omega_2||_2 the device
    spectral norm;
  * the reference SVD of A (bounds.hpp:274, "analysis-side oracle") is thin QR
    + Jacobi SVD of R on the device for n <= 512; for wider matrices the
    caller passes (sigma, V) -- for the generated test families they are known
    by construction;
  * the bound formulas are scalar arithmetic on the host, as in the reference.
No CPU fallback: without the CUDA library every device step raises.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import (ParameterError, ShapeError, SketchConfig, approx_error, full_svd, gaussian_matrix, matmul, norm,
               sor_svd_power_batch, thin_qr)

DBL_EPSILON = float(np.finfo(np.float64).eps)


class BoundInapplicableError(ArithmeticError):
    """errors.hpp: bound_inapplicable_error (Omega_1 not of full row rank)."""


@dataclass
class BoundParams:
    """bounds.hpp:20-33. Requires 2 <= p + k <= ell; the average-case bounds need p >= 2."""
    k: int = 0
    ell: int = 0
    p: int = 0
    q: int = 0

    def validate(self) -> None:
        if self.k < 1:
            raise ParameterError("bound params: k must be positive")
        if self.q < 0:
            raise ParameterError("bound params: q must be nonnegative")
        if self.p < 0:
            raise ParameterError("bound params: p must be nonnegative")
        if self.p + self.k < 2 or self.p + self.k > self.ell:
            raise ParameterError("bound params: need 2 <= p + k <= ell")


@dataclass
class OmegaSplit:
    """bounds.hpp:38-44 (omega1 / omega2 stay on the device)."""
    omega1: object
    omega2: object
    norm_omega2: float
    norm_omega1_pinv: float
    full_row_rank: bool


def _sigma_at(sigma: Sequence[float], index1: int) -> float:  # bounds.hpp:85-88
    return float(sigma[index1 - 1]) if index1 <= len(sigma) else 0.0


def _tail_norm(sigma: Sequence[float], k: int, kind: str) -> float:  # bounds.hpp:75-83
    if k >= len(sigma):
        return 0.0
    if kind == "spectral":
        return float(sigma[k])
    return math.sqrt(float(np.sum(np.asarray(sigma[k:], dtype=np.longdouble) ** 2)))


def _check_kind(kind: str, who: str) -> None:
    if kind not in ("frobenius", "spectral"):
        raise ParameterError(f"{who} supports frobenius and spectral norms")


def singular_values_wide(mat, ctx=None):
    """dense.hpp singular_values of an r x c device matrix with r <= c <= 512:
    the Jacobi SVD of the matrix padded with zero rows to c x c (its spectrum
    plus c - r zeros); returns the leading r values on the host."""
    import torch
    r, c = mat.shape
    if r > c:
        raise ShapeError("singular_values_wide expects rows <= cols")
    sq = torch.zeros((c, c), dtype=torch.float64, device=mat.device)
    sq[:r] = mat
    _, s, _, _ = full_svd(sq, ctx=ctx)
    return s[:r].cpu().numpy()


def omega_split(v, omega, params: BoundParams, ctx=None) -> OmegaSplit:
    """bounds.hpp:50-71: Omega_1 = V_1^T Omega ((ell-p) x ell), Omega_2 = V_2^T Omega,
    V_1 the first ell-p columns of the n x n right singular basis (device tensors)."""
    import torch
    params.validate()
    n = v.shape[0]
    if v.shape[1] != n:
        raise ShapeError("omega_split expects a full n x n singular basis")
    if omega.shape[0] != n or omega.shape[1] != params.ell:
        raise ShapeError("omega_split: test matrix must be n x ell")
    lead = params.ell - params.p
    if lead > n:
        raise ParameterError("omega_split: ell - p exceeds n")
    v = torch.as_tensor(v, dtype=torch.float64, device="cuda") if not hasattr(v, "is_cuda") or not v.is_cuda else v
    omega = torch.as_tensor(omega, dtype=torch.float64, device=v.device)
    omega1 = matmul(v[:, :lead].contiguous(), omega, transpose_a=True, ctx=ctx)
    if n > lead:
        omega2 = matmul(v[:, lead:].contiguous(), omega, transpose_a=True, ctx=ctx)
        n2 = norm(omega2, "spectral", ctx=ctx)
    else:
        omega2 = torch.zeros((0, params.ell), dtype=torch.float64, device=v.device)
        n2 = 0.0
    s1 = singular_values_wide(omega1, ctx=ctx)
    smax = float(s1[0]) if len(s1) else 0.0
    smin = float(s1[-1]) if len(s1) else 0.0
    frr = smin > n * DBL_EPSILON * smax
    return OmegaSplit(omega1, omega2, n2, 1.0 / smin if frr else math.inf, frr)


def det_sv_lower_bound(sigma, params: BoundParams, split: OmegaSplit) -> List[float]:
    """bounds.hpp:94-115: sigma_j / sqrt(1 + Phi (sigma_{ell-p+1}/sigma_j)^(4q+4)), j = 1..k."""
    params.validate()
    if not split.full_row_rank:
        raise BoundInapplicableError("Omega_1 is not full row rank")
    phi = split.norm_omega2 * split.norm_omega2 * split.norm_omega1_pinv * split.norm_omega1_pinv
    s_tail = _sigma_at(sigma, params.ell - params.p + 1)
    expo = 4.0 * params.q + 4.0
    out = []
    for j in range(1, params.k + 1):
        sj = _sigma_at(sigma, j)
        if sj <= 0.0:
            out.append(0.0)
            continue
        gamma = s_tail / sj
        out.append(sj / math.sqrt(1.0 + phi * math.pow(gamma, expo)))
    return out


def det_lowrank_bound(sigma, params: BoundParams, split: OmegaSplit, kind: str) -> float:
    """bounds.hpp:121-150 (Theorem 5's alpha / beta / eta / tau form)."""
    params.validate()
    _check_kind(kind, "det_lowrank_bound")
    if not split.full_row_rank:
        raise BoundInapplicableError("Omega_1 is not full row rank")
    a0 = _tail_norm(sigma, params.k, kind)
    s1 = _sigma_at(sigma, 1)
    sk = _sigma_at(sigma, params.k)
    st = _sigma_at(sigma, params.ell - params.p + 1)
    if st <= 0.0 or s1 <= 0.0:
        return a0
    phi = split.norm_omega2 * split.norm_omega2 * split.norm_omega1_pinv * split.norm_omega1_pinv
    rootk = math.sqrt(float(params.k))
    if params.q == 0:
        alpha = rootk * st * st / sk
        beta = st * st / (s1 * sk)
        eta = rootk * st
        tau = st / s1
    else:
        g = math.pow(st / sk, 2.0 * params.q)
        alpha = rootk * (st * st / sk) * g
        beta = (st * st / (s1 * sk)) * g
        eta = (sk / st) * alpha
        tau = (1.0 / st) * beta
    return a0 + math.sqrt(alpha * alpha * phi / (1.0 + beta * beta * phi)) + \
        math.sqrt(eta * eta * phi / (1.0 + tau * tau * phi))


def avg_nu1(n: int, ell: int, p: int) -> float:  # bounds.hpp:154-156
    return math.sqrt(float(n) - ell + p) + math.sqrt(float(ell)) + 7.0


def avg_nu2(ell: int, p: int) -> float:  # bounds.hpp:160-162
    return 4.0 * math.e * math.sqrt(float(ell)) / float(p + 1)


def avg_sv_lower_bound(sigma, params: BoundParams) -> List[float]:
    """bounds.hpp:168-188 (the spectrum length is the ambient column dimension n)."""
    params.validate()
    if params.p < 2:
        raise ParameterError("average-case bounds need p >= 2")
    n = len(sigma)
    nu = avg_nu1(n, params.ell, params.p) * avg_nu2(params.ell, params.p)
    st = _sigma_at(sigma, params.ell - params.p + 1)
    expo = 4.0 * params.q + 4.0
    out = []
    for j in range(1, params.k + 1):
        sj = _sigma_at(sigma, j)
        if sj <= 0.0:
            out.append(0.0)
            continue
        gamma = st / sj
        out.append(sj / math.sqrt(1.0 + nu * nu * math.pow(gamma, expo)))
    return out


def avg_lowrank_bound(sigma, params: BoundParams, kind: str) -> float:
    """bounds.hpp:192-209."""
    params.validate()
    if params.p < 2:
        raise ParameterError("average-case bounds need p >= 2")
    _check_kind(kind, "avg_lowrank_bound")
    a0 = _tail_norm(sigma, params.k, kind)
    sk = _sigma_at(sigma, params.k)
    st = _sigma_at(sigma, params.ell - params.p + 1)
    if st <= 0.0 or sk <= 0.0:
        return a0
    n = len(sigma)
    nu = avg_nu1(n, params.ell, params.p) * avg_nu2(params.ell, params.p)
    gamma_k = st / sk
    extra = (1.0 + gamma_k) * math.sqrt(float(params.k)) * nu * st
    if params.q > 0:
        extra *= math.pow(gamma_k, 2.0 * params.q)
    return a0 + extra


def avg_lowrank_bound_best_p(sigma, k: int, ell: int, q: int, kind: str) -> float:
    """bounds.hpp:212-222: the tightest admissible bound over p in {2, ..., ell-k}."""
    best = math.inf
    p = 2
    while p + k <= ell:
        best = min(best, avg_lowrank_bound(sigma, BoundParams(k, ell, p, q), kind))
        p += 1
    if not math.isfinite(best):
        raise ParameterError("no admissible p in {2, ..., ell-k}")
    return best


@dataclass
class BoundTrial:
    """bounds.hpp:227-238."""
    trial: int
    seed: int
    err_f: float = 0.0
    err_2: float = 0.0
    bound_f: float = 0.0
    bound_2: float = 0.0
    satisfied_f: bool = False
    satisfied_2: bool = False
    full_row_rank: bool = False
    sigma_hat: List[float] = field(default_factory=list)
    sv_lower: List[float] = field(default_factory=list)
    sv_satisfied: bool = False


@dataclass
class BoundReport:
    """bounds.hpp:245-256. bound_satisfied: [0, k) singular values, [k] Frobenius, [k+1] spectral."""
    kind: str
    trials: int
    sv_lower_bounds: List[float] = field(default_factory=list)
    lowrank_bound_frobenius: float = 0.0
    lowrank_bound_spectral: float = 0.0
    realized_error_frobenius: float = 0.0
    realized_error_spectral: float = 0.0
    realized_sigmas: List[float] = field(default_factory=list)
    bound_satisfied: List[bool] = field(default_factory=list)
    records: List[BoundTrial] = field(default_factory=list)


def reference_svd(a, ctx=None):
    """The analysis-side SVD of a (bounds.hpp:274) for rows >= cols, cols <= 512:
    a = Q R (device TSQR / CholeskyQR), R = U_r diag(sigma) V^T (device Jacobi).
    Returns (sigma as a host array of length n, V as an n x n device tensor)."""
    m, n = a.shape
    if m < n:
        raise ParameterError("bound analysis assumes rows >= cols")
    if n > 512:
        raise ParameterError("reference_svd: n > 512 needs (sigma, v) passed in (ref_svd=...)")
    _, r = thin_qr(a.double().contiguous(), ctx=ctx)
    _, s, v, _ = full_svd(r, ctx=ctx)
    return s.cpu().numpy(), v


def bound_tightness_experiment(a, k: int, params: BoundParams, trials: int, seed: int,
                               kind: str = "deterministic", ref_svd=None, ctx=None,
                               batch: int = 8) -> BoundReport:
    """bounds.hpp:265-379. a: CUDA float64 (or host) matrix with rows >= cols.
    ref_svd = (sigma[n], V[n x n]) of a when known (required for cols > 512)."""
    import torch
    params.validate()
    if k != params.k:
        raise ParameterError("bound_tightness_experiment: k differs from params.k")
    if trials < 1:
        raise ParameterError("bound_tightness_experiment needs trials >= 1")
    if kind not in ("deterministic", "average"):
        raise ParameterError("bound kind must be deterministic or average")
    if not (hasattr(a, "is_cuda") and a.is_cuda):
        a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
    m, n = a.shape
    if m < n:
        raise ParameterError("bound analysis assumes rows >= cols")
    if ref_svd is None:
        sigma, v = reference_svd(a, ctx=ctx)
    else:
        sigma = np.asarray(ref_svd[0], dtype=np.float64)
        v = torch.as_tensor(ref_svd[1], dtype=torch.float64, device=a.device)
    sigma = [float(x) for x in sigma]
    slack = 1e-9 * sigma[0] if sigma else 0.0
    mask = 2**64 - 1

    rep = BoundReport(kind=kind, trials=trials)
    mean_sigma = [0.0] * k
    mean_sv_bound = [0.0] * k
    sv_all_ok = [True] * k
    ss_sigma = [0.0] * k
    mean_err_f = mean_err_2 = mean_bound_f = mean_bound_2 = 0.0
    ss_err_f = ss_err_2 = 0.0
    all_f = all_2 = True
    frr_trials = 0

    cfg = SketchConfig(ell=params.ell, q=params.q, seed=seed & mask)
    for t0 in range(0, trials, max(1, batch)):
        nt = min(max(1, batch), trials - t0)
        seeds = [(seed + t0 + i) & mask for i in range(nt)]
        xs = sor_svd_power_batch(a, k, cfg, nt, seeds=seeds, ctx=ctx)  # bounds.hpp:288, batched
        for i, x in enumerate(xs):
            t = t0 + i
            rec = BoundTrial(trial=t, seed=seeds[i])
            rec.err_f = approx_error(a, x, "frobenius", ctx=ctx)
            rec.err_2 = approx_error(a, x, "spectral", ctx=ctx)
            rec.sigma_hat = [float(z) for z in x.sigma.cpu().numpy()]
            omega = torch.from_numpy(gaussian_matrix(n, params.ell, seeds[i])).to(a.device)
            split = omega_split(v, omega, params, ctx=ctx)
            rec.full_row_rank = split.full_row_rank
            if split.full_row_rank:
                frr_trials += 1
                rec.sv_lower = det_sv_lower_bound(sigma, params, split)
                rec.bound_f = det_lowrank_bound(sigma, params, split, "frobenius")
                rec.bound_2 = det_lowrank_bound(sigma, params, split, "spectral")
                rec.satisfied_f = rec.err_f <= rec.bound_f + slack
                rec.satisfied_2 = rec.err_2 <= rec.bound_2 + slack
                rec.sv_satisfied = True
                for j in range(k):
                    shat, lo, hi = rec.sigma_hat[j], rec.sv_lower[j], _sigma_at(sigma, j + 1)
                    if not (shat >= lo - slack and shat <= hi + slack):
                        rec.sv_satisfied = False
                        sv_all_ok[j] = False
                    mean_sv_bound[j] += lo
                all_f = all_f and rec.satisfied_f
                all_2 = all_2 and rec.satisfied_2
                mean_bound_f += rec.bound_f
                mean_bound_2 += rec.bound_2
            else:
                rec.bound_f = rec.bound_2 = math.inf
                rec.satisfied_f = rec.satisfied_2 = True  # hypothesis vacuous
                rec.sv_satisfied = True
            mean_err_f += rec.err_f
            mean_err_2 += rec.err_2
            ss_err_f += rec.err_f * rec.err_f
            ss_err_2 += rec.err_2 * rec.err_2
            for j in range(k):
                mean_sigma[j] += rec.sigma_hat[j]
                ss_sigma[j] += rec.sigma_hat[j] * rec.sigma_hat[j]
            rep.records.append(rec)

    nt_f = float(trials)
    mean_err_f /= nt_f
    mean_err_2 /= nt_f
    mean_sigma = [x / nt_f for x in mean_sigma]
    rep.realized_error_frobenius = mean_err_f
    rep.realized_error_spectral = mean_err_2
    rep.realized_sigmas = mean_sigma
    if kind == "deterministic":
        d = float(frr_trials) if frr_trials > 0 else 1.0
        rep.sv_lower_bounds = [x / d for x in mean_sv_bound]
        rep.lowrank_bound_frobenius = mean_bound_f / d
        rep.lowrank_bound_spectral = mean_bound_2 / d
        rep.bound_satisfied = [bool(x) for x in sv_all_ok] + [all_f, all_2]
    else:
        rep.sv_lower_bounds = avg_sv_lower_bound(sigma, params)
        rep.lowrank_bound_frobenius = avg_lowrank_bound(sigma, params, "frobenius")
        rep.lowrank_bound_spectral = avg_lowrank_bound(sigma, params, "spectral")

        def se(ss, mean):
            return math.sqrt(max(0.0, ss / nt_f - mean * mean) / nt_f)

        sat = [mean_sigma[j] + 3.0 * se(ss_sigma[j], mean_sigma[j]) >= rep.sv_lower_bounds[j] for j in range(k)]
        sat.append(mean_err_f - 3.0 * se(ss_err_f, mean_err_f) <= rep.lowrank_bound_frobenius)
        sat.append(mean_err_2 - 3.0 * se(ss_err_2, mean_err_2) <= rep.lowrank_bound_spectral)
        rep.bound_satisfied = sat
    return rep


def bound_report_csv(rep: BoundReport) -> str:
    """bounds.hpp:383-404: one row per trial plus a summary row (%.17g numbers)."""
    def g(x: float) -> str:
        return "inf" if math.isinf(x) and x > 0 else "%.17g" % x

    out = ["trial,seed,err_f,err_2,bound_f,bound_2,satisfied_f,satisfied_2\n"]
    for r in rep.records:
        out.append("%d,%d,%s,%s,%s,%s,%d,%d\n" % (r.trial, r.seed, g(r.err_f), g(r.err_2), g(r.bound_f), g(r.bound_2),
                                                  1 if r.satisfied_f else 0, 1 if r.satisfied_2 else 0))
    k = len(rep.sv_lower_bounds)
    sf = len(rep.bound_satisfied) >= k + 2 and rep.bound_satisfied[k]
    s2 = len(rep.bound_satisfied) >= k + 2 and rep.bound_satisfied[k + 1]
    out.append("summary,%d,%s,%s,%s,%s,%d,%d\n" % (rep.trials, g(rep.realized_error_frobenius),
                                                    g(rep.realized_error_spectral), g(rep.lowrank_bound_frobenius),
                                                    g(rep.lowrank_bound_spectral), 1 if sf else 0, 1 if s2 else 0))
    return "".join(out)
