"""B200-native SOR-SVD (arXiv 1804.00462) and ALM-RPCA — Python host API.

Mirrors the reference C++ API (/root/reference/proj/include/sorsvd):

    sor_svd_power(a, k, cfg)  -> LowRankApprox      sketch.hpp:87
    sor_svd(a, k, cfg)        -> LowRankApprox      sketch.hpp:116
    r_svd(a, ell, q, seed)    -> LowRankApprox      sketch.hpp:124 (baseline)
    tsr_svd(a, ell, seed)     -> LowRankApprox      sketch.hpp:139 (baseline)
    truncate(x, k)                                  sketch.hpp:152
    SketchConfig / LowRankApprox / SketchMethod      sketch.hpp:13-48
    flop_estimate / FlopVariant                      sketch.hpp:176-196
    gaussian_matrix / sub_seed                       random.hpp:24,60
    thin_qr / full_svd / matmul (device, skinny)     dense.hpp:114,65,20
    rpca_alm / RpcaConfig / RpcaResult
    ShapeError / ParameterError / NumericalError     errors.hpp:9-26

Every call goes through the C ABI of the sm_100a library
(include/sorsvd_b200.h, paper_1804_00462_b200/_lib/libsorsvd_b200.so). Host
(numpy) inputs use the host-buffer entry points (H2D/D2H inside); CUDA torch
tensors use the device entry points on torch's current stream. There is no
CPU fallback: without the library or a GPU every compute call raises.
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi as C

__all__ = [
    "SketchMethod", "SketchConfig", "LowRankApprox", "FlopVariant", "RpcaConfig", "RpcaResult", "Context",
    "ShapeError", "ParameterError", "NumericalError", "CudaError", "NcclError", "UnsupportedError", "EmuGroup",
    "sor_svd_power", "sor_svd", "sor_svd_power_batch", "r_svd", "tsr_svd", "truncate", "approx_error", "sord_header", "load_sord", "save_sord", "rpca_alm", "rpca_default_config", "estimate_rank_bound", "norm", "gaussian_matrix_device", "gen_lowrank_device", "gen_rpca_instance_device", "gaussian_matrix", "sub_seed",
    "flop_estimate", "validate_sketch", "thin_qr", "full_svd", "matmul", "default_context", "version",
]


# ----------------------------------------------------------------- errors --
class ShapeError(ValueError):
    """sorsvd::shape_error (errors.hpp:9)"""


class ParameterError(ValueError):
    """sorsvd::parameter_error (errors.hpp:14)"""


class NumericalError(RuntimeError):
    """sorsvd::numerical_error (errors.hpp:24)"""


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


class UnsupportedError(NotImplementedError):
    pass


_ERRORS = {C.ERR_SHAPE: ShapeError, C.ERR_PARAMETER: ParameterError, C.ERR_NUMERICAL: NumericalError,
           C.ERR_CUDA: CudaError, C.ERR_NCCL: NcclError, C.ERR_OOM: MemoryError,
           C.ERR_UNSUPPORTED: UnsupportedError, C.ERR_INTERNAL: RuntimeError}


def _check(rc: int, ctx=None):
    if rc != C.OK:
        msg = C.lib().sorsvd_last_error(ctx).decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


# ------------------------------------------------------------------ types --
class SketchMethod(enum.IntEnum):
    """sketch.hpp:13"""
    sor = 0
    sor_power = 1
    rsvd = 2
    tsr = 3


class FlopVariant(enum.IntEnum):
    """sketch.hpp:176"""
    sor_3pass = 0
    sor_2pass = 1
    sor_power_2q3 = 2
    sor_power_2q2 = 3


@dataclass
class SketchConfig:
    """sketch.hpp:29-34"""
    ell: int = 0
    q: int = 0
    seed: int = 0
    single_pass: bool = False


@dataclass
class LowRankApprox:
    """sketch.hpp:39-48 (u: m x k, sigma: k, v: n x k)."""
    u: object
    sigma: object
    v: object
    method: SketchMethod
    passes: int
    ell: int
    q: int
    seed: int
    stats: dict = field(default_factory=dict)


@dataclass
class RpcaConfig:
    """SPEC.md:356-360 (ledger: SURVEY.md Appendix B). lam/mu0 <= 0 select
    the defaults 1/sqrt(max(m,n)) and 1.25/sigma_1(X)."""
    lam: float = 0.0
    mu0: float = 0.0
    mu_bar_factor: float = 1e7
    rho: float = 1.6
    tol: float = 1e-7
    max_iter: int = 500
    ell: int = 10
    q: int = 1
    seed: int = 0


@dataclass
class RpcaResult:
    """SPEC.md:361-365"""
    l: object
    s: object
    iterations: int
    rel_error: float
    rank_l: int
    nnz_s: int
    converged: bool
    mu0: float = 0.0
    stats: dict = field(default_factory=dict)
    telemetry: object = None  # (iterations, 5) array: iter, mu, rel_error, rank_l, nnz_s

    def telemetry_csv(self) -> str:
        """the per-iteration telemetry CSV (iter, mu, rel_error, rank_l, nnz_s)."""
        rows = ["iter,mu,rel_error,rank_l,nnz_s\n"]
        for r in (self.telemetry if self.telemetry is not None else []):
            rows.append("%d,%.17g,%.17g,%d,%d\n" % (int(r[0]), r[1], r[2], int(r[3]), int(r[4])))
        return "".join(rows)


# ---------------------------------------------------------------- context --
class Context:
    """Owns a device context (streams, workspaces, cached CUDA graphs).

    Multi-GPU: Context(device, rank=r, world=w, nccl_id=bytes) with the id from
    Context.nccl_unique_id() on rank 0, broadcast by the caller."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 emu_group: Optional["EmuGroup"] = None):
        h = ctypes.c_void_p()
        if emu_group is not None:
            world = emu_group.world
            _check(C.lib().sorsvd_ctx_create_emulated(device, rank, emu_group.handle, ctypes.byref(h)))
        elif world > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ParameterError("parameter: world > 1 needs the 128-byte NCCL unique id")
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            _check(C.lib().sorsvd_ctx_create_dist(device, rank, world, ctypes.cast(buf, ctypes.c_void_p),
                                                   ctypes.byref(h)))
        else:
            _check(C.lib().sorsvd_ctx_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device
        self.rank = rank
        self.world = world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(C.lib().sorsvd_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
        return buf.raw

    @staticmethod
    def nccl_selftest(device: int = 0, count: int = 1 << 16) -> float:
        """One-rank NCCL communicator on `device`: all-reduce + all-gather of `count` doubles through the
        library's dlopen binding; returns the largest deviation from the input (0.0 expected)."""
        err = ctypes.c_double(-1.0)
        _check(C.lib().sorsvd_nccl_selftest(device, count, ctypes.byref(err)))
        return err.value

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int):
        _check(C.lib().sorsvd_set_stream(self._h, ctypes.c_void_p(stream_ptr)), self._h)

    # sorsvd_ctx_set_option keys / Jacobi variants (include/sorsvd_b200.h)
    OPT_JACOBI, OPT_SORD_CHUNK_MB, OPT_OZAKI_PLANES, OPT_FUSED_PAIR, OPT_UPLOAD_CHUNK_MB, OPT_OZAKI_MULTICAST, OPT_OZAKI_OVERLAP, OPT_UPLOAD_TN, OPT_NCCL_GRAPH = 1, 2, 3, 4, 5, 6, 7, 8, 9
    JACOBI_AUTO, JACOBI_BARRIER, JACOBI_ROTLOG = 0, 1, 2

    def set_option(self, key: int, value: int):
        """Per-context algorithm option (tests cross-check kernel variants with it)."""
        _check(C.lib().sorsvd_ctx_set_option(self._h, int(key), int(value)), self._h)

    def close(self):
        if getattr(self, "_h", None):
            C.lib().sorsvd_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class EmuGroup:
    """In-process emulation of `world` ranks on one GPU (one Context and one
    host thread per rank); the multi-GPU schedule with host-barrier collectives."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        _check(C.lib().sorsvd_emu_group_create(world, ctypes.byref(h)))
        self.handle = h
        self.world = world

    def close(self):
        if getattr(self, "handle", None):
            C.lib().sorsvd_emu_group_destroy(self.handle)
            self.handle = None


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def version() -> str:
    return C.lib().sorsvd_version().decode()


# ---------------------------------------------------------- host helpers --
def sub_seed(seed: int, stream: int) -> int:
    """random.hpp:24"""
    return int(C.lib().sorsvd_sub_seed(seed & (2**64 - 1), stream & (2**64 - 1)))


def gaussian_matrix(rows: int, cols: int, seed: int, nthreads: int = 0) -> np.ndarray:
    """random.hpp:60 — bit-identical to the reference draw (host, threaded)."""
    if rows < 1 or cols < 1:
        raise ShapeError("shape: matrix dimensions must be positive")
    out = np.empty((rows, cols), dtype=np.float64)
    _check(C.lib().sorsvd_gaussian_matrix(rows, cols, seed & (2**64 - 1), out.ctypes.data_as(C.c_dp), nthreads))
    return out


def flop_estimate(m: int, n: int, ell: int, k: int, q: int, variant: FlopVariant) -> int:
    """sketch.hpp:178"""
    v = C.lib().sorsvd_flop_estimate(m, n, ell, k, q, int(variant))
    if v < 0:
        raise ParameterError("parameter: flop_estimate requires positive dimensions and q >= 0")
    return int(v)


def validate_sketch(m: int, n: int, k: int, ell: int, q: int) -> None:
    """sketch.hpp:62-69"""
    _check(C.lib().sorsvd_validate_sketch(m, n, k, ell, q))


# ------------------------------------------------------------- internals --
def _is_torch_cuda(x) -> bool:
    try:
        import torch
    except ImportError:
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _torch_stream(ctx: Context, dev_tensor):
    import torch
    ctx.set_stream(torch.cuda.current_stream(dev_tensor.device).cuda_stream)


def _desc(m, n, lda, k, cfg: SketchConfig, flags: int, m_global: int = 0, dtype: int = C.F64) -> C.SorsvdDesc:
    return C.SorsvdDesc(m, n, lda, k, cfg.ell, cfg.q, int(cfg.single_pass), cfg.seed & (2**64 - 1), dtype,
                        flags, m_global)


def _host_out(shape):
    """float64 numpy array for a host-API result. Page-locked (from torch's
    caching host allocator) when torch is importable, so the device-to-host
    copy runs at full PCIe rate instead of through the driver's pageable
    staging; a plain numpy array otherwise."""
    try:
        import torch
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    except Exception:
        return np.empty(shape)


# -------------------------------------------------------------- hot path --
def _decompose(kind: str, a, k: int, cfg: SketchConfig, flags: int, omega, psi2, ctx, m_global: int = 0):
    """One call of sor_svd_power ("sor"), r_svd ("rsvd") or tsr_svd ("tsr")
    through the host-buffer or device entry point; returns (stats, u, sigma, v)."""
    host_fn = {"sor": "sorsvd_sor_svd_power", "rsvd": "sorsvd_r_svd", "tsr": "sorsvd_tsr_svd"}[kind]
    if omega is not None:
        flags |= C.FLAG_OMEGA_GIVEN
    st = C.SorsvdStats()
    if _is_torch_cuda(a):
        import torch
        if a.dtype not in (torch.float64, torch.float32) or a.dim() != 2 or a.stride(1) != 1:
            raise ShapeError("shape: device input must be a row-major float64 or float32 matrix")
        ctx = ctx or default_context(a.device.index or 0)
        _torch_stream(ctx, a)
        m, n = a.shape
        lda = a.stride(0)
        d = _desc(m, n, lda, k, cfg, flags, m_global, C.F32 if a.dtype == torch.float32 else C.F64)
        u = torch.empty((m, k), dtype=torch.float64, device=a.device)
        s = torch.empty((k,), dtype=torch.float64, device=a.device)
        v = torch.empty((n, k), dtype=torch.float64, device=a.device)
        ptrs = []
        keep = []
        for x, rows in ((omega, n), (psi2, m)):
            if x is None:
                ptrs.append(None)
                continue
            t = torch.as_tensor(x, dtype=torch.float64, device=a.device).contiguous()
            if tuple(t.shape) != (rows, cfg.ell):
                raise ShapeError("shape: test matrix must be (rows, ell)")
            keep.append(t)
            ptrs.append(t.data_ptr())
        fn = getattr(C.lib(), host_fn + "_device")
        args = [ctx.handle, ctypes.byref(d), a.data_ptr(), ptrs[0]] + ([ptrs[1]] if kind == "tsr" else [])
        _check(fn(*args, u.data_ptr(), s.data_ptr(), v.data_ptr(), ctypes.byref(st)), ctx.handle)
    else:
        a = np.asarray(a)
        a = np.ascontiguousarray(a, dtype=np.float32 if a.dtype == np.float32 else np.float64)
        if a.ndim != 2:
            raise ShapeError("shape: input must be a matrix")
        ctx = ctx or default_context(0)
        m, n = a.shape
        d = _desc(m, n, n, k, cfg, flags, m_global, C.F32 if a.dtype == np.float32 else C.F64)
        u = _host_out((m, k))
        s = _host_out((k,))
        v = _host_out((n, k))
        ptrs = []
        keep = []
        for x, rows in ((omega, n), (psi2, m)):
            if x is None:
                ptrs.append(None)
                continue
            t = np.ascontiguousarray(x, dtype=np.float64)
            if t.shape != (rows, cfg.ell):
                raise ShapeError("shape: test matrix must be (rows, ell)")
            keep.append(t)
            ptrs.append(t.ctypes.data_as(C.c_dp))
        fn = getattr(C.lib(), host_fn)
        args = [ctx.handle, ctypes.byref(d), a.ctypes.data_as(ctypes.c_void_p), ptrs[0]] + (
            [ptrs[1]] if kind == "tsr" else [])
        _check(fn(*args, u.ctypes.data_as(C.c_dp), s.ctypes.data_as(C.c_dp), v.ctypes.data_as(C.c_dp),
                  ctypes.byref(st)), ctx.handle)
    return st, u, s, v


def sor_svd_power(a, k: int, cfg: SketchConfig, omega=None, ctx: Optional[Context] = None,
                  stage_times: bool = False, use_graph: bool = True, m_global: int = 0,
                  _basic: bool = False, fp32_mode: str = "fp64", fp64_mode: str = "auto") -> LowRankApprox:
    """Subspace-orbit randomized SVD with q power iterations (sketch.hpp:87).

    a: numpy (m, n) on the host or a CUDA torch tensor; float64 runs the FP64
    path. float32 input is kept in FP32 (half the bytes); fp32_mode="fp64"
    (default) computes the passes in FP64 on the DMMA pipe, fp32_mode="tf32"
    on the TF32 tensor cores (fast; ~1e-3 relative and only the sketch
    directions above the TF32 rounding level are resolved). QR and
    the core SVD are FP64 and results are FP64 either way.
    fp64_mode: how the FP64 passes are computed: "dmma" (the FP64 tensor pipe),
    "ozaki" (exact int8 slice products on the tcgen05 tensor cores, ozaki_i8.cuh),
    or "auto" (default: ozaki for large passes, ell >= 32 and m*n*ell >= 2^30.5 with the
    per-call digit planes of A, >= 2^36 without).
    omega: optional (n, ell) test matrix; default gaussian_matrix(n, ell, seed)
    exactly as the reference draws it (sketch.hpp:90)."""
    if fp32_mode not in ("fp64", "tf32"):
        raise ParameterError("parameter: fp32_mode must be 'fp64' or 'tf32'")
    if fp64_mode not in ("auto", "dmma", "ozaki"):
        raise ParameterError("parameter: fp64_mode must be 'auto', 'dmma' or 'ozaki'")
    flags = C.FLAG_TF32 if fp32_mode == "tf32" else 0
    flags |= {"auto": 0, "dmma": C.FLAG_DMMA, "ozaki": C.FLAG_OZAKI}[fp64_mode]
    if stage_times:
        flags |= C.FLAG_STAGE_TIMES
    if not use_graph:
        flags |= C.FLAG_NO_GRAPH
    if _basic:
        flags |= C.FLAG_BASIC
    st, u, s, v = _decompose("sor", a, k, cfg, flags, omega, None, ctx, m_global)
    method = SketchMethod.sor if cfg.q == 0 else SketchMethod.sor_power
    return LowRankApprox(u, s, v, method, st.passes, cfg.ell, cfg.q, cfg.seed, st.as_dict())


def sor_svd_power_batch(a, k: int, cfg: SketchConfig, trials: int, seeds=None, omegas=None,
                        ctx: Optional[Context] = None, m_global: int = 0) -> list:
    """`trials` independent sor_svd_power calls on one A (the Monte-Carlo loop of
    bounds.hpp:262-379): trial t uses seeds[t], default cfg.seed + t
    (bounds.hpp:288), or omegas[t] (trials, n, ell). Every pass over A serves
    all trials in one launch. Returns one LowRankApprox per trial."""
    if trials < 1:
        raise ParameterError("parameter: trials must be positive")
    seed_list = [(cfg.seed + t) & (2**64 - 1) for t in range(trials)] if seeds is None else \
        [int(x) & (2**64 - 1) for x in seeds]
    if len(seed_list) != trials:
        raise ShapeError("shape: need one seed per trial")
    sarr = (C.c_u64 * trials)(*seed_list)
    flags = C.FLAG_OMEGA_GIVEN if omegas is not None else 0
    st = C.SorsvdStats()
    if _is_torch_cuda(a):
        import torch
        if a.dtype not in (torch.float64, torch.float32) or a.dim() != 2 or a.stride(1) != 1:
            raise ShapeError("shape: device input must be a row-major float64 or float32 matrix")
        ctx = ctx or default_context(a.device.index or 0)
        _torch_stream(ctx, a)
        m, n = a.shape
        d = _desc(m, n, a.stride(0), k, cfg, flags, m_global, C.F32 if a.dtype == torch.float32 else C.F64)
        u = torch.empty((trials, m, k), dtype=torch.float64, device=a.device)
        s = torch.empty((trials, k), dtype=torch.float64, device=a.device)
        v = torch.empty((trials, n, k), dtype=torch.float64, device=a.device)
        om = None
        if omegas is not None:
            om = torch.as_tensor(omegas, dtype=torch.float64, device=a.device).contiguous()
            if tuple(om.shape) != (trials, n, cfg.ell):
                raise ShapeError("shape: omegas must be (trials, n, ell)")
        _check(C.lib().sorsvd_sor_svd_power_batch_device(ctx.handle, ctypes.byref(d), trials, sarr, a.data_ptr(),
                                                         om.data_ptr() if om is not None else None, u.data_ptr(),
                                                         s.data_ptr(), v.data_ptr(), ctypes.byref(st)), ctx.handle)
    else:
        a = np.asarray(a)
        a = np.ascontiguousarray(a, dtype=np.float32 if a.dtype == np.float32 else np.float64)
        ctx = ctx or default_context(0)
        m, n = a.shape
        d = _desc(m, n, n, k, cfg, flags, m_global, C.F32 if a.dtype == np.float32 else C.F64)
        u = _host_out((trials, m, k))
        s = _host_out((trials, k))
        v = _host_out((trials, n, k))
        om_p = None
        if omegas is not None:
            om = np.ascontiguousarray(omegas, dtype=np.float64)
            if om.shape != (trials, n, cfg.ell):
                raise ShapeError("shape: omegas must be (trials, n, ell)")
            om_p = om.ctypes.data_as(C.c_dp)
        _check(C.lib().sorsvd_sor_svd_power_batch(ctx.handle, ctypes.byref(d), trials, sarr,
                                                  a.ctypes.data_as(ctypes.c_void_p), om_p, u.ctypes.data_as(C.c_dp),
                                                  s.ctypes.data_as(C.c_dp), v.ctypes.data_as(C.c_dp),
                                                  ctypes.byref(st)), ctx.handle)
    method = SketchMethod.sor if cfg.q == 0 else SketchMethod.sor_power
    stats = st.as_dict()
    return [LowRankApprox(u[t], s[t], v[t], method, st.passes, cfg.ell, cfg.q, seed_list[t], dict(stats))
            for t in range(trials)]


def sor_svd(a, k: int, cfg: SketchConfig, **kw) -> LowRankApprox:
    """Basic form; requires cfg.q == 0 (sketch.hpp:116-119)."""
    if cfg.q != 0:
        raise ParameterError("parameter: sor_svd requires q == 0; use sor_svd_power")
    return sor_svd_power(a, k, cfg, _basic=True, **kw)


def r_svd(a, ell: int, q: int, seed: int, omega=None, ctx: Optional[Context] = None,
          use_graph: bool = True, m_global: int = 0) -> LowRankApprox:
    """One-sided randomized SVD baseline (sketch.hpp:124-136): all ell triplets,
    passes 2q+2. omega (n, ell) defaults to gaussian_matrix(n, ell, seed)."""
    cfg = SketchConfig(ell=ell, q=q, seed=seed)
    flags = 0 if use_graph else C.FLAG_NO_GRAPH
    st, u, s, v = _decompose("rsvd", a, ell, cfg, flags, omega, None, ctx, m_global)
    return LowRankApprox(u, s, v, SketchMethod.rsvd, st.passes, ell, q, seed, st.as_dict())


def tsr_svd(a, ell: int, seed: int, psi1=None, psi2=None, ctx: Optional[Context] = None,
            use_graph: bool = True, m_global: int = 0) -> LowRankApprox:
    """Two-sided randomized SVD baseline (sketch.hpp:139-149): Psi1 (n, ell) from
    seed, Psi2 (m, ell) from seed ^ 1 unless both are given; pseudo-inverse core;
    all ell triplets, passes 1."""
    if (psi1 is None) != (psi2 is None):
        raise ParameterError("parameter: give both psi1 and psi2 or neither")
    cfg = SketchConfig(ell=ell, q=0, seed=seed)
    flags = 0 if use_graph else C.FLAG_NO_GRAPH
    st, u, s, v = _decompose("tsr", a, ell, cfg, flags, psi1, psi2, ctx, m_global)
    return LowRankApprox(u, s, v, SketchMethod.tsr, st.passes, ell, 0, seed, st.as_dict())


def approx_error(a, x: LowRankApprox, kind: str = "frobenius", ctx: Optional[Context] = None) -> float:
    """sketch.hpp:168-172: ||a - reconstruct(x)||. kind "frobenius": one fused pass
    over a on the device (the m x n reconstruction is never formed). kind
    "spectral": the difference is formed on the device and its sigma_1 comes from
    `norm(., "spectral")` (the reference: dgesdd of the dense difference). On a row-sharded
    context a and x.u are the rank's rows (spectral: n <= 1024)."""
    import torch
    if kind not in ("frobenius", "spectral"):
        raise ParameterError("parameter: approx_error supports frobenius and spectral norms")
    dev = a.device if _is_torch_cuda(a) else torch.device("cuda", 0)
    A = a if _is_torch_cuda(a) else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if A.dtype not in (torch.float64, torch.float32) or A.dim() != 2 or A.stride(1) != 1:
        raise ShapeError("shape: approx_error expects a row-major float64 or float32 matrix")
    u = torch.as_tensor(x.u, dtype=torch.float64, device=dev).contiguous()
    s = torch.as_tensor(x.sigma, dtype=torch.float64, device=dev).contiguous()
    v = torch.as_tensor(x.v, dtype=torch.float64, device=dev).contiguous()
    m, n = A.shape
    if u.shape[0] != m or v.shape[0] != n:
        raise ShapeError("approx_error: approximation does not match matrix dims")
    ctx = ctx or default_context(dev.index or 0)
    _torch_stream(ctx, A)
    out = ctypes.c_double()
    fn = C.lib().sorsvd_approx_error_fro_device if kind == "frobenius" else C.lib().sorsvd_approx_error_spectral_device
    _check(fn(ctx.handle, m, n, A.data_ptr(), A.stride(0), C.F32 if A.dtype == torch.float32 else C.F64, s.shape[0],
              u.data_ptr(), u.shape[1], s.data_ptr(), v.data_ptr(), v.shape[1], ctypes.byref(out)), ctx.handle)
    return out.value


def norm(a, kind: str = "frobenius", ctx: Optional[Context] = None, seed: int = 0) -> float:
    """dense.hpp:163-176 on a CUDA (or host) float64 matrix: "frobenius" or "spectral"
    (sigma_1 by Gram squaring + Rayleigh-Ritz for min(m, n) <= 1024, else block
    subspace iteration; the reference runs dgesdd on the whole matrix). On a row-sharded
    context a is the rank's row block (spectral: n <= 1024, the Gram matrix is summed over ranks)."""
    import torch
    if kind not in ("frobenius", "spectral"):
        raise ParameterError("parameter: norm supports frobenius and spectral")
    dev = a.device if _is_torch_cuda(a) else torch.device("cuda", 0)
    A = (a if _is_torch_cuda(a) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev))
    if A.dtype != torch.float64 or A.dim() != 2 or A.stride(1) != 1:
        raise ShapeError("shape: norm expects a row-major float64 matrix")
    ctx = ctx or default_context(dev.index or 0)
    _torch_stream(ctx, A)
    m, n = A.shape
    if kind == "frobenius":  # ||A - 0||_F through the fused error pass (deterministic reduction)
        zs = torch.zeros((1,), dtype=torch.float64, device=dev)
        zu = torch.zeros((m, 1), dtype=torch.float64, device=dev)
        zv = torch.zeros((n, 1), dtype=torch.float64, device=dev)
        out = ctypes.c_double()
        _check(C.lib().sorsvd_approx_error_fro_device(ctx.handle, m, n, A.data_ptr(), A.stride(0), C.F64, 1,
                                                      zu.data_ptr(), 1, zs.data_ptr(), zv.data_ptr(), 1,
                                                      ctypes.byref(out)), ctx.handle)
        return out.value
    out = ctypes.c_double()
    _check(C.lib().sorsvd_norm_spectral_device(ctx.handle, m, n, A.data_ptr(), A.stride(0), seed & (2**64 - 1),
                                               ctypes.byref(out)), ctx.handle)
    return out.value


# ------------------------------------------------- generators on the device --
def gaussian_matrix_device(rows: int, cols: int, seed: int, device: int = 0, ctx: Optional[Context] = None):
    """random.hpp:60-65 filled on the device (reference words / uniforms, device log / sincos:
    a few ulp from `gaussian_matrix`, which is bit-identical to the reference)."""
    import torch
    out = torch.empty((rows, cols), dtype=torch.float64, device=torch.device("cuda", device))
    ctx = ctx or default_context(device)
    _torch_stream(ctx, out)
    _check(C.lib().sorsvd_gaussian_matrix_device(ctx.handle, rows, cols, seed & (2**64 - 1), out.data_ptr(), cols),
           ctx.handle)
    return out


def gen_lowrank_device(m: int, n: int, sigma, noise_std: float, seed: int, x_scale: float = 1.0, y_scale: float = 1.0,
                       dtype=None, row0: int = 0, m_global: int = 0, device: int = 0, ctx: Optional[Context] = None):
    """Rows [row0, row0 + m) of (x_scale X) diag(sigma) (y_scale Y)^T + noise_std E, the low-rank-plus-noise
    family of BASELINE.json configs 1 / 3 / 5, generated in HBM (see sorsvd_gen_lowrank_device)."""
    import torch
    dtype = dtype or torch.float64
    if dtype not in (torch.float64, torch.float32):
        raise ParameterError("parameter: dtype must be float64 or float32")
    sg = np.ascontiguousarray(sigma, dtype=np.float64)
    out = torch.empty((m, n), dtype=dtype, device=torch.device("cuda", device))
    ctx = ctx or default_context(device)
    _torch_stream(ctx, out)
    _check(C.lib().sorsvd_gen_lowrank_device(ctx.handle, m, n, sg.size, sg.ctypes.data_as(C.c_dp), x_scale, y_scale,
                                             noise_std, seed & (2**64 - 1), row0, m_global,
                                             C.F32 if dtype == torch.float32 else C.F64, out.data_ptr(), n), ctx.handle)
    return out


def gen_rpca_instance_device(n: int, r: int, s: int, seed: int, device: int = 0, ctx: Optional[Context] = None):
    """matrixgen.hpp:99-124 on the device: (x, l_true, s_true) as CUDA float64 n x n tensors."""
    import torch
    dev = torch.device("cuda", device)
    x, l, sp = (torch.empty((n, n), dtype=torch.float64, device=dev) for _ in range(3))
    ctx = ctx or default_context(device)
    _torch_stream(ctx, x)
    _check(C.lib().sorsvd_gen_rpca_instance_device(ctx.handle, n, r, s, seed & (2**64 - 1), x.data_ptr(), l.data_ptr(),
                                                   sp.data_ptr()), ctx.handle)
    return x, l, sp


def sord_header(path: str):
    """(rows, cols) of a SORD matrix file (no GPU needed)."""
    r, c = C.c_i64(), C.c_i64()
    _check(C.lib().sorsvd_sord_header(path.encode(), ctypes.byref(r), ctypes.byref(c)))
    return r.value, c.value


def load_sord(path: str, device: int = 0, dtype=None, ctx: Optional[Context] = None):
    """Stream a SORD file into a CUDA tensor (float64, or float32 rounded on
    the device) without holding the matrix on the host."""
    import torch
    dtype = dtype or torch.float64
    if dtype not in (torch.float64, torch.float32):
        raise ParameterError("parameter: dtype must be float64 or float32")
    rows, cols = sord_header(path)
    out = torch.empty((rows, cols), dtype=dtype, device=torch.device("cuda", device))
    ctx = ctx or default_context(device)
    _torch_stream(ctx, out)
    _check(C.lib().sorsvd_load_sord_device(ctx.handle, path.encode(), out.data_ptr(), cols,
                                           C.F32 if dtype == torch.float32 else C.F64), ctx.handle)
    return out


def save_sord(path: str, a, ctx: Optional[Context] = None) -> None:
    """Write a CUDA float64 matrix as a SORD file, streamed through pinned buffers."""
    import torch
    if not _is_torch_cuda(a) or a.dtype != torch.float64 or a.dim() != 2 or a.stride(1) != 1:
        raise ShapeError("shape: save_sord expects a row-major CUDA float64 matrix")
    ctx = ctx or default_context(a.device.index or 0)
    _torch_stream(ctx, a)
    _check(C.lib().sorsvd_save_sord_device(ctx.handle, path.encode(), a.data_ptr(), a.shape[0], a.shape[1],
                                           a.stride(0)), ctx.handle)


def truncate(x: LowRankApprox, k: int) -> LowRankApprox:
    """sketch.hpp:152-160: the leading k triplets (views of the same storage)."""
    if k < 1 or k > len(x.sigma):
        raise ParameterError("truncate rank out of range")
    return LowRankApprox(x.u[:, :k], x.sigma[:k], x.v[:, :k], x.method, x.passes, x.ell, x.q, x.seed,
                         dict(x.stats))


# ----------------------------------------------------- stage entry points --
def thin_qr(t, ctx: Optional[Context] = None):
    """dense.hpp:114 on a CUDA float64 tensor (tall-skinny, k <= 512): (q, r)."""
    import torch
    if not _is_torch_cuda(t) or t.dtype != torch.float64:
        raise ShapeError("shape: thin_qr expects a CUDA float64 tensor")
    ctx = ctx or default_context(t.device.index or 0)
    _torch_stream(ctx, t)
    t = t.contiguous()
    m, k = t.shape
    q = torch.empty((m, k), dtype=torch.float64, device=t.device)
    r = torch.empty((k, k), dtype=torch.float64, device=t.device)
    _check(C.lib().sorsvd_thin_qr_device(ctx.handle, m, k, t.data_ptr(), k, q.data_ptr(), k, r.data_ptr(), k),
           ctx.handle)
    return q, r


def full_svd(mat, ctx: Optional[Context] = None):
    """dense.hpp:65 for a small square CUDA float64 matrix: (u, sigma, v, sweeps)."""
    import torch
    if not _is_torch_cuda(mat) or mat.dtype != torch.float64 or mat.shape[0] != mat.shape[1]:
        raise ShapeError("shape: full_svd expects a square CUDA float64 tensor")
    ctx = ctx or default_context(mat.device.index or 0)
    _torch_stream(ctx, mat)
    mat = mat.contiguous()
    k = mat.shape[0]
    u = torch.empty((k, k), dtype=torch.float64, device=mat.device)
    v = torch.empty((k, k), dtype=torch.float64, device=mat.device)
    s = torch.empty((k,), dtype=torch.float64, device=mat.device)
    sw = C.c_i32()
    _check(C.lib().sorsvd_small_svd_device(ctx.handle, k, mat.data_ptr(), k, u.data_ptr(), k, s.data_ptr(),
                                           v.data_ptr(), k, ctypes.byref(sw)), ctx.handle)
    return u, s, v, sw.value


def matmul(a, b, transpose_a: bool = False, ctx: Optional[Context] = None):
    """dense.hpp:20 restricted to skinny products: op(a) @ b with b narrow.
    float64 -> FP64 DMMA kernel; float32 -> tcgen05 TF32 kernel (FP32 accumulate)."""
    import torch
    if not (_is_torch_cuda(a) and _is_torch_cuda(b)):
        raise ShapeError("shape: matmul expects CUDA float64 tensors")
    ctx = ctx or default_context(a.device.index or 0)
    _torch_stream(ctx, a)
    a = a.contiguous()
    b = b.contiguous()
    M, K = (a.shape[1], a.shape[0]) if transpose_a else a.shape
    if b.shape[0] != K:
        raise ShapeError(f"shape: matmul inner dimensions {K} and {b.shape[0]} differ")
    N = b.shape[1]
    if a.dtype == torch.float32:
        # FP32 operands go to the tcgen05 TF32 tensor-core kernel (FP32 accumulation)
        b = b.to(torch.float32)
        c = torch.empty((M, N), dtype=torch.float32, device=a.device)
        _check(C.lib().sorsvd_matmul_f32_device(ctx.handle, int(transpose_a), M, K, N, a.data_ptr(), a.shape[1],
                                                b.data_ptr(), N, c.data_ptr(), N), ctx.handle)
        return c
    c = torch.empty((M, N), dtype=torch.float64, device=a.device)
    _check(C.lib().sorsvd_matmul_device(ctx.handle, int(transpose_a), M, K, N, a.data_ptr(), a.shape[1],
                                        b.data_ptr(), N, c.data_ptr(), N), ctx.handle)
    return c


# ------------------------------------------------------------------- RPCA --
def estimate_rank_bound(x, ctx: Optional[Context] = None) -> int:
    """SPEC.md:377-385 (PAPER Eq. 66): ceil((||X||_* / ||X||_F)^2); the spectrum comes from
    thin QR + Jacobi SVD on the device (min(m, n) <= 512). Zero matrix -> ParameterError.
    Row-sharded context: x is the rank's rows (n <= 256, at least n rows per rank)."""
    import torch
    dev = x.device if _is_torch_cuda(x) else torch.device("cuda", 0)
    X = x if _is_torch_cuda(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
    if X.dtype != torch.float64 or X.dim() != 2 or X.stride(1) != 1:
        raise ShapeError("shape: estimate_rank_bound expects a row-major float64 matrix")
    ctx = ctx or default_context(dev.index or 0)
    _torch_stream(ctx, X)
    out = C.c_i64()
    _check(C.lib().sorsvd_estimate_rank_bound_device(ctx.handle, X.shape[0], X.shape[1], X.data_ptr(), X.stride(0),
                                                     ctypes.byref(out), None, None), ctx.handle)
    return int(out.value)


def rpca_default_config(x_or_m, n: Optional[int] = None, ell: Optional[int] = None, q: int = 1, seed: int = 0,
                        ctx: Optional[Context] = None, m_global: int = 0) -> RpcaConfig:
    """lambda = 1/sqrt(max(m,n)), mu0 = 1.25/sigma_1(X) (estimated on the device by
    rpca_alm: mu0 = 0 here), mu_bar = 1e7 mu0, rho = 1.6, tol = 1e-7, max_iter = 500, q = 1 and
    ell = min(2 * estimate_rank_bound(x), min(m,n) - 1). Call with the matrix (the spec's form),
    or with (m, n, ell) when the sketch size is chosen by the caller. Row-sharded: the rank's
    row block with ctx and m_global (lambda and the ell cap use the global row count)."""
    if hasattr(x_or_m, "shape"):
        m, nn = x_or_m.shape
        m = m_global or m
        if ell is None:
            ell = max(1, min(2 * estimate_rank_bound(x_or_m, ctx=ctx), min(m, nn) - 1))
    else:
        m, nn = int(x_or_m), int(n)
        ell = 10 if ell is None else ell
    return RpcaConfig(lam=1.0 / math.sqrt(max(m, nn)), mu0=0.0, mu_bar_factor=1e7, rho=1.6, tol=1e-7,
                      max_iter=500, ell=ell, q=q, seed=seed)


def rpca_alm(x, cfg: RpcaConfig, ctx: Optional[Context] = None, want_l: bool = True,
             m_global: int = 0) -> RpcaResult:
    """Inexact ALM RPCA with SOR-SVD per iteration.
    Multi-GPU: x is this rank's row block of D, m_global the total rows; L and
    S come back row-sharded, the scalars (iterations, rel_error, rank, nnz)
    are global."""
    res = C.RpcaRes()
    if _is_torch_cuda(x):
        import torch
        ctx = ctx or default_context(x.device.index or 0)
        _torch_stream(ctx, x)
        m, n = x.shape
        d = C.RpcaDesc(m, n, x.stride(0), cfg.lam, cfg.mu0, cfg.mu_bar_factor, cfg.rho, cfg.tol, cfg.max_iter,
                       cfg.ell, cfg.q, C.F64, cfg.seed & (2**64 - 1), 0, 0, m_global)
        s = torch.empty((m, n), dtype=torch.float64, device=x.device)
        l = torch.empty((m, n), dtype=torch.float64, device=x.device) if want_l else None
        _check(C.lib().sorsvd_rpca_alm_device(ctx.handle, ctypes.byref(d), x.data_ptr(),
                                              l.data_ptr() if l is not None else None, s.data_ptr(),
                                              ctypes.byref(res)), ctx.handle)
    else:
        x = np.ascontiguousarray(x, dtype=np.float64)
        ctx = ctx or default_context(0)
        m, n = x.shape
        d = C.RpcaDesc(m, n, n, cfg.lam, cfg.mu0, cfg.mu_bar_factor, cfg.rho, cfg.tol, cfg.max_iter, cfg.ell,
                       cfg.q, C.F64, cfg.seed & (2**64 - 1), 0, 0, m_global)
        s = _host_out((m, n))
        l = _host_out((m, n)) if want_l else None
        _check(C.lib().sorsvd_rpca_alm(ctx.handle, ctypes.byref(d), x.ctypes.data_as(C.c_dp),
                                       l.ctypes.data_as(C.c_dp) if l is not None else None,
                                       s.ctypes.data_as(C.c_dp), ctypes.byref(res)), ctx.handle)
    stats = {f: getattr(res, f) for f, _ in res._fields_}
    rows = C.c_i32()
    _check(C.lib().sorsvd_rpca_telemetry(ctx.handle, 0, None, ctypes.byref(rows)), ctx.handle)
    tele = np.zeros((rows.value, 5))
    if rows.value:
        _check(C.lib().sorsvd_rpca_telemetry(ctx.handle, rows.value, tele.ctypes.data_as(C.c_dp), ctypes.byref(rows)),
               ctx.handle)
    return RpcaResult(l, s, res.iterations, res.rel_error, res.rank_l, res.nnz_s, bool(res.converged), res.mu0,
                      stats, tele)
