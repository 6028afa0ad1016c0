"""ctypes binding of include/sorsvd_b200.h (the C ABI of libsorsvd_b200.so).

No fallback: if the sm_100a library is missing or no CUDA device is present,
every entry point raises. The CPU oracles under oracle/ are never imported
from here.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libsorsvd_b200.so")

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_u64 = ctypes.c_uint64
c_u32 = ctypes.c_uint32
c_dp = ctypes.POINTER(ctypes.c_double)
c_vp = ctypes.c_void_p

# sorsvd_status (include/sorsvd_b200.h)
OK, ERR_SHAPE, ERR_PARAMETER, ERR_NUMERICAL, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_UNSUPPORTED, ERR_INTERNAL = range(9)
F64, F32 = 0, 1
FLAG_OMEGA_GIVEN = 0x1
FLAG_NO_GRAPH = 0x2
FLAG_STAGE_TIMES = 0x4
FLAG_BASIC = 0x8
FLAG_TF32 = 0x10
FLAG_OZAKI = 0x20
FLAG_DMMA = 0x40


class SorsvdDesc(ctypes.Structure):
    _fields_ = [("m", c_i64), ("n", c_i64), ("lda", c_i64), ("k", c_i32), ("ell", c_i32), ("q", c_i32),
                ("single_pass", c_i32), ("seed", c_u64), ("dtype", c_i32), ("flags", c_u32), ("m_global", c_i64)]


class SorsvdStats(ctypes.Structure):
    _fields_ = [("ms_total", ctypes.c_double), ("ms_h2d", ctypes.c_double), ("ms_d2h", ctypes.c_double),
                ("ms_passes", ctypes.c_double), ("ms_qr", ctypes.c_double), ("ms_project", ctypes.c_double),
                ("ms_svd", ctypes.c_double), ("ms_basis", ctypes.c_double), ("flops_passes", ctypes.c_double),
                ("bytes_passes", ctypes.c_double), ("passes", c_i32), ("method", c_i32), ("launches", c_i32),
                ("jacobi_sweeps", c_i32), ("pass_kind", c_i32), ("oz_planes", c_i32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class RpcaDesc(ctypes.Structure):
    _fields_ = [("m", c_i64), ("n", c_i64), ("ldd", c_i64), ("lam", ctypes.c_double), ("mu0", ctypes.c_double),
                ("mu_bar_factor", ctypes.c_double), ("rho", ctypes.c_double), ("tol", ctypes.c_double),
                ("max_iter", c_i32), ("ell", c_i32), ("q", c_i32), ("dtype", c_i32), ("seed", c_u64),
                ("flags", c_u32), ("pad_", c_i32), ("m_global", c_i64)]


class RpcaRes(ctypes.Structure):
    _fields_ = [("iterations", c_i32), ("rank_l", c_i32), ("converged", c_i32), ("launches", c_i32),
                ("nnz_s", c_i64), ("rel_error", ctypes.c_double), ("mu0", ctypes.c_double),
                ("ms_total", ctypes.c_double), ("ms_h2d", ctypes.c_double), ("ms_d2h", ctypes.c_double)]


# Every symbol the header declares: (name, restype, argtypes)
SIGNATURES = [
    ("sorsvd_ctx_create", c_i32, [ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("sorsvd_nccl_unique_id", c_i32, [c_vp]),
    ("sorsvd_ozaki_products", c_i32, []),
    ("sorsvd_nccl_selftest", c_i32, [c_i32, c_i64, c_dp]),
    ("sorsvd_ctx_create_dist", c_i32, [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp, ctypes.POINTER(c_vp)]),
    ("sorsvd_ctx_destroy", None, [c_vp]),
    ("sorsvd_emu_group_create", c_i32, [ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("sorsvd_emu_group_destroy", None, [c_vp]),
    ("sorsvd_ctx_create_emulated", c_i32, [ctypes.c_int, ctypes.c_int, c_vp, ctypes.POINTER(c_vp)]),
    ("sorsvd_last_error", ctypes.c_char_p, [c_vp]),
    ("sorsvd_set_stream", c_i32, [c_vp, c_vp]),
    ("sorsvd_ctx_set_option", c_i32, [c_vp, c_i32, c_i64]),
    ("sorsvd_ctx_rank", c_i32, [c_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("sorsvd_sor_svd_power", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_vp, c_dp, c_dp, c_dp, c_dp,
                                     ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_sor_svd_power_device", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_vp, c_vp, c_vp, c_vp, c_vp,
                                            ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_sor_svd_power_batch", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_i32, ctypes.POINTER(c_u64), c_vp,
                                           c_dp, c_dp, c_dp, c_dp, ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_sor_svd_power_batch_device", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_i32, ctypes.POINTER(c_u64),
                                                  c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_r_svd", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_vp, c_dp, c_dp, c_dp, c_dp,
                             ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_r_svd_device", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_vp, c_vp, c_vp, c_vp, c_vp,
                                    ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_tsr_svd", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_vp, c_dp, c_dp, c_dp, c_dp, c_dp,
                               ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_tsr_svd_device", c_i32, [c_vp, ctypes.POINTER(SorsvdDesc), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      ctypes.POINTER(SorsvdStats)]),
    ("sorsvd_rpca_alm", c_i32, [c_vp, ctypes.POINTER(RpcaDesc), c_dp, c_dp, c_dp, ctypes.POINTER(RpcaRes)]),
    ("sorsvd_rpca_alm_device", c_i32, [c_vp, ctypes.POINTER(RpcaDesc), c_vp, c_vp, c_vp, ctypes.POINTER(RpcaRes)]),
    ("sorsvd_approx_error_fro_device", c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_i32, c_i32, c_vp, c_i64, c_vp,
                                               c_vp, c_i64, c_dp]),
    ("sorsvd_approx_error_spectral_device", c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_i32, c_i32, c_vp, c_i64, c_vp,
                                                    c_vp, c_i64, c_dp]),
    ("sorsvd_norm_spectral_device", c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_u64, c_dp]),
    ("sorsvd_gaussian_matrix_device", c_i32, [c_vp, c_i64, c_i64, c_u64, c_vp, c_i64]),
    ("sorsvd_gen_lowrank_device", c_i32, [c_vp, c_i64, c_i64, c_i32, c_dp, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, c_u64, c_i64, c_i64, c_i32, c_vp, c_i64]),
    ("sorsvd_gen_rpca_instance_device", c_i32, [c_vp, c_i64, c_i32, ctypes.c_longlong, c_u64, c_vp, c_vp, c_vp]),
    ("sorsvd_rpca_telemetry", c_i32, [c_vp, c_i32, c_dp, ctypes.POINTER(c_i32)]),
    ("sorsvd_estimate_rank_bound", c_i32, [c_vp, c_i64, c_i64, c_dp, c_i64, ctypes.POINTER(c_i64), c_dp, c_dp]),
    ("sorsvd_estimate_rank_bound_device", c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, ctypes.POINTER(c_i64), c_dp, c_dp]),
    ("sorsvd_sord_header", c_i32, [ctypes.c_char_p, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    ("sorsvd_load_sord_device", c_i32, [c_vp, ctypes.c_char_p, c_vp, c_i64, c_i32]),
    ("sorsvd_save_sord_device", c_i32, [c_vp, ctypes.c_char_p, c_vp, c_i64, c_i64, c_i64]),
    ("sorsvd_thin_qr_device", c_i32, [c_vp, c_i64, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64]),
    ("sorsvd_small_svd_device", c_i32, [c_vp, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64,
                                        ctypes.POINTER(c_i32)]),
    ("sorsvd_matmul_device", c_i32, [c_vp, c_i32, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64]),
    ("sorsvd_matmul_f32_device", c_i32, [c_vp, c_i32, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64]),
    ("sorsvd_measure_peaks", c_i32, [c_vp, c_dp, c_dp]),
    ("sorsvd_debug_buffer", c_i32, [c_vp, ctypes.c_char_p, c_vp, c_i64]),
    ("sorsvd_ozaki_scales_device", c_i32, [c_vp, c_i64, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp]),
    ("sorsvd_pass_ozaki_device", c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32,
                                         c_dp, c_dp]),
    ("sorsvd_pass_device", c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_dp,
                                   ctypes.POINTER(c_i32)]),
    ("sorsvd_pass_f32_device", c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_dp,
                                       ctypes.POINTER(c_i32)]),
    ("sorsvd_pass_f32a_device", c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32, c_dp,
                                        ctypes.POINTER(c_i32)]),
    ("sorsvd_sub_seed", c_u64, [c_u64, c_u64]),
    ("sorsvd_gaussian_matrix", c_i32, [c_i64, c_i64, c_u64, c_dp, ctypes.c_int]),
    ("sorsvd_gaussian_rows", c_i32, [c_i64, c_i64, c_i64, c_u64, c_dp, ctypes.c_int]),
    ("sorsvd_flop_estimate", ctypes.c_longlong, [ctypes.c_longlong] * 5 + [ctypes.c_int]),
    ("sorsvd_validate_sketch", c_i32, [c_i64, c_i64, c_i32, c_i32, c_i32]),
    ("sorsvd_version", ctypes.c_char_p, []),
]

_lib = None


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"sm_100a library not found at {LIB_PATH}; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib
