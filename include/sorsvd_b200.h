/*
 * sorsvd_b200.h — C ABI of the B200-native SOR-SVD hot path.
 *
 * This is the drop-in boundary for the reference's header-only C++ API
 * (/root/reference/proj/include/sorsvd). Plain pointers and sizes only; no
 * torch or C++ types cross it. Matrices are row-major, element (i,j) at
 * p[i*ld + j], exactly the reference Matrix layout (matrix.hpp:61).
 *
 * Error convention: every entry point returns a sorsvd_status. The codes
 * mirror the reference exception taxonomy (errors.hpp:9-26):
 *   SORSVD_ERR_SHAPE     <-> sorsvd::shape_error      (errors.hpp:9)
 *   SORSVD_ERR_PARAMETER <-> sorsvd::parameter_error  (errors.hpp:14)
 *   SORSVD_ERR_NUMERICAL <-> sorsvd::numerical_error  (errors.hpp:24)
 * plus device-side failures. sorsvd_last_error() returns the message of the
 * last failure on a context (the reference's exception what()).
 *
 * Threading: a context is bound to one device and is not thread-safe; use one
 * per host thread (the reference functions are pure and re-entrant,
 * the context only owns streams, workspaces and graphs).
 */
#ifndef SORSVD_B200_H
#define SORSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sorsvd_status {
    SORSVD_OK = 0,
    SORSVD_ERR_SHAPE = 1,
    SORSVD_ERR_PARAMETER = 2,
    SORSVD_ERR_NUMERICAL = 3,
    SORSVD_ERR_CUDA = 4,
    SORSVD_ERR_NCCL = 5,
    SORSVD_ERR_OOM = 6,
    SORSVD_ERR_UNSUPPORTED = 7,
    SORSVD_ERR_INTERNAL = 8
} sorsvd_status;

typedef enum sorsvd_dtype { SORSVD_F64 = 0, SORSVD_F32 = 1 } sorsvd_dtype;

/* SketchMethod (sketch.hpp:13) */
typedef enum sorsvd_method { SORSVD_SOR = 0, SORSVD_SOR_POWER = 1, SORSVD_RSVD = 2, SORSVD_TSR = 3 } sorsvd_method;

/* FlopVariant (sketch.hpp:176) */
typedef enum sorsvd_flop_variant {
    SORSVD_FLOPS_SOR_3PASS = 0,
    SORSVD_FLOPS_SOR_2PASS = 1,
    SORSVD_FLOPS_SOR_POWER_2Q3 = 2,
    SORSVD_FLOPS_SOR_POWER_2Q2 = 3
} sorsvd_flop_variant;

/* desc.flags */
#define SORSVD_FLAG_OMEGA_GIVEN 0x1u  /* use the caller's Omega instead of gaussian_matrix(n,ell,seed) */
#define SORSVD_FLAG_NO_GRAPH 0x2u     /* issue kernels directly (no CUDA-graph replay) */
#define SORSVD_FLAG_STAGE_TIMES 0x4u  /* per-stage CUDA-event times in stats (implies NO_GRAPH) */
#define SORSVD_FLAG_BASIC 0x8u        /* sor_svd semantics: require q == 0 (sketch.hpp:116-119) */
#define SORSVD_FLAG_TF32 0x10u        /* dtype F32: passes on the TF32 tensor cores (fast; ~1e-3 relative,
                                         resolves only sketch directions above the TF32 rounding level).
                                         Default for F32: FP64 arithmetic on the FP32-stored A. */
#define SORSVD_FLAG_OZAKI 0x20u       /* FP64 arithmetic (F64, or F32 storage) with the A-streaming passes
                                         computed as exact int8 slice products on the tcgen05 tensor cores
                                         (Ozaki scheme: 7 signed byte digits of a 55-bit fixed point, the 34
                                         products with digit levels >= 5): error at or below the reference
                                         dgemm's own sum rounding. Default for large passes: ell >= 32 and
                                         m n ell >= 2^30.5 when the call's int8 digit planes of A fit in HBM
                                         (SORSVD_OPT_OZAKI_PLANES), >= 2^36 otherwise; this flag forces it */
#define SORSVD_FLAG_DMMA 0x40u        /* force the FP64 DMMA passes (the default below that size) */

typedef struct sorsvd_ctx sorsvd_ctx;

/* Problem descriptor: SketchConfig (sketch.hpp:29-34) + the matrix shape. */
typedef struct sorsvd_desc {
    int64_t m;        /* rows of A held by this rank (all rows when world == 1) */
    int64_t n;        /* columns of A */
    int64_t lda;      /* leading dimension of A (>= n) */
    int32_t k;        /* target rank */
    int32_t ell;      /* sketch size, k <= ell < min(m_global, n) */
    int32_t q;        /* power iterations */
    int32_t single_pass; /* SketchConfig::single_pass: M_approx core, 2q+2 passes (sketch.hpp:100-104) */
    uint64_t seed;    /* Omega = gaussian_matrix(n, ell, seed) unless OMEGA_GIVEN */
    int32_t dtype;    /* sorsvd_dtype of A: SORSVD_F64, or SORSVD_F32 (FP32 storage; see SORSVD_FLAG_TF32) */
    uint32_t flags;
    int64_t m_global; /* total rows over all ranks (0 -> m) */
} sorsvd_desc;

typedef struct sorsvd_stats {
    double ms_total;     /* device time of the call (CUDA events) */
    double ms_h2d;       /* host->device copies (host-buffer entry points) */
    double ms_d2h;       /* device->host copies */
    double ms_passes;    /* STAGE_TIMES only: the 2q+2 sketch passes */
    double ms_qr;        /* STAGE_TIMES only: TSQR of T1 and T2 */
    double ms_project;   /* STAGE_TIMES only: M = Q1^T A Q2 */
    double ms_svd;       /* STAGE_TIMES only: Jacobi SVD of M */
    double ms_basis;     /* STAGE_TIMES only: U = Q1 Ut, V = Q2 Vt */
    double flops_passes; /* 2*m*n*ell*passes (BASELINE metric numerator) */
    double bytes_passes; /* m*n*sizeof(A)*passes */
    int32_t passes;      /* LowRankApprox::passes (sketch.hpp:104) */
    int32_t method;      /* sorsvd_method */
    int32_t launches;    /* kernel launches issued for the call */
    int32_t jacobi_sweeps;
    int32_t pass_kind;   /* how the passes over A ran: 0 FP64 DMMA, 1 Ozaki int8 (FP64), 2 TF32 */
    int32_t oz_planes;   /* pass_kind 1: 1 = the passes streamed digit planes of A cut once per call
                            (SORSVD_OPT_OZAKI_PLANES), 0 = A converted inside every pass */
} sorsvd_stats;

/* ---- context -------------------------------------------------------------- */
int sorsvd_ctx_create(int device, sorsvd_ctx** out);
/* Multi-GPU: one context per rank (one process per GPU). unique_id is the
 * 128-byte NCCL id produced by sorsvd_nccl_unique_id on rank 0 and broadcast
 * by the caller (e.g. torch.distributed). */
int sorsvd_nccl_unique_id(void* out128);
/* int8 digit products per FP64 multiply-add in this build's Ozaki passes (bench.py's int8 op count). */
int sorsvd_ozaki_products(void);
/* One-GPU check of the NCCL binding (dlopen of libnccl.so.2, call signatures, stream order): a
 * one-rank communicator on `device`, in-place all-reduce + all-gather of `count` doubles; both must
 * return the input (max_abs_err = 0). Only one GPU is reachable in the build environment, so this
 * is the hardware test of the calls the row-sharded contexts issue. */
int sorsvd_nccl_selftest(int device, int64_t count, double* max_abs_err);
int sorsvd_ctx_create_dist(int device, int rank, int world, const void* unique_id128, sorsvd_ctx** out);
void sorsvd_ctx_destroy(sorsvd_ctx* ctx);
/* Per-context algorithm options (defaults are the tuned choices; tests use
 * these to cross-check kernel variants against each other). */
#define SORSVD_OPT_JACOBI 1          /* value: sorsvd_jacobi_variant */
#define SORSVD_OPT_SORD_CHUNK_MB 2   /* value: staging chunk of the SORD loader, MiB (default 64) */
#define SORSVD_OPT_OZAKI_MULTICAST 6 /* value: 1 = the planes passes run the column-chunk CTAs of a row tile as one thread-block
                                        cluster and load each A plane once per cluster (TMA multicast, multicast commits);
                                        0 (default) = every CTA loads all 7 planes itself. Same results; measured no
                                        faster on B200 (the pass is bound by shared-memory bandwidth, not by L2 -> SM) */
#define SORSVD_OPT_OZAKI_OVERLAP 7   /* value: 1 (default) = device-resident calls of the planes engine cut row chunk i + 1 into
                                        planes on a second stream while the first pass sweeps chunk i; 0 = convert all of A,
                                        then pass (same bits) */
#define SORSVD_OPT_UPLOAD_TN 8       /* value: 1 (default) = the pipelined host upload also runs the first A^T T1 pass chunk by chunk
                                        (one K range per row chunk, added in chunk order): same accuracy, last bits differ
                                        from the device-resident call; 0 = only the first pass rides under the upload and
                                        the host call returns the device call's bits */
#define SORSVD_OPT_NCCL_GRAPH 9      /* value: 0 (default) = contexts with an NCCL communicator enqueue every call stream-ordered
                                        (the schedule the emulated-group tests cover); 1 = capture the call, collectives
                                        included, in a CUDA graph like single-GPU contexts do */
#define SORSVD_OPT_UPLOAD_CHUNK_MB 5 /* value: MiB per row chunk of A in host-buffer calls of the Ozaki planes engine (default
                                        1536): A uploads in chunks on a copy stream and each chunk is converted and swept
                                        by the first pass T1 = A Omega while the next one crosses PCIe */
#define SORSVD_OPT_FUSED_PAIR 4      /* value: 1 (default) = narrow sketches over narrow matrices (ell <= 16, n <= 512, FP64)
                                        run each power step T1 = A X, T2 = A^T T1 and the projection as ONE sweep over A
                                        (skinny_pair_f64.cuh); 0 = separate NN / TN GEMM passes */
#define SORSVD_OPT_OZAKI_PLANES 3    /* value: 1 (default) = the Ozaki engine cuts A into int8 digit planes once per
                                        call (7/8 of an FP64 A of extra HBM, taken when it fits) and its passes
                                        stream them; 0 = always convert A inside every pass */
#define SORSVD_JACOBI_AUTO 0         /* by k: CTA / point-to-point ring / barrier ring / rotation log */
#define SORSVD_JACOBI_BARRIER 1      /* barrier cluster ring instead of the point-to-point ring */
#define SORSVD_JACOBI_ROTLOG 2       /* the k > 256 rotation-log kernel at any k >= 8 */
int sorsvd_ctx_set_option(sorsvd_ctx* ctx, int32_t key, int64_t value);
/* In-process emulation of `world` ranks on one device (tests): one context
 * per rank, each driven by its own host thread; collectives become host
 * barriers plus device sums. Same schedule as the NCCL path, graphs off. */
typedef struct sorsvd_emu_group sorsvd_emu_group;
int sorsvd_emu_group_create(int world, sorsvd_emu_group** out);
void sorsvd_emu_group_destroy(sorsvd_emu_group* group);
int sorsvd_ctx_create_emulated(int device, int rank, sorsvd_emu_group* group, sorsvd_ctx** out);
const char* sorsvd_last_error(const sorsvd_ctx* ctx);
/* Bind the context to a caller stream (cudaStream_t). NULL (the default for a
 * new context) means the legacy default stream: the context computes on its own
 * stream and every call is ordered after the work already queued on the
 * default stream, and before anything queued there after the call. */
int sorsvd_set_stream(sorsvd_ctx* ctx, void* stream);
int sorsvd_ctx_rank(const sorsvd_ctx* ctx, int* rank, int* world);

/* ---- sor_svd_power (sketch.hpp:87) / sor_svd (sketch.hpp:116) ---------------
 * Host buffers: A (m x lda), omega (n x ell, or NULL -> drawn from seed),
 * outputs U (m x k), sigma (k), V (n x k). Includes H2D/D2H. */
int sorsvd_sor_svd_power(sorsvd_ctx* ctx, const sorsvd_desc* desc, const void* A, const double* omega,
                         double* U, double* sigma, double* V, sorsvd_stats* stats);
/* Device buffers (already resident in HBM on the context's device). When
 * omega is NULL the host draws gaussian_matrix(n, ell, seed) and uploads it. */
int sorsvd_sor_svd_power_device(sorsvd_ctx* ctx, const sorsvd_desc* desc, const void* dA,
                                const double* dOmega, double* dU, double* dSigma, double* dV,
                                sorsvd_stats* stats);

/* ---- batched trials (the Monte-Carlo loop of bounds.hpp:262-379) -------------
 * `trials` independent sor_svd_power calls on the same A, trial t drawn from
 * seeds[t] (or desc.seed + t when seeds is NULL, the harness's convention,
 * bounds.hpp:288), or from omegas (trials x n x ell) with OMEGA_GIVEN. Every
 * pass over A serves all trials in one launch. Outputs are stacked per trial:
 * U trials x m x k, sigma trials x k, V trials x n x k. Each trial matches the
 * single call with its seed to the parity tolerances (not bitwise: the wider
 * passes sum in a different order). Row-sharded contexts: every rank passes its
 * row block (desc.m local, desc.m_global total) and the same seeds; U comes back
 * row-sharded per trial. ell <= 256; no TF32, no single_pass. */
int sorsvd_sor_svd_power_batch(sorsvd_ctx* ctx, const sorsvd_desc* desc, int32_t trials, const uint64_t* seeds,
                               const void* A, const double* omegas, double* U, double* sigma, double* V,
                               sorsvd_stats* stats);
int sorsvd_sor_svd_power_batch_device(sorsvd_ctx* ctx, const sorsvd_desc* desc, int32_t trials,
                                      const uint64_t* seeds, const void* dA, const double* dOmegas, double* dU,
                                      double* dSigma, double* dV, sorsvd_stats* stats);

/* ---- baselines: r_svd (sketch.hpp:124) / tsr_svd (sketch.hpp:139) -----------
 * Same descriptor; desc.k is ignored (all ell triplets are returned: U m x ell,
 * sigma ell, V n x ell), single_pass and BASIC are ignored, tsr ignores q.
 * r_svd: Omega = gaussian_matrix(n, ell, seed) unless OMEGA_GIVEN; passes 2q+2.
 * tsr_svd: Psi1 = gaussian_matrix(n, ell, seed), Psi2 = gaussian_matrix(m, ell,
 * seed ^ 1) unless OMEGA_GIVEN (then both must be given); passes 1 (the two
 * sketches are two launches over A in this build). Row-sharded contexts
 * (desc.m_global): the rank's rows of A, and for tsr_svd the rank's rows of Psi2
 * (drawn as rows [row0, row0 + m) of the m_global x ell matrix, sorsvd_gaussian_rows);
 * U row-sharded, sigma and V replicated. No TF32. */
int sorsvd_r_svd(sorsvd_ctx* ctx, const sorsvd_desc* desc, const void* A, const double* omega, double* U,
                 double* sigma, double* V, sorsvd_stats* stats);
int sorsvd_r_svd_device(sorsvd_ctx* ctx, const sorsvd_desc* desc, const void* dA, const double* dOmega,
                        double* dU, double* dSigma, double* dV, sorsvd_stats* stats);
int sorsvd_tsr_svd(sorsvd_ctx* ctx, const sorsvd_desc* desc, const void* A, const double* psi1, const double* psi2,
                   double* U, double* sigma, double* V, sorsvd_stats* stats);
int sorsvd_tsr_svd_device(sorsvd_ctx* ctx, const sorsvd_desc* desc, const void* dA, const double* dPsi1,
                          const double* dPsi2, double* dU, double* dSigma, double* dV, sorsvd_stats* stats);

/* ---- RPCA by inexact ALM --------------- */
typedef struct sorsvd_rpca_desc {
    int64_t m, n, ldd;
    double lambda;        /* <= 0 -> 1/sqrt(max(m,n)) */
    double mu0;           /* <= 0 -> 1.25/sigma_1(D) estimated on the device */
    double mu_bar_factor; /* mu_bar = mu_bar_factor * mu0 (default 1e7) */
    double rho;           /* 1.6 */
    double tol;           /* 1e-7 */
    int32_t max_iter;
    int32_t ell;          /* sketch size = truncation rank */
    int32_t q;
    int32_t dtype;
    uint64_t seed;        /* iteration it uses seed + it */
    uint32_t flags;
    int32_t pad_;
    int64_t m_global;     /* multi-GPU: total rows (m = this rank's row block); <= 0 -> m */
} sorsvd_rpca_desc;

typedef struct sorsvd_rpca_result {
    int32_t iterations;
    int32_t rank_l;      /* count of shrunk sigma > 1e-8 * max */
    int32_t converged;
    int32_t launches;
    int64_t nnz_s;
    double rel_error;    /* ||D-L-S||_F / ||D||_F */
    double mu0;
    double ms_total;
    double ms_h2d;
    double ms_d2h;
} sorsvd_rpca_result;

/* Host buffers D (m x ldd) -> L, S (m x n, dense row-major). */
int sorsvd_rpca_alm(sorsvd_ctx* ctx, const sorsvd_rpca_desc* desc, const double* D, double* L, double* S,
                    sorsvd_rpca_result* res);
/* Device buffers. L may be NULL (factors only). */
int sorsvd_rpca_alm_device(sorsvd_ctx* ctx, const sorsvd_rpca_desc* desc, const double* dD, double* dL,
                           double* dS, sorsvd_rpca_result* res);

/* Per-iteration telemetry of the context's last rpca_alm call ("per-iteration telemetry
 * CSV (iter, mu, rel_error, rank_l, nnz_s)"): *rows = iterations run; up to cap_rows rows of those 5
 * values (as doubles) are written to out (may be NULL to query the count). Multi-rank: nnz_s is the
 * global count. */
int sorsvd_rpca_telemetry(sorsvd_ctx* ctx, int32_t cap_rows, double* out, int32_t* rows);

/* estimate_rank_bound(x) = ceil((||X||_* / ||X||_F)^2) (PAPER Eq. 66), the input of
 * rpca_default_config's ell = min(2 * bound, min(m,n) - 1). Device FP64 X, min(m,n) <=
 * 512 (thin QR + Jacobi SVD of R). Zero matrix -> SORSVD_ERR_PARAMETER. nuclear / frobenius (may be
 * NULL) receive the two norms. Row-sharded contexts (dX = this rank's rows, m >= n on every rank,
 * n <= 256): the ranks' R factors are gathered and factored again; every rank gets the same bound. */
int sorsvd_estimate_rank_bound_device(sorsvd_ctx* ctx, int64_t m, int64_t n, const double* dX, int64_t ldx,
                                      int64_t* bound, double* nuclear, double* frobenius);
/* The same on a host matrix (uploaded inside). */
int sorsvd_estimate_rank_bound(sorsvd_ctx* ctx, int64_t m, int64_t n, const double* X, int64_t ldx, int64_t* bound,
                               double* nuclear, double* frobenius);

/* approx_error(a, x, NormKind::frobenius) (sketch.hpp:168-172) on device
 * buffers: ||A - U diag(sigma) V^T||_F in one fused pass over A (A m x lda,
 * FP64 or FP32 by dtype; U m x ldu, V n x ldv, first k columns). Multi-rank:
 * A and U are this rank's row block and the sum of squares is reduced over
 * ranks. */
int sorsvd_approx_error_fro_device(sorsvd_ctx* ctx, int64_t m, int64_t n, const void* dA, int64_t lda, int32_t dtype,
                                   int32_t k, const double* dU, int64_t ldu, const double* dSigma, const double* dV,
                                   int64_t ldv, double* err);

/* approx_error(a, x, NormKind::spectral) (sketch.hpp:168-172; the reference: dgesdd 'N' of the
 * dense difference, dense.hpp:173-176): E = A - U diag(sigma) V^T is formed on the device and
 * sigma_1(E) comes from norm(spectral) below. Row-sharded contexts (A, U = this rank's rows;
 * n <= 1024): the Gram matrix of E is summed over the ranks. The bound harness
 * (bounds.hpp:289-290) asks for both norms per trial. */
int sorsvd_approx_error_spectral_device(sorsvd_ctx* ctx, int64_t m, int64_t n, const void* dA, int64_t lda,
                                        int32_t dtype, int32_t k, const double* dU, int64_t ldu,
                                        const double* dSigma, const double* dV, int64_t ldv, double* err);

/* norm(a, NormKind::spectral) (dense.hpp:173-176) of a device FP64 matrix: min(m, n) <= 1024 ->
 * Gram matrix, 12 rescaled squarings and a 16-column Rayleigh-Ritz step (<= 1e-12 relative
 * against dgesdd, clustered leading values included); larger -> block subspace iteration with
 * Rayleigh-Ritz to a stationary value (seed draws its start block). Also RPCA's mu0.
 * Row-sharded contexts (dA = this rank's rows): n <= 1024, G = sum over ranks of A_r^T A_r. */
int sorsvd_norm_spectral_device(sorsvd_ctx* ctx, int64_t m, int64_t n, const double* dA, int64_t lda, uint64_t seed,
                                double* out);

/* ---- test-matrix generators on the device (matrixgen.hpp) ---------------
 * gaussian_matrix(rows, cols, seed) (random.hpp:60-65) filled on the device: the reference's
 * splitmix64 words and uniforms, with the device's log / sincos (a few ulp from the host draw of
 * sorsvd_gaussian_matrix, which is bit-identical to the reference). */
int sorsvd_gaussian_matrix_device(sorsvd_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, double* dOut, int64_t ld);
/* Rows [row0, row0 + m) of the m_global x n matrix (x_scale X) diag(sigma) (y_scale Y)^T + noise_std E
 * (BASELINE.json configs 1, 3, 5): X = gaussian_matrix(m_global, r, sub_seed(seed, 1)) and
 * Y = gaussian_matrix(n, r, sub_seed(seed, 2)) drawn on the host (reference-exact) and uploaded; row i of E =
 * NormalStream(sub_seed(sub_seed(seed, 3), i)) drawn in the kernel. sigma: r host values. dtype selects
 * FP64 or FP32 storage of A (lda in elements). m_global <= 0 -> row0 + m. */
int sorsvd_gen_lowrank_device(sorsvd_ctx* ctx, int64_t m, int64_t n, int32_t r, const double* sigma, double x_scale,
                              double y_scale, double noise_std, uint64_t seed, int64_t row0, int64_t m_global,
                              int32_t dtype, void* dA, int64_t lda);
/* gen_rpca_instance(n, r, s, seed) (matrixgen.hpp:99-124): X = L + S (n x n, dense) on the device; dL / dS
 * (may be NULL) receive the two components. The support and signs of S are identical to the reference's. */
int sorsvd_gen_rpca_instance_device(sorsvd_ctx* ctx, int64_t n, int32_t r, long long s, uint64_t seed, double* dX,
                                    double* dL, double* dS);

/* ---- SORD matrix files ----------------------------------------
 * "SORD", u32 version = 1, u64 rows, u64 cols, then rows*cols little-endian
 * float64, row-major. The loader streams the file into device memory through two
 * pinned staging buffers (the disk read of one chunk overlaps the copy of the
 * other; the host never holds the matrix), optionally rounding to FP32 on the
 * device (dtype SORSVD_F32, e.g. a 137 GB FP64 file into 68.7 GB of HBM). */
int sorsvd_sord_header(const char* path, int64_t* rows, int64_t* cols);
int sorsvd_load_sord_device(sorsvd_ctx* ctx, const char* path, void* dA, int64_t lda, int32_t dtype);
int sorsvd_save_sord_device(sorsvd_ctx* ctx, const char* path, const double* dA, int64_t rows, int64_t cols,
                            int64_t lda);

/* ---- stage-level entry points (kernel unit tests) ------------------------- */
/* thin_qr (dense.hpp:114): dT (m x ldt) -> dQ (m x ldq), dR (k x ldr); device. */
int sorsvd_thin_qr_device(sorsvd_ctx* ctx, int64_t m, int32_t k, const double* dT, int64_t ldt, double* dQ,
                          int64_t ldq, double* dR, int64_t ldr);
/* full_svd of a square k x k (dense.hpp:65): device buffers, row-major. */
int sorsvd_small_svd_device(sorsvd_ctx* ctx, int32_t k, const double* dM, int64_t ldm, double* dU,
                            int64_t ldu, double* dS, double* dV, int64_t ldv, int32_t* sweeps);
/* matmul (dense.hpp:20) restricted to the skinny shapes of the path:
 * C = op(A) * B, op(A) = A (ta=0, A is M x K) or A^T (ta=1, A is K x M). */
int sorsvd_matmul_device(sorsvd_ctx* ctx, int32_t ta, int64_t M, int64_t K, int32_t N, const double* dA,
                         int64_t lda, const double* dB, int64_t ldb, double* dC, int64_t ldc);

/* FP32 operands on the tensor cores (tcgen05 kind::tf32, FP32 accumulation);
 * A must be 16-byte aligned with lda % 4 == 0. */
int sorsvd_matmul_f32_device(sorsvd_ctx* ctx, int32_t ta, int64_t M, int64_t K, int32_t N, const float* dA,
                             int64_t lda, const float* dB, int64_t ldb, float* dC, int64_t ldc);

/* ---- measurement (bench.py roofline) --------------------------------------- */
/* Live FP64 DMMA peak (TFLOP/s, burst) and streaming HBM read (GB/s). */
int sorsvd_measure_peaks(sorsvd_ctx* ctx, double* fp64_tflops, double* hbm_read_gbs);
/* One A-streaming pass (sketch.hpp:95 when ta = 0, :96 when ta = 1) repeated
 * `reps` times between CUDA events; dX / dT padded to ld = ell rounded up to 8
 * (or to 128 when ell > 128). Reports the average pass time. */
/* Test hook: copy count doubles of the context workspace buffer `name` ("T1", "T2", "Q1", "Q2",
 * "Mk", ...) to the device pointer dst. */
int sorsvd_debug_buffer(sorsvd_ctx* ctx, const char* name, double* dst, int64_t count);
/* The Ozaki scale exponents of A (tests): row_e[m], col_e[n] (device), max|.| < 2^e. */
int sorsvd_ozaki_scales_device(sorsvd_ctx* ctx, int64_t m, int64_t n, int64_t lda, int32_t dtype, const void* dA,
                               int32_t* row_e, int32_t* col_e);
/* One Ozaki pass (SORSVD_FLAG_OZAKI's kernels) C = op(A) X for tests / timing; dtype of A F64 or F32,
 * X and C FP64 padded like sorsvd_pass_device. ms_scales: the per-call max|A| read. */
int sorsvd_pass_ozaki_device(sorsvd_ctx* ctx, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell,
                             int32_t dtype, const void* dA, const double* dX, double* dT, int32_t reps,
                             double* ms_avg, double* ms_scales);
int sorsvd_pass_device(sorsvd_ctx* ctx, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell, const double* dA,
                       const double* dX, double* dT, int32_t reps, double* ms_avg, int32_t* launches_per_pass);

/* The same for an fp32 A on the TF32 tensor cores (dX / dT padded to ell
 * rounded up to 32, or to 256 when ell > 256). */
int sorsvd_pass_f32_device(sorsvd_ctx* ctx, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell,
                           const float* dA, const float* dX, float* dT, int32_t reps, double* ms_avg,
                           int32_t* launches_per_pass);

/* FP32-stored A with FP64 arithmetic (the default F32 sor path): dX / dT are
 * FP64 with the sorsvd_pass_device padding. */
int sorsvd_pass_f32a_device(sorsvd_ctx* ctx, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell,
                            const float* dA, const double* dX, double* dT, int32_t reps, double* ms_avg,
                            int32_t* launches_per_pass);

/* ---- host helpers mirroring random.hpp / sketch.hpp ----------------------- */
uint64_t sorsvd_sub_seed(uint64_t seed, uint64_t stream);                    /* random.hpp:24 */
int sorsvd_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out, int nthreads);
/* Rows [row0, row0 + rows) of gaussian_matrix(., cols, seed) (the splitmix64 stream is counter based: a row
 * block of a larger draw, e.g. one rank's rows of a sharded factor, is drawn without its prefix). */
int sorsvd_gaussian_rows(int64_t cols, int64_t row0, int64_t rows, uint64_t seed, double* out, int nthreads); /* random.hpp:60 */
long long sorsvd_flop_estimate(long long m, long long n, long long ell, long long k, long long q,
                               int variant);                                  /* sketch.hpp:178 */
int sorsvd_validate_sketch(int64_t m, int64_t n, int32_t k, int32_t ell, int32_t q); /* sketch.hpp:62 */
const char* sorsvd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SORSVD_B200_H */
