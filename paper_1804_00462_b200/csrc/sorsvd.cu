// Host runtime + C ABI for the B200 SOR-SVD hot path (include/sorsvd_b200.h).
//
// The context owns one CUDA stream (plus a side stream for the concurrent
// TSQRs), grow-only device workspaces, per-shape TSQR plans and a cache of
// captured CUDA graphs, so a repeated sor_svd_power call (benchmarks, every
// RPCA iteration) is a single cudaGraphLaunch. With world > 1 (one process
// per GPU) A is row-sharded; the Aᵀ·T1 partials and the projected core are
// summed with NCCL all-reduce and the TSQR R factors cross GPUs as an
// all-gather of k x k blocks. An in-process "emulated"
// mode runs G row shards on one GPU with the same schedule, replacing NCCL by
// on-device sums, for tests on a single B200.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sorsvd_b200.h"
#include "common.cuh"
#include "gemm_f64.cuh"
#include "host_api.hpp"
#include "jacobi_f64.cuh"
#include "peaks.cuh"
#include "rpca_f64.cuh"
#include "tc_gemm_f32.cuh"
#include "cholqr_f64.cuh"
#include "cqr_f64.cuh"
#include "mapprox_f64.cuh"
#include "jacobi_big_f64.cuh"
#include "cholc_f64.cuh"
#include "ozaki_i8.cuh"
#include "ozaki_planes_i8.cuh"
#include "gen_f64.cuh"
#include "skinny_pair_f64.cuh"
#include "smallk_f64.cuh"
#include <cfloat>

using namespace sorsvd_dev;

namespace {

struct Error {
    int status;
    std::string msg;
};

thread_local std::string g_global_err;

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw Error{e_ == cudaErrorMemoryAllocation ? SORSVD_ERR_OOM : SORSVD_ERR_CUDA,        \
                        std::string("cuda: ") + cudaGetErrorString(e_) + " at " #call};           \
    } while (0)


// NCCL is resolved lazily with dlopen so the library never pins an NCCL
// version into a process: inside torch the already-loaded libnccl.so.2 is
// reused (RTLD_NOLOAD first); elsewhere the system one is opened on first
// multi-GPU use. nccl.h is used for types only.
struct NcclApi {
    bool tried = false;
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.tried) {
        api.tried = true;
        api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!api.h) api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) api.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (api.h) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
            api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
            api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
        }
    }
    if (!api.h || !api.AllReduce || !api.CommInitRank)
        throw Error{SORSVD_ERR_NCCL, "nccl: libnccl.so.2 not loadable"};
    return api;
}

#define NCK(call)                                                                                  \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw Error{SORSVD_ERR_NCCL, std::string("nccl: ") + nccl().GetErrorString(r_) + " at " #call}; \
    } while (0)

inline int pad8(int k) { return (k + 7) & ~7; }
inline int npad(int ell) { return ell <= 128 ? pad8(ell) : ((ell + 127) / 128) * 128; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct QrPlan {
    int64_t rows = 0;
    int k = 0, Np = 0;
    bool smem = true;
    int P = 1;
    std::vector<int64_t> row0;
    std::vector<int> rcnt;
    std::vector<int> nodes;  // nodes[0] = P leaves, ..., nodes[L] = 1
    int max_leaf_rows = 0;
    // device tables
    int64_t* d_row0 = nullptr;
    int* d_rows = nullptr;
    // segmented GEMM tile tables: [0] leaves, [l] level l (l >= 1)
    std::vector<int*> t_row0, t_rows, t_seg;
    std::vector<int> t_count;
    // buffers
    std::vector<double*> R;      // per level: nodes[l] * k * k
    std::vector<double*> QN;     // per level l >= 1: nodes[l] * 2k * Np
    std::vector<double*> C;      // per level l in [0, L-1): children C's of level l+1 nodes
    std::vector<double*> SN;     // per level l >= 1: stacked [R_2i; R_2i+1] node inputs (2k x k)
    std::vector<int64_t*> n_row0;
    std::vector<int*> n_rows;
    int rb_max = 0, cmax = 1, leaf_cs = 1, node_cs = 1;
    // CholeskyQR2 fast path
    double *G1 = nullptr, *G2 = nullptr, *Ri1 = nullptr, *Ri2 = nullptr, *R1 = nullptr, *Qtmp = nullptr,
           *cwork = nullptr;
    int* flag = nullptr;
    bool hint_house = false;  // the CholeskyQR2 gate rejected this plan's last operands (RPCA reads the flag back
                              // between batches): go straight to the Householder TSQR, skip the doomed attempt
    // k > 256: shifted CholeskyQR3 (cholc_f64.cuh); R lands in R[0] with row pitch ldR
    bool big = false;
    int ldR = 0;
    double* Rp[3] = {nullptr, nullptr, nullptr};
    double* Rtmp = nullptr;
    double* Wtrsm = nullptr;  // rows x 32 GEMM part of the blocked TRSM
    double *wy_tau = nullptr, *wy_sgn = nullptr;  // compact-WY Q of a single-block Householder QR
    std::string ws_name;  // per-plan split-K workspace (the two sketches' QRs run concurrently)
    std::vector<void*> owned;
};

struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
};

}  // namespace

// In-process multi-rank emulation on one device: `world` contexts (one host
// thread each) share a group; the collectives become a host barrier plus
// device sums in fixed rank order. Exercises the multi-GPU schedule (sharded
// passes, cross-rank TSQR tree, all-reduce placement) on a single GPU; CUDA
// graphs are disabled for emulated contexts (host barriers cannot be captured).
struct sorsvd_emu_group {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    std::vector<void*> bufs;  // per-rank buffer registered for the current collective
    bool broken = false;      // a rank failed: its peers must not wait for it forever
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) throw Error{SORSVD_ERR_INTERNAL, "emulated group: a peer rank failed"};
        const long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen || broken; });
            if (generation == gen) throw Error{SORSVD_ERR_INTERNAL, "emulated group: a peer rank failed"};
        }
    }
    void poison() {
        std::lock_guard<std::mutex> lk(mu);
        broken = true;
        cv.notify_all();
    }
};

struct sorsvd_ctx {
    int opt_jacobi = SORSVD_JACOBI_AUTO;  // sorsvd_ctx_set_option(SORSVD_OPT_JACOBI)
    int opt_oz_overlap = 1;               // sorsvd_ctx_set_option(SORSVD_OPT_OZAKI_OVERLAP): conversion of row chunk i + 1
                                          // under the first pass over chunk i (device-resident calls)
    int opt_oz_multicast = 0;             // sorsvd_ctx_set_option(SORSVD_OPT_OZAKI_MULTICAST): cluster + TMA multicast of the A planes
                                          // (measured: no gain, the pass is shared-memory-bandwidth bound)
    int opt_nccl_graph = 0;               // sorsvd_ctx_set_option(SORSVD_OPT_NCCL_GRAPH): capture NCCL collectives in the call's CUDA graph
    int opt_upload_tn = 1;                // sorsvd_ctx_set_option(SORSVD_OPT_UPLOAD_TN): host-buffer planes calls also run the
                                          // first A^T pass chunk by chunk under the upload (results differ from the
                                          // device-resident call in the last bits: K ranges summed in chunk order)
    int64_t opt_upload_chunk_mb = 1536;   // sorsvd_ctx_set_option(SORSVD_OPT_UPLOAD_CHUNK_MB): host-buffer calls of the planes engine
    int opt_fused_pair = 1;               // sorsvd_ctx_set_option(SORSVD_OPT_FUSED_PAIR): 0 = separate NN / TN GEMM passes
    int64_t opt_oz_planes = 1;                // sorsvd_ctx_set_option(SORSVD_OPT_OZAKI_PLANES): 0 = convert inside every pass
    int64_t opt_sord_chunk_mb = 64;       // sorsvd_ctx_set_option(SORSVD_OPT_SORD_CHUNK_MB)
    int device = 0;
    int rank = 0, world = 1;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr, stream = nullptr, side = nullptr;
    cudaStream_t comm_stream = nullptr;  // multi-rank: all-reduces of finished T2 blocks, under the next blocks' GEMMs
    // Ordered with the legacy default stream (the caller passed no stream, e.g. torch's default
    // stream): every entry point waits for the work already queued there and makes it wait for
    // the call's own work (events), while the context computes on its own non-blocking stream
    // (CUDA graphs cannot be captured on the legacy stream).
    bool legacy_order = true;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    static constexpr int kTnBlocks = 4;
    cudaEvent_t ev_blk[kTnBlocks] = {}, ev_comm = nullptr;
    std::vector<cudaStream_t> tstreams;  // batched trials (created on first use)
    std::vector<cudaEvent_t> tevents;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_a = nullptr, ev_b = nullptr;
    cudaEvent_t ev_st[8] = {};
    cudaEvent_t ev_h[4] = {};
    std::string err;
    std::map<std::string, Buf> bufs;
    std::map<std::string, std::unique_ptr<QrPlan>> plans;
    std::map<std::string, GraphEntry> graphs;
    struct SkTable {
        std::vector<int*> dev;  // cta_seg, seg_tile, seg_k0, seg_k1, split_slot0, split_tiles, seg_slot
        int nsplit = 0, nseg = 0, nslot = 0;
    };
    std::map<std::string, SkTable> sk_tables;  // stream-K segment tables, by shape
    ncclComm_t comm = nullptr;
    sorsvd_emu_group* emu = nullptr;  // in-process multi-rank emulation (tests)
    int launches = 0;
    bool capturing = false;
    std::vector<double> host_omega;
    std::vector<cudaEvent_t> up_ev;  // pipelined host upload: one event per row chunk of A
    std::vector<double> rpca_tele;  // last rpca_alm: iterations x {mu, rel_error, rank_l, nnz_s}
    std::vector<double> host_psi2;  // tsr_svd's second test matrix (host draw)
    double* om_pin = nullptr;       // host-buffer calls: page-locked Omega draw
    size_t om_pin_n = 0;
    const int* pred = nullptr;  // predication of every launch (CholeskyQR2 vs Householder)
    int pred_skip = 0;
};

namespace {

void invalidate_graphs(sorsvd_ctx* c) {
    for (auto& kv : c->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    c->graphs.clear();
}

double* dbuf(sorsvd_ctx* c, const std::string& name, size_t count, bool zero = false) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(double);
    Buf& b = c->bufs[name];
    if (b.bytes < bytes) {
        if (c->capturing) throw Error{SORSVD_ERR_INTERNAL, "workspace growth during graph capture: " + name};
        invalidate_graphs(c);
        if (b.p) CK(cudaFree(b.p));
        b.p = nullptr;
        CK(cudaMalloc(&b.p, bytes));
        b.bytes = bytes;
        // the zero fill runs on the legacy stream, which does not order with the
        // context's non-blocking streams: wait for it here (allocation is rare)
        CK(cudaMemset(b.p, 0, bytes));
        CK(cudaStreamSynchronize(0));
    } else if (zero) {
        CK(cudaMemsetAsync(b.p, 0, bytes, c->stream));
    }
    return static_cast<double*>(b.p);
}

// Kernel attributes are process-wide (per device), and contexts may live on
// several host threads (one per emulated rank, or a caller's thread pool):
// every kernel that takes dynamic shared memory is opened up ONCE to the
// device's opt-in maximum (plus non-portable cluster sizes where it needs
// them), instead of being set to each launch's size right before the launch,
// which another thread could undo in between (a launch failure, or a
// different occupancy answer and so a different cluster shape on one rank).
std::mutex g_attr_mu;

template <typename... Args>
void allow_smem(void (*fn)(Args...), bool cluster = false) {
    static std::set<std::pair<const void*, int>> done;  // guarded by g_attr_mu
    thread_local std::set<std::pair<const void*, int>> seen;  // this thread's fast path
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const std::pair<const void*, int> key{reinterpret_cast<const void*>(fn), dev};
    if (seen.count(key)) return;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    seen.insert(key);
    if (!done.insert(key).second) return;
    int mx = 0;
    CK(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, fn));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes));
    if (cluster) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

void check_launch(sorsvd_ctx* c) {
    CK(cudaGetLastError());
    c->launches++;
}

// ---------------------------------------------------------------- GEMM ----
struct GemmCall {
    bool ta = false;
    const double* A = nullptr;
    int64_t lda = 0;
    int64_t M = 0, K = 0;
    const double* B = nullptr;
    int64_t ldb = 0;
    int N = 0;  // padded column count (multiple of 8, or of 128 when > 128)
    double* C = nullptr;
    int64_t ldc = 0;
    double alpha = 1.0;
    // segmented
    const int* tile_row0 = nullptr;
    const int* tile_rows = nullptr;
    const int* tile_seg = nullptr;
    int ntiles = 0;
    int64_t b_seg_stride = 0;
    int force_splits = 0;
    const char* ws_name = "gemm_ws";
    const float* Af = nullptr;  // FP32-storage A (FP64 arithmetic); overrides A
    // stream-K is taken when its modelled cost is below sk_bias x split-K's; the
    // A-streaming passes with one column chunk use 1.0 (measured: C2 pass 145 -> 137 us),
    // everything else keeps the margin its numerics were pinned with (the k = 512 parity
    // tests sit within 1.5x of their floor-based tolerance)
    double sk_bias = 0.95;
};

template <int FM, int FN, bool TA, bool V16, typename AT>
void launch_gemm_t(const GemmArgs& a, dim3 grid, cudaStream_t s) {
    using S = GemmShape<FM, FN, TA, AT>;
    allow_smem(gemm_f64_kernel<FM, FN, TA, V16, AT>);
    gemm_f64_kernel<FM, FN, TA, V16, AT><<<grid, kGemmThreads, S::SMEM, s>>>(a);
}

template <int FN>
void dispatch_fn(bool ta, bool v16, bool f32a, const GemmArgs& a, dim3 grid, cudaStream_t s) {
    constexpr int FM = FN <= 4 ? 4 : 2;
    if (f32a) {  // FP32-storage A: 16-byte rows required (validated by the caller)
        if (ta) launch_gemm_t<FM, FN, true, true, float>(a, grid, s);
        else launch_gemm_t<FM, FN, false, true, float>(a, grid, s);
        return;
    }
    if (ta) {
        if (v16) launch_gemm_t<FM, FN, true, true, double>(a, grid, s);
        else launch_gemm_t<FM, FN, true, false, double>(a, grid, s);
    } else {
        if (v16) launch_gemm_t<FM, FN, false, true, double>(a, grid, s);
        else launch_gemm_t<FM, FN, false, false, double>(a, grid, s);
    }
}

int gemm_bk_for(int N) {
    const int FN = N <= 128 ? N / 8 : 16;
    return gemm_bk(FN <= 4 ? 4 : 2);
}

int gemm_bm_for(int N) {
    const int FN = N <= 128 ? N / 8 : 16;
    return 64 * (FN <= 4 ? 4 : 2);
}

void run_gemm(sorsvd_ctx* c, const GemmCall& g, cudaStream_t s) {
    if (g.N <= 0 || g.N % 8 != 0 || (g.N > 128 && g.N % 128 != 0))
        throw Error{SORSVD_ERR_INTERNAL, "gemm: bad padded N"};
    const int FN = g.N <= 128 ? g.N / 8 : 16;
    const int gy = g.N <= 128 ? 1 : g.N / 128;
    const int BM = gemm_bm_for(g.N);
    const int64_t gx = g.tile_row0 ? g.ntiles : cdiv(g.M, BM);
    if (gx == 0) return;
    int S = 1;
    if (g.force_splits > 0) {
        S = g.force_splits;
    } else if (!g.tile_row0) {
        const int64_t base = gx * gy;
        const int64_t maxS = std::max<int64_t>(1, std::min<int64_t>(512, g.K / 128));
        double best = 1e300;
        // tiny outputs (Gram matrices of the CholeskyQR gates, C1 / C4 shapes): the split
        // reduction is a chain of dependent L2 round trips (16 partials per trip in
        // reduce_splits_kernel), ~48 K-rows each, not a bandwidth term
        // (reduce_splits_warp_kernel from 32 splits: 128 partials per trip; 1.0 measured
        // best of 3.0 / 1.0 / 0.375: C4 solve 9.21 / 8.89 / 8.87 ms, C1 call 0.323 / 0.312 / 0.319 ms)
        constexpr double trip_w = 1.0;
        const bool tiny = g.M * g.N <= 4096;
        for (int64_t cand = 1; cand <= maxS; ++cand) {
            const double waves = (double)cdiv(base * cand, c->num_sms);
            const double trip = tiny ? (cand >= 32 ? trip_w : 3.0) : 0.0;
            const double cost = waves * ((double)g.K / cand + 96.0) +
                                (cand > 1 ? 0.02 * cand * g.M * g.N / (double)c->num_sms + trip * cand : 0.0);
            if (cost < best * 0.999) {
                best = cost;
                S = (int)cand;
            }
        }
    }
    // stream-K when whole tiles x splits leave SMs idle: equal BK-unit shares per
    // CTA across tile boundaries, partial tiles summed by streamk_fixup_kernel
    bool streamk = false;
    const int BK = gemm_bk_for(g.N);
    const int64_t units = cdiv(g.K, BK);
    const int64_t tiles = gx * gy;
    // stream-K from 16 BK-units per tile (C1: 0.333 -> 0.321 ms per call); tiny outputs keep
    // split-K: a stream-K tile spread over ~all SMs has a fix-up that is
    // a chain of ~num_sms / 16 dependent L2 round trips per element
    // Also past one wave of tiles (the A-streaming passes: C3's NN pass is 3126 tiles =
    // 21.12 waves, so a whole-tile schedule idles 88% of the SMs for the last wave): every
    // CTA then runs ~tiles/n whole tiles plus a partial one at each end of its unit
    // range, and only those <= 2n boundary tiles go through the fix-up.
    const bool tiny_out = g.M * g.N <= 4096;
    if (!g.tile_row0 && g.force_splits == 0 && units >= 16 && !tiny_out) {
        const int64_t n = c->num_sms;
        const int BNk = g.N <= 128 ? g.N : 128;
        const double fix_elems = tiles < n ? (double)g.M * g.N : (double)std::min<int64_t>(tiles, 2 * n) * BM * BNk;
        const double sk_cost = (double)cdiv(tiles * units, n) * BK + 2 * 96.0 + 0.02 * 3 * fix_elems / (double)n;
        const double cur_cost = (double)cdiv(tiles * S, n) * ((double)g.K / S + 96.0) +
                                (S > 1 ? 0.02 * S * g.M * g.N / (double)n : 0.0);
        streamk = sk_cost < g.sk_bias * cur_cost;
    }
    GemmArgs a{};
    a.A = g.Af ? static_cast<const void*>(g.Af) : static_cast<const void*>(g.A);
    a.lda = g.lda;
    a.B = g.B;
    a.ldb = g.ldb;
    a.b_seg_stride = g.b_seg_stride;
    a.M = g.M;
    a.K = g.K;
    a.alpha = g.alpha;
    a.tile_row0 = g.tile_row0;
    a.tile_rows = g.tile_rows;
    a.tile_seg = g.tile_seg;
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    const int64_t kchunk = cdiv(cdiv(g.K, S), BK) * BK;
    a.k_chunk = std::max<int64_t>(kchunk, BK);
    double* ws = nullptr;
    if (S > 1) {
        ws = dbuf(c, g.ws_name, (size_t)S * g.M * g.ldc);
        a.C = ws;
        a.ldc = g.ldc;
        a.c_split_stride = g.M * g.ldc;
    } else {
        a.C = g.C;
        a.ldc = g.ldc;
        a.c_split_stride = 0;
    }
    std::vector<int> sk_split_tiles_h;
    const int* sk_split_slot0 = nullptr;
    const int* sk_split_tiles = nullptr;
    if (streamk) {
        const int n = c->num_sms;
        const int64_t T = tiles * units;
        char key[128];
        snprintf(key, sizeof key, "%lld:%lld:%d:%d", (long long)tiles, (long long)units, n, (int)gy);
        auto it = c->sk_tables.find(key);
        if (it == c->sk_tables.end()) {
            if (c->capturing) throw Error{SORSVD_ERR_INTERNAL, "stream-K table creation during capture"};
            std::vector<int> cta_seg{0}, seg_tile, seg_k0, seg_k1, tile_seg0(tiles + 1, 0), split, seg_slot,
                split_slot0;
            for (int cc = 0; cc < n; ++cc) {
                int64_t u0 = cc * T / n, u1 = (cc + 1) * T / n;
                while (u0 < u1) {
                    const int64_t t = u0 / units, k0 = u0 - t * units, k1 = std::min<int64_t>(units, k0 + (u1 - u0));
                    seg_tile.push_back((int)t);
                    seg_k0.push_back((int)k0);
                    seg_k1.push_back((int)k1);
                    u0 += k1 - k0;
                }
                cta_seg.push_back((int)seg_tile.size());
            }
            for (size_t q = 0; q < seg_tile.size(); ++q) tile_seg0[seg_tile[q] + 1]++;
            for (int64_t t = 0; t < tiles; ++t) {
                if (tile_seg0[t + 1] > 1) split.push_back((int)t);
                tile_seg0[t + 1] += tile_seg0[t];
            }
            // partial segments get compact workspace slots, in segment order: the slots of
            // one split tile are then a contiguous range, and the ranges follow `split`
            int slot = 0;
            for (size_t q = 0; q < seg_tile.size(); ++q) {
                const bool whole = seg_k0[q] == 0 && seg_k1[q] == units;
                seg_slot.push_back(whole ? -1 : slot);
                if (!whole) {
                    if (split_slot0.empty() || seg_tile[q] != seg_tile[q - 1] || seg_slot[q - 1] < 0)
                        split_slot0.push_back(slot);
                    ++slot;
                }
            }
            split_slot0.push_back(slot);
            if (split_slot0.size() != split.size() + 1)
                throw Error{SORSVD_ERR_INTERNAL, "stream-K: slot table mismatch"};
            auto up = [&](const std::vector<int>& v) {
                int* d = nullptr;
                CK(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(int)));
                if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
                return d;
            };
            sorsvd_ctx::SkTable t;
            t.dev = {up(cta_seg), up(seg_tile), up(seg_k0), up(seg_k1), up(split_slot0), up(split), up(seg_slot)};
            t.nsplit = (int)split.size();
            t.nseg = (int)seg_tile.size();
            t.nslot = slot;
            it = c->sk_tables.emplace(key, t).first;
        }
        const std::vector<int*>& tab = it->second.dev;
        a.sk_cta_seg = tab[0];
        a.sk_seg_tile = tab[1];
        a.sk_seg_k0 = tab[2];
        a.sk_seg_k1 = tab[3];
        sk_split_slot0 = tab[4];
        sk_split_tiles = tab[5];
        a.sk_seg_slot = tab[6];
        a.sk_units = (int)units;
        a.sk_gy = (int)gy;
        const int BN = g.N <= 128 ? g.N : 128;
        a.sk_ws = dbuf(c, std::string(g.ws_name) + "_sk", (size_t)std::max(it->second.nslot, 1) * BM * BN);
        sk_split_tiles_h.resize((size_t)it->second.nsplit);
    }
    const bool f32a = g.Af != nullptr;
    const bool aligned = f32a ? (((uintptr_t)g.Af % 16) == 0 && (g.lda % 4) == 0)
                              : (((uintptr_t)g.A % 16) == 0 && (g.lda % 2) == 0);
    if (f32a && !aligned) throw Error{SORSVD_ERR_SHAPE, "shape: fp32 A needs 16-byte aligned rows (lda % 4 == 0)"};
    const bool v16 = aligned;
    dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)S);
    if (!g.tile_row0 && gy > 1) {
        a.gy_fused = (int)gy;
        grid = dim3((unsigned)(gx * gy), 1, (unsigned)S);
    }
    if (streamk) {
        grid = dim3((unsigned)c->num_sms, 1, 1);
        a.C = g.C;
        a.ldc = g.ldc;
        a.c_split_stride = 0;
    }
    switch (FN) {
#define FN_CASE(n) \
    case n: dispatch_fn<n>(g.ta, v16, f32a, a, grid, s); break;
        FN_CASE(1) FN_CASE(2) FN_CASE(3) FN_CASE(4) FN_CASE(5) FN_CASE(6) FN_CASE(7) FN_CASE(8)
        FN_CASE(9) FN_CASE(10) FN_CASE(11) FN_CASE(12) FN_CASE(13) FN_CASE(14) FN_CASE(15) FN_CASE(16)
#undef FN_CASE
        default: throw Error{SORSVD_ERR_INTERNAL, "gemm: FN"};
    }
    check_launch(c);
    if (streamk) {
        const int nsplit = (int)sk_split_tiles_h.size();
        if (nsplit > 0) {
            const int BN = g.N <= 128 ? g.N : 128;
            const dim3 fgrid((unsigned)cdiv((int64_t)BM * BN, 256), (unsigned)std::min(nsplit, 65535));
            streamk_fixup_kernel<<<fgrid, 256, 0, s>>>(
                a.sk_ws, sk_split_slot0, sk_split_tiles, nsplit, BM, BN, (int)gy, g.M, g.C, g.ldc, c->pred,
                c->pred_skip);
            check_launch(c);
        }
        return;
    }
    if (S > 1) {
        if (g.ldc % 2) throw Error{SORSVD_ERR_INTERNAL, "gemm: odd ldc with splits"};
        const int64_t count2 = g.M * g.ldc / 2;
        if (S >= 32 && count2 <= 8192) {
            const int blocks = (int)cdiv(count2 * 32, 256);
            reduce_splits_warp_kernel<<<blocks, 256, 0, s>>>(ws, count2, S, g.M * g.ldc, g.C, c->pred,
                                                             c->pred_skip);
        } else {
            const int blocks = (int)std::min<int64_t>(cdiv(count2, 256), (int64_t)c->num_sms * 8);
            reduce_splits_kernel<<<blocks, 256, 0, s>>>(ws, count2, S, g.M * g.ldc, g.C, c->pred, c->pred_skip);
        }
        check_launch(c);
    }
}

// ------------------------------------------------------ TF32 tcgen05 GEMM ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
        if (!ptr || q != cudaDriverEntryPointSuccess)
            throw Error{SORSVD_ERR_CUDA, "cuda: cuTensorMapEncodeTiled unavailable"};
        fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

// 2-D fp32 tensor map over a row-major (rows x cols, ld) matrix, box {bx (inner), by}, 128B swizzle.
CUtensorMap make_map_f32(const float* base, int64_t rows, int64_t cols, int64_t ld, int bx, int by, bool mn_major) {
    if (((uintptr_t)base % 16) || ((ld * 4) % 16)) throw Error{SORSVD_ERR_SHAPE, "shape: fp32 operand must be 16B aligned (ld % 4 == 0)"};
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE,
                                mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error{SORSVD_ERR_CUDA, "cuda: cuTensorMapEncodeTiled failed " + std::to_string((int)r)};
    return m;
}

inline int npad32(int ell) { return ell <= 256 ? ((ell + 31) / 32) * 32 : ((ell + 255) / 256) * 256; }

template <int BN, bool TA>
void launch_tc_t(const CUtensorMap& ma, const CUtensorMap& mb, const TcArgs& a, dim3 grid, cudaStream_t s) {
    using S = TcShape<BN>;
    allow_smem(tc_gemm_tf32_kernel<BN, TA>);
    tc_gemm_tf32_kernel<BN, TA><<<grid, kTcThreads, S::SMEM, s>>>(ma, mb, a);
}

template <bool TA>
void dispatch_tc(int BN, const CUtensorMap& ma, const CUtensorMap& mb, const TcArgs& a, dim3 grid, cudaStream_t s) {
    switch (BN) {
        case 32: launch_tc_t<32, TA>(ma, mb, a, grid, s); break;
        case 64: launch_tc_t<64, TA>(ma, mb, a, grid, s); break;
        case 96: launch_tc_t<96, TA>(ma, mb, a, grid, s); break;
        case 128: launch_tc_t<128, TA>(ma, mb, a, grid, s); break;
        case 160: launch_tc_t<160, TA>(ma, mb, a, grid, s); break;
        case 192: launch_tc_t<192, TA>(ma, mb, a, grid, s); break;
        case 224: launch_tc_t<224, TA>(ma, mb, a, grid, s); break;
        case 256: launch_tc_t<256, TA>(ma, mb, a, grid, s); break;
        default: throw Error{SORSVD_ERR_INTERNAL, "tc gemm: BN"};
    }
}

// C (M x N fp32, ldc) = op(A) * B on the tensor cores (TF32 in, FP32 accumulate).
// op(A) = A (A: M x K row-major) or A^T (A: K x M row-major); B: K x N row-major,
// N a multiple of 32 (<= 256) or of 256.
void run_tc_gemm(sorsvd_ctx* c, bool ta, const float* A, int64_t lda, int64_t M, int64_t K, const float* B,
                 int64_t ldb, int N, float* C, int64_t ldc, cudaStream_t s, const char* ws_name = "tc_ws") {
    if (N % 32 || (N > 256 && N % 256)) throw Error{SORSVD_ERR_INTERNAL, "tc gemm: bad N"};
    const int BN = N <= 256 ? N : 256;
    const int gy = N / BN;
    const int64_t gx = cdiv(M, kTcBM);
    int S = 1;
    {
        const int64_t base = gx * gy;
        const int64_t maxS = std::max<int64_t>(1, std::min<int64_t>(64, K / 512));
        double best = 1e300;
        for (int64_t cand = 1; cand <= maxS; ++cand) {
            const double waves = (double)cdiv(base * cand, c->num_sms);
            const double cost = waves * ((double)K / cand + 256.0) + (cand > 1 ? 0.02 * cand * M * N / (double)c->num_sms : 0.0);
            if (cost < best * 0.999) {
                best = cost;
                S = (int)cand;
            }
        }
    }
    const CUtensorMap ma = ta ? make_map_f32(A, K, M, lda, 32, kTcBK, true) : make_map_f32(A, M, K, lda, kTcBK, kTcBM, false);
    const CUtensorMap mb = make_map_f32(B, K, N, ldb, 32, kTcBK, true);
    TcArgs a{};
    a.M = M;
    a.K = K;
    a.k_chunk = std::max<int64_t>(kTcBK, cdiv(cdiv(K, S), kTcBK) * kTcBK);
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    float* ws = nullptr;
    if (S > 1) {
        ws = reinterpret_cast<float*>(dbuf(c, ws_name, (size_t)S * M * ldc / 2 + 1));
        a.C = ws;
        a.ldc = ldc;
        a.c_split_stride = M * ldc;
    } else {
        a.C = C;
        a.ldc = ldc;
    }
    dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)S);
    if (ta) dispatch_tc<true>(BN, ma, mb, a, grid, s);
    else dispatch_tc<false>(BN, ma, mb, a, grid, s);
    check_launch(c);
    if (S > 1) {
        const int64_t count4 = M * ldc / 4;
        const int blocks = (int)std::min<int64_t>(cdiv(count4, 256), (int64_t)c->num_sms * 8);
        reduce_splits_f32_kernel<<<blocks, 256, 0, s>>>(ws, count4, S, M * ldc, C, c->pred, c->pred_skip);
        check_launch(c);
    }
}

void cast_to_f64(sorsvd_ctx* c, const float* in, int64_t ldi, double* out, int64_t ldo, int64_t rows, int cols,
                 cudaStream_t s) {
    const int blocks = (int)std::min<int64_t>(cdiv(rows * cols, 256), (int64_t)c->num_sms * 8);
    cast_f32_to_f64_kernel<<<blocks, 256, 0, s>>>(in, ldi, out, ldo, rows, cols);
    check_launch(c);
}
void cast_to_f32(sorsvd_ctx* c, const double* in, int64_t ldi, float* out, int64_t ldo, int64_t rows, int cols,
                 cudaStream_t s) {
    const int blocks = (int)std::min<int64_t>(cdiv(rows * cols, 256), (int64_t)c->num_sms * 8);
    cast_f64_to_f32_kernel<<<blocks, 256, 0, s>>>(in, ldi, out, ldo, rows, cols);
    check_launch(c);
}

// ---------------------------------------------------------------- TSQR ----
// Leaves and tree nodes are factored by the cluster Householder kernel
// (cqr_f64.cuh). A leaf is as many rows as one cluster of up to 16 CTAs can
// hold, so the sketches of C1, C2 and C4 are a single leaf (no tree).
constexpr int kCqrMaxCluster = 16;

int cqr_rows_per_cta(int k) {
    const int64_t avail = kCqrSmemBudget / 8 - 3 * (int64_t)cqr_rw(k) - 2 * (int64_t)k - 8;
    return (int)std::max<int64_t>(1, avail / k - 1);
}

int cqr_max_cluster(sorsvd_ctx* c, int k) {
    static std::map<int, int> cache;  // guarded by g_attr_mu (process-wide, shared by all contexts)
    {
        std::lock_guard<std::mutex> lk(g_attr_mu);
        auto it = cache.find(k);
        if (it != cache.end()) return it->second;
    }
    const size_t sm = cqr_smem_bytes(cqr_rows_per_cta(k), k);
    allow_smem(cqr_kernel, true);
    int best = 1;
    for (int cs = kCqrMaxCluster; cs >= 1; cs /= 2) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kCqrThreads);
        cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, cqr_kernel, &cfg) == cudaSuccess && n > 0) {
            best = cs;
            break;
        }
        cudaGetLastError();
    }
    (void)c;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    cache.emplace(k, best);
    return cache[k];
}

struct RegCfg {
    int ch = 0, threads = 0, csize = 0;
};

template <int CH>
int cqr_reg_max_threads() {
    static int t = -1;
    if (t < 0) {
        cudaFuncAttributes fa{};
        CK(cudaFuncGetAttributes(&fa, cqr_reg_kernel<CH>));
        t = std::min(1024, fa.maxThreadsPerBlock) / 32 * 32;
    }
    return t;
}

int cqr_reg_threads_for(int ch) {
    switch (ch) {
        case 16: return cqr_reg_max_threads<16>();
        case 24: return cqr_reg_max_threads<24>();
        case 32: return cqr_reg_max_threads<32>();
        case 48: return cqr_reg_max_threads<48>();
        default: return cqr_reg_max_threads<64>();
    }
}

// Register-resident configuration for a block of `rows` x k over at most
// `cmax` CTAs: smallest chunk (shortest per-thread stream) that fits.
RegCfg cqr_reg_choose(int k, int64_t rows, int cmax) {
    RegCfg best;
    for (int ch : {16, 24, 32, 48, 64}) {
        const int tmax = cqr_reg_threads_for(ch);
        const int nch_max = tmax / k;
        if (nch_max < 1) continue;
        const int64_t rows_cta = (int64_t)nch_max * ch;
        const int64_t C = cdiv(rows, rows_cta);
        if (C > cmax) continue;
        const int Rb = (int)cdiv(rows, C);
        const int nch = (Rb + ch - 1) / ch;
        const int threads = (k * nch + 31) / 32 * 32;
        if (cqr_reg_smem_bytes(Rb, k, ch) > 200 * 1024 || threads > tmax) continue;
        best.ch = ch;
        best.threads = threads;
        best.csize = (int)C;
        return best;
    }
    return best;
}

int64_t cqr_reg_capacity(int k, int cmax) {
    int64_t cap = 0;
    for (int ch : {16, 24, 32, 48, 64}) {
        const int nch_max = cqr_reg_threads_for(ch) / k;
        cap = std::max<int64_t>(cap, (int64_t)cmax * nch_max * ch);
    }
    return cap;
}

template <int CH>
void launch_cqr_reg_t(sorsvd_ctx* c, const CqrArgs& a, int nblocks, const RegCfg& rc, int Rb, cudaStream_t s) {
    const size_t sm = cqr_reg_smem_bytes(Rb, a.k, CH);
    allow_smem(cqr_reg_kernel<CH>, true);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nblocks * rc.csize));
    cfg.blockDim = dim3((unsigned)rc.threads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = rc.csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, cqr_reg_kernel<CH>, a));
    check_launch(c);
}

// Factor + explicit Q of `nblocks` blocks of at most `rows_max` rows each:
// register-resident kernel when a configuration fits, shared-memory kernel
// otherwise.
void launch_cqr(sorsvd_ctx* c, const CqrArgs& a0, int nblocks, int rows_max, int cmax_smem, int rb_smem,
                cudaStream_t s) {
    CqrArgs a = a0;
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    const RegCfg rc = a.wy ? RegCfg{} : cqr_reg_choose(a.k, rows_max, kCqrMaxCluster);
    if (rc.ch) {
        const int Rb = (int)cdiv(rows_max, rc.csize);
        switch (rc.ch) {
            case 16: launch_cqr_reg_t<16>(c, a, nblocks, rc, Rb, s); break;
            case 24: launch_cqr_reg_t<24>(c, a, nblocks, rc, Rb, s); break;
            case 32: launch_cqr_reg_t<32>(c, a, nblocks, rc, Rb, s); break;
            case 48: launch_cqr_reg_t<48>(c, a, nblocks, rc, Rb, s); break;
            default: launch_cqr_reg_t<64>(c, a, nblocks, rc, Rb, s); break;
        }
        return;
    }
    const int csize = (int)std::min<int64_t>(cmax_smem, cdiv(rows_max, rb_smem));
    const int Rb = (int)cdiv(rows_max, csize);
    const size_t sm = cqr_smem_bytes(Rb, a.k);
    allow_smem(cqr_kernel, true);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nblocks * csize));
    cfg.blockDim = dim3(kCqrThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, cqr_kernel, a));
    check_launch(c);
}

void build_seg_tiles(const std::vector<int64_t>& seg_row0, const std::vector<int>& seg_rows, int BM,
                     std::vector<int>& r0, std::vector<int>& rc, std::vector<int>& sg) {
    for (size_t s = 0; s < seg_row0.size(); ++s)
        for (int off = 0; off < seg_rows[s]; off += BM) {
            r0.push_back((int)(seg_row0[s] + off));
            rc.push_back(std::min(BM, seg_rows[s] - off));
            sg.push_back((int)s);
        }
}

template <typename T>
T* upload(QrPlan* p, const std::vector<T>& v) {
    T* d = nullptr;
    CK(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(T)));
    if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    p->owned.push_back(d);
    return d;
}

double* dalloc(QrPlan* p, size_t count) {
    double* d = nullptr;
    CK(cudaMalloc(&d, std::max<size_t>(count, 1) * sizeof(double)));
    CK(cudaMemset(d, 0, std::max<size_t>(count, 1) * sizeof(double)));
    CK(cudaStreamSynchronize(0));  // legacy-stream fill vs the non-blocking streams (see dbuf)
    p->owned.push_back(d);
    return d;
}

constexpr int kHouseMaxK = 256;  // largest k of the cluster Householder TSQR (2k x k node in one cluster)
constexpr int kBigQrPasses = 5;  // adaptive CholeskyQR passes for k > 256 (cholc_f64.cuh); odd -> ends in Q

// Build (or fetch) the TSQR plan for `rows` x k. leaves_given > 0 builds a
// plan whose level-0 "leaves" are external k x k R blocks (the cross-GPU tree).
QrPlan* get_qr_plan(sorsvd_ctx* c, int64_t rows, int k, int leaves_given, const char* tag) {
    const std::string key = std::string(tag) + ":" + std::to_string(rows) + "x" + std::to_string(k) + "g" + std::to_string(leaves_given);
    auto it = c->plans.find(key);
    if (it != c->plans.end()) return it->second.get();
    if (c->capturing) throw Error{SORSVD_ERR_INTERNAL, "qr plan creation during capture"};
    invalidate_graphs(c);
    auto p = std::make_unique<QrPlan>();
    p->ws_name = "ws_" + key;
    p->rows = rows;
    p->k = k;
    p->Np = npad(k);
    p->ldR = k;
    if (k > kHouseMaxK) {
        if (leaves_given > 0) throw Error{SORSVD_ERR_INTERNAL, "tsqr tree plan requested for k > 256"};
        const int Np = p->Np;
        p->big = true;
        p->ldR = Np;
        p->nodes.push_back(1);
        p->R.assign(1, dalloc(p.get(), (size_t)k * Np));
        p->G1 = dalloc(p.get(), (size_t)Np * Np);
        p->Ri1 = dalloc(p.get(), (size_t)Np * Np);
        for (auto& r : p->Rp) r = dalloc(p.get(), (size_t)Np * Np);
        p->Rtmp = dalloc(p.get(), (size_t)Np * Np);
        p->Qtmp = dalloc(p.get(), (size_t)rows * Np);
        p->Wtrsm = dalloc(p.get(), (size_t)rows * kCholcB);
        p->flag = reinterpret_cast<int*>(dalloc(p.get(), 1));  // [0] breakdown, [1] done
        QrPlan* raw = p.get();
        c->plans[key] = std::move(p);
        return raw;
    }
    p->rb_max = cqr_rows_per_cta(k);
    p->cmax = cqr_max_cluster(c, k);
    if (leaves_given > 0) {
        p->P = leaves_given;
    } else {
        // the per-reflector latency (cluster reduction) dominates, so the
        // fewest tree levels win: leaves as large as either kernel can hold
        const int64_t reg_cap = cqr_reg_capacity(k, kCqrMaxCluster);
        int64_t leaf_max = std::max<int64_t>(reg_cap, (int64_t)p->cmax * p->rb_max);
        p->P = (int)std::max<int64_t>(1, cdiv(rows, leaf_max));
        const int64_t base = rows / p->P, extra = rows % p->P;
        int64_t r = 0;
        for (int i = 0; i < p->P; ++i) {
            const int cnt = (int)(base + (i < extra ? 1 : 0));
            p->row0.push_back(r);
            p->rcnt.push_back(cnt);
            p->max_leaf_rows = std::max(p->max_leaf_rows, cnt);
            r += cnt;
        }
        if (p->P > 1 && base < k) throw Error{SORSVD_ERR_INTERNAL, "tsqr: leaf shorter than k"};
        p->leaf_cs = (int)std::min<int64_t>(p->cmax, cdiv(p->max_leaf_rows, p->rb_max));
        p->d_row0 = upload(p.get(), p->row0);
        p->d_rows = upload(p.get(), p->rcnt);
    }
    p->nodes.push_back(p->P);
    while (p->nodes.back() > 1) p->nodes.push_back((p->nodes.back() + 1) / 2);
    const int L = (int)p->nodes.size() - 1;
    const int Np = p->Np;
    const int BM = gemm_bm_for(Np);
    p->node_cs = (int)std::min<int64_t>(p->cmax, cdiv(2 * k, p->rb_max));
    p->t_row0.assign(L + 1, nullptr);
    p->t_rows.assign(L + 1, nullptr);
    p->t_seg.assign(L + 1, nullptr);
    p->t_count.assign(L + 1, 0);
    p->R.assign(L + 1, nullptr);
    p->QN.assign(L + 1, nullptr);
    p->C.assign(L + 1, nullptr);
    p->SN.assign(L + 1, nullptr);
    p->n_row0.assign(L + 1, nullptr);
    p->n_rows.assign(L + 1, nullptr);
    for (int l = 0; l <= L; ++l) p->R[l] = dalloc(p.get(), (size_t)p->nodes[l] * k * k);
    for (int l = 1; l <= L; ++l) {
        p->QN[l] = dalloc(p.get(), (size_t)p->nodes[l] * 2 * k * Np);
        p->SN[l] = dalloc(p.get(), (size_t)p->nodes[l] * 2 * k * k);
        std::vector<int64_t> r0;
        std::vector<int> rc;
        for (int i = 0; i < p->nodes[l]; ++i) {
            r0.push_back((int64_t)i * 2 * k);
            rc.push_back(2 * k);
        }
        p->n_row0[l] = upload(p.get(), r0);
        p->n_rows[l] = upload(p.get(), rc);
    }
    for (int l = 0; l < L; ++l) p->C[l] = dalloc(p.get(), (size_t)p->nodes[l + 1] * 2 * k * Np);
    if (leaves_given == 0 && L >= 1) {
        std::vector<int> r0, rc, sg;
        build_seg_tiles(p->row0, p->rcnt, BM, r0, rc, sg);
        p->t_row0[0] = upload(p.get(), r0);
        p->t_rows[0] = upload(p.get(), rc);
        p->t_seg[0] = upload(p.get(), sg);
        p->t_count[0] = (int)r0.size();
    }
    for (int l = 1; l < L; ++l) {
        std::vector<int64_t> sr0;
        std::vector<int> src;
        for (int i = 0; i < p->nodes[l]; ++i) {
            sr0.push_back((int64_t)i * 2 * k);
            src.push_back(2 * k);
        }
        std::vector<int> r0, rc, sg;
        build_seg_tiles(sr0, src, BM, r0, rc, sg);
        p->t_row0[l] = upload(p.get(), r0);
        p->t_rows[l] = upload(p.get(), rc);
        p->t_seg[l] = upload(p.get(), sg);
        p->t_count[l] = (int)r0.size();
    }
    if (leaves_given == 0) {
        p->G1 = dalloc(p.get(), (size_t)Np * Np);
        p->G2 = dalloc(p.get(), (size_t)Np * Np);
        p->Ri1 = dalloc(p.get(), (size_t)Np * Np);
        p->Ri2 = dalloc(p.get(), (size_t)Np * Np);
        p->R1 = dalloc(p.get(), (size_t)k * k);
        p->cwork = dalloc(p.get(), (size_t)k * k);
        p->Qtmp = dalloc(p.get(), (size_t)rows * Np);
        p->flag = reinterpret_cast<int*>(dalloc(p.get(), 1));
        p->wy_tau = dalloc(p.get(), (size_t)k);
        p->wy_sgn = dalloc(p.get(), (size_t)k);
    }
    QrPlan* raw = p.get();
    c->plans[key] = std::move(p);
    return raw;
}

// Factor: leaves (from T) + tree levels. root_sign: the plan's root is the
// global root (diag(R) >= 0). Leaf explicit Qs are written in place in T (or
// straight into Q when the single leaf is the final root).
void qr_factor(sorsvd_ctx* c, QrPlan* p, double* T, int64_t ldt, double* Q, int64_t ldq, bool root_sign,
               cudaStream_t s, const double* Rleaves = nullptr) {
    const int k = p->k;
    const int L = (int)p->nodes.size() - 1;
    if (!Rleaves) {
        CqrArgs a{};
        const bool direct = (L == 0 && root_sign);
        // one block, explicit Q wanted: factor only, then Q by compact WY (two GEMMs)
        const bool wy = direct && k >= 48 && p->wy_tau;  // small k: in-kernel form-Q wins
        a.in = T;
        a.ldi = ldt;
        a.qout = wy ? p->Qtmp : (direct ? Q : T);
        a.ldq = wy ? p->Np : (direct ? ldq : ldt);
        a.row0 = p->d_row0;
        a.rows = p->d_rows;
        a.k = k;
        a.R = p->R[0];
        a.ldr = k;
        a.root_sign = (L == 0 && root_sign) ? 1 : 0;
        a.wy = wy ? 1 : 0;
        a.tau_out = p->wy_tau;
        a.sgn_out = p->wy_sgn;
        launch_cqr(c, a, p->P, p->max_leaf_rows, p->cmax, p->rb_max, s);
        if (wy) {
            const int Np = p->Np;
            GemmCall g;  // G = V^T V
            g.ta = true;
            g.A = p->Qtmp;
            g.lda = Np;
            g.M = k;
            g.K = p->rows;
            g.B = p->Qtmp;
            g.ldb = Np;
            g.N = Np;
            g.C = p->G2;
            g.ldc = Np;
            g.ws_name = p->ws_name.c_str();
            run_gemm(c, g, s);
            // U = T^{-1} (into Ri1), B = V1^T diag(sgn) (into Ri2); T = U^{-1} (into R1... via trinv)
            wy_prep_kernel<<<16, 256, 0, s>>>(p->G2, Np, p->wy_tau, p->wy_sgn, p->Qtmp, Np, k, p->Ri1, p->Ri2, Np,
                                              c->pred, c->pred_skip);
            check_launch(c);
            const int wpb = 4;  // (a shared-memory staged variant measured slower: issue bound on the shuffles)
            trinv_kernel<<<(k + wpb - 1) / wpb, 32 * wpb, (size_t)wpb * k * sizeof(double), s>>>(
                p->Ri1, Np, k, p->G1, Np, c->pred, c->pred_skip);
            check_launch(c);
            {
                GemmCall x;  // X = T B  (k x Np) into Ri1 (U is no longer needed)
                x.A = p->G1;
                x.lda = Np;
                x.M = k;
                x.K = k;
                x.B = p->Ri2;
                x.ldb = Np;
                x.N = Np;
                x.C = p->Ri1;
                x.ldc = Np;
                x.ws_name = p->ws_name.c_str();
                run_gemm(c, x, s);
            }
            GemmCall h;  // Q = -V X  (+ E diag(sgn) below)
            h.A = p->Qtmp;
            h.lda = Np;
            h.M = p->rows;
            h.K = k;
            h.B = p->Ri1;
            h.ldb = Np;
            h.N = Np;
            h.C = Q;
            h.ldc = ldq;
            h.alpha = -1.0;
            h.ws_name = p->ws_name.c_str();
            run_gemm(c, h, s);
            wy_diag_kernel<<<1, 128, 0, s>>>(Q, ldq, p->wy_sgn, k, c->pred, c->pred_skip);
            check_launch(c);
        }
    }
    for (int l = 1; l <= L; ++l) {
        const double* Rin = (l == 1 && Rleaves) ? Rleaves : p->R[l - 1];
        stack_r_kernel<<<p->nodes[l], 256, 0, s>>>(Rin, p->nodes[l - 1], k, k, p->SN[l], k, c->pred, c->pred_skip);
        check_launch(c);
        CqrArgs a{};
        a.in = p->SN[l];
        a.ldi = k;
        a.qout = p->QN[l];
        a.ldq = p->Np;
        a.row0 = p->n_row0[l];
        a.rows = p->n_rows[l];
        a.k = k;
        a.R = p->R[l];
        a.ldr = k;
        a.root_sign = (l == L && root_sign) ? 1 : 0;
        launch_cqr(c, a, p->nodes[l], 2 * k, p->cmax, p->rb_max, s);
    }
}

// Top-down: push C factors down the tree, finish with Q = Q_leaf * C_leaf.
// Cin (k x Np, optional) multiplies the plan's root from the right (the
// cross-GPU path factor); without it the root Q already carries the signs.
// Returns the level-0 C array (one k x Np block per leaf) when leaf_out is
// null (used by the cross-GPU tree to hand each rank its factor).
void qr_formq(sorsvd_ctx* c, QrPlan* p, double* T, int64_t ldt, double* Q, int64_t ldq, const double* Cin,
              cudaStream_t s, bool leaves_are_blocks = false) {
    const int k = p->k, Np = p->Np;
    const int L = (int)p->nodes.size() - 1;
    if (L == 0) {
        if (Cin) {  // local root is a single leaf: Q = Qleaf * Cin
            GemmCall g;
            g.A = T;
            g.lda = ldt;
            g.M = p->rows;
            g.K = k;
            g.B = Cin;
            g.ldb = Np;
            g.N = Np;
            g.C = Q;
            g.ldc = ldq;
            g.force_splits = 1;
            run_gemm(c, g, s);
        }
        return;
    }
    // level L-1 children factors: root Q (2k x Np), optionally times Cin
    const double* Ccur;
    if (Cin) {
        GemmCall g;
        g.A = p->QN[L];
        g.lda = Np;
        g.M = 2 * k;
        g.K = k;
        g.B = Cin;
        g.ldb = Np;
        g.N = Np;
        g.C = p->C[L - 1];
        g.ldc = Np;
        g.force_splits = 1;
        run_gemm(c, g, s);
        Ccur = p->C[L - 1];
    } else {
        Ccur = p->QN[L];
    }
    for (int l = L - 1; l >= 1; --l) {
        GemmCall g;
        g.A = p->QN[l];
        g.lda = Np;
        g.M = (int64_t)p->nodes[l] * 2 * k;
        g.K = k;
        g.B = Ccur;
        g.ldb = Np;
        g.b_seg_stride = (int64_t)k * Np;
        g.N = Np;
        g.C = p->C[l - 1];
        g.ldc = Np;
        g.tile_row0 = p->t_row0[l];
        g.tile_rows = p->t_rows[l];
        g.tile_seg = p->t_seg[l];
        g.ntiles = p->t_count[l];
        g.force_splits = 1;
        run_gemm(c, g, s);
        Ccur = p->C[l - 1];
    }
    if (leaves_are_blocks) {
        // caller reads the per-leaf factors from p->C[0] (or QN[L] when L == 1 and no Cin)
        return;
    }
    GemmCall g;
    g.A = T;
    g.lda = ldt;
    g.M = p->rows;
    g.K = k;
    g.B = Ccur;
    g.ldb = Np;
    g.b_seg_stride = (int64_t)k * Np;
    g.N = Np;
    g.C = Q;
    g.ldc = ldq;
    g.tile_row0 = p->t_row0[0];
    g.tile_rows = p->t_rows[0];
    g.tile_seg = p->t_seg[0];
    g.ntiles = p->t_count[0];
    g.force_splits = 1;
    run_gemm(c, g, s);
}

struct PredScope {
    sorsvd_ctx* c;
    const int* saved;
    int saved_skip;
    PredScope(sorsvd_ctx* c_, const int* flag, int skip) : c(c_), saved(c_->pred), saved_skip(c_->pred_skip) {
        c->pred = flag;
        c->pred_skip = skip;
    }
    ~PredScope() {
        c->pred = saved;
        c->pred_skip = saved_skip;
    }
};

void launch_chol(sorsvd_ctx* c, const CholArgs& a0, cudaStream_t s) {
    CholArgs a = a0;
    a.outer = c->pred;  // enclosing predicate (RPCA): a skipped iteration marks the QR flag dead
    a.outer_skip = c->pred_skip;
    // the factor in shared memory when it fits, plus the back-substitution columns when both fit
    const size_t kk8 = (size_t)a.k * a.k * sizeof(double);
    const size_t sm = 2 * kk8 <= kCholSmemBytes ? 2 * kk8 : kk8 <= kCholSmemBytes ? kk8 : 0;
    allow_smem(chol_inv_kernel);
    // small k: fewer threads (cheaper barriers); the per-element operation order is unchanged
    const int threads = a.k <= 16 ? 128 : a.k <= 48 ? 256 : kCholThreads;
    chol_inv_kernel<<<1, threads, sm, s>>>(a);
    check_launch(c);
}

// k > 256: adaptive (shifted) CholeskyQR passes (cholc_f64.cuh). T (rows x k,
// pitch Np) is left intact; Q gets the orthonormal factor, p->R[0] (pitch Np)
// R = R_p ... R_1.
// distributed: T is this rank's row block; the Gram matrices are summed over
// ranks (the shift uses the global row count) and every rank forms its own
// rows of Q.
void allreduce_sum(sorsvd_ctx* c, double* buf, size_t count, cudaStream_t s);

// cholc_kernel over a ceil(k/32)-CTA cluster (CTA r holds rows [32r, 32r+32) of L).
void launch_cholc(sorsvd_ctx* c, const CholcArgs& a, cudaStream_t s) {
    const int C = (a.k + kCholcB - 1) / kCholcB;
    allow_smem(cholc_kernel, true);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)C);
    cfg.blockDim = dim3(kCholcThreads);
    cfg.dynamicSmemBytes = cholc_smem_bytes(a.k);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, cholc_kernel, a));
    check_launch(c);
}

void qr_run_big(sorsvd_ctx* c, QrPlan* p, const double* T, int64_t ldt, double* Q, int64_t ldq, cudaStream_t s,
                int64_t rows_global = 0, bool distributed = false) {
    const int k = p->k, Np = p->Np;
    if (ldt != Np || ldq != Np) throw Error{SORSVD_ERR_INTERNAL, "qr_run_big: T and Q must be padded to Np"};
    const int64_t mg = rows_global > 0 ? rows_global : p->rows;
    auto gram = [&](const double* X, double* G) {
        GemmCall g;
        g.ta = true;
        g.A = X;
        g.lda = Np;
        g.M = k;
        g.K = p->rows;
        g.B = X;
        g.ldb = Np;
        g.N = Np;
        g.C = G;
        g.ldc = Np;
        g.ws_name = p->ws_name.c_str();
        run_gemm(c, g, s);
        if (distributed) allreduce_sum(c, G, (size_t)k * Np, s);
    };
    // Out R = X (blocked TRSM: the GEMM part X_{<J} R_{<J,J} on the DMMA engine)
    double* W = p->Wtrsm;
    auto trsm = [&](const double* X, const double* R, double* Out) {
        const int nblk = (k + kCholcB - 1) / kCholcB;
        const unsigned grid = (unsigned)cdiv(p->rows, 256);
        for (int J = 0; J < nblk; ++J) {
            const int c0 = J * kCholcB, nb = std::min(kCholcB, k - c0);
            if (J > 0) {
                GemmCall g;
                g.A = Out;
                g.lda = Np;
                g.M = p->rows;
                g.K = c0;
                g.B = R + c0;
                g.ldb = Np;
                g.N = (nb + 7) & ~7;  // stays inside R's Np-wide rows
                g.C = W;
                g.ldc = kCholcB;
                g.ws_name = p->ws_name.c_str();
                run_gemm(c, g, s);
            }
            trsm_rows_kernel<<<grid, 256, 0, s>>>(X + c0, Np, J > 0 ? W : nullptr, kCholcB, R + (size_t)c0 * Np + c0,
                                                  Np, nb, Out + c0, Np, p->rows, c->pred, c->pred_skip);
            check_launch(c);
        }
    };
    auto chol = [&](double* R) {
        CholcArgs a{};
        a.G = p->G1;
        a.ldg = Np;
        a.k = k;
        a.shift_coef = 11.0 * ((double)mg * k + (double)k * (k + 1)) * DBL_EPSILON;
        a.R = R;
        a.ldr = Np;
        a.flag = p->flag;
        a.done = p->flag + 1;
        a.done_tol = 1e-13;
        launch_cholc(c, a, s);
    };
    int* done = p->flag + 1;
    qr_flags_init_kernel<<<1, 32, 0, s>>>(p->flag, c->pred, c->pred_skip);  // dead when the caller is off
    check_launch(c);
    set_identity_kernel<<<64, 256, 0, s>>>(p->R[0], Np, k);
    check_launch(c);
    const double* X = T;
    double* outs[2] = {Q, p->Qtmp};
    const int blocks = (int)std::min<int64_t>(cdiv(p->rows * Np, 256), (int64_t)c->num_sms * 8);
    for (int pass = 0; pass < kBigQrPasses; ++pass) {
        double* out = outs[pass & 1];
        {
            PredScope ps(c, done, 1);
            gram(X, p->G1);
        }
        chol(p->Rp[0]);  // sets *done when X is already orthonormal
        {
            PredScope ps(c, done, 1);
            trsm(X, p->Rp[0], out);
            GemmCall g;  // R <- R_pass * R
            g.A = p->Rp[0];
            g.lda = Np;
            g.M = k;
            g.K = k;
            g.B = p->R[0];
            g.ldb = Np;
            g.N = Np;
            g.C = p->Rtmp;
            g.ldc = Np;
            g.ws_name = p->ws_name.c_str();
            run_gemm(c, g, s);
            copy_rows_kernel<<<64, 256, 0, s>>>(p->Rtmp, Np, p->R[0], Np, k, Np, done, 1);
            check_launch(c);
        }
        // converged earlier: carry X through unchanged
        copy_rows_kernel<<<blocks, 256, 0, s>>>(X, Np, out, Np, p->rows, Np, done, 0);
        check_launch(c);
        X = out;
    }
}

// After a synchronised run: a failed shifted Cholesky (cond(T) beyond ~1/eps
// or non-finite input) is reported as the reference's numerical_error.
void check_big_qr(QrPlan* p) {
    if (!p || !p->big) return;
    int f = 0;
    CK(cudaMemcpy(&f, p->flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (f) throw Error{SORSVD_ERR_NUMERICAL, "numerical: thin_qr (shifted CholeskyQR) broke down"};
}

// Full single-GPU thin QR of T (rows x k): CholeskyQR2 when the sketch is well
// conditioned, the cluster Householder TSQR otherwise (device-side choice,
// cholqr_f64.cuh). T is left intact by the CholeskyQR2 path; the Householder
// path may overwrite it. Final R (diag >= 0) lands in p->R[L].
void qr_run(sorsvd_ctx* c, QrPlan* p, double* T, int64_t ldt, double* Q, int64_t ldq, cudaStream_t s) {
    if (p->big) {
        qr_run_big(c, p, T, ldt, Q, ldq, s);
        return;
    }
    const int k = p->k, Np = p->Np;
    const int L = (int)p->nodes.size() - 1;
    auto gram = [&](const double* X, int64_t ldx, double* G) {
        if (k <= 32) {  // one launch: per-warp register partials, last-CTA ordered sum (smallk_f64.cuh)
            const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(c->num_sms, cdiv(p->rows, 128)));
            double* ws = dbuf(c, p->ws_name + ":gram", (size_t)c->num_sms * 32 * 32);
            unsigned int* ticket = reinterpret_cast<unsigned int*>(dbuf(c, p->ws_name + ":ticket", 1));
            if (k <= 16)
                gram_tall_kernel<16><<<grid, kGramThreads, 0, s>>>(X, ldx, p->rows, k, ws, ticket, G, Np, c->pred,
                                                                   c->pred_skip);
            else
                gram_tall_kernel<32><<<grid, kGramThreads, 0, s>>>(X, ldx, p->rows, k, ws, ticket, G, Np, c->pred,
                                                                   c->pred_skip);
            check_launch(c);
            return;
        }
        GemmCall g;
        g.ta = true;
        g.A = X;
        g.lda = ldx;
        g.M = k;
        g.K = p->rows;
        g.B = X;
        g.ldb = ldx;
        g.N = Np;
        g.C = G;
        g.ldc = Np;
        g.ws_name = p->ws_name.c_str();
        run_gemm(c, g, s);
    };
    auto rmul = [&](const double* X, int64_t ldx, const double* Ri, double* Out, int64_t ldo) {
        GemmCall g;
        g.A = X;
        g.lda = ldx;
        g.M = p->rows;
        g.K = k;
        g.B = Ri;
        g.ldb = Np;
        g.N = Np;
        g.C = Out;
        g.ldc = ldo;
        g.ws_name = p->ws_name.c_str();
        run_gemm(c, g, s);
    };
    if (ldt != Np) throw Error{SORSVD_ERR_INTERNAL, "qr_run: T must be padded to Np"};
    if (p->hint_house) {  // Gram + Cholesky attempt skipped (it was rejected on the previous operands of this plan)
        qr_factor(c, p, T, ldt, Q, ldq, true, s);
        qr_formq(c, p, T, ldt, Q, ldq, nullptr, s);
        return;
    }
    // k > 160: the factor no longer fits one CTA's shared memory and chol_inv_kernel would run
    // its k sequential steps out of global memory (k = 256: 3.7 ms per factorisation); the
    // factor is then spread over a cluster (cholc_kernel in CholeskyQR2 mode, same gates) and
    // R^{-1} comes from a column-parallel back substitution
    const bool cluster_chol = (size_t)k * k * sizeof(double) > kCholSmemBytes;
    auto cluster_pass = [&](int pass, const double* G, double* R, double* Ri) {
        CholcArgs a{};
        a.G = G;
        a.ldg = Np;
        a.k = k;
        a.R = R;
        a.ldr = k;
        a.flag = p->flag;
        a.mode = pass;
        a.outer = c->pred;
        a.outer_skip = c->pred_skip;
        launch_cholc(c, a, s);
        const int wpb = 8;
        trinv_kernel<<<(k + wpb - 1) / wpb, 32 * wpb, (size_t)wpb * k * sizeof(double), s>>>(R, k, k, Ri, Np,
                                                                                             p->flag, 1);
        check_launch(c);
    };
    gram(T, ldt, p->G1);
    if (cluster_chol) {
        cluster_pass(1, p->G1, p->R1, p->Ri1);
        {
            PredScope ps(c, p->flag, 1);  // skipped when pass 1 rejected
            rmul(T, ldt, p->Ri1, p->Qtmp, Np);
            gram(p->Qtmp, Np, p->G2);
        }
        cluster_pass(2, p->G2, p->cwork, p->Ri2);
        triu_mul_kernel<<<std::min<int>((k * k + 255) / 256, c->num_sms * 4), 256, 0, s>>>(p->cwork, k, p->R1, k,
                                                                                           p->R[L], k, k, p->flag, 1);
        check_launch(c);
        {
            PredScope ps(c, p->flag, 1);
            rmul(p->Qtmp, Np, p->Ri2, Q, ldq);
        }
        {
            PredScope ps(c, p->flag, 0);  // Householder only when CholeskyQR2 was rejected
            qr_factor(c, p, T, ldt, Q, ldq, true, s);
            qr_formq(c, p, T, ldt, Q, ldq, nullptr, s);
        }
        return;
    }
    CholArgs a1{};
    a1.G = p->G1;
    a1.ldg = Np;
    a1.k = k;
    a1.Rinv = p->Ri1;
    a1.ldr = Np;
    a1.work = p->cwork;
    a1.flag = p->flag;
    a1.pass = 1;
    a1.Rf = p->R1;
    a1.ldf = k;
    launch_chol(c, a1, s);
    {
        PredScope ps(c, p->flag, 1);  // skipped when pass 1 rejected
        rmul(T, ldt, p->Ri1, p->Qtmp, Np);
        gram(p->Qtmp, Np, p->G2);
    }
    CholArgs a2 = a1;
    a2.G = p->G2;
    a2.Rinv = p->Ri2;
    a2.pass = 2;
    a2.Rf = nullptr;
    a2.R1 = p->R1;
    a2.ldr1 = k;
    a2.Rout = p->R[L];
    a2.ldo = k;
    launch_chol(c, a2, s);
    {
        PredScope ps(c, p->flag, 1);
        rmul(p->Qtmp, Np, p->Ri2, Q, ldq);
    }
    {
        PredScope ps(c, p->flag, 0);  // Householder only when CholeskyQR2 was rejected
        qr_factor(c, p, T, ldt, Q, ldq, true, s);
        qr_formq(c, p, T, ldt, Q, ldq, nullptr, s);
    }
}

const double* qr_leaf_factors(QrPlan* p, bool had_cin) {
    const int L = (int)p->nodes.size() - 1;
    if (L == 1 && !had_cin) return p->QN[1];
    return p->C[0];
}

// ---------------------------------------------------------------- Jacobi --
template <int KP>
void launch_jacobi_p2p_t(sorsvd_ctx* c, const JacobiArgs& a, int csize, cudaStream_t s) {
    const size_t sm = jacobi_p2p_smem_bytes(KP, a.ppc);
    allow_smem(jacobi_p2p_kernel<KP>, true);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)csize);
    cfg.blockDim = dim3((unsigned)(32 * a.ppc));
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, jacobi_p2p_kernel<KP>, a));
    check_launch(c);
}

template <int KP>
void launch_jacobi_t(sorsvd_ctx* c, const JacobiArgs& a, int csize, cudaStream_t s) {
    const size_t sm = jacobi_smem_bytes(a.k, a.ppc);
    allow_smem(jacobi_cluster_kernel<KP>, true);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)csize);
    cfg.blockDim = dim3((unsigned)(32 * a.ppc));
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel<KP>, a));
    check_launch(c);
}

template <int KP>
void launch_jacobi_big_t(const JacobiBigArgs& a, int csize, cudaStream_t s) {
    const size_t sm = (size_t)3 * kJbWarps * 2 * (32 * KP) * sizeof(double);  // mailboxes x2 parities + outbox
    allow_smem(jacobi_big_kernel<KP>, true);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)csize);
    cfg.blockDim = dim3(kJbWarps * 32);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, jacobi_big_kernel<KP>, a));
}

// 256 < k <= 512: G-only ring with a rotation log, V rebuilt row-parallel
// (jacobi_big_f64.cuh).
void run_jacobi_big(sorsvd_ctx* c, int k, const double* M, int ldm, double* U, int ldu, double* S, double* V,
                    int ldv, int* sweeps, cudaStream_t s) {
    const int kk = (k + 3) & ~3, P = kk / 2, W = P / 2;
    const int csize = (W + kJbWarps - 1) / kJbWarps;
    if (csize > 16) throw Error{SORSVD_ERR_UNSUPPORTED, "jacobi: k > 512"};
    const int max_sweeps = 40;
    JacobiBigArgs a{};
    a.M = M;
    a.ldm = ldm;
    a.k = k;
    a.kk = kk;
    a.Gout = dbuf(c, "jb_G", (size_t)kk * kk);
    a.tlog = dbuf(c, "jb_log", (size_t)max_sweeps * (kk - 1) * P);
    a.max_sweeps = max_sweeps;
    a.info = reinterpret_cast<int*>(dbuf(c, "jb_info", 1));
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    double* sig = dbuf(c, "jb_sig", (size_t)k);
    double* sgn = dbuf(c, "jb_sgn", (size_t)k);
    int* perm = reinterpret_cast<int*>(dbuf(c, "jb_perm", (size_t)k));
    if (kk <= 384) launch_jacobi_big_t<12>(a, csize, s);
    else launch_jacobi_big_t<16>(a, csize, s);
    check_launch(c);
    const int wpb = 8;
    jb_sigma_kernel<<<(k + wpb - 1) / wpb, 32 * wpb, 0, s>>>(a.Gout, k, kk, sig);
    check_launch(c);
    jb_rank_kernel<<<(k + wpb - 1) / wpb, 32 * wpb, 0, s>>>(a.Gout, k, kk, sig, U, ldu, S, perm, sgn);
    check_launch(c);
    const size_t sm = (size_t)kJbRows * kk * sizeof(double);
    jb_vrec_kernel<<<(k + kJbRows - 1) / kJbRows, P, sm, s>>>(a.tlog, a.info, k, kk, perm, sgn, V, ldv);
    check_launch(c);
    if (sweeps) CK(cudaMemcpyAsync(sweeps, a.info, sizeof(int), cudaMemcpyDeviceToDevice, s));
}

void run_jacobi(sorsvd_ctx* c, int k, const double* M, int ldm, double* U, int ldu, double* S, double* V, int ldv,
                int* sweeps, cudaStream_t s) {
    if (k > 256 || (c->opt_jacobi == SORSVD_JACOBI_ROTLOG && k >= 8)) {
        run_jacobi_big(c, k, M, ldm, U, ldu, S, V, ldv, sweeps, s);
        return;
    }
    JacobiArgs a{};
    a.M = M;
    a.ldm = ldm;
    a.k = k;
    a.U = U;
    a.ldu = ldu;
    a.S = S;
    a.V = V;
    a.ldv = ldv;
    a.max_sweeps = 60;
    a.sweeps_out = sweeps;
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    const int kp = (k + 31) / 32;
    const int KP = kp <= 1 ? 1 : kp <= 2 ? 2 : kp <= 4 ? 4 : 8;
    const int P = ((k + 1) & ~1) / 2;
    if (k > 16 && k <= 32 && c->opt_jacobi != SORSVD_JACOBI_BARRIER) {
        // 16 < k <= 32: the point-to-point ring, one warp per CTA over a P-CTA cluster
        // (measured C1, k = 20: 0.118 -> 0.087 ms); k <= 16 keeps the single CTA (RPCA's
        // k = 10 is faster there)
        const int Pk = ((k + 1) & ~1) / 2;
        a.ppc = 1;
        launch_jacobi_p2p_t<2>(c, a, Pk, s);
        return;
    }
    if (k <= 32 && jacobi_cta_smem_bytes(k) <= 212 * 1024) {
        // small k: one CTA, G and V in shared memory (no cluster barrier needed;
        // measured 4x slower than the cluster ring at k = 100)
        const int warps = std::min(P, 32);
        const size_t sm = jacobi_cta_smem_bytes(k);
        allow_smem(jacobi_cta_kernel<1, 1>);
        jacobi_cta_kernel<1, 1><<<1, 32 * warps, sm, s>>>(a);
        check_launch(c);
        return;
    }
    cudaFuncAttributes fa{};
    switch (KP) {
        case 1: CK(cudaFuncGetAttributes(&fa, jacobi_cluster_kernel<1>)); break;
        case 2: CK(cudaFuncGetAttributes(&fa, jacobi_cluster_kernel<2>)); break;
        case 4: CK(cudaFuncGetAttributes(&fa, jacobi_cluster_kernel<4>)); break;
        default: CK(cudaFuncGetAttributes(&fa, jacobi_cluster_kernel<8>)); break;
    }
    // spread the pair slots over up to 16 CTAs (per-round work is issue bound,
    // so more SMs per round win over the cost of the cluster barrier)
    int ppc = std::min(32, fa.maxThreadsPerBlock / 32);  // register-limited warps per CTA
    while (ppc > 1 && jacobi_smem_bytes(k, ppc) > 200 * 1024) --ppc;
    ppc = std::min(ppc, std::max(1, (P + 15) / 16));
    const int csize = (P + ppc - 1) / ppc;
    if (csize > 16) throw Error{SORSVD_ERR_UNSUPPORTED, "jacobi: cluster too large"};
    a.ppc = (P + csize - 1) / csize;
    // point-to-point ring (mbarrier / st.async, no barrier per round) for 32 < k <= 128:
    // measured k = 100: 0.98 vs 1.17 ms; at k = 256 (KP = 8, 8 warps per CTA) the
    // barrier ring stays faster (5.0 vs 7.4 ms)
    if ((KP == 2 || KP == 4) && c->opt_jacobi != SORSVD_JACOBI_BARRIER &&
        jacobi_p2p_smem_bytes(KP, a.ppc) <= 200 * 1024) {
        if (KP == 2) launch_jacobi_p2p_t<2>(c, a, csize, s);
        else launch_jacobi_p2p_t<4>(c, a, csize, s);
        return;
    }
    switch (KP) {
        case 1: launch_jacobi_t<1>(c, a, csize, s); break;
        case 2: launch_jacobi_t<2>(c, a, csize, s); break;
        case 4: launch_jacobi_t<4>(c, a, csize, s); break;
        default: launch_jacobi_t<8>(c, a, csize, s); break;
    }
}

// ------------------------------------------------------------- pipeline ----
struct SorBuffers {
    double *T1, *T2, *Q1, *Q2, *Y, *Mk, *Uk, *Vk, *Sk, *Uo, *Vo;
    double *T2pre = nullptr, *Lhs = nullptr, *Core = nullptr, *Uc = nullptr, *Vc = nullptr, *Sc = nullptr,
           *Pinv = nullptr;  // single_pass (m_approx)
    double *Psi2 = nullptr, *Y2 = nullptr;  // tsr_svd: second test matrix (m x Np) and row sketch (n x Np)
    float *T1f = nullptr, *T2f = nullptr, *Q2f = nullptr, *Yf = nullptr;  // FP32 path
    int* sweeps;
};

struct SorProblem {
    const double* A;   // FP64 A (dtype F64)
    const float* Af;   // FP32 A (dtype F32): passes on the TF32 tensor cores
    int dtype;
    int64_t m, n, lda;
    int k, ell, q;
    int Np;            // FP64 padded width (npad)
    int Np32;          // FP32 padded width for the tcgen05 passes (npad32)
    int64_t m_global;
    bool single_pass;
    bool tf32;         // dtype F32 with SORSVD_FLAG_TF32: passes on the tcgen05 tensor cores
    bool ozaki;        // SORSVD_FLAG_OZAKI: FP64 passes as int8 slice products on the tcgen05 tensor cores
    bool oz_planes = false;  // ... from digit planes of A cut once per call (ozaki_planes_i8.cuh), memory permitting
    int64_t oz_pm = 0;       // rows [0, oz_pm) of A have planes (== m: all; less: the rest is converted in the passes)
    bool pre_tn = false;     // ... and the first T2 = A^T T1 too (chunk by chunk, K ranges added in order)
    bool pre_first = false;  // host-buffer call: planes and the first T1 = A Omega were produced chunk by chunk
                             // while A was uploading (sor_device's pipelined upload)
    int method = SORSVD_SOR_POWER;  // SORSVD_RSVD / SORSVD_TSR: the baselines of sketch.hpp:124-149
};

SorBuffers prepare_sor(sorsvd_ctx* c, const SorProblem& P, QrPlan** p1, QrPlan** p2, QrPlan** pg) {
    SorBuffers b{};
    const int Np = P.Np;
    b.T1 = dbuf(c, "T1", (size_t)P.m * Np);
    b.T2 = dbuf(c, "T2", (size_t)P.n * Np);
    b.Q1 = dbuf(c, "Q1", (size_t)P.m * Np);
    b.Q2 = dbuf(c, "Q2", (size_t)P.n * Np);
    b.Y = dbuf(c, "Y", (size_t)P.m * Np);
    b.Mk = dbuf(c, "Mk", (size_t)Np * Np);
    b.Uk = dbuf(c, "Uk", (size_t)Np * Np);
    b.Vk = dbuf(c, "Vk", (size_t)Np * Np);
    b.Sk = dbuf(c, "Sk", (size_t)Np);
    b.Uo = dbuf(c, "Uo", (size_t)P.m * Np);
    b.Vo = dbuf(c, "Vo", (size_t)P.n * Np);
    b.sweeps = reinterpret_cast<int*>(dbuf(c, "sweeps", 1));
    if (P.method == SORSVD_TSR) {
        b.Psi2 = dbuf(c, "Psi2", (size_t)P.m * Np);
        b.Y2 = dbuf(c, "Y2", (size_t)P.n * Np);
    }
    if (P.single_pass || P.method == SORSVD_TSR) {
        b.T2pre = dbuf(c, "T2pre", (size_t)P.n * Np);
        b.Lhs = dbuf(c, "Lhs", (size_t)Np * Np);
        b.Core = dbuf(c, "Core", (size_t)Np * Np);
        b.Uc = dbuf(c, "Uc", (size_t)Np * Np);
        b.Vc = dbuf(c, "Vc", (size_t)Np * Np);
        b.Sc = dbuf(c, "Sc", (size_t)Np);
        b.Pinv = dbuf(c, "Pinv", (size_t)Np * Np);
    }
    if (P.tf32) {
        auto fbuf = [&](const char* nm, size_t count) { return reinterpret_cast<float*>(dbuf(c, nm, count / 2 + 2, true)); };
        b.T1f = fbuf("T1f", (size_t)P.m * P.Np32);
        b.T2f = fbuf("T2f", (size_t)P.n * P.Np32);
        b.Q2f = fbuf("Q2f", (size_t)P.n * P.Np32);
        b.Yf = fbuf("Yf", (size_t)P.m * P.Np32);
    }
    *p1 = get_qr_plan(c, P.m, P.ell, 0, "T1");
    *p2 = get_qr_plan(c, P.n, P.ell, 0, "T2");
    *pg = (c->world > 1 && P.ell <= kHouseMaxK) ? get_qr_plan(c, (int64_t)c->world * P.ell, P.ell, c->world, "G")
                                                 : nullptr;
    if (c->world > 1 && P.ell <= kHouseMaxK) {
        dbuf(c, "Rg", (size_t)c->world * P.ell * P.ell);
        dbuf(c, "CinLocal", (size_t)P.ell * Np);
    }
    return b;
}

__global__ void emu_sum_kernel(void* const* bufs, int world, size_t count, int f32) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        if (f32) {
            float acc = 0.f;
            for (int r = 0; r < world; ++r) acc += static_cast<float*>(bufs[r])[i];
            for (int r = 0; r < world; ++r) static_cast<float*>(bufs[r])[i] = acc;
        } else {
            double acc = 0.0;
            for (int r = 0; r < world; ++r) acc += static_cast<double*>(bufs[r])[i];
            for (int r = 0; r < world; ++r) static_cast<double*>(bufs[r])[i] = acc;
        }
    }
}

// Sum-all-reduce of a device buffer across ranks (NCCL, or the emulation group).
void comm_allreduce(sorsvd_ctx* c, void* buf, size_t count, bool f32, cudaStream_t s) {
    if (c->world <= 1) return;
    if (c->comm) {
        NCK(nccl().AllReduce(buf, buf, count, f32 ? ncclFloat : ncclDouble, ncclSum, c->comm, s));
        return;
    }
    if (!c->emu) throw Error{SORSVD_ERR_INTERNAL, "multi-rank context without a communicator"};
    sorsvd_emu_group* g = c->emu;
    CK(cudaStreamSynchronize(s));
    g->bufs[c->rank] = buf;
    g->barrier();
    if (c->rank == 0) {
        void** dp = nullptr;
        CK(cudaMalloc(&dp, sizeof(void*) * g->world));
        CK(cudaMemcpy(dp, g->bufs.data(), sizeof(void*) * g->world, cudaMemcpyHostToDevice));
        emu_sum_kernel<<<std::min<size_t>(cdiv(count, 256), (size_t)c->num_sms * 4), 256, 0, s>>>(dp, g->world, count,
                                                                                                    f32 ? 1 : 0);
        check_launch(c);
        CK(cudaStreamSynchronize(s));
        CK(cudaFree(dp));
    }
    g->barrier();
}

// All-gather of `count` doubles per rank into recv (rank r at r*count).
void comm_allgather(sorsvd_ctx* c, const double* send, double* recv, size_t count, cudaStream_t s) {
    if (c->comm) {
        NCK(nccl().AllGather(send, recv, count, ncclDouble, c->comm, s));
        return;
    }
    sorsvd_emu_group* g = c->emu;
    CK(cudaStreamSynchronize(s));
    g->bufs[c->rank] = const_cast<double*>(send);
    g->barrier();
    for (int r = 0; r < g->world; ++r)
        CK(cudaMemcpyAsync(recv + (size_t)r * count, g->bufs[r], count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    g->barrier();
}

void allreduce_sum(sorsvd_ctx* c, double* buf, size_t count, cudaStream_t s) { comm_allreduce(c, buf, count, false, s); }

void record_stage(sorsvd_ctx* c, bool timing, int idx) {
    if (timing) CK(cudaEventRecord(c->ev_st[idx], c->stream));
}

// M_approx = (Q1^T T1) pinv(Q2^T T2pre)   (sketch.hpp:54-58,100-101; dense.hpp:138-157).
// No pass over A: the single-pass variant trades the projection for the
// pseudo-inverse correction of the ell x ell core.
void enqueue_m_approx(sorsvd_ctx* c, const SorProblem& P, const SorBuffers& b, cudaStream_t s) {
    const int Np = P.Np, ell = P.ell;
    GemmCall g;  // lhs = Q1^T T1 (row-sharded operands: summed over ranks)
    g.ta = true;
    g.A = b.Q1;
    g.lda = Np;
    g.M = ell;
    g.K = P.m;
    g.B = b.T1;
    g.ldb = Np;
    g.N = Np;
    g.C = b.Lhs;
    g.ldc = Np;
    run_gemm(c, g, s);
    allreduce_sum(c, b.Lhs, (size_t)ell * Np, s);
    GemmCall h;  // core = Q2^T W (replicated operands)
    h.ta = true;
    h.A = b.Q2;
    h.lda = Np;
    h.M = ell;
    h.K = P.n;
    h.B = b.T2pre;
    h.ldb = Np;
    h.N = Np;
    h.C = b.Core;
    h.ldc = Np;
    run_gemm(c, h, s);
    run_jacobi(c, ell, b.Core, Np, b.Uc, Np, b.Sc, b.Vc, Np, b.sweeps, s);
    const dim3 grid((unsigned)cdiv(ell, 128), (unsigned)ell);
    const double tol = (double)ell * DBL_EPSILON;  // pseudo_inverse default cutoff (dense.hpp:155-157)
    small_gemm_kernel<<<grid, 128, 0, s>>>(b.Vc, Np, b.Uc, Np, true, b.Sc, tol, b.Pinv, Np, ell);
    check_launch(c);
    small_gemm_kernel<<<grid, 128, 0, s>>>(b.Lhs, Np, b.Pinv, Np, false, nullptr, 0.0, b.Mk, Np, ell);
    check_launch(c);
}

// ------------------------------------------------------ Ozaki (int8) passes --
// Left-operand exponents of A for both orientations (rows for NN, columns for
// TN) from one read of A (ozaki_i8.cuh). Once per call: A is fixed across the
// call's 2q+3 passes.
struct OzScales {
    const int* row_e = nullptr;  // m
    const int* col_e = nullptr;  // n
    // the call's digit planes of A (ozaki_planes_i8.cuh), or null: converted inside every pass
    int8_t* planes = nullptr;
    int64_t pitch = 0, plane_stride = 0;
    int64_t pm = 0, pn = 0;      // the planes' matrix (tensor-map extents)
};

int64_t oz_planes_pitch(int64_t n) { return (n + 15) / 16 * 16; }

// How many leading rows of A can keep their 7 digit planes (7/8 of an FP64 A) beside A? All m when
// they fit with room for the call's other workspaces; else as many whole 128-row tiles as fit, when
// that is at least a quarter of A (config 5 on one GPU: 68.7 GB of FP32 A leaves room for the planes
// of ~5/6 of its rows; the passes convert the remaining rows themselves); else 0. Decided before
// anything is enqueued (the answer is baked into the captured graph).
int64_t oz_planes_rows(sorsvd_ctx* c, const SorProblem& P) {
    if (c->opt_oz_planes == 0 || P.m >= INT_MAX || P.n >= INT_MAX) return 0;
    const size_t row_bytes = (size_t)kOzSlices * (size_t)oz_planes_pitch(P.n);
    int64_t want = P.m;
    if (c->opt_oz_planes > 1) want = std::min<int64_t>(want, c->opt_oz_planes / kOzBM * kOzBM);  // tests: cap the rows
    auto it = c->bufs.find("oz_planes");
    const size_t have = it == c->bufs.end() ? 0 : it->second.bytes;
    if (have >= row_bytes * (size_t)want) return want;
    if (c->capturing) return 0;
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    // growing frees the old buffer first; keep room for the call's other workspaces
    const size_t reserve = ((size_t)6 << 30) + (size_t)(P.m + P.n) * P.Np * 8 * 4;
    const size_t avail = fr + have > reserve ? fr + have - reserve : 0;
    if (avail >= row_bytes * (size_t)want) return want;
    // partial cover: what fits now, but never fewer rows than the workspace this context already
    // holds (a later call on the same A then splits its rows where the earlier one did: same bits)
    int64_t rows = (int64_t)(avail / row_bytes) / kOzBM * kOzBM;
    if (rows < std::max<int64_t>(P.m / 4, 1024)) rows = 0;
    const int64_t rows_have = (int64_t)(have / row_bytes) / kOzBM * kOzBM;
    return std::min(std::max(rows, rows_have), want);
}
bool oz_planes_fit(sorsvd_ctx* c, const SorProblem& P) { return oz_planes_rows(c, P) == P.m; }

template <typename AT>
void launch_rowplanes(sorsvd_ctx* c, const AT* A, const SorProblem& P, int* re, const OzScales& oz, cudaStream_t s) {
    const int vec = ((uintptr_t)A % 16) == 0 && (P.lda * (int64_t)sizeof(AT)) % 16 == 0;
    if (P.n >= 4096) {  // a block per row
        // 2 x 512 threads per SM measured best (C3, per call): 12.9 ms; 4 x 256: 14.8 (the rows in
        // flight outgrow L2 between the two reads); 1 x 1024: 16.0 (the two phases of a row serialise)
        const unsigned blocks = (unsigned)std::min<int64_t>(P.m, (int64_t)c->num_sms * 2);
        ozaki_rowplanes_kernel<AT, 512><<<blocks, 512, 0, s>>>(A, P.lda, P.m, P.n, re, oz.planes, oz.pitch,
                                                               oz.plane_stride, vec, c->pred, c->pred_skip);
    } else {  // a warp per row
        const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(P.m, 16), (int64_t)c->num_sms * 2);
        ozaki_rowplanes_kernel<AT, 32><<<blocks, 512, 0, s>>>(A, P.lda, P.m, P.n, re, oz.planes, oz.pitch,
                                                              oz.plane_stride, vec, c->pred, c->pred_skip);
    }
}

// The call's planes workspace (no kernels): exponents and the 7 digit planes of an m x n A.
OzScales oz_planes_of(sorsvd_ctx* c, const SorProblem& P) {
    OzScales oz{reinterpret_cast<int*>(dbuf(c, "oz_rowe", (size_t)(P.m + 1) / 2)), nullptr};
    const int64_t pm = P.oz_pm > 0 ? P.oz_pm : P.m;
    oz.pitch = oz_planes_pitch(P.n);
    oz.plane_stride = oz.pitch * pm;
    oz.pm = pm;
    oz.pn = P.n;
    oz.planes = reinterpret_cast<int8_t*>(dbuf(c, "oz_planes", (size_t)(kOzSlices * oz.plane_stride + 7) / 8));
    return oz;
}

// Rows [r0, r0 + rows) of A -> their exponents and digit planes (a row chunk of the call's planes).
void oz_convert_rows(sorsvd_ctx* c, const SorProblem& P, const OzScales& oz, int64_t r0, int64_t rows, cudaStream_t s) {
    SorProblem Q = P;
    Q.m = rows;
    OzScales o = oz;
    o.planes = oz.planes + r0 * oz.pitch;
    int* re = const_cast<int*>(oz.row_e) + r0;
    if (P.dtype == SORSVD_F32) launch_rowplanes<float>(c, P.Af + r0 * P.lda, Q, re, o, s);
    else launch_rowplanes<double>(c, P.A + r0 * P.lda, Q, re, o, s);
    check_launch(c);
}

OzScales oz_prepare_a(sorsvd_ctx* c, const SorProblem& P, cudaStream_t s) {
    int* re = reinterpret_cast<int*>(dbuf(c, "oz_rowe", (size_t)(P.m + 1) / 2));
    OzScales oz{re, nullptr};
    int64_t r0 = 0;  // first row without planes
    if (P.oz_planes) {
        // cut A into its row-scaled digit planes once (row maxima and digits in one read of A);
        // every pass of the call streams the planes, TN passes fold the row scales into T1
        oz = oz_planes_of(c, P);
        oz_convert_rows(c, P, oz, 0, oz.pm, s);
        if (oz.pm >= P.m) return oz;
        r0 = oz.pm;  // the planes cover rows [0, pm) only: the rest keeps the in-pass converter's scales
    }
    // rows [r0, m): row exponents, and the column exponents over those rows (the TN left operand)
    const int64_t mb = P.m - r0;
    auto* rmax = reinterpret_cast<unsigned long long*>(dbuf(c, "oz_rowmax", (size_t)mb));
    auto* cmax = reinterpret_cast<unsigned long long*>(dbuf(c, "oz_colmax", (size_t)P.n));
    int* ce = reinterpret_cast<int*>(dbuf(c, "oz_cole", (size_t)(P.n + 1) / 2));
    CK(cudaMemsetAsync(rmax, 0, (size_t)mb * 8, s));
    CK(cudaMemsetAsync(cmax, 0, (size_t)P.n * 8, s));
    const dim3 grid((unsigned)cdiv(P.n, 512), (unsigned)cdiv(mb, 64));
    if (P.dtype == SORSVD_F32)
        ozaki_absmax_kernel<float><<<grid, 256, 0, s>>>(P.Af + r0 * P.lda, P.lda, mb, P.n, rmax, cmax);
    else
        ozaki_absmax_kernel<double><<<grid, 256, 0, s>>>(P.A + r0 * P.lda, P.lda, mb, P.n, rmax, cmax);
    check_launch(c);
    ozaki_exp_kernel<<<(unsigned)std::min<int64_t>(cdiv(mb, 256), c->num_sms * 8), 256, 0, s>>>(rmax, mb, re + r0);
    check_launch(c);
    ozaki_exp_kernel<<<(unsigned)std::min<int64_t>(cdiv(P.n, 256), c->num_sms * 8), 256, 0, s>>>(cmax, P.n, ce);
    check_launch(c);
    oz.col_e = ce;
    return oz;
}

template <bool TA, typename AT>
void launch_ozaki_t(const OzArgs& a0, unsigned grid, cudaStream_t s) {
    OzArgs a = a0;
    // A tiles by TMA when its rows are 16-byte aligned (the tensor map's stride rule), else
    // the converters load them from global memory themselves
    const bool tma = ((uintptr_t)a.A % 16) == 0 && ((a.lda * (int64_t)sizeof(AT)) % 16) == 0;
    CUtensorMap map{};
    if (tma) {
        const int64_t rows = TA ? a.K : a.M, cols = TA ? a.M : a.K;  // A is rows x cols row-major either way
        cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)(a.lda * (int64_t)sizeof(AT))};
        const int e16 = 128 / (int)sizeof(AT);  // elements per 128-byte swizzle row
        cuuint32_t box[2] = {(cuuint32_t)e16, (cuuint32_t)(TA ? kOzBK : kOzBM)};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode_tiled()(&map, sizeof(AT) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                    2, const_cast<void*>(a.A), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error{SORSVD_ERR_CUDA, "cuda: cuTensorMapEncodeTiled failed " + std::to_string((int)r)};
        allow_smem(ozaki_gemm_kernel<TA, AT, true>);
        ozaki_gemm_kernel<TA, AT, true><<<grid, kOzThreads, kOzSmem, s>>>(map, a);
    } else {
        allow_smem(ozaki_gemm_kernel<TA, AT, false>);
        ozaki_gemm_kernel<TA, AT, false><<<grid, kOzThreads, kOzSmem, s>>>(map, a);
    }
}

// Split-K for the planes engine: the number of K splits that minimises the modelled pass
// time on `sms` SMs (waves x (steps per split + fixed cost per CTA) + the partial sum).
int oz_pick_splits(int64_t tiles, int KT, int64_t out_bytes, int sms) {
    const double t_step = 0.62, t_fixed = 12.0;  // us: one 32-deep K step (34 digit MMAs); CTA prologue + drain
    int best = 1;
    double best_cost = 1e300;
    for (int S = 1; S <= 16; ++S) {
        const int per = (int)cdiv(KT, S);
        if (S > 1 && per < 24) break;
        const int Se = (int)cdiv(KT, per);
        const double waves = (double)cdiv(tiles * Se, sms);
        double cost = waves * (per * t_step + t_fixed);
        if (Se > 1) cost += 5.0 + (double)(Se + 1) * (double)out_bytes / 5.0e6;  // reduce: 5 TB/s
        if (cost < best_cost * 0.98) {
            best_cost = cost;
            best = Se;
        }
    }
    return best;
}

// The K partition of the one-launch NN pass T1 = A X of problem P (its row chunks reuse it).
int oz_nn_splits(sorsvd_ctx* c, const SorProblem& P) {
    return oz_pick_splits(cdiv(P.m, kOzBM) * cdiv(P.Np, kOzBN), (int)cdiv(P.n, kOzBK), P.m * P.Np * 8, c->num_sms);
}

// C (M x Np) = op(A) X with X (K x Np row-major): NN (M = m, K = n, left rows = rows
// of A) or TN (M = n, K = m, left rows = columns [n0, n0 + P.n) of the call's A; P
// describes that column block). X is cut into digit planes first. With the call's
// digit planes of A (oz.planes) the pass streams them (ozaki_planes_i8.cuh), else A
// is converted inside the pass kernel (ozaki_i8.cuh).
// The right operand X (K x Np) cut into its digit planes (per-column exponents): shared by every
// launch over the same X.
struct OzX {
    int8_t* Xd = nullptr;
    int* xexp = nullptr;
};

OzX oz_cut_x(sorsvd_ctx* c, const SorProblem& P, bool ta, const OzScales& oz, const double* X, cudaStream_t s) {
    const int Np = P.Np;
    const int NC = (int)cdiv(Np, kOzBN);
    const int64_t K = ta ? P.m : P.n;
    const int64_t KT = cdiv(K, kOzBK);
    const bool planes = oz.planes != nullptr;
    auto* xmax = reinterpret_cast<unsigned long long*>(dbuf(c, ta ? "oz_xmax_tn" : "oz_xmax_nn", (size_t)Np));
    OzX x;
    x.xexp = reinterpret_cast<int*>(dbuf(c, ta ? "oz_xexp_tn" : "oz_xexp_nn", (size_t)(Np + 1) / 2));
    x.Xd = reinterpret_cast<int8_t*>(dbuf(c, ta ? "oz_xd_tn" : "oz_xd_nn", (size_t)(KT * NC * kOzXStep + 7) / 8));
    CK(cudaMemsetAsync(xmax, 0, (size_t)Np * 8, s));
    const dim3 cgrid((unsigned)cdiv(Np, 32), (unsigned)std::min<int64_t>(cdiv(K, kOzCmRows), 32768));
    const int64_t items = KT * 2 * (int64_t)NC * kOzBN;
    const unsigned xblocks = (unsigned)std::min<int64_t>(cdiv(items, 256), (int64_t)c->num_sms * 16);
    if (planes && ta) {  // the planes are row-scaled: A's row scales ride on the right operand
        ozaki_colmax_scaled_kernel<<<cgrid, 256, 0, s>>>(X, Np, K, Np, oz.row_e, xmax);
        check_launch(c);
        ozaki_exp_kernel<<<1, 256, 0, s>>>(xmax, Np, x.xexp);
        check_launch(c);
        ozaki_xdigits_scaled_kernel<<<xblocks, 256, 0, s>>>(X, Np, K, Np, NC, oz.row_e, x.xexp, x.Xd);
        check_launch(c);
    } else {
        ozaki_colmax_kernel<<<cgrid, 256, 0, s>>>(X, Np, K, Np, xmax);
        check_launch(c);
        ozaki_exp_kernel<<<1, 256, 0, s>>>(xmax, Np, x.xexp);
        check_launch(c);
        ozaki_xdigits_kernel<<<xblocks, 256, 0, s>>>(X, Np, K, Np, NC, x.xexp, x.Xd);
        check_launch(c);
    }
    return x;
}

// One launch of the planes engine over left rows [l0, l0 + M) of the planes (NN: rows of A; TN:
// columns of A): C (M x Np, the caller's pointer to the block's first row) = op(A)[l0 ..] X.
// TN only: k0 = first row of the K range this launch contracts over (P.m = its length), acc = add to C.
void oz_launch_planes(sorsvd_ctx* c, const SorProblem& P, bool ta, const OzScales& oz, const OzX& x, double* C,
                      int64_t l0, int64_t M, cudaStream_t s, int dbg = 0, int64_t k0 = 0, bool acc = false,
                      int splits = 0) {
    const int Np = P.Np;
    const int NC = (int)cdiv(Np, kOzBN);
    const int64_t K = ta ? P.m : P.n;
    const int64_t KT = cdiv(K, kOzBK);
    OzpArgs a{};
    a.M = M;
    a.K = K;
    a.mn0 = (int)l0;
    a.kt0 = (int)(k0 / kOzBK);
    a.acc0 = (acc && true) ? 1 : 0;
    a.lexp = ta ? nullptr : oz.row_e + l0;
    a.Xd = x.Xd;
    a.xexp = x.xexp;
    a.NC = NC;
    a.N = Np;
    a.ldc = Np;
    a.dbg = dbg;
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    const int64_t tiles = cdiv(M, kOzBM) * NC;
    // splits > 0: the caller's K partition (a row chunk of a pass keeps the whole pass's, so that
    // its rows come out with the same bits as from the one-launch pass)
    const int S = splits > 0 ? splits : oz_pick_splits(tiles, (int)KT, M * Np * 8, c->num_sms);
    a.kt_split = (int)cdiv(KT, S);
    a.c_split_stride = M * Np;
    double* ws = S > 1 ? dbuf(c, "oz_split", (size_t)S * M * Np) : nullptr;
    a.C = S > 1 ? ws : C;
    if (S > 1) a.acc0 = 0;  // the partials start from zero; the reduction adds them to C
    // NC column-chunk CTAs of a row tile as one cluster sharing the A planes by TMA multicast
    const bool mc = c->opt_oz_multicast && NC >= 2 && NC <= 8;
    CUtensorMap map{};
    cuuint64_t dims[3] = {(cuuint64_t)oz.pn, (cuuint64_t)oz.pm, (cuuint64_t)kOzSlices};
    cuuint64_t strides[2] = {(cuuint64_t)oz.pitch, (cuuint64_t)oz.plane_stride};
    cuuint32_t box[3] = {(cuuint32_t)(ta ? kOzBM : kOzBK), (cuuint32_t)(ta ? kOzBK : kOzBM),
                         (cuuint32_t)(mc ? 1 : kOzSlices)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, oz.planes, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, ta ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error{SORSVD_ERR_CUDA, "cuda: cuTensorMapEncodeTiled (planes) failed " + std::to_string((int)r)};
    const dim3 grid((unsigned)tiles, (unsigned)S);
    if (mc) {
        auto kern = ta ? ozaki_planes_gemm_kernel<true, true> : ozaki_planes_gemm_kernel<false, true>;
        allow_smem(kern, true);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kOzpThreads);
        cfg.dynamicSmemBytes = kOzpSmem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)NC;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, kern, map, a));
    } else if (ta) {
        allow_smem(ozaki_planes_gemm_kernel<true, false>);
        ozaki_planes_gemm_kernel<true, false><<<grid, kOzpThreads, kOzpSmem, s>>>(map, a);
    } else {
        allow_smem(ozaki_planes_gemm_kernel<false, false>);
        ozaki_planes_gemm_kernel<false, false><<<grid, kOzpThreads, kOzpSmem, s>>>(map, a);
    }
    check_launch(c);
    if (S > 1 && acc) {
        const int blocks = (int)std::min<int64_t>(cdiv(M * Np, 256), (int64_t)c->num_sms * 8);
        oz_reduce_acc_kernel<<<blocks, 256, 0, s>>>(ws, M * Np, S, M * Np, C, 1, c->pred, c->pred_skip);
        check_launch(c);
    } else if (S > 1) {
        const int64_t count2 = M * Np / 2;
        const int blocks = (int)std::min<int64_t>(cdiv(count2, 256), (int64_t)c->num_sms * 8);
        reduce_splits_kernel<<<blocks, 256, 0, s>>>(ws, count2, S, M * Np, C, c->pred, c->pred_skip);
        check_launch(c);
    }
}

// The in-pass converter engine (ozaki_i8.cuh) over rows [r0, m) of A (r0 = 0: all of A): NN writes
// C's rows [r0, m); TN contracts over those rows only and, with acc, adds to C (the planes engine
// wrote the contribution of rows [0, r0) first).
void oz_launch_convert(sorsvd_ctx* c, const SorProblem& P, bool ta, const OzScales& oz, const OzX& x, double* C,
                       int64_t r0, int64_t n0, bool acc, cudaStream_t s, int dbg) {
    const int Np = P.Np;
    const int NC = (int)cdiv(Np, kOzBN);
    const int64_t mb = P.m - r0;
    const int64_t M = ta ? P.n : mb, K = ta ? mb : P.n;
    OzArgs a{};
    a.A = P.dtype == SORSVD_F32 ? static_cast<const void*>(P.Af + r0 * P.lda) : static_cast<const void*>(P.A + r0 * P.lda);
    a.lda = P.lda;
    a.M = M;
    a.K = K;
    a.lexp = ta ? oz.col_e + n0 : oz.row_e + r0;
    a.Xd = x.Xd;
    a.xexp = x.xexp;
    a.NC = NC;
    a.N = Np;
    a.C = ta ? C : C + r0 * Np;
    a.ldc = Np;
    a.dbg = dbg;
    a.acc0 = acc ? 1 : 0;
    a.vec = ((uintptr_t)a.A % 16) == 0 && (P.dtype == SORSVD_F32 ? P.lda % 4 : P.lda % 2) == 0;
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    const unsigned grid = (unsigned)(cdiv(M, kOzBM) * NC);
    if (P.dtype == SORSVD_F32) {
        if (ta) launch_ozaki_t<true, float>(a, grid, s);
        else launch_ozaki_t<false, float>(a, grid, s);
    } else {
        if (ta) launch_ozaki_t<true, double>(a, grid, s);
        else launch_ozaki_t<false, double>(a, grid, s);
    }
    check_launch(c);
}

void run_ozaki(sorsvd_ctx* c, const SorProblem& P, bool ta, const OzScales& oz, const double* X, double* C,
               cudaStream_t s, int dbg = 0, int64_t n0 = 0) {
    const int64_t M = ta ? P.n : P.m;
    const int64_t pm = oz.planes ? std::min(oz.pm, P.m) : 0;  // rows with planes
    if (pm >= P.m) {  // all of A from its digit planes
        const OzX ox = oz_cut_x(c, P, ta, oz, X, s);
        oz_launch_planes(c, P, ta, oz, ox, C, ta ? n0 : 0, M, s, dbg);
        return;
    }
    if (pm == 0) {  // A converted inside the pass
        const OzX ox = oz_cut_x(c, P, ta, oz, X, s);
        oz_launch_convert(c, P, ta, oz, ox, C, 0, n0, false, s, dbg);
        return;
    }
    // planes for rows [0, pm), the in-pass converter for rows [pm, m)
    if (!ta) {  // the two row ranges are independent outputs; X is cut once (plain per-column cut)
        OzScales plain = oz;
        plain.planes = nullptr;
        const OzX ox = oz_cut_x(c, P, false, plain, X, s);
        oz_launch_planes(c, P, false, oz, ox, C, 0, pm, s, dbg);
        oz_launch_convert(c, P, false, oz, ox, C, pm, 0, false, s, dbg);
        return;
    }
    // TN: T2 = A_top^T T1_top (planes; the top rows' scales ride on T1_top) + A_bot^T T1_bot
    SorProblem Qt = P;
    Qt.m = pm;
    const OzX xt = oz_cut_x(c, Qt, true, oz, X, s);
    oz_launch_planes(c, Qt, true, oz, xt, C, n0, M, s, dbg);
    SorProblem Qb = P;
    Qb.m = P.m - pm;
    OzScales plain = oz;
    plain.planes = nullptr;
    const OzX xb = oz_cut_x(c, Qb, true, plain, X + pm * P.Np, s);  // stream order: after the top launch read xt
    oz_launch_convert(c, P, true, oz, xb, C, pm, n0, true, s, dbg);
}

// Q = thin_qr(T).q of a row-sharded m x ell operand (the sketch T1 / Y; sketch.hpp:98, :129, :145):
// single rank -> the plain QR; multi-rank -> the local TSQR runs to one R per rank, the k x k R's
// cross ranks by all-gather, every rank solves the small cross-rank tree redundantly and applies
// its own k x k factor to its local leaves (k > 256: the CholeskyQR Gram matrices are summed).
void qr_rows(sorsvd_ctx* c, const SorProblem& P, QrPlan* p1, QrPlan* pg, double* T, double* Q, cudaStream_t s) {
    const int Np = P.Np, ell = P.ell;
    if (c->world > 1 && p1->big) {
        qr_run_big(c, p1, T, Np, Q, Np, s, P.m_global, true);
    } else if (c->world > 1) {
        qr_factor(c, p1, T, Np, Q, Np, false, s);
        const int L1 = (int)p1->nodes.size() - 1;
        double* Rg = dbuf(c, "Rg", (size_t)c->world * ell * ell);
        comm_allgather(c, p1->R[L1], Rg, (size_t)ell * ell, s);
        qr_factor(c, pg, nullptr, 0, nullptr, 0, true, s, Rg);
        qr_formq(c, pg, nullptr, 0, nullptr, 0, nullptr, s, true);
        const double* Cg = qr_leaf_factors(pg, false) + (size_t)c->rank * ell * Np;
        qr_formq(c, p1, T, Np, Q, Np, Cg, s);
    } else {
        qr_run(c, p1, T, Np, Q, Np, s);
    }
}

// T2 = A^T T1 summed over the ranks' row blocks (sketch.hpp:96). Single rank: one
// launch. Multi-rank: the pass runs as kTnBlocks launches over column blocks of A
// (row blocks of T2), and each finished block's all-reduce is issued on the comm
// stream while the next block's GEMM runs, so only the last block's reduction
// is exposed; the compute stream joins the comm stream before T2 is used.
void tn_pass_reduced(sorsvd_ctx* c, const SorProblem& P, const double* T1, double* T2, cudaStream_t s,
                     const OzScales* oz = nullptr) {
    const int Np = P.Np;
    auto tn = [&](int64_t n0, int64_t n1) {
        if (P.ozaki) {  // the column block [n0, n1) of A as its own TN problem (its columns' exponents)
            SorProblem Q = P;
            Q.A = P.A ? P.A + n0 : nullptr;
            Q.Af = P.Af ? P.Af + n0 : nullptr;
            Q.n = n1 - n0;
            run_ozaki(c, Q, true, *oz, T1, T2 + n0 * Np, s, 0, n0);
            return;
        }
        GemmCall g2;
        g2.ta = true;
        g2.A = P.A ? P.A + n0 : nullptr;
        g2.Af = P.Af ? P.Af + n0 : nullptr;
        g2.lda = P.lda;
        g2.M = n1 - n0;
        g2.K = P.m;
        g2.B = T1;
        g2.ldb = Np;
        g2.N = Np;
        g2.C = T2 + n0 * Np;
        g2.ldc = Np;
        g2.sk_bias = Np <= 128 ? 1.0 : 0.95;
        run_gemm(c, g2, s);
    };
    constexpr int NB = sorsvd_ctx::kTnBlocks;
    const int BM = P.ozaki ? kOzBM : gemm_bm_for(Np);
    if (c->world <= 1 || P.n < (int64_t)NB * BM) {
        tn(0, P.n);
        allreduce_sum(c, T2, (size_t)P.n * Np, s);
        return;
    }
    // block edges on tile boundaries (multiples of BM keep A's column offset 16-byte aligned)
    const int64_t tiles = cdiv(P.n, BM);
    for (int bi = 0; bi < NB; ++bi) {
        const int64_t n0 = std::min<int64_t>(P.n, tiles * bi / NB * BM);
        const int64_t n1 = bi == NB - 1 ? P.n : std::min<int64_t>(P.n, tiles * (bi + 1) / NB * BM);
        if (n1 <= n0) continue;
        tn(n0, n1);
        CK(cudaEventRecord(c->ev_blk[bi], s));
        CK(cudaStreamWaitEvent(c->comm_stream, c->ev_blk[bi], 0));
        comm_allreduce(c, T2 + n0 * Np, (size_t)(n1 - n0) * Np, false, c->comm_stream);
    }
    CK(cudaEventRecord(c->ev_comm, c->comm_stream));
    CK(cudaStreamWaitEvent(s, c->ev_comm, 0));
}

// ---------------------------------------------- fused NN + TN sweeps (narrow) --
// One power step T1 = A X, T2 = A^T T1 (or the projection M = Q1^T (A Q2)) in one sweep over A for
// narrow sketches over narrow matrices (skinny_pair_f64.cuh): FP64 A, ell <= 16, n <= 512.
bool pair_ok(const sorsvd_ctx* c, const SorProblem& P) {
    return c->opt_fused_pair && P.dtype == SORSVD_F64 && !P.tf32 && !P.ozaki && P.Np <= kPairNP && P.n <= 512 && P.n >= 2;
}

// T1 (m x Np) = A X; out2 = A^T T1 (n x Np, proj = false) or L^T T1 (Np x Np, proj = true: L = Q1).
void run_pair(sorsvd_ctx* c, const SorProblem& P, const double* X, double* T1, double* out2, bool proj,
              const double* L, cudaStream_t s) {
    PairArgs a{};
    a.A = P.A;
    a.lda = P.lda;
    a.m = P.m;
    a.n = (int)P.n;
    a.X = X;
    a.ldx = P.Np;
    a.np = P.Np;
    a.T1 = T1;
    a.ldt = P.Np;
    a.L = L;
    a.ldl = P.Np;
    a.vec = ((uintptr_t)P.A % 16) == 0 && P.lda % 2 == 0;
    a.pred = c->pred;
    a.pred_skip = c->pred_skip;
    // n <= 320: two independent 8-warp halves per CTA on alternate 16-row blocks (skinny_pair2_kernel)
    const bool two = c->opt_fused_pair == 1 && a.n <= 320 && pair2_smem_bytes(a.n, proj) <= (size_t)227 * 1024;
    a.rb = two ? kPair2Rb : pair_smem_bytes(a.n, 32, proj) <= (size_t)227 * 1024 ? 32 : 16;
    const size_t smem = two ? pair2_smem_bytes(a.n, proj) : pair_smem_bytes(a.n, a.rb, proj);
    const int rows2 = proj ? kPairNP : a.n;
    const int grid = (int)std::min<int64_t>(c->num_sms, cdiv(P.m, two ? 2 * a.rb : a.rb));
    a.part = dbuf(c, proj ? "pair_part_p" : "pair_part", (size_t)grid * rows2 * kPairNP);
    if (two && proj) {
        allow_smem(skinny_pair2_kernel<true>);
        skinny_pair2_kernel<true><<<grid, kPairThreads, smem, s>>>(a);
    } else if (two) {
        allow_smem(skinny_pair2_kernel<false>);
        skinny_pair2_kernel<false><<<grid, kPairThreads, smem, s>>>(a);
    } else if (proj) {
        allow_smem(skinny_pair_kernel<true>);
        skinny_pair_kernel<true><<<grid, kPairThreads, smem, s>>>(a);
    } else {
        allow_smem(skinny_pair_kernel<false>);
        skinny_pair_kernel<false><<<grid, kPairThreads, smem, s>>>(a);
    }
    check_launch(c);
    pair_reduce_kernel<<<(unsigned)cdiv((int64_t)rows2 * kPairNP, 32), 256, 0, s>>>(
        a.part, grid, rows2, proj ? P.Np : rows2, P.Np, out2, P.Np, c->pred, c->pred_skip);
    check_launch(c);
}

// Enqueue one sor_svd_power on c->stream (T2 must already hold Omega, padded).
void enqueue_sor(sorsvd_ctx* c, const SorProblem& P, const SorBuffers& b, QrPlan* p1, QrPlan* p2, QrPlan* pg,
                 bool timing) {
    cudaStream_t s = c->stream;
    const int Np = P.Np, ell = P.ell;
    record_stage(c, timing, 0);
    OzScales oz;
    bool first_done = P.pre_first;  // T1 = A Omega of pass 0 already produced (with the planes)
    if (P.ozaki && P.pre_first) {
        oz = oz_planes_of(c, P);
    } else if (P.ozaki && P.oz_pm == P.m && c->opt_oz_overlap && !P.single_pass) {
        // Conversion and first pass interleaved by row chunks: chunk i + 1 is cut into planes on the side
        // stream (HBM-bound, one 512-thread block fits beside a pass CTA: the pass kernel is capped at 96
        // registers for this) while the first pass T1 = A Omega sweeps chunk i (tensor-bound). Rows are
        // independent, so the bits are those of convert-all-then-pass.
        oz = oz_planes_of(c, P);
        const OzX ox = oz_cut_x(c, P, false, oz, b.T2, s);
        const int NC = (int)cdiv(Np, kOzBN);
        int g = c->num_sms, h = NC;
        while (h) {
            const int t = g % h;
            g = h;
            h = t;
        }
        const int s_full = oz_nn_splits(c, P);
        const int64_t unit_rows = (int64_t)(c->num_sms / g) * kOzBM;  // whole waves of 128-row tiles
        const int64_t units = cdiv(P.m, unit_rows);
        const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(10, units));
        const int64_t rows_per = cdiv(units, nch) * unit_rows;
        const int nchunks = (int)cdiv(P.m, rows_per);
        while ((int)c->up_ev.size() < nchunks) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->up_ev.push_back(e);
        }
        CK(cudaEventRecord(c->ev_fork, s));
        CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
        oz_convert_rows(c, P, oz, 0, std::min(rows_per, P.m), c->side);
        CK(cudaEventRecord(c->up_ev[0], c->side));
        for (int i = 0; i < nchunks; ++i) {
            const int64_t r0 = (int64_t)i * rows_per, rows = std::min(rows_per, P.m - r0);
            if (i + 1 < nchunks) {
                const int64_t r1 = r0 + rows_per;
                oz_convert_rows(c, P, oz, r1, std::min(rows_per, P.m - r1), c->side);
                CK(cudaEventRecord(c->up_ev[(size_t)i + 1], c->side));
            }
            CK(cudaStreamWaitEvent(s, c->up_ev[(size_t)i], 0));
            oz_launch_planes(c, P, false, oz, ox, b.T1 + r0 * Np, r0, rows, s, 0, 0, false, s_full);
        }
        first_done = true;
    } else if (P.ozaki) {
        oz = oz_prepare_a(c, P, s);
    }
    for (int i = 0; i <= P.q; ++i) {
        if (P.single_pass && i == P.q) {  // t2_pre: the row sketch entering the last iteration (sketch.hpp:94)
            if (P.tf32)
                cast_to_f64(c, b.T2f, P.Np32, b.T2pre, Np, P.n, ell, s);
            else
                CK(cudaMemcpyAsync(b.T2pre, b.T2, (size_t)P.n * Np * 8, cudaMemcpyDeviceToDevice, s));
        }
        if (P.tf32) {  // TF32 tensor-core passes (tc_gemm_f32.cuh)
            run_tc_gemm(c, false, P.Af, P.lda, P.m, P.n, b.T2f, P.Np32, P.Np32, b.T1f, P.Np32, s);
            run_tc_gemm(c, true, P.Af, P.lda, P.n, P.m, b.T1f, P.Np32, P.Np32, b.T2f, P.Np32, s);
            comm_allreduce(c, b.T2f, (size_t)P.n * P.Np32, true, s);
            continue;
        }
        if (P.ozaki) {  // FP64 passes as int8 slice products (ozaki_i8.cuh)
            if (!(first_done && i == 0)) run_ozaki(c, P, false, oz, b.T2, b.T1, s);  // T1 = A T2   (sketch.hpp:95)
            if (!(P.pre_tn && i == 0)) tn_pass_reduced(c, P, b.T1, b.T2, s, &oz);  // T2 = A^T T1 (sketch.hpp:96), summed over ranks
            continue;
        }
        if (pair_ok(c, P)) {  // T1 = A T2 and T2 = A^T T1 in one sweep over A (skinny_pair_f64.cuh)
            run_pair(c, P, b.T2, b.T1, b.T2, false, nullptr, s);
            allreduce_sum(c, b.T2, (size_t)P.n * Np, s);
            continue;
        }
        GemmCall g1;  // T1 = A * T2     (sketch.hpp:95); FP32 A widened to FP64 in the kernel
        g1.A = P.A;
        g1.Af = P.Af;
        g1.lda = P.lda;
        g1.M = P.m;
        g1.K = P.n;
        g1.B = b.T2;
        g1.ldb = Np;
        g1.N = Np;
        g1.C = b.T1;
        g1.ldc = Np;
        g1.sk_bias = Np <= 128 ? 1.0 : 0.95;
        run_gemm(c, g1, s);
        tn_pass_reduced(c, P, b.T1, b.T2, s);  // T2 = A^T * T1   (sketch.hpp:96), summed over ranks
    }
    if (P.tf32) {  // the QR / SVD stages run in FP64
        cast_to_f64(c, b.T1f, P.Np32, b.T1, Np, P.m, ell, s);
        cast_to_f64(c, b.T2f, P.Np32, b.T2, Np, P.n, ell, s);
    }
    record_stage(c, timing, 1);
    // Q1 = thin_qr(T1).q, Q2 = thin_qr(T2).q concurrently (sketch.hpp:98-99)
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    const bool keep_t1 = P.single_pass && c->world > 1;  // the sharded TSQR factors T1 in place
    if (keep_t1) CK(cudaMemcpyAsync(b.Y, b.T1, (size_t)P.m * Np * 8, cudaMemcpyDeviceToDevice, s));
    qr_rows(c, P, p1, pg, b.T1, b.Q1, s);
    qr_run(c, p2, b.T2, Np, b.Q2, Np, c->side);
    CK(cudaEventRecord(c->ev_join, c->side));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    record_stage(c, timing, 2);
    if (P.single_pass) {
        SorBuffers bm = b;
        if (keep_t1) bm.T1 = b.Y;
        enqueue_m_approx(c, P, bm, s);
    } else {
    // M = Q1^T (A Q2)   (sketch.hpp:100-102)
    if (P.tf32) {
        cast_to_f32(c, b.Q2, Np, b.Q2f, P.Np32, P.n, ell, s);
        run_tc_gemm(c, false, P.Af, P.lda, P.m, P.n, b.Q2f, P.Np32, P.Np32, b.Yf, P.Np32, s);
        cast_to_f64(c, b.Yf, P.Np32, b.Y, Np, P.m, ell, s);
    }
    {
        GemmCall g;
        g.A = P.A;
        g.lda = P.lda;
        g.M = P.m;
        g.K = P.n;
        g.B = b.Q2;
        g.ldb = Np;
        g.N = Np;
        g.C = b.Y;
        g.ldc = Np;
        g.Af = P.Af;
        g.sk_bias = Np <= 128 ? 1.0 : 0.95;
        if (pair_ok(c, P)) {  // Y = A Q2 and M = Q1^T Y in one sweep over A (skinny_pair_f64.cuh)
            CK(cudaMemsetAsync(b.Mk, 0, (size_t)Np * Np * 8, s));
            run_pair(c, P, b.Q2, b.Y, b.Mk, true, b.Q1, s);
        } else {
        if (P.ozaki) run_ozaki(c, P, false, oz, b.Q2, b.Y, s);
        else if (!P.tf32) run_gemm(c, g, s);
        GemmCall h;
        h.ta = true;
        h.A = b.Q1;
        h.lda = Np;
        h.M = ell;
        h.K = P.m;
        h.B = b.Y;
        h.ldb = Np;
        h.N = Np;
        h.C = b.Mk;
        h.ldc = Np;
        run_gemm(c, h, s);
        }
        allreduce_sum(c, b.Mk, (size_t)ell * Np, s);
    }
    }
    record_stage(c, timing, 3);
    // truncated_svd(M, k)   (sketch.hpp:103)
    run_jacobi(c, ell, b.Mk, Np, b.Uk, Np, b.Sk, b.Vk, Np, b.sweeps, s);
    record_stage(c, timing, 4);
    // U = Q1 Ut_k, V = Q2 Vt_k   (sketch.hpp:105,107), the two products side by side
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    {
        GemmCall g;
        g.A = b.Q1;
        g.lda = Np;
        g.M = P.m;
        g.K = ell;
        g.B = b.Uk;
        g.ldb = Np;
        g.N = Np;
        g.C = b.Uo;
        g.ldc = Np;
        run_gemm(c, g, s);
        GemmCall h;
        h.A = b.Q2;
        h.lda = Np;
        h.M = P.n;
        h.K = ell;
        h.B = b.Vk;
        h.ldb = Np;
        h.N = Np;
        h.C = b.Vo;
        h.ldc = Np;
        h.ws_name = "gemm_ws_side";
        run_gemm(c, h, c->side);
    }
    CK(cudaEventRecord(c->ev_join, c->side));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    record_stage(c, timing, 5);
}

__global__ void transpose_pad_kernel(const double* __restrict__ src, int64_t lds, int k, double* __restrict__ dst,
                                     int ldd) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ldd * ldd; e += gridDim.x * blockDim.x) {
        const int i = e / ldd, j = e - i * ldd;
        dst[e] = (i < k && j < k) ? src[(int64_t)j * lds + i] : 0.0;
    }
}

// One skinny GEMM C = op(A) B over the whole A (the sketch passes of the baselines).
void pass_gemm(sorsvd_ctx* c, const SorProblem& P, bool ta, const double* B, double* C, cudaStream_t s) {
    GemmCall g;
    g.ta = ta;
    g.A = P.A;
    g.Af = P.Af;
    g.lda = P.lda;
    g.M = ta ? P.n : P.m;
    g.K = ta ? P.m : P.n;
    g.B = B;
    g.ldb = P.Np;
    g.N = P.Np;
    g.C = C;
    g.ldc = P.Np;
    g.sk_bias = P.Np <= 128 ? 1.0 : 0.95;
    run_gemm(c, g, s);
}

// U = Q1 Uk (m x Np), V = Q2 Vk (n x Np)   (sketch.hpp:105,107 / :135 / :147)
void enqueue_basis(sorsvd_ctx* c, const SorProblem& P, const SorBuffers& b, cudaStream_t s) {
    for (int h = 0; h < 2; ++h) {
        GemmCall g;
        g.A = h ? b.Q2 : b.Q1;
        g.lda = P.Np;
        g.M = h ? P.n : P.m;
        g.K = P.ell;
        g.B = h ? b.Vk : b.Uk;
        g.ldb = P.Np;
        g.N = P.Np;
        g.C = h ? b.Vo : b.Uo;
        g.ldc = P.Np;
        run_gemm(c, g, s);
    }
}

// r_svd (sketch.hpp:124-136): Y = (A A^T)^q A Omega, Qy = thin_qr(Y).q,
// B = Qy^T A, full_svd(B), U = Qy U_B. T2 holds Omega on entry.
// full_svd of the ell x n B (dense.hpp:65) runs as B^T = A^T Qy = Qb Rb
// (one more TN pass + a thin QR), then the ell x ell one-sided Jacobi on
// Rb^T = U_B S (Vj)^T, so U_B comes out of the Jacobi kernel with the
// reference sign canonicalisation (dense.hpp:80-95) and V = Qb Vj.
// Row-sharded A: Y and Qy are row blocks (local passes, the sharded TSQR), every A^T product is summed
// over ranks, B^T's QR / the Jacobi SVD / V are replicated.
void enqueue_rsvd(sorsvd_ctx* c, const SorProblem& P, const SorBuffers& b, QrPlan* p1, QrPlan* p2, QrPlan* pg,
                  bool timing) {
    cudaStream_t s = c->stream;
    record_stage(c, timing, 0);
    pass_gemm(c, P, false, b.T2, b.T1, s);  // Y = A Omega        (:127)
    for (int i = 0; i < P.q; ++i) {         // Y = A (A^T Y)      (:128)
        tn_pass_reduced(c, P, b.T1, b.T2, s);
        pass_gemm(c, P, false, b.T2, b.T1, s);
    }
    record_stage(c, timing, 1);
    qr_rows(c, P, p1, pg, b.T1, b.Q1, s);      // Qy = thin_qr(Y).q   (:129)
    record_stage(c, timing, 2);
    tn_pass_reduced(c, P, b.Q1, b.T2, s);      // B^T = A^T Qy       (:130)
    qr_run(c, p2, b.T2, P.Np, b.Q2, P.Np, s);  // B^T = Qb Rb
    const int L = (int)p2->nodes.size() - 1;
    transpose_pad_kernel<<<std::min(cdiv((int64_t)P.Np * P.Np, 256), (int64_t)c->num_sms), 256, 0, s>>>(
        p2->R[L], p2->ldR, P.ell, b.Mk, P.Np);  // Rb^T = B Qb
    check_launch(c);
    record_stage(c, timing, 3);
    run_jacobi(c, P.ell, b.Mk, P.Np, b.Uk, P.Np, b.Sk, b.Vk, P.Np, b.sweeps, s);  // full_svd(B)   (:131)
    record_stage(c, timing, 4);
    enqueue_basis(c, P, b, s);  // U = Qy U_B (:132), V = Qb Vj
    record_stage(c, timing, 5);
}

// tsr_svd (sketch.hpp:139-149): Y1 = A Psi1, Y2 = A^T Psi2 (Psi2 from seed^1),
// Q1 = thin_qr(Y1).q, Q2 = thin_qr(Y2).q, B = m_approx(Q1, Y1, Q2, Psi1),
// full_svd(B), U = Q1 U_B, V = Q2 V_B. T2 holds Psi1, b.Psi2 holds Psi2.
// The two sketches are two launches over A here (the reference counts the
// pair as its one pass, sketch.hpp:148).
// Row-sharded A: Psi2's rows are this rank's rows of gaussian_matrix(m_global, ell, seed ^ 1); Y2 is
// summed over ranks; Q1 by the sharded TSQR; m_approx sums Q1^T Y1 over ranks.
void enqueue_tsr(sorsvd_ctx* c, const SorProblem& P, const SorBuffers& b, QrPlan* p1, QrPlan* p2, QrPlan* pg,
                 bool timing) {
    cudaStream_t s = c->stream;
    record_stage(c, timing, 0);
    pass_gemm(c, P, false, b.T2, b.T1, s);       // Y1 = A Psi1     (:143)
    tn_pass_reduced(c, P, b.Psi2, b.Y2, s);      // Y2 = A^T Psi2   (:144)
    record_stage(c, timing, 1);
    if (c->world > 1) {  // collectives stay on one stream: the two QRs run one after the other
        // the sharded TSQR factors its operand in place: keep Y1 for m_approx's Q1^T Y1
        CK(cudaMemcpyAsync(b.Y, b.T1, (size_t)P.m * P.Np * 8, cudaMemcpyDeviceToDevice, s));
        qr_rows(c, P, p1, pg, b.T1, b.Q1, s);
        qr_run(c, p2, b.Y2, P.Np, b.Q2, P.Np, s);
        record_stage(c, timing, 2);
        SorBuffers bb = b;
        bb.T2pre = b.T2;
        bb.T1 = b.Y;
        enqueue_m_approx(c, P, bb, s);
        record_stage(c, timing, 3);
        run_jacobi(c, P.ell, b.Mk, P.Np, b.Uk, P.Np, b.Sk, b.Vk, P.Np, b.sweeps, s);
        record_stage(c, timing, 4);
        enqueue_basis(c, P, b, s);
        record_stage(c, timing, 5);
        return;
    }
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    qr_run(c, p1, b.T1, P.Np, b.Q1, P.Np, s);        // (:145)
    qr_run(c, p2, b.Y2, P.Np, b.Q2, P.Np, c->side);  // (:146)
    CK(cudaEventRecord(c->ev_join, c->side));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    record_stage(c, timing, 2);
    SorBuffers bb = b;
    bb.T2pre = b.T2;  // m_approx's W is Psi1 itself (:147)
    enqueue_m_approx(c, P, bb, s);
    record_stage(c, timing, 3);
    run_jacobi(c, P.ell, b.Mk, P.Np, b.Uk, P.Np, b.Sk, b.Vk, P.Np, b.sweeps, s);  // full_svd(B)  (:148)
    record_stage(c, timing, 4);
    enqueue_basis(c, P, b, s);
    record_stage(c, timing, 5);
}

// Count of non-finite entries of a row-major FP64 / FP32 matrix (failure path
// only: the reference rejects such input in the Matrix constructor,
// matrix.hpp:32-33, before any arithmetic).
template <typename T>
__global__ void nonfinite_count_kernel(const T* __restrict__ a, int64_t m, int64_t n, int64_t lda,
                                       unsigned long long* out) {
    unsigned long long cnt = 0;
    const int64_t total = m * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        cnt += isfinite((double)a[i * lda + j]) ? 0ull : 1ull;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

// True when any rank's A block holds a NaN / Inf.
bool matrix_has_nonfinite(sorsvd_ctx* c, const void* A, int dtype, int64_t m, int64_t n, int64_t lda) {
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(dbuf(c, "nf_cnt", 1));
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c->stream));
    const int blocks = c->num_sms * 4;
    if (dtype == SORSVD_F32)
        nonfinite_count_kernel<<<blocks, 256, 0, c->stream>>>(static_cast<const float*>(A), m, n, lda, cnt);
    else
        nonfinite_count_kernel<<<blocks, 256, 0, c->stream>>>(static_cast<const double*>(A), m, n, lda, cnt);
    check_launch(c);
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    double flag = h ? 1.0 : 0.0;
    if (c->world > 1) {
        double* dv = dbuf(c, "nf_flag", 1);
        CK(cudaMemcpyAsync(dv, &flag, sizeof flag, cudaMemcpyHostToDevice, c->stream));
        comm_allreduce(c, dv, 1, false, c->stream);
        CK(cudaMemcpyAsync(&flag, dv, sizeof flag, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    return flag != 0.0;
}

// After a call: a non-finite sigma means either non-finite input (the
// reference's parameter_error, raised before any arithmetic) or a breakdown
// (numerical_error). Any NaN / Inf entry of A reaches sigma: Inf * 0 and
// NaN * x are NaN, so the entry's row of T1 = A Omega is non-finite and so is
// every later stage. The check costs one read of k doubles on the happy path.
void check_result_finite(sorsvd_ctx* c, const double* dS, int k, const void* A, int dtype, int64_t m, int64_t n,
                         int64_t lda) {
    std::vector<double> hs(k);
    CK(cudaMemcpyAsync(hs.data(), dS, (size_t)k * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    bool ok = true;
    for (double v : hs) ok = ok && std::isfinite(v);
    if (c->world > 1) {  // every rank takes the same branch (the scan below is collective)
        double* dv = dbuf(c, "nf_ok", 1);
        const double bad = ok ? 0.0 : 1.0;
        CK(cudaMemcpyAsync(dv, &bad, sizeof bad, cudaMemcpyHostToDevice, c->stream));
        comm_allreduce(c, dv, 1, false, c->stream);
        double tot = 0.0;
        CK(cudaMemcpyAsync(&tot, dv, sizeof tot, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        ok = tot == 0.0;
    }
    if (ok) return;
    if (matrix_has_nonfinite(c, A, dtype, m, n, lda))
        throw Error{SORSVD_ERR_PARAMETER, "parameter: matrix entries must be finite"};
    throw Error{SORSVD_ERR_NUMERICAL, "numerical: non-finite singular values"};
}

// Graph cache key: everything baked into the captured kernel arguments that
// can differ between calls on the same A -- including the launch predicate
// (an RPCA iteration's graph carries the RPCA stop flag; a later plain call
// on the same A must not replay it).
std::string sor_key(const SorProblem& P, const int* pred, int pred_skip) {
    char buf[320];
    snprintf(buf, sizeof buf, "sor%d:%d:%d:%d%d%lld:%p:%lld:%lld:%lld:%d:%d:%d", P.method, P.dtype, (int)P.single_pass,
             (int)P.tf32, (int)P.ozaki, (long long)P.oz_pm,
             P.dtype == SORSVD_F32 ? (const void*)P.Af : (const void*)P.A, (long long)P.m, (long long)P.n,
             (long long)P.lda, P.k, P.ell, P.q);
    if (pred) snprintf(buf + strlen(buf), sizeof buf - strlen(buf), ":pred%p/%d", (const void*)pred, pred_skip);
    return buf;
}

void validate(const sorsvd_desc* d) {
    if (!d) throw Error{SORSVD_ERR_PARAMETER, "parameter: null descriptor"};
    const int64_t mg = d->m_global > 0 ? d->m_global : d->m;
    if (d->m < 1 || d->n < 1) throw Error{SORSVD_ERR_SHAPE, "shape: matrix dimensions must be positive"};
    if (d->lda < d->n) throw Error{SORSVD_ERR_SHAPE, "shape: lda < n"};
    if (const char* e = sorsvd_host::validate_sketch(mg, d->n, d->k, d->ell, d->q))
        throw Error{SORSVD_ERR_PARAMETER, e};
    if ((d->flags & SORSVD_FLAG_BASIC) && d->q != 0)
        throw Error{SORSVD_ERR_PARAMETER, "parameter: sor_svd requires q == 0; use sor_svd_power"};
    if (d->dtype != SORSVD_F64 && d->dtype != SORSVD_F32) throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown dtype"};
    if (d->dtype == SORSVD_F32 && (d->lda % 4))
        throw Error{SORSVD_ERR_SHAPE, "shape: fp32 A needs lda % 4 == 0 (16-byte rows for TMA)"};
    if (d->ell > 512) throw Error{SORSVD_ERR_UNSUPPORTED, "ell > 512 is not supported (core SVD / QR limit)"};
}

// FP64 passes on the int8 tensor cores by default when a pass is big enough to amortise the
// per-call conversion of A and the per-pass digit cutting of the skinny operand. Measured call
// times, Ozaki / DMMA (tools/oz_threshold.py, profiles/r02_oz_threshold.jsonl): with the per-call
// digit planes 0.93 at m n ell = 2^30.6 (C2's shape), 0.86 at 2^31.8, 0.70-0.81 from 2^32.9 up, 0.49 on
// C3; converting inside every pass (planes do not fit) pays from ~2^36 (C5 1.65x faster). So: auto =
// m n ell >= 2^30.5 when the planes fit, >= 2^36 otherwise, and ell >= 32 (oz_auto_keep below).
// SORSVD_FLAG_OZAKI / SORSVD_FLAG_DMMA force either.
bool ozaki_wanted(uint32_t flags, int64_t m, int64_t n, int ell) {
    if (flags & SORSVD_FLAG_DMMA) return false;
    if (flags & SORSVD_FLAG_OZAKI) return true;
    return (double)m * (double)n * (double)ell >= 1518500250.0 /* 2^30.5 */ && ell >= 32;
}
// The automatic choice stands without the planes only from 2^36 up.
bool oz_auto_keep(uint32_t flags, int64_t m, int64_t n, int ell, bool planes) {
    if (flags & SORSVD_FLAG_OZAKI) return true;
    return planes || (double)m * (double)n * (double)ell >= 68719476736.0 /* 2^36 */;
}

// Host-buffer calls: A's upload as row chunks on the copy stream (one event per chunk), so that the
// Ozaki planes engine can convert chunk i and run the first pass T1 = A Omega over it while chunk
// i + 1 is still crossing PCIe (sor_device). rows_per_chunk is a whole number of 128-row tiles
// whose CTAs fill whole waves of the device.
struct HostUpload {
    bool chunked = false;
    int64_t rows_per_chunk = 0;
    int nchunks = 0;
    int issued = 0;  // chunks whose copies are enqueued so far
};

// Enqueue the copies of chunks [up.issued, upto) on the copy stream. Chunk 0 goes first; the host
// draws Omega while it crosses and enqueues Omega's (small) upload on the same stream before the
// remaining chunks, so the compute stream has Omega when chunk 0 lands.
void upload_issue(sorsvd_ctx* c, HostUpload& up, const void* A, void* dA, int64_t m, int64_t lda, size_t esz, int upto) {
    const size_t row_bytes = (size_t)lda * esz;
    for (int i = up.issued; i < upto && i < up.nchunks; ++i) {
        const int64_t r0 = (int64_t)i * up.rows_per_chunk, rows = std::min(up.rows_per_chunk, m - r0);
        CK(cudaMemcpyAsync(static_cast<char*>(dA) + (size_t)r0 * row_bytes, static_cast<const char*>(A) + (size_t)r0 * row_bytes,
                           (size_t)rows * row_bytes, cudaMemcpyHostToDevice, c->comm_stream));
        CK(cudaEventRecord(c->up_ev[(size_t)i], c->comm_stream));
        up.issued = i + 1;
    }
}

HostUpload upload_chunked(sorsvd_ctx* c, const void* A, void* dA, int64_t m, int64_t lda, size_t esz, int Np) {
    HostUpload up;
    const int NC = (int)cdiv(Np, kOzBN);
    int g = c->num_sms, h = NC;  // gcd(num_sms, NC)
    while (h) {
        const int t = g % h;
        g = h;
        h = t;
    }
    const int64_t unit_rows = (int64_t)(c->num_sms / g) * kOzBM;  // tiles x NC CTAs = whole waves
    const size_t row_bytes = (size_t)lda * esz;
    int64_t units = std::max<int64_t>(
        1, (int64_t)(((size_t)std::max<int64_t>(1, c->opt_upload_chunk_mb) << 20) / std::max<size_t>(1, unit_rows * row_bytes)));
    up.rows_per_chunk = units * unit_rows;
    up.nchunks = (int)cdiv(m, up.rows_per_chunk);
    while ((int)c->up_ev.size() < up.nchunks) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->up_ev.push_back(e);
    }
    // the copy stream starts after whatever the compute stream has queued (the previous call's reads of dA)
    CK(cudaEventRecord(c->ev_comm, c->stream));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_comm, 0));
    up.chunked = true;
    upload_issue(c, up, A, dA, m, lda, esz, 1);  // chunk 0 now; the rest after Omega's upload is enqueued
    return up;
}

// First global row of this rank's block: the exclusive prefix sum of the ranks' row counts
// (one small all-reduce of a world-long vector; 0 on a single rank).
int64_t rank_row0(sorsvd_ctx* c, int64_t m) {
    if (c->world <= 1) return 0;
    double* dv = dbuf(c, "row_counts", (size_t)c->world);
    std::vector<double> h((size_t)c->world, 0.0);
    h[(size_t)c->rank] = (double)m;
    CK(cudaMemcpyAsync(dv, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream));
    comm_allreduce(c, dv, (size_t)c->world, false, c->stream);
    CK(cudaMemcpyAsync(h.data(), dv, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    int64_t r0 = 0;
    for (int r = 0; r < c->rank; ++r) r0 += (int64_t)h[(size_t)r];
    return r0;
}

// Core device-side call. dOmega: n x ell dense (or null: drawn on the host).
void sor_device(sorsvd_ctx* c, const sorsvd_desc* d, const void* dA, const double* dOmega, double* dU,
                double* dS, double* dV, sorsvd_stats* st, int method = SORSVD_SOR_POWER,
                const double* dPsi2 = nullptr, const HostUpload* up = nullptr) {
    validate(d);
    const bool baseline = method == SORSVD_RSVD || method == SORSVD_TSR;
    if (baseline) {
        if (d->flags & SORSVD_FLAG_TF32) throw Error{SORSVD_ERR_UNSUPPORTED, "r_svd / tsr_svd: no TF32 mode"};
    }
    SorProblem P{};
    P.method = method;
    P.dtype = d->dtype;
    P.A = d->dtype == SORSVD_F64 ? static_cast<const double*>(dA) : nullptr;
    P.Af = d->dtype == SORSVD_F32 ? static_cast<const float*>(dA) : nullptr;
    P.Np32 = npad32(d->ell);
    P.m = d->m;
    P.n = d->n;
    P.lda = d->lda;
    P.k = d->k;
    P.ell = d->ell;
    P.q = d->q;
    P.Np = npad(d->ell);
    P.m_global = d->m_global > 0 ? d->m_global : d->m;
    P.single_pass = d->single_pass != 0 && !baseline;
    P.tf32 = d->dtype == SORSVD_F32 && (d->flags & SORSVD_FLAG_TF32);
    P.ozaki = !P.tf32 && !baseline && ozaki_wanted(d->flags, P.m, P.n, P.ell);
    QrPlan *p1, *p2, *pg;
    SorBuffers b = prepare_sor(c, P, &p1, &p2, &pg);
    P.oz_pm = P.ozaki ? oz_planes_rows(c, P) : 0;
    P.oz_planes = P.oz_pm > 0;
    if (P.ozaki && !oz_auto_keep(d->flags, P.m, P.n, P.ell, P.oz_planes)) P.ozaki = false;
    double* psi2_in = nullptr;
    if (method == SORSVD_TSR) {  // Psi2 = gaussian_matrix(m, ell, seed ^ 1)   (sketch.hpp:142)
        psi2_in = dbuf(c, "psi2_in", (size_t)P.m * P.ell);
        if (dPsi2 && (d->flags & SORSVD_FLAG_OMEGA_GIVEN)) {
            CK(cudaMemcpyAsync(psi2_in, dPsi2, (size_t)P.m * P.ell * 8, cudaMemcpyDeviceToDevice, c->stream));
        } else {
            // this rank's rows [row0, row0 + m) of the m_global x ell draw
            const int64_t row0 = rank_row0(c, P.m);
            c->host_psi2.resize((size_t)P.m * P.ell);
            sorsvd_host::gaussian_fill_range(c->host_psi2.data(), (uint64_t)row0 * P.ell, (uint64_t)(row0 + P.m) * P.ell,
                                             d->seed ^ 1ULL, 0);
            CK(cudaMemcpyAsync(psi2_in, c->host_psi2.data(), (size_t)P.m * P.ell * 8, cudaMemcpyHostToDevice,
                               c->stream));
        }
    }
    // Omega and the outputs stay outside the captured graph (so the graph is
    // keyed on A alone): Omega is staged into a context buffer before the
    // launch, U / sigma / V are copied out after it.
    double* om_in = dbuf(c, "omega_in", (size_t)P.n * P.ell);
    if (dOmega && (d->flags & SORSVD_FLAG_OMEGA_GIVEN)) {
        CK(cudaMemcpyAsync(om_in, dOmega, (size_t)P.n * P.ell * 8, cudaMemcpyDeviceToDevice, c->stream));
    } else {
        c->host_omega.resize((size_t)P.n * P.ell);
        sorsvd_host::gaussian_fill(c->host_omega.data(), (uint64_t)P.n * P.ell, d->seed, 0);
        CK(cudaMemcpyAsync(om_in, c->host_omega.data(), (size_t)P.n * P.ell * 8, cudaMemcpyHostToDevice, c->stream));
    }
    const double* om = om_in;
    const bool timing = (d->flags & SORSVD_FLAG_STAGE_TIMES) != 0;
    // host-buffer call with A arriving in row chunks: the planes engine converts and sweeps chunk i
    // (first pass T1 = A Omega, rows independent) while chunk i + 1 uploads
    const bool pipe = up && up->chunked && P.ozaki && P.oz_pm == P.m && c->world == 1 && !baseline;
    if (up && up->chunked && !pipe)  // not eligible after all: wait for the whole upload
        CK(cudaStreamWaitEvent(c->stream, c->up_ev[(size_t)up->nchunks - 1], 0));
    // NCCL contexts enqueue stream-ordered calls by default: collectives captured into a graph (two
    // streams, fork/join) could not be run in the one-GPU build environment, the plain form is the
    // schedule the emulated-group tests run; SORSVD_OPT_NCCL_GRAPH opts in.
    const bool use_graph = !timing && !c->emu && !(c->comm && !c->opt_nccl_graph) &&
                           !(d->flags & SORSVD_FLAG_NO_GRAPH) && !pipe;
    CK(cudaEventRecord(c->ev_a, c->stream));
    const int launches0 = c->launches;
    int launches = 0;
    auto stage_omega = [&]() {
        // T2 <- Omega (padded; rounded to fp32 for the TF32 passes)
        if (P.tf32) {
            cast_to_f32(c, om, P.ell, b.T2f, P.Np32, P.n, P.ell, c->stream);
        } else {
            CK(cudaMemsetAsync(b.T2, 0, (size_t)P.n * P.Np * 8, c->stream));
            CK(cudaMemcpy2DAsync(b.T2, (size_t)P.Np * 8, om, (size_t)P.ell * 8, (size_t)P.ell * 8, (size_t)P.n,
                                 cudaMemcpyDeviceToDevice, c->stream));
        }
    };
    auto enqueue_all = [&]() {
        stage_omega();
        if (pipe) {
            const OzScales oz = oz_planes_of(c, P);
            const OzX ox = oz_cut_x(c, P, false, oz, b.T2, c->stream);  // Omega's digit planes: once for all chunks
            const int s_full = oz_nn_splits(c, P);
            // the first T2 = A^T T1 as well, one K range per chunk (its rows of T1 exist as soon as the chunk's
            // first pass is done), into a second buffer (T2 still holds Omega for the later chunks' first pass)
            const bool tn_too = c->opt_upload_tn && P.q >= 1 && !P.single_pass;
            double* T2n = tn_too ? dbuf(c, "T2_next", (size_t)P.n * P.Np) : nullptr;
            for (int i = 0; i < up->nchunks; ++i) {
                const int64_t r0 = (int64_t)i * up->rows_per_chunk, rows = std::min(up->rows_per_chunk, P.m - r0);
                CK(cudaStreamWaitEvent(c->stream, c->up_ev[(size_t)i], 0));
                oz_convert_rows(c, P, oz, r0, rows, c->stream);
                oz_launch_planes(c, P, false, oz, ox, b.T1 + r0 * P.Np, r0, rows, c->stream, 0, 0, false, s_full);
                if (tn_too) {
                    SorProblem Qc = P;
                    Qc.m = rows;
                    OzScales ozc = oz;
                    ozc.row_e = oz.row_e + r0;  // the chunk's rows' scales ride on its rows of T1
                    const OzX xt = oz_cut_x(c, Qc, true, ozc, b.T1 + r0 * P.Np, c->stream);
                    oz_launch_planes(c, Qc, true, oz, xt, T2n, 0, P.n, c->stream, 0, r0, i > 0);
                }
            }
            SorProblem Q = P;
            Q.pre_first = true;
            if (tn_too) {
                CK(cudaMemcpyAsync(b.T2, T2n, (size_t)P.n * P.Np * 8, cudaMemcpyDeviceToDevice, c->stream));
                Q.pre_tn = true;
            }
            enqueue_sor(c, Q, b, p1, p2, pg, timing);
            return;
        }
        if (method == SORSVD_TSR) {
            CK(cudaMemsetAsync(b.Psi2, 0, (size_t)P.m * P.Np * 8, c->stream));
            CK(cudaMemcpy2DAsync(b.Psi2, (size_t)P.Np * 8, psi2_in, (size_t)P.ell * 8, (size_t)P.ell * 8,
                                 (size_t)P.m, cudaMemcpyDeviceToDevice, c->stream));
            enqueue_tsr(c, P, b, p1, p2, pg, timing);
        } else if (method == SORSVD_RSVD) {
            enqueue_rsvd(c, P, b, p1, p2, pg, timing);
        } else {
            enqueue_sor(c, P, b, p1, p2, pg, timing);
        }
    };
    auto copy_out = [&]() {
        CK(cudaMemcpy2DAsync(dU, (size_t)P.k * 8, b.Uo, (size_t)P.Np * 8, (size_t)P.k * 8, (size_t)P.m,
                             cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpy2DAsync(dV, (size_t)P.k * 8, b.Vo, (size_t)P.Np * 8, (size_t)P.k * 8, (size_t)P.n,
                             cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(dS, b.Sk, (size_t)P.k * 8, cudaMemcpyDeviceToDevice, c->stream));
    };
    if (use_graph) {
        const std::string key = sor_key(P, c->pred, c->pred_skip) + (p1->hint_house ? ":h1" : "") + (p2->hint_house ? ":h2" : "");
        auto it = c->graphs.find(key);
        if (it == c->graphs.end()) {
            if (c->graphs.size() >= 32) invalidate_graphs(c);  // bound the cache (keys carry A's address)
            // warm-up run outside capture sets kernel attributes
            enqueue_all();
            CK(cudaStreamSynchronize(c->stream));
            const int l0 = c->launches;
            cudaGraph_t graph;
            c->capturing = true;
            CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue_all();
            } catch (...) {
                cudaStreamEndCapture(c->stream, &graph);
                c->capturing = false;
                throw;
            }
            CK(cudaStreamEndCapture(c->stream, &graph));
            c->capturing = false;
            GraphEntry ge;
            CK(cudaGraphInstantiate(&ge.exec, graph, 0));
            CK(cudaGraphDestroy(graph));
            ge.launches = c->launches - l0;
            c->graphs[key] = ge;
            it = c->graphs.find(key);
            CK(cudaEventRecord(c->ev_a, c->stream));
        }
        CK(cudaGraphLaunch(it->second.exec, c->stream));
        launches = it->second.launches;
    } else {
        enqueue_all();
        launches = c->launches - launches0;
    }
    copy_out();
    CK(cudaEventRecord(c->ev_b, c->stream));
    if (!c->pred)  // inside RPCA (predicated iterations) the driver runs its own finiteness test
        check_result_finite(c, b.Sk, P.k, dA, P.dtype, P.m, P.n, P.lda);
    if (p1->big || p2->big) {
        CK(cudaEventSynchronize(c->ev_b));
        check_big_qr(p1);
        check_big_qr(p2);
    }
    if (st) {
        CK(cudaEventSynchronize(c->ev_b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
        st->ms_total = ms;
        const int passes = method == SORSVD_RSVD ? 2 * d->q + 2                       // sketch.hpp:134
                           : method == SORSVD_TSR ? 1                                  // sketch.hpp:148
                           : d->single_pass     ? 2 * d->q + 2 : 2 * d->q + 3;        // sketch.hpp:104
        st->passes = passes;
        st->method = baseline ? method : d->q == 0 ? SORSVD_SOR : SORSVD_SOR_POWER;
        const int launched = method == SORSVD_TSR ? 2 : passes;  // tsr: A Psi1 and A^T Psi2 are two sweeps here
        st->flops_passes = 2.0 * (double)d->m * d->n * d->ell * launched;
        st->bytes_passes = (double)d->m * d->n * (d->dtype == SORSVD_F32 ? 4.0 : 8.0) * launched;
        st->launches = launches;
        st->pass_kind = P.tf32 ? 2 : P.ozaki ? 1 : 0;
        st->oz_planes = !P.ozaki ? 0 : P.oz_pm >= P.m ? 1 : P.oz_pm > 0 ? 2 : 0;
        int sw = 0;
        CK(cudaMemcpy(&sw, b.sweeps, sizeof(int), cudaMemcpyDeviceToHost));
        st->jacobi_sweeps = sw;
        if (timing) {
            float t[5];
            for (int i = 0; i < 5; ++i) CK(cudaEventElapsedTime(&t[i], c->ev_st[i], c->ev_st[i + 1]));
            st->ms_passes = t[0];
            st->ms_qr = t[1];
            st->ms_project = t[2];
            st->ms_svd = t[3];
            st->ms_basis = t[4];
        }
    }
}

// ------------------------------------------------------- batched trials ----
// T independent sor_svd_power calls on one A (bounds.hpp:262-379 runs one per
// Monte-Carlo trial, seed + t) sharing every pass over A: the T test matrices
// sit side by side as the columns of one n x (T Np) operand, so each of the
// 2q+2 sketch passes and the projection pass is ONE launch over A for all
// trials (A read once, a T-times wider and better-fed DMMA tile). The
// per-trial QRs, core SVDs and basis products are latency-bound chains; they
// run on up to kTrialStreams streams side by side.
constexpr int kTrialStreams = 8;

void ensure_trial_streams(sorsvd_ctx* c, int n) {
    while ((int)c->tstreams.size() < n) {
        cudaStream_t t;
        cudaEvent_t e;
        CK(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->tstreams.push_back(t);
        c->tevents.push_back(e);
    }
}

void batch_device(sorsvd_ctx* c, const sorsvd_desc* d, int trials, const uint64_t* seeds, const void* dA,
                  const double* dOmegas, double* dU, double* dS, double* dV, sorsvd_stats* st) {
    validate(d);
    if (trials < 1) throw Error{SORSVD_ERR_PARAMETER, "parameter: trials must be positive"};
    if (d->flags & SORSVD_FLAG_TF32) throw Error{SORSVD_ERR_UNSUPPORTED, "batched trials: no TF32 mode"};
    if (d->single_pass) throw Error{SORSVD_ERR_UNSUPPORTED, "batched trials: single_pass not supported"};
    if (d->ell > kHouseMaxK) throw Error{SORSVD_ERR_UNSUPPORTED, "batched trials: ell <= 256"};
    SorProblem P{};
    P.dtype = d->dtype;
    P.A = d->dtype == SORSVD_F64 ? static_cast<const double*>(dA) : nullptr;
    P.Af = d->dtype == SORSVD_F32 ? static_cast<const float*>(dA) : nullptr;
    P.m = d->m;
    P.n = d->n;
    P.lda = d->lda;
    P.k = d->k;
    P.ell = d->ell;
    P.q = d->q;
    P.Np = npad(d->ell);
    P.m_global = d->m_global > 0 ? d->m_global : P.m;
    const bool multi = c->world > 1;  // row-sharded A: partial sums all-reduced, T1's QR by the sharded TSQR
    const int Np = P.Np, ell = P.ell, k = P.k;
    const int64_t m = P.m, n = P.n;
    const int Wt = trials * Np;                       // the trials' columns side by side
    const int W = Wt <= 128 ? Wt : ((Wt + 127) / 128) * 128;  // padded for the GEMM's column chunks
    double* X = dbuf(c, "b_X", (size_t)n * W);      // Omega_all, then T2_all, then Q2_all
    double* T1b = dbuf(c, "b_T1", (size_t)m * W);
    double* Yb = dbuf(c, "b_Y", (size_t)m * W);
    double* om_in = dbuf(c, "b_om", (size_t)trials * n * ell);
    cudaStream_t s = c->stream;
    // test matrices: gaussian_matrix(n, ell, seed_t) per trial (sketch.hpp:90), or given
    if (dOmegas && (d->flags & SORSVD_FLAG_OMEGA_GIVEN)) {
        CK(cudaMemcpyAsync(om_in, dOmegas, (size_t)trials * n * ell * 8, cudaMemcpyDeviceToDevice, s));
    } else {
        c->host_omega.resize((size_t)trials * n * ell);
        for (int t = 0; t < trials; ++t)
            sorsvd_host::gaussian_fill(c->host_omega.data() + (size_t)t * n * ell, (uint64_t)n * ell,
                                       seeds ? seeds[t] : d->seed + (uint64_t)t, 0);
        CK(cudaMemcpyAsync(om_in, c->host_omega.data(), (size_t)trials * n * ell * 8, cudaMemcpyHostToDevice, s));
    }
    CK(cudaEventRecord(c->ev_a, s));
    const int l0 = c->launches;
    CK(cudaMemsetAsync(X, 0, (size_t)n * W * 8, s));
    for (int t = 0; t < trials; ++t)
        CK(cudaMemcpy2DAsync(X + (size_t)t * Np, (size_t)W * 8, om_in + (size_t)t * n * ell, (size_t)ell * 8,
                             (size_t)ell * 8, (size_t)n, cudaMemcpyDeviceToDevice, s));
    auto pass = [&](bool ta, const double* B, double* C) {
        GemmCall g;
        g.ta = ta;
        g.A = P.A;
        g.Af = P.Af;
        g.lda = P.lda;
        g.M = ta ? n : m;
        g.K = ta ? m : n;
        g.B = B;
        g.ldb = W;
        g.N = W;
        g.C = C;
        g.ldc = W;
        g.sk_bias = W <= 128 ? 1.0 : 0.95;
        run_gemm(c, g, s);
    };
    for (int i = 0; i <= P.q; ++i) {  // sketch.hpp:93-97, all trials per launch
        pass(false, X, T1b);
        pass(true, T1b, X);
        if (multi) comm_allreduce(c, X, (size_t)n * W, false, s);  // T2_all summed over the row blocks
    }
    // per-trial QRs (sketch.hpp:98-99) side by side on the trial streams (multi-rank: one after
    // the other on the context stream, so that every rank issues its collectives in the same order)
    const int S = multi ? 1 : std::min(trials, kTrialStreams);
    ensure_trial_streams(c, S);
    QrPlan* pgm = multi ? get_qr_plan(c, (int64_t)c->world * ell, ell, c->world, "G") : nullptr;
    if (multi) {
        dbuf(c, "Rg", (size_t)c->world * ell * ell);
        dbuf(c, "CinLocal", (size_t)ell * Np);
    }
    auto tstream = [&](int t) { return multi ? s : c->tstreams[t % S]; };
    struct Trial {
        double *T1, *T2, *Q1, *Q2, *Mk, *Uk, *Vk, *Sk, *Uo, *Vo;
        int* sweeps;
        QrPlan *p1, *p2;
    };
    // Q1_t, Q2_t live from the QR phase to the basis products (one pair per trial);
    // everything else is scratch of the trial's stream (trials t and t + S run one
    // after the other on stream t % S), so memory grows by (m + n) Np per trial
    std::vector<Trial> tr(trials);
    for (int t = 0; t < trials; ++t) {
        const std::string tag = "b" + std::to_string(t) + "_";
        const std::string sl = "bs" + std::to_string(t % S) + "_";
        Trial& x = tr[t];
        x.Q1 = dbuf(c, tag + "Q1", (size_t)m * Np);
        x.Q2 = dbuf(c, tag + "Q2", (size_t)n * Np);
        x.T1 = dbuf(c, sl + "T1", (size_t)m * Np);
        x.T2 = dbuf(c, sl + "T2", (size_t)n * Np);
        x.Mk = dbuf(c, sl + "Mk", (size_t)Np * Np);
        x.Uk = dbuf(c, sl + "Uk", (size_t)Np * Np);
        x.Vk = dbuf(c, sl + "Vk", (size_t)Np * Np);
        x.Sk = dbuf(c, sl + "Sk", (size_t)Np);
        x.Uo = dbuf(c, sl + "Uo", (size_t)m * Np);
        x.Vo = dbuf(c, sl + "Vo", (size_t)n * Np);
        x.sweeps = reinterpret_cast<int*>(dbuf(c, tag + "sw", 1));
        x.p1 = get_qr_plan(c, m, ell, 0, (sl + "T1").c_str());
        x.p2 = get_qr_plan(c, n, ell, 0, (sl + "T2").c_str());
    }
    auto fork = [&]() {
        if (multi) return;
        CK(cudaEventRecord(c->ev_fork, s));
        for (int j = 0; j < S; ++j) CK(cudaStreamWaitEvent(c->tstreams[j], c->ev_fork, 0));
    };
    auto join = [&]() {
        if (multi) return;
        for (int j = 0; j < S; ++j) {
            CK(cudaEventRecord(c->tevents[j], c->tstreams[j]));
            CK(cudaStreamWaitEvent(s, c->tevents[j], 0));
        }
    };
    fork();
    for (int t = 0; t < trials; ++t) {
        cudaStream_t ts = tstream(t);
        Trial& x = tr[t];
        CK(cudaMemcpy2DAsync(x.T1, (size_t)Np * 8, T1b + (size_t)t * Np, (size_t)W * 8, (size_t)Np * 8, (size_t)m,
                             cudaMemcpyDeviceToDevice, ts));
        CK(cudaMemcpy2DAsync(x.T2, (size_t)Np * 8, X + (size_t)t * Np, (size_t)W * 8, (size_t)Np * 8, (size_t)n,
                             cudaMemcpyDeviceToDevice, ts));
        qr_rows(c, P, x.p1, pgm, x.T1, x.Q1, ts);
        qr_run(c, x.p2, x.T2, Np, x.Q2, Np, ts);
        CK(cudaMemcpy2DAsync(X + (size_t)t * Np, (size_t)W * 8, x.Q2, (size_t)Np * 8, (size_t)Np * 8, (size_t)n,
                             cudaMemcpyDeviceToDevice, ts));
    }
    join();
    pass(false, X, Yb);  // Y_t = A Q2_t for all trials in one launch (sketch.hpp:100-102)
    fork();
    for (int t = 0; t < trials; ++t) {
        cudaStream_t ts = tstream(t);
        Trial& x = tr[t];
        const std::string ws = "bws" + std::to_string(t % S);
        GemmCall h;  // M_t = Q1_t^T Y_t
        h.ta = true;
        h.A = x.Q1;
        h.lda = Np;
        h.M = ell;
        h.K = m;
        h.B = Yb + (size_t)t * Np;
        h.ldb = W;
        h.N = Np;
        h.C = x.Mk;
        h.ldc = Np;
        h.ws_name = ws.c_str();
        run_gemm(c, h, ts);
        if (multi) comm_allreduce(c, x.Mk, (size_t)ell * Np, false, ts);
        run_jacobi(c, ell, x.Mk, Np, x.Uk, Np, x.Sk, x.Vk, Np, x.sweeps, ts);  // sketch.hpp:103
        for (int hh = 0; hh < 2; ++hh) {  // U = Q1 Ut_k, V = Q2 Vt_k   (sketch.hpp:105,107)
            GemmCall g;
            g.A = hh ? x.Q2 : x.Q1;
            g.lda = Np;
            g.M = hh ? n : m;
            g.K = ell;
            g.B = hh ? x.Vk : x.Uk;
            g.ldb = Np;
            g.N = Np;
            g.C = hh ? x.Vo : x.Uo;
            g.ldc = Np;
            g.ws_name = ws.c_str();
            run_gemm(c, g, ts);
        }
        CK(cudaMemcpy2DAsync(dU + (size_t)t * m * k, (size_t)k * 8, x.Uo, (size_t)Np * 8, (size_t)k * 8, (size_t)m,
                             cudaMemcpyDeviceToDevice, ts));
        CK(cudaMemcpy2DAsync(dV + (size_t)t * n * k, (size_t)k * 8, x.Vo, (size_t)Np * 8, (size_t)k * 8, (size_t)n,
                             cudaMemcpyDeviceToDevice, ts));
        CK(cudaMemcpyAsync(dS + (size_t)t * k, x.Sk, (size_t)k * 8, cudaMemcpyDeviceToDevice, ts));
    }
    join();
    CK(cudaEventRecord(c->ev_b, s));
    if (st) {
        CK(cudaEventSynchronize(c->ev_b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
        st->ms_total = ms;
        st->passes = 2 * d->q + 3;
        st->method = d->q == 0 ? SORSVD_SOR : SORSVD_SOR_POWER;
        st->flops_passes = 2.0 * (double)m * n * ell * st->passes * trials;
        st->bytes_passes = (double)m * n * (d->dtype == SORSVD_F32 ? 4.0 : 8.0) * st->passes;  // A read once per pass
        st->launches = c->launches - l0;
        int sw = 0;
        CK(cudaMemcpy(&sw, tr[0].sweeps, sizeof(int), cudaMemcpyDeviceToHost));
        st->jacobi_sweeps = sw;
    }
}


// ------------------------------------------------------------ SORD files ----
// "SORD", u32 version = 1, u64 rows, u64 cols, rows*cols little-endian
// float64, row-major. Streamed through two pinned staging buffers so that the disk
// read (write) of one chunk overlaps the host<->device copy of the other and the
// host never holds the whole matrix (a 137 GB FP64 file can land as 68.7 GB FP32).
struct SordHeader {
    int64_t rows = 0, cols = 0;
};

SordHeader sord_read_header(int fd, const char* path) {
    unsigned char h[24];
    if (pread(fd, h, 24, 0) != 24) throw Error{SORSVD_ERR_SHAPE, std::string("shape: SORD header truncated: ") + path};
    if (memcmp(h, "SORD", 4) != 0) throw Error{SORSVD_ERR_PARAMETER, std::string("parameter: not a SORD file: ") + path};
    uint32_t ver;
    uint64_t r, cc;
    memcpy(&ver, h + 4, 4);
    memcpy(&r, h + 8, 8);
    memcpy(&cc, h + 16, 8);
    if (ver != 1) throw Error{SORSVD_ERR_PARAMETER, "parameter: unsupported SORD version " + std::to_string(ver)};
    if (r == 0 || cc == 0 || r > (1ull << 40) || cc > (1ull << 40))
        throw Error{SORSVD_ERR_SHAPE, "shape: SORD dimensions out of range"};
    struct stat st;
    if (fstat(fd, &st) != 0 || (uint64_t)st.st_size != 24 + r * cc * 8)
        throw Error{SORSVD_ERR_SHAPE, std::string("shape: SORD payload size does not match rows x cols: ") + path};
    return SordHeader{(int64_t)r, (int64_t)cc};
}

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

int64_t sord_chunk_rows(const sorsvd_ctx* c, int64_t cols) {
    const int64_t mb = std::max<int64_t>(1, c->opt_sord_chunk_mb);
    return std::max<int64_t>(1, (mb << 20) / (cols * 8));
}

struct PinnedPair {  // two pinned staging buffers + their reuse events
    double* h[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    explicit PinnedPair(size_t bytes) {
        for (int i = 0; i < 2; ++i) {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&h[i]), bytes, cudaHostAllocDefault));
            CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
    }
    ~PinnedPair() {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) {
                cudaEventSynchronize(ev[i]);
                cudaEventDestroy(ev[i]);
            }
            if (h[i]) cudaFreeHost(h[i]);
        }
    }
};

void sord_load(sorsvd_ctx* c, const char* path, void* dA, int64_t lda, int dtype) {
    Fd f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) throw Error{SORSVD_ERR_PARAMETER, std::string("parameter: cannot open ") + path};
    const SordHeader hd = sord_read_header(f.fd, path);
    if (lda < hd.cols) throw Error{SORSVD_ERR_SHAPE, "shape: lda < cols"};
    if (dtype != SORSVD_F64 && dtype != SORSVD_F32) throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown dtype"};
    const int64_t cr = std::min(sord_chunk_rows(c, hd.cols), hd.rows);
    const size_t cbytes = (size_t)cr * hd.cols * 8;
    PinnedPair pp(cbytes);
    double* stage[2] = {nullptr, nullptr};
    if (dtype == SORSVD_F32) {
        stage[0] = dbuf(c, "sord_stage0", (size_t)cr * hd.cols);
        stage[1] = dbuf(c, "sord_stage1", (size_t)cr * hd.cols);
    }
    cudaStream_t s = c->stream;
    int64_t r0 = 0;
    for (int64_t ch = 0; r0 < hd.rows; ++ch, r0 += cr) {
        const int b = (int)(ch & 1);
        const int64_t nr = std::min(cr, hd.rows - r0);
        const size_t nb = (size_t)nr * hd.cols * 8;
        CK(cudaEventSynchronize(pp.ev[b]));  // the copy out of this buffer two chunks ago is done
        size_t got = 0;
        while (got < nb) {
            const ssize_t k = pread(f.fd, reinterpret_cast<char*>(pp.h[b]) + got, nb - got,
                                    (off_t)(24 + (size_t)r0 * hd.cols * 8 + got));
            if (k <= 0) throw Error{SORSVD_ERR_SHAPE, std::string("shape: SORD read failed: ") + path};
            got += (size_t)k;
        }
        if (dtype == SORSVD_F64) {
            double* dst = static_cast<double*>(dA) + r0 * lda;
            CK(cudaMemcpy2DAsync(dst, (size_t)lda * 8, pp.h[b], (size_t)hd.cols * 8, (size_t)hd.cols * 8, (size_t)nr,
                                 cudaMemcpyHostToDevice, s));
        } else {
            CK(cudaMemcpyAsync(stage[b], pp.h[b], nb, cudaMemcpyHostToDevice, s));
            cast_to_f32(c, stage[b], hd.cols, static_cast<float*>(dA) + r0 * lda, lda, nr, (int)hd.cols, s);
        }
        CK(cudaEventRecord(pp.ev[b], s));
    }
    CK(cudaStreamSynchronize(s));
}

void sord_save(sorsvd_ctx* c, const char* path, const double* dA, int64_t rows, int64_t cols, int64_t lda) {
    if (rows < 1 || cols < 1 || lda < cols) throw Error{SORSVD_ERR_SHAPE, "shape: SORD save dimensions"};
    Fd f;
    f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) throw Error{SORSVD_ERR_PARAMETER, std::string("parameter: cannot create ") + path};
    unsigned char h[24];
    memcpy(h, "SORD", 4);
    const uint32_t ver = 1;
    const uint64_t r = (uint64_t)rows, cc = (uint64_t)cols;
    memcpy(h + 4, &ver, 4);
    memcpy(h + 8, &r, 8);
    memcpy(h + 16, &cc, 8);
    if (pwrite(f.fd, h, 24, 0) != 24) throw Error{SORSVD_ERR_INTERNAL, "SORD write failed"};
    const int64_t cr = std::min(sord_chunk_rows(c, cols), rows);
    PinnedPair pp((size_t)cr * cols * 8);
    cudaStream_t s = c->stream;
    auto issue = [&](int64_t ch) {  // device -> pinned buffer ch & 1
        const int64_t a0 = ch * cr, nr = std::min(cr, rows - a0);
        CK(cudaMemcpy2DAsync(pp.h[ch & 1], (size_t)cols * 8, dA + a0 * lda, (size_t)lda * 8, (size_t)cols * 8,
                             (size_t)nr, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(pp.ev[ch & 1], s));
    };
    const int64_t nch = cdiv(rows, cr);
    issue(0);
    for (int64_t ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) issue(ch + 1);  // next chunk's copy overlaps this chunk's disk write
        CK(cudaEventSynchronize(pp.ev[ch & 1]));
        const int64_t a0 = ch * cr, nr = std::min(cr, rows - a0);
        const size_t nb = (size_t)nr * cols * 8;
        size_t put = 0;
        while (put < nb) {
            const ssize_t k = pwrite(f.fd, reinterpret_cast<const char*>(pp.h[ch & 1]) + put, nb - put,
                                     (off_t)(24 + (size_t)a0 * cols * 8 + put));
            if (k <= 0) throw Error{SORSVD_ERR_INTERNAL, std::string("SORD write failed: ") + path};
            put += (size_t)k;
        }
    }
}

// ----------------------------------------------------------------- RPCA ----
double device_sumsq(sorsvd_ctx* c, const double* x, int64_t m, int64_t n, int64_t ld) {
    const int blocks = c->num_sms * 4;
    double* part = dbuf(c, "rp_part2", (size_t)blocks);
    double* tot = dbuf(c, "rp_tot2", 2);
    sumsq_partials_kernel<<<blocks, 256, 0, c->stream>>>(x, m, n, ld, part);
    check_launch(c);
    sum_partials_kernel<<<1, 1024, 0, c->stream>>>(part, blocks, tot);
    check_launch(c);
    comm_allreduce(c, tot, 1, false, c->stream);  // multi-rank: sum over the row blocks
    double h[2];
    CK(cudaMemcpyAsync(h, tot, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return h[0];
}

// sigma_1(A) when min(m, n) <= 1024: G = A^T A (or A A^T), 12 squarings (each
// rescaled by its max entry) give P ~ G^(4096), whose range is the top
// eigenspace to working precision; a Rayleigh-Ritz step on span(P Omega)
// (16 columns: QR, Q^T G Q, Jacobi) gives lambda_1 = sigma_1^2 to ~eps
// relative. ~25 launches instead of a subspace iteration on A whose step
// count depends on sigma_2 / sigma_1.
double estimate_sigma1_gram(sorsvd_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda) {
    const bool tall = m >= n || c->world > 1;  // row-sharded D: G = sum_r D_r^T D_r
    const int s = (int)(tall ? n : m);
    const int Np = npad(s);
    double* G = dbuf(c, "est_G", (size_t)Np * Np, true);
    double* P0 = dbuf(c, "est_P0", (size_t)Np * Np, true);
    double* P1 = dbuf(c, "est_P1", (size_t)Np * Np, true);
    cudaStream_t st = c->stream;
    if (tall) {
        // G = A^T A: TN with B = A needs B padded to Np columns -> copy A's rows? use A^T A via TN on A
        // directly when n is already a multiple of 8 and lda == n, else stage A padded.
        const double* Ap = A;
        int64_t ldp = lda;
        if (lda % 2 || n % 8 || lda != n) {
            double* Ad = dbuf(c, "est_Apad", (size_t)m * Np, true);
            CK(cudaMemcpy2DAsync(Ad, (size_t)Np * 8, A, (size_t)lda * 8, (size_t)n * 8, (size_t)m,
                                 cudaMemcpyDeviceToDevice, st));
            Ap = Ad;
            ldp = Np;
        }
        GemmCall g;
        g.ta = true;
        g.A = Ap;
        g.lda = ldp;
        g.M = s;
        g.K = m;
        g.B = Ap;
        g.ldb = ldp;
        g.N = Np;
        g.C = G;
        g.ldc = Np;
        g.ws_name = "est_ws";
        run_gemm(c, g, st);
        comm_allreduce(c, G, (size_t)s * Np, false, st);
    } else {
        // G = A A^T: NN with B = A^T (staged transposed, padded)
        double* At = dbuf(c, "est_At", (size_t)n * Np, true);
        dim3 tb(32, 8), tg((unsigned)cdiv(m, 32), (unsigned)cdiv(n, 32));
        transpose_kernel<<<tg, tb, 0, st>>>(A, lda, m, n, At, Np);
        check_launch(c);
        GemmCall g;
        g.A = A;
        g.lda = lda;
        g.M = s;
        g.K = n;
        g.B = At;
        g.ldb = Np;
        g.N = Np;
        g.C = G;
        g.ldc = Np;
        g.ws_name = "est_ws";
        run_gemm(c, g, st);
    }
    CK(cudaMemcpyAsync(P0, G, (size_t)s * Np * 8, cudaMemcpyDeviceToDevice, st));
    double* cur = P0;
    double* nxt = P1;
    unsigned long long* mx = reinterpret_cast<unsigned long long*>(dbuf(c, "est_mx", 16));
    CK(cudaMemsetAsync(mx, 0, 16 * sizeof(unsigned long long), st));
    const int sg = (int)std::min<int64_t>(cdiv((int64_t)s * s, 256), 2 * c->num_sms);
    auto rescale = [&](int slot) {
        maxabs_kernel<<<sg, 256, 0, st>>>(cur, s, s, Np, mx + slot);
        check_launch(c);
        scale_by_kernel<<<sg, 256, 0, st>>>(cur, s, s, Np, mx + slot);
        check_launch(c);
    };
    for (int it = 0; it < 12; ++it) {
        rescale(it);
        GemmCall g;
        g.A = cur;
        g.lda = Np;
        g.M = s;
        g.K = s;
        g.B = cur;
        g.ldb = Np;
        g.N = Np;
        g.C = nxt;
        g.ldc = Np;
        g.ws_name = "est_ws";
        run_gemm(c, g, st);
        std::swap(cur, nxt);
    }
    rescale(12);
    // Rayleigh-Ritz on span(G^(4096) Omega), b = 16 columns: the Ritz value is
    // exact to working precision unless lambda_17 / lambda_1 > ~0.99
    const int b = std::min(16, s);
    const int Nb = npad(b);
    double* Om = dbuf(c, "est_Om", (size_t)s * Nb, true);
    double* X = dbuf(c, "est_X2", (size_t)s * Nb, true);
    double* Qb = dbuf(c, "est_Qb", (size_t)s * Nb, true);
    double* GQ = dbuf(c, "est_GQ", (size_t)s * Nb, true);
    double* H = dbuf(c, "est_H", (size_t)b * Nb, true);
    double* Uh = dbuf(c, "est_Uh", (size_t)b * b);
    double* Vh = dbuf(c, "est_Vh", (size_t)b * b);
    double* Sh = dbuf(c, "est_Sh", (size_t)b);
    int* sw = reinterpret_cast<int*>(dbuf(c, "est_sw2", 1));
    {
        std::vector<double> h((size_t)s * b);
        sorsvd_host::gaussian_fill(h.data(), h.size(), 0x5eed5eedULL, 0);
        CK(cudaMemcpy2DAsync(Om, (size_t)Nb * 8, h.data(), (size_t)b * 8, (size_t)b * 8, (size_t)s,
                             cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    auto mm = [&](bool ta, const double* Am, int64_t ldam, int64_t M, int64_t K, const double* Bm, double* Cm) {
        GemmCall g;
        g.ta = ta;
        g.A = Am;
        g.lda = ldam;
        g.M = M;
        g.K = K;
        g.B = Bm;
        g.ldb = Nb;
        g.N = Nb;
        g.C = Cm;
        g.ldc = Nb;
        g.ws_name = "est_ws";
        run_gemm(c, g, st);
    };
    mm(false, cur, Np, s, s, Om, X);   // X = P Omega
    QrPlan* pq = get_qr_plan(c, s, b, 0, "est_b");
    qr_run(c, pq, X, Nb, Qb, Nb, st);  // Q = orth(X)
    mm(false, G, Np, s, s, Qb, GQ);    // G Q
    mm(true, Qb, Nb, b, s, GQ, H);     // H = Q^T G Q  (b x b, symmetric PSD)
    run_jacobi(c, b, H, Nb, Uh, b, Sh, Vh, b, sw, st);
    double h = 0.0;
    CK(cudaMemcpyAsync(&h, Sh, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!std::isfinite(h) || h < 0.0) throw Error{SORSVD_ERR_NUMERICAL, "numerical: sigma_1 estimate not finite"};
    return std::sqrt(h);
}

// sigma_1(A) for mu0 = 1.25/||D||_2: block subspace iteration
// with re-orthonormalisation (TSQR each step) and a Rayleigh-Ritz value from
// the Jacobi SVD of R(A X); iterates until the Ritz value is stationary to
// 1e-14 relative. The reference uses dgesdd on all of D (dense.hpp:173).
double estimate_sigma1(sorsvd_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, uint64_t seed) {
    const int ell = (int)std::max<int64_t>(1, std::min<int64_t>(16, std::min(m, n) - 1));
    const int Np = npad(ell);
    QrPlan* pn = get_qr_plan(c, n, ell, 0, "est_n");
    QrPlan* pm = get_qr_plan(c, m, ell, 0, "est_m");
    double* X = dbuf(c, "est_X", (size_t)n * Np, true);
    double* T1 = dbuf(c, "est_T1", (size_t)m * Np);
    double* T2 = dbuf(c, "est_T2", (size_t)n * Np);
    double* Uk = dbuf(c, "est_U", (size_t)ell * ell);
    double* Vk = dbuf(c, "est_V", (size_t)ell * ell);
    double* Sk = dbuf(c, "est_S", (size_t)ell);
    int* sw = reinterpret_cast<int*>(dbuf(c, "est_sw", 1));
    std::vector<double> h((size_t)n * ell);
    sorsvd_host::gaussian_fill(h.data(), h.size(), seed, 0);
    CK(cudaMemcpy2DAsync(X, (size_t)Np * 8, h.data(), (size_t)ell * 8, (size_t)ell * 8, (size_t)n,
                         cudaMemcpyHostToDevice, c->stream));
    cudaStream_t s = c->stream;
    auto mul = [&](bool ta, const double* B, double* Cout) {
        GemmCall g;
        g.ta = ta;
        g.A = A;
        g.lda = lda;
        g.M = ta ? n : m;
        g.K = ta ? m : n;
        g.B = B;
        g.ldb = Np;
        g.N = Np;
        g.C = Cout;
        g.ldc = Np;
        run_gemm(c, g, s);
    };
    double prev = -1.0, cur = 0.0;
    const int L = (int)pm->nodes.size() - 1;
    for (int it = 1; it <= 400; ++it) {
        mul(false, X, T1);
        mul(true, T1, T2);
        qr_factor(c, pn, T2, Np, X, Np, true, s);
        qr_formq(c, pn, T2, Np, X, Np, nullptr, s);
        if (it % 4 == 0) {
            mul(false, X, T1);
            qr_factor(c, pm, T1, Np, T1, Np, true, s);
            run_jacobi(c, ell, pm->R[L], ell, Uk, ell, Sk, Vk, ell, sw, s);
            CK(cudaMemcpyAsync(&cur, Sk, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (!std::isfinite(cur)) throw Error{SORSVD_ERR_NUMERICAL, "numerical: sigma_1 estimate not finite"};
            if (std::fabs(cur - prev) <= 1e-14 * cur) break;
            prev = cur;
        }
    }
    return cur;
}

void rpca_device(sorsvd_ctx* c, const sorsvd_rpca_desc* d, const double* dD, double* dL, double* dSout,
                 sorsvd_rpca_result* res) {
    if (!d) throw Error{SORSVD_ERR_PARAMETER, "parameter: null descriptor"};
    const int64_t m = d->m, n = d->n, ldd = d->ldd;
    if (m < 2 || n < 2 || ldd < n) throw Error{SORSVD_ERR_SHAPE, "shape: bad RPCA matrix shape"};
    if (d->rho <= 1.0 || d->tol <= 0.0 || d->ell < 1 || d->max_iter < 1)
        throw Error{SORSVD_ERR_PARAMETER, "parameter: rpca config invalid (rho > 1, tol > 0, ell >= 1)"};
    if (const char* e = sorsvd_host::validate_sketch(m, n, d->ell, d->ell, d->q)) throw Error{SORSVD_ERR_PARAMETER, e};
    if (d->dtype != SORSVD_F64) throw Error{SORSVD_ERR_UNSUPPORTED, "only SORSVD_F64 is implemented"};
    const int ell = d->ell;
    const int64_t mg = d->m_global > 0 ? d->m_global : m;
    if (c->world == 1 && mg != m) throw Error{SORSVD_ERR_SHAPE, "shape: m_global != m on a single-rank context"};
    const double lambda = d->lambda > 0 ? d->lambda : 1.0 / std::sqrt((double)std::max(mg, n));
    CK(cudaEventRecord(c->ev_h[2], c->stream));
    const int launches0 = c->launches;
    double* S = dSout ? dSout : dbuf(c, "rp_S", (size_t)m * n);
    double* Y = dbuf(c, "rp_Y", (size_t)m * n);
    double* W = dbuf(c, "rp_W", (size_t)m * n);
    double* U = dbuf(c, "rp_U", (size_t)m * ell);
    double* V = dbuf(c, "rp_V", (size_t)n * ell);
    double* sig = dbuf(c, "rp_sig", (size_t)ell);
    const double dnorm = std::sqrt(device_sumsq(c, dD, m, n, ldd));
    if (!std::isfinite(dnorm)) {
        if (matrix_has_nonfinite(c, dD, SORSVD_F64, m, n, ldd))
            throw Error{SORSVD_ERR_PARAMETER, "parameter: matrix entries must be finite"};
        throw Error{SORSVD_ERR_NUMERICAL, "numerical: ||D||_F overflows"};
    }
    sorsvd_rpca_result r{};
    if (dnorm == 0.0) {  // X = 0 -> L = S = 0 in one iteration
        CK(cudaMemsetAsync(S, 0, (size_t)m * n * 8, c->stream));
        if (dL) CK(cudaMemsetAsync(dL, 0, (size_t)m * n * 8, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        r.iterations = 1;
        r.converged = 1;
        c->rpca_tele.assign(4, 0.0);
        if (res) *res = r;
        return;
    }
    double mu = d->mu0;
    if (!(mu > 0.0)) {
        const bool gram = c->world > 1 ? n <= 1024 : std::min(m, n) <= 1024;
        if (c->world > 1 && !gram)
            throw Error{SORSVD_ERR_UNSUPPORTED, "multi-rank rpca with n > 1024 needs mu0 passed in"};
        mu = 1.25 / (gram ? estimate_sigma1_gram(c, dD, m, n, ldd)
                         : estimate_sigma1(c, dD, m, n, ldd, d->seed ^ 0x5bd1e995ULL));
    }
    r.mu0 = mu;
    const double mu_bar = (d->mu_bar_factor > 0 ? d->mu_bar_factor : 1e7) * mu;
    CK(cudaMemsetAsync(S, 0, (size_t)m * n * 8, c->stream));
    CK(cudaMemsetAsync(Y, 0, (size_t)m * n * 8, c->stream));
    const dim3 grid((unsigned)cdiv(n, 64), (unsigned)cdiv(m, 64));
    const int64_t nblk = (int64_t)grid.x * grid.y;
    double* part = dbuf(c, "rp_part", (size_t)nblk);
    double* tot = dbuf(c, "rp_tot", 4);
    auto* nnzp = reinterpret_cast<unsigned int*>(dbuf(c, "rp_nnzp", (size_t)(nblk + 1) / 2));
    double* tele = dbuf(c, "rp_tele", (size_t)4 * d->max_iter);  // per-iteration telemetry rows
    // Iterations are enqueued kBatch at a time without a host round trip: the
    // stopping test runs on the device (rpca_check_kernel) and every kernel of
    // an iteration after convergence is predicated off, so the result is the
    // same as stopping on the host. mu follows its data-independent schedule
    // (min(rho mu, mu_bar)); each in-flight iteration has its own
    // U / sigma / V slot so the last executed one survives for the final L.
    constexpr int kBatch = 4;
    double* Us = dbuf(c, "rp_Us", (size_t)kBatch * m * ell);
    double* Vs = dbuf(c, "rp_Vs", (size_t)kBatch * n * ell);
    double* sigs = dbuf(c, "rp_sigs", (size_t)kBatch * ell);
    int* stf = reinterpret_cast<int*>(dbuf(c, "rp_state", 2));  // [0] done, [1] iterations, [2] error
    double* rels = dbuf(c, "rp_rel", 1);
    CK(cudaMemsetAsync(stf, 0, 4 * sizeof(int), c->stream));
    for (const char* tag : {"T1", "T2"}) get_qr_plan(c, tag[1] == '1' ? m : n, ell, 0, tag)->hint_house = false;
    std::vector<double> mus;
    mus.push_back(mu);
    int it = 0;
    double rel = 0.0;
    int rank = 0;
    bool conv = false;
    int executed = 0;
    while (it < d->max_iter) {
        const int nb = std::min(kBatch, d->max_iter - it);
        for (int bi = 0; bi < nb; ++bi) {
            const int j = it + bi;
            while ((int)mus.size() <= j + 1) mus.push_back(std::min(d->rho * mus.back(), mu_bar));
            double* Uj = Us + (size_t)(j % kBatch) * m * ell;
            double* Vj = Vs + (size_t)(j % kBatch) * n * ell;
            double* sj = sigs + (size_t)(j % kBatch) * ell;
            PredScope ps(c, stf, 1);  // everything below is skipped once stf[0] == 1
            sorsvd_desc sd{};
            sd.m = m;
            sd.n = n;
            sd.lda = j == 0 ? ldd : n;
            sd.k = ell;
            sd.ell = ell;
            sd.q = d->q;
            sd.seed = d->seed + (uint64_t)j;
            sd.dtype = SORSVD_F64;
            sd.flags = d->flags & SORSVD_FLAG_NO_GRAPH;
            sd.m_global = mg;
            sor_device(c, &sd, j == 0 ? dD : W, nullptr, Uj, sj, Vj, nullptr);
            RpcaArgs a{};
            a.D = dD;
            a.ldd = ldd;
            a.S = S;
            a.Y = Y;
            a.W = W;
            a.ldx = n;
            a.U = Uj;
            a.ldu = ell;
            a.V = Vj;
            a.ldv = ell;
            a.sig = sj;
            a.m = m;
            a.n = n;
            a.k = ell;
            a.mu = mus[j];
            a.mu_next = mus[j + 1];
            a.eps = lambda / mus[j];
            a.partial = part;
            a.nnz_partial = nnzp;
            a.mode = 0;
            a.pred = stf;
            a.pred_skip = 1;
            rpca_update_kernel<<<grid, kRpcaThreads, 0, c->stream>>>(a);
            check_launch(c);
            sum_partials_kernel<<<1, 1024, 0, c->stream>>>(part, nblk, tot, stf, 1, nnzp);
            check_launch(c);
            comm_allreduce(c, tot, 3, false, c->stream);  // residual and nonzero count over all row blocks
            rpca_check_kernel<<<1, 1, 0, c->stream>>>(tot, dnorm, d->tol, j, stf, rels, stf, 1, tele + 4 * (size_t)j, sj,
                                                      ell, mus[j]);
            check_launch(c);
        }
        int hst[3];
        CK(cudaMemcpyAsync(hst, stf, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&rel, rels, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        executed = hst[1];
        if (hst[2]) throw Error{SORSVD_ERR_NUMERICAL, "numerical: rpca produced a non-finite iterate"};
        if (c->world == 1) {
            // W's sketches are ill-conditioned from the first iterations on (a dominant low-rank part over the
            // sparse residue): once the CholeskyQR2 gate has rejected them, later iterations of this solve go
            // straight to the Householder TSQR (the attempt costs a Gram + a factorisation per QR)
            for (const char* tag : {"T1", "T2"}) {
                QrPlan* qp = get_qr_plan(c, tag[1] == '1' ? m : n, ell, 0, tag);
                if (qp->big || qp->hint_house || !qp->flag) continue;
                int fl = 0;
                CK(cudaMemcpy(&fl, qp->flag, sizeof(int), cudaMemcpyDeviceToHost));
                if (fl == 1) qp->hint_house = true;
            }
        }
        if (hst[0]) {
            conv = true;
            break;
        }
        it += nb;
    }
    it = executed;
    for (const char* tag : {"T1", "T2"}) get_qr_plan(c, tag[1] == '1' ? m : n, ell, 0, tag)->hint_house = false;
    // rank of the last executed iteration's shrunk spectrum
    const int fl = it - 1;
    U = Us + (size_t)(fl % kBatch) * m * ell;
    V = Vs + (size_t)(fl % kBatch) * n * ell;
    sig = sigs + (size_t)(fl % kBatch) * ell;
    std::vector<double> hsig(ell);
    CK(cudaMemcpy(hsig.data(), sig, ell * sizeof(double), cudaMemcpyDeviceToHost));
    const double mu_last = mus[fl];
    {
        const double z0 = std::max(hsig[0] - 1.0 / mu_last, 0.0);
        for (int jj = 0; jj < ell; ++jj)
            if (std::max(hsig[jj] - 1.0 / mu_last, 0.0) > 1e-8 * z0) ++rank;
    }
    if (dL) {
        RpcaArgs a{};
        a.L = dL;
        a.ldl = n;
        a.U = U;
        a.ldu = ell;
        a.V = V;
        a.ldv = ell;
        a.sig = sig;
        a.m = m;
        a.n = n;
        a.k = ell;
        a.mu = mu_last;
        a.mode = 1;
        rpca_update_kernel<<<grid, kRpcaThreads, 0, c->stream>>>(a);
        check_launch(c);
    }
    const int blocks = c->num_sms * 4;
    unsigned long long* np = reinterpret_cast<unsigned long long*>(dbuf(c, "rp_nnz", (size_t)blocks));
    nnz_partials_kernel<<<blocks, 256, 0, c->stream>>>(S, m, n, n, np);
    check_launch(c);
    std::vector<unsigned long long> hn(blocks);
    CK(cudaMemcpyAsync(hn.data(), np, blocks * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaEventRecord(c->ev_h[3], c->stream));
    CK(cudaStreamSynchronize(c->stream));
    long long nnz = 0;
    for (auto v : hn) nnz += (long long)v;
    if (c->world > 1) {  // global count (exact in double below 2^53)
        double* dn = dbuf(c, "rp_nnz_g", 1);
        const double hv = (double)nnz;
        CK(cudaMemcpyAsync(dn, &hv, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        comm_allreduce(c, dn, 1, false, c->stream);
        double tot_nnz = 0.0;
        CK(cudaMemcpyAsync(&tot_nnz, dn, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        nnz = (long long)tot_nnz;
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev_h[2], c->ev_h[3]));
    c->rpca_tele.assign((size_t)4 * it, 0.0);
    CK(cudaMemcpy(c->rpca_tele.data(), tele, (size_t)4 * it * sizeof(double), cudaMemcpyDeviceToHost));
    r.iterations = it;
    r.rank_l = rank;
    r.converged = conv ? 1 : 0;
    r.nnz_s = nnz;
    r.rel_error = rel;
    r.ms_total = ms;
    r.launches = c->launches - launches0;
    if (res) *res = r;
}

int fail(sorsvd_ctx* c, const Error& e) {
    if (c) c->err = e.msg;
    g_global_err = e.msg;
    if (c && c->capturing) c->capturing = false;
    return e.status;
}

template <typename F>
int guarded(sorsvd_ctx* c, F&& f) {
    try {
        if (c) CK(cudaSetDevice(c->device));
        const bool order = c && c->legacy_order && c->ev_in && !c->capturing;
        if (order) {
            CK(cudaEventRecord(c->ev_in, cudaStreamLegacy));
            CK(cudaStreamWaitEvent(c->stream, c->ev_in, 0));
        }
        f();
        if (order) {
            CK(cudaEventRecord(c->ev_out, c->stream));
            CK(cudaStreamWaitEvent(cudaStreamLegacy, c->ev_out, 0));
        }
        return SORSVD_OK;
    } catch (const Error& e) {
        if (c && c->emu) c->emu->poison();  // release peers blocked in a collective
        return fail(c, e);
    } catch (const std::bad_alloc&) {
        return fail(c, Error{SORSVD_ERR_OOM, "host allocation failed"});
    } catch (const std::exception& e) {
        return fail(c, Error{SORSVD_ERR_INTERNAL, e.what()});
    }
}

void ctx_init(sorsvd_ctx* c, int device) {
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    for (auto& e : c->ev_blk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    c->stream = c->own_stream;
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreate(&c->ev_a));
    CK(cudaEventCreate(&c->ev_b));
    for (auto& e : c->ev_st) CK(cudaEventCreate(&e));
    for (auto& e : c->ev_h) CK(cudaEventCreate(&e));
}

}  // namespace

// ================================================================ C ABI ====
extern "C" {

const char* sorsvd_version(void) { return "sorsvd-b200 0.2 (sm_100a: tcgen05 int8 digit-plane passes, FP64 DMMA, TF32)"; }

int sorsvd_ctx_create(int device, sorsvd_ctx** out) {
    if (!out) return SORSVD_ERR_PARAMETER;
    auto* c = new sorsvd_ctx();
    int rc = guarded(nullptr, [&] { ctx_init(c, device); });
    if (rc != SORSVD_OK) {
        delete c;
        *out = nullptr;
        return rc;
    }
    *out = c;
    return SORSVD_OK;
}

// Digit products per FP64 multiply-add of this build's Ozaki engines (34: pairs t + u >= 5; 28: >= 6).
int sorsvd_ozaki_products(void) { return kOzProducts; }

int sorsvd_nccl_unique_id(void* out128) {
    return guarded(nullptr, [&] {
        ncclUniqueId id;
        NCK(nccl().GetUniqueId(&id));
        static_assert(sizeof(id) == 128, "nccl id size");
        std::memcpy(out128, &id, sizeof(id));
    });
}

// One-GPU check of the NCCL binding the multi-rank contexts use (libnccl resolved by dlopen, the
// entry points' signatures, ncclDouble / ncclSum, stream-ordered calls): a communicator of ONE rank on
// `device`, an in-place all-reduce and an all-gather of `count` doubles on a fresh stream; both must
// return the input. max_abs_err receives the largest deviation (0 expected).
int sorsvd_nccl_selftest(int device, int64_t count, double* max_abs_err) {
    if (count < 1 || !max_abs_err) return SORSVD_ERR_PARAMETER;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        ncclUniqueId id;
        NCK(nccl().GetUniqueId(&id));
        ncclComm_t comm = nullptr;
        NCK(nccl().CommInitRank(&comm, 1, id, 0));
        cudaStream_t st = nullptr;
        double *a = nullptr, *b = nullptr;
        std::vector<double> h((size_t)count), r((size_t)count), g((size_t)count);
        for (int64_t i = 0; i < count; ++i) h[(size_t)i] = 1.0 / (double)(i + 1) - 0.25 * (double)(i % 7);
        try {
            CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            CK(cudaMalloc(&a, (size_t)count * 8));
            CK(cudaMalloc(&b, (size_t)count * 8));
            CK(cudaMemcpyAsync(a, h.data(), (size_t)count * 8, cudaMemcpyHostToDevice, st));
            NCK(nccl().AllReduce(a, a, (size_t)count, ncclDouble, ncclSum, comm, st));
            NCK(nccl().AllGather(a, b, (size_t)count, ncclDouble, comm, st));
            CK(cudaMemcpyAsync(r.data(), a, (size_t)count * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(g.data(), b, (size_t)count * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } catch (...) {
            cudaFree(a);
            cudaFree(b);
            if (st) cudaStreamDestroy(st);
            nccl().CommDestroy(comm);
            throw;
        }
        cudaFree(a);
        cudaFree(b);
        cudaStreamDestroy(st);
        NCK(nccl().CommDestroy(comm));
        double e = 0.0;
        for (int64_t i = 0; i < count; ++i)
            e = std::max(e, std::max(std::fabs(r[(size_t)i] - h[(size_t)i]), std::fabs(g[(size_t)i] - h[(size_t)i])));
        *max_abs_err = e;
    });
}

int sorsvd_ctx_create_dist(int device, int rank, int world, const void* unique_id128, sorsvd_ctx** out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return SORSVD_ERR_PARAMETER;
    auto* c = new sorsvd_ctx();
    int rc = guarded(nullptr, [&] {
        ctx_init(c, device);
        c->rank = rank;
        c->world = world;
        if (world > 1) {
            ncclUniqueId id;
            std::memcpy(&id, unique_id128, sizeof(id));
            NCK(nccl().CommInitRank(&c->comm, world, id, rank));
        }
    });
    if (rc != SORSVD_OK) {
        delete c;
        *out = nullptr;
        return rc;
    }
    *out = c;
    return SORSVD_OK;
}

int sorsvd_emu_group_create(int world, sorsvd_emu_group** out) {
    if (!out || world < 1) return SORSVD_ERR_PARAMETER;
    auto* g = new sorsvd_emu_group();
    g->world = world;
    g->bufs.assign(world, nullptr);
    *out = g;
    return SORSVD_OK;
}

void sorsvd_emu_group_destroy(sorsvd_emu_group* g) { delete g; }

int sorsvd_ctx_create_emulated(int device, int rank, sorsvd_emu_group* g, sorsvd_ctx** out) {
    if (!out || !g || rank < 0 || rank >= g->world) return SORSVD_ERR_PARAMETER;
    auto* c = new sorsvd_ctx();
    int rc = guarded(nullptr, [&] {
        ctx_init(c, device);
        c->rank = rank;
        c->world = g->world;
        c->emu = g;
    });
    if (rc != SORSVD_OK) {
        delete c;
        *out = nullptr;
        return rc;
    }
    *out = c;
    return SORSVD_OK;
}

void sorsvd_ctx_destroy(sorsvd_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    invalidate_graphs(c);
    for (auto& kv : c->plans)
        for (void* p : kv.second->owned) cudaFree(p);
    for (auto& kv : c->bufs)
        if (kv.second.p) cudaFree(kv.second.p);
    if (c->comm) nccl().CommDestroy(c->comm);
    cudaEventDestroy(c->ev_fork);
    cudaEventDestroy(c->ev_join);
    cudaEventDestroy(c->ev_a);
    cudaEventDestroy(c->ev_b);
    for (auto& e : c->ev_st) cudaEventDestroy(e);
    for (auto& e : c->ev_h) cudaEventDestroy(e);
    for (auto& kv : c->sk_tables)
        for (int* d : kv.second.dev) cudaFree(d);
    if (c->om_pin) cudaFreeHost(c->om_pin);
    for (cudaStream_t t : c->tstreams) cudaStreamDestroy(t);
    for (cudaEvent_t e : c->tevents) cudaEventDestroy(e);
    for (cudaEvent_t e : c->up_ev) cudaEventDestroy(e);
    cudaStreamSynchronize(c->comm_stream);
    for (auto& e : c->ev_blk) cudaEventDestroy(e);
    cudaEventDestroy(c->ev_comm);
    cudaEventDestroy(c->ev_in);
    cudaEventDestroy(c->ev_out);
    cudaStreamDestroy(c->comm_stream);
    cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->own_stream);
    delete c;
}

const char* sorsvd_last_error(const sorsvd_ctx* c) { return c ? c->err.c_str() : g_global_err.c_str(); }

int sorsvd_set_stream(sorsvd_ctx* c, void* stream) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        // NULL: the caller's work is on the legacy default stream (torch's default stream):
        // compute on the own stream, ordered with it by events (see legacy_order)
        cudaStream_t s = stream ? (cudaStream_t)stream : c->own_stream;
        if (s != c->stream) invalidate_graphs(c);
        c->stream = s;
        c->legacy_order = stream == nullptr;
    });
}

int sorsvd_ctx_set_option(sorsvd_ctx* c, int32_t key, int64_t value) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        switch (key) {
            case SORSVD_OPT_JACOBI:
                if (value < SORSVD_JACOBI_AUTO || value > SORSVD_JACOBI_ROTLOG)
                    throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown Jacobi variant"};
                c->opt_jacobi = (int)value;
                invalidate_graphs(c);  // captured calls baked the previous variant in
                break;
            case SORSVD_OPT_OZAKI_OVERLAP:
                c->opt_oz_overlap = value != 0;
                invalidate_graphs(c);
                break;
            case SORSVD_OPT_OZAKI_MULTICAST:
                c->opt_oz_multicast = value != 0;
                invalidate_graphs(c);
                break;
            case SORSVD_OPT_UPLOAD_TN:
                c->opt_upload_tn = value != 0;
                break;
            case SORSVD_OPT_NCCL_GRAPH:
                c->opt_nccl_graph = value != 0;
                invalidate_graphs(c);
                break;
            case SORSVD_OPT_UPLOAD_CHUNK_MB:
                if (value < 1) throw Error{SORSVD_ERR_PARAMETER, "parameter: upload chunk must be >= 1 MiB"};
                c->opt_upload_chunk_mb = value;
                break;
            case SORSVD_OPT_FUSED_PAIR:
                if (value < 0 || value > 2) throw Error{SORSVD_ERR_PARAMETER, "parameter: FUSED_PAIR is 0, 1 or 2"};
                c->opt_fused_pair = (int)value;  // 2: the one-pipeline kernel also for n <= 320 (A/B timing)
                invalidate_graphs(c);
                break;
            case SORSVD_OPT_OZAKI_PLANES:
                if (value < 0) throw Error{SORSVD_ERR_PARAMETER, "parameter: OZAKI_PLANES must be >= 0"};
                c->opt_oz_planes = (int64_t)value;
                invalidate_graphs(c);
                break;
            case SORSVD_OPT_SORD_CHUNK_MB:
                if (value < 1) throw Error{SORSVD_ERR_PARAMETER, "parameter: SORD chunk must be >= 1 MiB"};
                c->opt_sord_chunk_mb = value;
                break;
            default: throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown context option"};
        }
    });
}

int sorsvd_ctx_rank(const sorsvd_ctx* c, int* rank, int* world) {
    if (!c) return SORSVD_ERR_PARAMETER;
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    return SORSVD_OK;
}

int sorsvd_sor_svd_power_device(sorsvd_ctx* c, const sorsvd_desc* d, const void* dA, const double* dOmega,
                                double* dU, double* dSigma, double* dV, sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (!dA || !dU || !dSigma || !dV) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        sor_device(c, d, dA, dOmega, dU, dSigma, dV, st);
    });
}

// Host-buffer call of one of the decompositions: A (and the given test
// matrices) uploaded, U / sigma / V downloaded, all inside the timed call.
static void host_call(sorsvd_ctx* c, const sorsvd_desc* d, const void* A, const double* omega, const double* psi2,
                      double* U, double* sigma, double* V, sorsvd_stats* st, int method) {
    validate(d);
    if (!A || !U || !sigma || !V) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
    const size_t esz = d->dtype == SORSVD_F32 ? 4 : 8;
    const size_t abytes = (size_t)d->m * d->lda * esz;
    cudaEvent_t e0 = c->ev_h[0], e1 = c->ev_h[1], e2 = c->ev_h[2], e3 = c->ev_h[3];
    CK(cudaEventRecord(e0, c->stream));
    {
        // the device copy of A comes first: a planes workspace left by an earlier (device-resident)
        // call is given back when A would not fit beside it
        auto ia = c->bufs.find("hostA");
        const size_t have_a = ia == c->bufs.end() ? 0 : ia->second.bytes;
        auto ip = c->bufs.find("oz_planes");
        if (have_a < abytes && ip != c->bufs.end() && ip->second.p) {
            size_t fr = 0, tot = 0;
            CK(cudaMemGetInfo(&fr, &tot));
            if (fr + have_a < abytes + ((size_t)8 << 30)) {
                CK(cudaStreamSynchronize(c->stream));
                invalidate_graphs(c);
                CK(cudaFree(ip->second.p));
                c->bufs.erase(ip);
            }
        }
    }
    double* dA = dbuf(c, "hostA", (abytes + 7) / 8);
    HostUpload up;
    // whatever happens below (a validation error, a CUDA failure), the caller's A is not read after
    // this function returns: the copy stream is drained on every exit path
    struct DrainCopies {
        sorsvd_ctx* c;
        ~DrainCopies() {
            cudaStreamSynchronize(c->comm_stream);
            cudaStreamSynchronize(c->stream);
        }
    } drain{c};
    {
        // Ozaki planes engine on one rank: upload A in row chunks on the copy stream and let the
        // device convert / sweep each chunk as it lands (sor_device); else one copy on the stream
        SorProblem P{};
        P.m = d->m;
        P.n = d->n;
        P.Np = npad(d->ell);
        const bool planes = method == SORSVD_SOR_POWER && c->world == 1 &&
                            !(d->dtype == SORSVD_F32 && (d->flags & SORSVD_FLAG_TF32)) &&
                            ozaki_wanted(d->flags, d->m, d->n, d->ell) && oz_planes_fit(c, P);
        if (planes) up = upload_chunked(c, A, dA, d->m, d->lda, esz, P.Np);
        else CK(cudaMemcpyAsync(dA, A, abytes, cudaMemcpyHostToDevice, c->stream));
    }
    // A copy engine drains one stream's queued copies before it turns to another stream's, so with a
    // chunked upload Omega's (small) copy rides the copy stream itself, between chunk 0 and the rest
    cudaStream_t om_stream = up.chunked ? c->comm_stream : c->stream;
    const double* dOm = nullptr;
    sorsvd_desc dd = *d;
    if (omega && (d->flags & SORSVD_FLAG_OMEGA_GIVEN)) {
        double* p = dbuf(c, "hostOm", (size_t)d->n * d->ell);
        CK(cudaMemcpyAsync(p, omega, (size_t)d->n * d->ell * 8, cudaMemcpyHostToDevice, om_stream));
        dOm = p;
    } else if (method != SORSVD_TSR) {
        // draw Omega = gaussian_matrix(n, ell, seed) (sketch.hpp:90) into a page-locked
        // buffer while A's transfer runs, and upload it asynchronously right behind A (a
        // pageable upload would stall the host behind A and then stage the copy); the call
        // is synchronous, so the buffer is free again when it returns
        const size_t cnt = (size_t)d->n * d->ell;
        if (c->om_pin_n < cnt) {
            if (c->om_pin) CK(cudaFreeHost(c->om_pin));
            c->om_pin = nullptr;
            CK(cudaHostAlloc(reinterpret_cast<void**>(&c->om_pin), cnt * sizeof(double), cudaHostAllocDefault));
            c->om_pin_n = cnt;
        }
        c->host_omega.resize(cnt);
        sorsvd_host::gaussian_fill(c->host_omega.data(), (uint64_t)cnt, d->seed, 0);
        memcpy(c->om_pin, c->host_omega.data(), cnt * sizeof(double));
        double* p = dbuf(c, "hostOm", cnt);
        CK(cudaMemcpyAsync(p, c->om_pin, cnt * 8, cudaMemcpyHostToDevice, om_stream));
        dOm = p;
        dd.flags |= SORSVD_FLAG_OMEGA_GIVEN;
    }
    if (up.chunked) {  // Omega rode the copy stream (behind chunk 0): the compute stream waits for it
        CK(cudaEventRecord(c->ev_comm, c->comm_stream));
        CK(cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
    }
    d = &dd;
    const double* dPsi2 = nullptr;
    if (psi2 && (d->flags & SORSVD_FLAG_OMEGA_GIVEN)) {
        double* p = dbuf(c, "hostPsi2", (size_t)d->m * d->ell);
        CK(cudaMemcpyAsync(p, psi2, (size_t)d->m * d->ell * 8, cudaMemcpyHostToDevice, c->stream));
        dPsi2 = p;
    }
    if (up.chunked) upload_issue(c, up, A, dA, d->m, d->lda, esz, up.nchunks);
    CK(cudaEventRecord(e1, c->stream));
    double* dU = dbuf(c, "hostU", (size_t)d->m * d->k);
    double* dS = dbuf(c, "hostS", (size_t)d->k);
    double* dV = dbuf(c, "hostV", (size_t)d->n * d->k);
    sorsvd_stats local{};
    sor_device(c, d, dA, dOm, dU, dS, dV, &local, method, dPsi2, up.chunked ? &up : nullptr);
    CK(cudaEventRecord(e2, c->stream));
    CK(cudaMemcpyAsync(U, dU, (size_t)d->m * d->k * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(V, dV, (size_t)d->n * d->k * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(sigma, dS, (size_t)d->k * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaEventRecord(e3, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float h2d = 0.f, d2h = 0.f;
    CK(cudaEventElapsedTime(&h2d, e0, e1));
    CK(cudaEventElapsedTime(&d2h, e2, e3));
    local.ms_h2d = h2d;
    local.ms_d2h = d2h;
    if (st) *st = local;
}

int sorsvd_sor_svd_power(sorsvd_ctx* c, const sorsvd_desc* d, const void* A, const double* omega, double* U,
                         double* sigma, double* V, sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] { host_call(c, d, A, omega, nullptr, U, sigma, V, st, SORSVD_SOR_POWER); });
}

// r_svd / tsr_svd take (ell, q, seed) / (ell, seed): the descriptor is
// normalised to k = ell (all ell triplets are returned, sketch.hpp:122,139),
// q = 0 for tsr and no single-pass core.
static sorsvd_desc baseline_desc(const sorsvd_desc* d, int method) {
    if (!d) throw Error{SORSVD_ERR_PARAMETER, "parameter: null descriptor"};
    sorsvd_desc e = *d;
    e.k = e.ell;
    e.single_pass = 0;
    e.flags &= ~SORSVD_FLAG_BASIC;
    if (method == SORSVD_TSR) e.q = 0;
    return e;
}

int sorsvd_r_svd(sorsvd_ctx* c, const sorsvd_desc* d, const void* A, const double* omega, double* U, double* sigma,
                 double* V, sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        const sorsvd_desc e = baseline_desc(d, SORSVD_RSVD);
        host_call(c, &e, A, omega, nullptr, U, sigma, V, st, SORSVD_RSVD);
    });
}

int sorsvd_r_svd_device(sorsvd_ctx* c, const sorsvd_desc* d, const void* dA, const double* dOmega, double* dU,
                        double* dSigma, double* dV, sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        const sorsvd_desc e = baseline_desc(d, SORSVD_RSVD);
        if (!dA || !dU || !dSigma || !dV) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        sor_device(c, &e, dA, dOmega, dU, dSigma, dV, st, SORSVD_RSVD);
    });
}

int sorsvd_tsr_svd(sorsvd_ctx* c, const sorsvd_desc* d, const void* A, const double* psi1, const double* psi2,
                   double* U, double* sigma, double* V, sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        const sorsvd_desc e = baseline_desc(d, SORSVD_TSR);
        if ((e.flags & SORSVD_FLAG_OMEGA_GIVEN) && (!psi1 || !psi2))
            throw Error{SORSVD_ERR_PARAMETER, "parameter: OMEGA_GIVEN needs both psi1 and psi2"};
        host_call(c, &e, A, psi1, psi2, U, sigma, V, st, SORSVD_TSR);
    });
}

int sorsvd_tsr_svd_device(sorsvd_ctx* c, const sorsvd_desc* d, const void* dA, const double* dPsi1,
                          const double* dPsi2, double* dU, double* dSigma, double* dV, sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        const sorsvd_desc e = baseline_desc(d, SORSVD_TSR);
        if (!dA || !dU || !dSigma || !dV) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        if ((e.flags & SORSVD_FLAG_OMEGA_GIVEN) && (!dPsi1 || !dPsi2))
            throw Error{SORSVD_ERR_PARAMETER, "parameter: OMEGA_GIVEN needs both psi1 and psi2"};
        sor_device(c, &e, dA, dPsi1, dU, dSigma, dV, st, SORSVD_TSR, dPsi2);
    });
}

int sorsvd_sor_svd_power_batch_device(sorsvd_ctx* c, const sorsvd_desc* d, int32_t trials, const uint64_t* seeds,
                                      const void* dA, const double* dOmegas, double* dU, double* dSigma, double* dV,
                                      sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (!dA || !dU || !dSigma || !dV) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        batch_device(c, d, trials, seeds, dA, dOmegas, dU, dSigma, dV, st);
    });
}

int sorsvd_sor_svd_power_batch(sorsvd_ctx* c, const sorsvd_desc* d, int32_t trials, const uint64_t* seeds,
                               const void* A, const double* omegas, double* U, double* sigma, double* V,
                               sorsvd_stats* st) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        validate(d);
        if (trials < 1) throw Error{SORSVD_ERR_PARAMETER, "parameter: trials must be positive"};
        if (!A || !U || !sigma || !V) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        const size_t esz = d->dtype == SORSVD_F32 ? 4 : 8;
        const size_t abytes = (size_t)d->m * d->lda * esz;
        cudaEvent_t e0 = c->ev_h[0], e1 = c->ev_h[1], e2 = c->ev_h[2], e3 = c->ev_h[3];
        CK(cudaEventRecord(e0, c->stream));
        double* dA = dbuf(c, "hostA", (abytes + 7) / 8);
        CK(cudaMemcpyAsync(dA, A, abytes, cudaMemcpyHostToDevice, c->stream));
        const double* dOm = nullptr;
        const size_t om_n = (size_t)trials * d->n * d->ell;
        if (omegas && (d->flags & SORSVD_FLAG_OMEGA_GIVEN)) {
            double* p = dbuf(c, "hostOmB", om_n);
            CK(cudaMemcpyAsync(p, omegas, om_n * 8, cudaMemcpyHostToDevice, c->stream));
            dOm = p;
        }
        CK(cudaEventRecord(e1, c->stream));
        const size_t un = (size_t)trials * d->m * d->k, vn = (size_t)trials * d->n * d->k, sn = (size_t)trials * d->k;
        double* dU = dbuf(c, "hostUB", un);
        double* dS = dbuf(c, "hostSB", sn);
        double* dV = dbuf(c, "hostVB", vn);
        sorsvd_stats local{};
        batch_device(c, d, trials, seeds, dA, dOm, dU, dS, dV, &local);
        CK(cudaEventRecord(e2, c->stream));
        CK(cudaMemcpyAsync(U, dU, un * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(V, dV, vn * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(sigma, dS, sn * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaEventRecord(e3, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        float h2d = 0.f, d2h = 0.f;
        CK(cudaEventElapsedTime(&h2d, e0, e1));
        CK(cudaEventElapsedTime(&d2h, e2, e3));
        local.ms_h2d = h2d;
        local.ms_d2h = d2h;
        if (st) *st = local;
    });
}

// approx_error(a, x, frobenius)   (sketch.hpp:168-172), fused single pass over A
int sorsvd_approx_error_fro_device(sorsvd_ctx* c, int64_t m, int64_t n, const void* dA, int64_t lda, int32_t dtype,
                                   int32_t k, const double* dU, int64_t ldu, const double* dSigma, const double* dV,
                                   int64_t ldv, double* err) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (m < 1 || n < 1 || k < 1 || lda < n || ldu < k || ldv < k)
            throw Error{SORSVD_ERR_SHAPE, "shape: approx_error: approximation does not match matrix dims"};
        if (!dA || !dU || !dSigma || !dV || !err) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        if (dtype != SORSVD_F64 && dtype != SORSVD_F32) throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown dtype"};
        const dim3 grid((unsigned)cdiv(n, 64), (unsigned)cdiv(m, 64));
        const int64_t nblk = (int64_t)grid.x * grid.y;
        double* part = dbuf(c, "ae_part", (size_t)nblk);
        double* tot = dbuf(c, "ae_tot", 2);
        if (dtype == SORSVD_F64)
            approx_err_kernel<double><<<grid, kRpcaThreads, 0, c->stream>>>(static_cast<const double*>(dA), lda, dU,
                                                                            ldu, dSigma, dV, ldv, m, n, k, part);
        else
            approx_err_kernel<float><<<grid, kRpcaThreads, 0, c->stream>>>(static_cast<const float*>(dA), lda, dU, ldu,
                                                                           dSigma, dV, ldv, m, n, k, part);
        check_launch(c);
        sum_partials_kernel<<<1, 1024, 0, c->stream>>>(part, nblk, tot);
        check_launch(c);
        comm_allreduce(c, tot, 1, false, c->stream);  // row-sharded A: sum of squares over ranks
        double h[2];
        CK(cudaMemcpyAsync(h, tot, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        *err = sqrt(h[0]);
    });
}

// norm(a, spectral)   (dense.hpp:173-176: dgesdd 'N' on the whole matrix): sigma_1 from the Gram
// squaring + Rayleigh-Ritz estimate (min(m, n) <= 1024; <= 1e-12 relative vs dgesdd) or the block
// subspace iteration above it.
int sorsvd_norm_spectral_device(sorsvd_ctx* c, int64_t m, int64_t n, const double* dA, int64_t lda, uint64_t seed,
                                double* out) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (m < 1 || n < 1 || lda < n) throw Error{SORSVD_ERR_SHAPE, "shape: matrix dimensions must be positive"};
        if (!dA || !out) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        // row-sharded A (dA = this rank's rows): the Gram path sums G = A_r^T A_r over the ranks
        if (c->world > 1 && n > 1024)
            throw Error{SORSVD_ERR_UNSUPPORTED, "norm(spectral): row-sharded contexts need n <= 1024"};
        const double ss = device_sumsq(c, dA, m, n, lda);
        if (!std::isfinite(ss)) throw Error{SORSVD_ERR_PARAMETER, "parameter: matrix entries must be finite"};
        if (ss == 0.0) {
            *out = 0.0;
            return;
        }
        *out = (std::min(m, n) <= 1024 || c->world > 1) ? estimate_sigma1_gram(c, dA, m, n, lda)
               : std::min(m, n) < 3  ? std::sqrt(ss)  // unreachable for the harness; rank-1-ish edge
                                      : estimate_sigma1(c, dA, m, n, lda, seed);
    });
}

// approx_error(a, x, spectral)   (sketch.hpp:168-172): E = a - reconstruct(x) formed on the device,
// then norm(E, spectral) as above. The bound harness (bounds.hpp:289-290) calls both norms per trial.
int sorsvd_approx_error_spectral_device(sorsvd_ctx* c, int64_t m, int64_t n, const void* dA, int64_t lda, int32_t dtype,
                                        int32_t k, const double* dU, int64_t ldu, const double* dSigma,
                                        const double* dV, int64_t ldv, double* err) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (m < 1 || n < 1 || k < 1 || lda < n || ldu < k || ldv < k)
            throw Error{SORSVD_ERR_SHAPE, "shape: approx_error: approximation does not match matrix dims"};
        if (!dA || !dU || !dSigma || !dV || !err) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        if (dtype != SORSVD_F64 && dtype != SORSVD_F32) throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown dtype"};
        if (c->world > 1 && n > 1024)  // dA, dU: this rank's rows; sigma, V replicated
            throw Error{SORSVD_ERR_UNSUPPORTED, "approx_error(spectral): row-sharded contexts need n <= 1024"};
        const int64_t lde = (n + 7) / 8 * 8;
        double* E = dbuf(c, "ae_E", (size_t)m * lde, true);
        const dim3 grid((unsigned)cdiv(n, 16), (unsigned)cdiv(m, 16));
        if (dtype == SORSVD_F64)
            residual_kernel<double><<<grid, 256, 0, c->stream>>>(static_cast<const double*>(dA), lda, dU, ldu, dSigma, dV,
                                                                ldv, m, n, k, E, lde);
        else
            residual_kernel<float><<<grid, 256, 0, c->stream>>>(static_cast<const float*>(dA), lda, dU, ldu, dSigma, dV,
                                                               ldv, m, n, k, E, lde);
        check_launch(c);
        const double ss = device_sumsq(c, E, m, n, lde);
        if (!std::isfinite(ss)) throw Error{SORSVD_ERR_NUMERICAL, "numerical: approximation error not finite"};
        if (ss == 0.0) {
            *err = 0.0;
            return;
        }
        *err = (std::min(m, n) <= 1024 || c->world > 1) ? estimate_sigma1_gram(c, E, m, n, lde)
                                                        : estimate_sigma1(c, E, m, n, lde, 0x5eedULL);
    });
}

int sorsvd_sord_header(const char* path, int64_t* rows, int64_t* cols) {
    try {
        if (!path || !rows || !cols) return SORSVD_ERR_PARAMETER;
        Fd f;
        f.fd = open(path, O_RDONLY);
        if (f.fd < 0) return SORSVD_ERR_PARAMETER;
        const SordHeader h = sord_read_header(f.fd, path);
        *rows = h.rows;
        *cols = h.cols;
        return SORSVD_OK;
    } catch (const Error& e) {
        g_global_err = e.msg;
        return e.status;
    }
}

int sorsvd_load_sord_device(sorsvd_ctx* c, const char* path, void* dA, int64_t lda, int32_t dtype) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (!path || !dA) throw Error{SORSVD_ERR_PARAMETER, "parameter: null argument"};
        sord_load(c, path, dA, lda, dtype);
    });
}

int sorsvd_save_sord_device(sorsvd_ctx* c, const char* path, const double* dA, int64_t rows, int64_t cols,
                            int64_t lda) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (!path || !dA) throw Error{SORSVD_ERR_PARAMETER, "parameter: null argument"};
        sord_save(c, path, dA, rows, cols, lda);
    });
}

int sorsvd_thin_qr_device(sorsvd_ctx* c, int64_t m, int32_t k, const double* dT, int64_t ldt, double* dQ,
                          int64_t ldq, double* dR, int64_t ldr) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (m < k || k < 1) throw Error{SORSVD_ERR_SHAPE, "shape: thin_qr requires rows >= cols"};
        if (k > 512) throw Error{SORSVD_ERR_UNSUPPORTED, "thin_qr: k > 512"};
        const int Np = npad(k);
        QrPlan* p = get_qr_plan(c, m, k, 0, "api");
        double* T = dbuf(c, "qrT", (size_t)m * Np, true);
        double* Q = dbuf(c, "qrQ", (size_t)m * Np, true);
        CK(cudaMemcpy2DAsync(T, (size_t)Np * 8, dT, (size_t)ldt * 8, (size_t)k * 8, (size_t)m,
                             cudaMemcpyDeviceToDevice, c->stream));
        qr_run(c, p, T, Np, Q, Np, c->stream);
        CK(cudaMemcpy2DAsync(dQ, (size_t)ldq * 8, Q, (size_t)Np * 8, (size_t)k * 8, (size_t)m,
                             cudaMemcpyDeviceToDevice, c->stream));
        const int L = (int)p->nodes.size() - 1;
        if (dR)
            CK(cudaMemcpy2DAsync(dR, (size_t)ldr * 8, p->R[L], (size_t)p->ldR * 8, (size_t)k * 8, (size_t)k,
                                 cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        check_big_qr(p);
    });
}

// estimate_rank_bound(x) = ceil((||X||_* / ||X||_F)^2)   (PAPER Eq. 66; spec only,
// no reference code): the spectrum of X from thin QR + the Jacobi SVD of R (min(m, n) <= 512; a
// wide X is transposed first). The quotient is shaved by 1e-12 before the ceiling so that exactly
// flat spectra (I_n -> n, rank 1 -> 1: the spec's examples) are not pushed up by rounding.
int sorsvd_estimate_rank_bound_device(sorsvd_ctx* c, int64_t m, int64_t n, const double* dX, int64_t ldx,
                                      int64_t* bound, double* nuclear, double* frobenius) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (m < 1 || n < 1 || ldx < n) throw Error{SORSVD_ERR_SHAPE, "shape: matrix dimensions must be positive"};
        if (!dX || !bound) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        // row-sharded X (dX = this rank's rows): local thin QR, the ranks' R factors gathered and
        // factored again (the TSQR of qr_rows without forming Q), so every rank gets the same spectrum
        const bool sharded = c->world > 1;
        if (sharded && (m < n || n > kHouseMaxK))
            throw Error{SORSVD_ERR_UNSUPPORTED, "estimate_rank_bound: row-sharded contexts need n <= 256 and >= n rows per rank"};
        const double ss = device_sumsq(c, dX, m, n, ldx);
        if (!std::isfinite(ss)) throw Error{SORSVD_ERR_PARAMETER, "parameter: matrix entries must be finite"};
        if (ss == 0.0) throw Error{SORSVD_ERR_PARAMETER, "parameter: estimate_rank_bound of the zero matrix"};
        const int64_t rows = std::max(m, n);
        const int k = (int)std::min(m, n);
        if (k > 512) throw Error{SORSVD_ERR_UNSUPPORTED, "estimate_rank_bound: min(m, n) > 512"};
        const int Np = npad(k);
        double* T = dbuf(c, "erT", (size_t)rows * Np, true);
        double* Q = dbuf(c, "erQ", (size_t)rows * Np, true);
        if (m >= n) {
            CK(cudaMemcpy2DAsync(T, (size_t)Np * 8, dX, (size_t)ldx * 8, (size_t)n * 8, (size_t)m,
                                 cudaMemcpyDeviceToDevice, c->stream));
        } else {
            dim3 tb(32, 8), tg((unsigned)cdiv(m, 32), (unsigned)cdiv(n, 32));
            transpose_kernel<<<tg, tb, 0, c->stream>>>(dX, ldx, m, n, T, Np);
            check_launch(c);
        }
        double fro = std::sqrt(ss), nuc = 0.0;
        std::vector<double> hs((size_t)k);
        if (k == 1) {
            nuc = fro;
        } else {
            QrPlan* p = get_qr_plan(c, rows, k, 0, "er");
            if (sharded) {
                qr_factor(c, p, T, Np, Q, Np, false, c->stream);
                const int L1 = (int)p->nodes.size() - 1;
                double* Rg = dbuf(c, "erRg", (size_t)c->world * k * k);
                comm_allgather(c, p->R[L1], Rg, (size_t)k * k, c->stream);
                p = get_qr_plan(c, (int64_t)c->world * k, k, c->world, "erG");
                qr_factor(c, p, nullptr, 0, nullptr, 0, true, c->stream, Rg);
            } else {
                qr_run(c, p, T, Np, Q, Np, c->stream);
            }
            const int L = (int)p->nodes.size() - 1;
            double* U = dbuf(c, "erU", (size_t)k * k);
            double* V = dbuf(c, "erV", (size_t)k * k);
            double* S = dbuf(c, "erS", (size_t)k);
            int* dsw = reinterpret_cast<int*>(dbuf(c, "sweeps_er", 1));
            run_jacobi(c, k, p->R[L], (int)p->ldR, U, k, S, V, k, dsw, c->stream);
            CK(cudaMemcpyAsync(hs.data(), S, (size_t)k * 8, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            check_big_qr(p);
            for (int j = k - 1; j >= 0; --j) nuc += hs[(size_t)j];  // small values first
        }
        if (!std::isfinite(nuc)) throw Error{SORSVD_ERR_NUMERICAL, "numerical: singular values not finite"};
        const double ratio = nuc / fro;
        *bound = (int64_t)std::max(1.0, std::ceil(ratio * ratio * (1.0 - 1e-12)));
        if (nuclear) *nuclear = nuc;
        if (frobenius) *frobenius = fro;
    });
}

// Host-buffer form of estimate_rank_bound (X uploaded into a context workspace).
int sorsvd_estimate_rank_bound(sorsvd_ctx* c, int64_t m, int64_t n, const double* X, int64_t ldx, int64_t* bound,
                               double* nuclear, double* frobenius) {
    if (!c) return SORSVD_ERR_PARAMETER;
    double* dX = nullptr;
    const int rc = guarded(c, [&] {
        if (m < 1 || n < 1 || ldx < n) throw Error{SORSVD_ERR_SHAPE, "shape: matrix dimensions must be positive"};
        if (!X || !bound) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        dX = dbuf(c, "er_host", (size_t)m * n);
        CK(cudaMemcpy2DAsync(dX, (size_t)n * 8, X, (size_t)ldx * 8, (size_t)n * 8, (size_t)m, cudaMemcpyHostToDevice,
                             c->stream));
    });
    if (rc != SORSVD_OK) return rc;
    return sorsvd_estimate_rank_bound_device(c, m, n, dX, n, bound, nuclear, frobenius);
}

int sorsvd_small_svd_device(sorsvd_ctx* c, int32_t k, const double* dM, int64_t ldm, double* dU, int64_t ldu,
                            double* dS, double* dV, int64_t ldv, int32_t* sweeps) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (k < 1 || k > 512) throw Error{SORSVD_ERR_PARAMETER, "parameter: k out of range [1, 512]"};
        int* dsw = reinterpret_cast<int*>(dbuf(c, "sweeps_svd", 1));
        run_jacobi(c, k, dM, (int)ldm, dU, (int)ldu, dS, dV, (int)ldv, dsw, c->stream);
        int sw = 0;
        CK(cudaMemcpyAsync(&sw, dsw, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (sweeps) *sweeps = sw;
    });
}

int sorsvd_matmul_device(sorsvd_ctx* c, int32_t ta, int64_t M, int64_t K, int32_t N, const double* dA,
                         int64_t lda, const double* dB, int64_t ldb, double* dC, int64_t ldc) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (M < 1 || K < 1 || N < 1) throw Error{SORSVD_ERR_SHAPE, "shape: matmul dims must be positive"};
        const int Np = npad(N);
        double* Bp = dbuf(c, "mmB", (size_t)K * Np, true);
        double* Cp = dbuf(c, "mmC", (size_t)M * Np);
        CK(cudaMemcpy2DAsync(Bp, (size_t)Np * 8, dB, (size_t)ldb * 8, (size_t)N * 8, (size_t)K,
                             cudaMemcpyDeviceToDevice, c->stream));
        GemmCall g;
        g.ta = ta != 0;
        g.A = dA;
        g.lda = lda;
        g.M = M;
        g.K = K;
        g.B = Bp;
        g.ldb = Np;
        g.N = Np;
        g.C = Cp;
        g.ldc = Np;
        run_gemm(c, g, c->stream);
        CK(cudaMemcpy2DAsync(dC, (size_t)ldc * 8, Cp, (size_t)Np * 8, (size_t)N * 8, (size_t)M,
                             cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sorsvd_rpca_alm_device(sorsvd_ctx* c, const sorsvd_rpca_desc* d, const double* dD, double* dL, double* dS,
                           sorsvd_rpca_result* res) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (!dD || !dS) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        rpca_device(c, d, dD, dL, dS, res);
    });
}

int sorsvd_rpca_alm(sorsvd_ctx* c, const sorsvd_rpca_desc* d, const double* D, double* L, double* S,
                    sorsvd_rpca_result* res) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (!d) throw Error{SORSVD_ERR_PARAMETER, "parameter: null descriptor"};
        if (!D || !S) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        const size_t cells = (size_t)d->m * d->n;
        CK(cudaEventRecord(c->ev_h[0], c->stream));
        double* dD = dbuf(c, "rp_hostD", (size_t)d->m * d->ldd);
        CK(cudaMemcpyAsync(dD, D, (size_t)d->m * d->ldd * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaEventRecord(c->ev_h[1], c->stream));
        double* dS = dbuf(c, "rp_hostS", cells);
        double* dL = L ? dbuf(c, "rp_hostL", cells) : nullptr;
        sorsvd_rpca_result r{};
        rpca_device(c, d, dD, dL, dS, &r);
        float h2d = 0.f;
        CK(cudaEventElapsedTime(&h2d, c->ev_h[0], c->ev_h[1]));
        CK(cudaEventRecord(c->ev_h[0], c->stream));
        CK(cudaMemcpyAsync(S, dS, cells * 8, cudaMemcpyDeviceToHost, c->stream));
        if (L) CK(cudaMemcpyAsync(L, dL, cells * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaEventRecord(c->ev_h[1], c->stream));
        CK(cudaStreamSynchronize(c->stream));
        float d2h = 0.f;
        CK(cudaEventElapsedTime(&d2h, c->ev_h[0], c->ev_h[1]));
        r.ms_h2d = h2d;
        r.ms_d2h = d2h;
        if (res) *res = r;
    });
}

// ---- f4: test-matrix generators on the device (gen_f64.cuh) ---------------------------------
// gaussian_matrix(rows, cols, seed) (random.hpp:60-65) written straight into device memory; the
// words and uniforms are the reference's, log / sincos are the device's (a few ulp from glibc's).
int sorsvd_gaussian_matrix_device(sorsvd_ctx* c, int64_t rows, int64_t cols, uint64_t seed, double* dOut, int64_t ld) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (rows < 1 || cols < 1 || ld < cols) throw Error{SORSVD_ERR_SHAPE, "shape: matrix dimensions must be positive"};
        if (!dOut) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        const int64_t pairs = (rows * cols + 1) / 2;
        gaussian_fill_kernel<<<(unsigned)std::min<int64_t>(cdiv(pairs, 256), (int64_t)c->num_sms * 16), 256, 0, c->stream>>>(
            dOut, rows, cols, ld, seed, 1.0);
        check_launch(c);
    });
}

// The low-rank-plus-noise family of BASELINE.json's configs 1, 3 and 5, rows [row0, row0 + m) of the
// m_global x n matrix A = (x_scale X) diag(sigma) (y_scale Y)^T + noise_std E:
//   X = gaussian_matrix(m_global, r, sub_seed(seed, 1)), Y = gaussian_matrix(n, r, sub_seed(seed, 2))
//   (drawn on the host, bit-identical to the reference stream, and uploaded: (m + n) r values),
//   E's global row i = the first n normals of NormalStream(sub_seed(sub_seed(seed, 3), i)), drawn in
//   the kernel (m n values). Each rank of a row-sharded run generates its own block.
int sorsvd_gen_lowrank_device(sorsvd_ctx* c, int64_t m, int64_t n, int32_t r, const double* sigma, double x_scale,
                              double y_scale, double noise_std, uint64_t seed, int64_t row0, int64_t m_global,
                              int32_t dtype, void* dA, int64_t lda) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (m < 1 || n < 1 || r < 1 || lda < n || row0 < 0) throw Error{SORSVD_ERR_SHAPE, "shape: bad generator shape"};
        if (m_global <= 0) m_global = row0 + m;
        if (row0 + m > m_global) throw Error{SORSVD_ERR_SHAPE, "shape: row block outside the matrix"};
        if (!sigma || !dA) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        if (dtype != SORSVD_F64 && dtype != SORSVD_F32) throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown dtype"};
        std::vector<double> hx((size_t)m * r), hy((size_t)n * r);
        sorsvd_host::gaussian_fill_range(hx.data(), (uint64_t)row0 * r, (uint64_t)(row0 + m) * r,
                                         sorsvd_host::sub_seed(seed, 1), 0);
        sorsvd_host::gaussian_fill(hy.data(), (uint64_t)n * r, sorsvd_host::sub_seed(seed, 2), 0);
        for (double& v : hx) v *= x_scale;
        for (double& v : hy) v *= y_scale;
        double* X = dbuf(c, "gen_X", (size_t)m * r);
        double* Y = dbuf(c, "gen_Y", (size_t)n * r);
        double* S = dbuf(c, "gen_S", (size_t)r);
        CK(cudaMemcpyAsync(X, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(Y, hy.data(), hy.size() * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(S, sigma, (size_t)r * 8, cudaMemcpyHostToDevice, c->stream));
        const dim3 grid((unsigned)cdiv(n, 64), (unsigned)cdiv(m, 64));
        const uint64_t ns = sorsvd_host::sub_seed(seed, 3);
        if (dtype == SORSVD_F64)
            gen_lowrank_kernel<double><<<grid, kRpcaThreads, 0, c->stream>>>(static_cast<double*>(dA), lda, m, n, X, r, S,
                                                                            Y, r, r, noise_std, ns, row0);
        else
            gen_lowrank_kernel<float><<<grid, kRpcaThreads, 0, c->stream>>>(static_cast<float*>(dA), lda, m, n, X, r, S, Y,
                                                                           r, r, noise_std, ns, row0);
        check_launch(c);
        CK(cudaStreamSynchronize(c->stream));  // the host staging vectors go out of scope
    });
}

// gen_rpca_instance(n, r, s, seed) (matrixgen.hpp:99-124) assembled on the device: L = U V^T from the
// host-drawn n x r factors (streams 1, 2) on DMMA tiles, the sparse support by Floyd's sampling and the
// +-50 signs on the host (integer arithmetic, identical to the reference), scattered into S and X.
int sorsvd_gen_rpca_instance_device(sorsvd_ctx* c, int64_t n, int32_t r, long long s, uint64_t seed, double* dX,
                                    double* dL, double* dS) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (r < 1 || r >= n) throw Error{SORSVD_ERR_PARAMETER, "parameter: gen_rpca_instance needs 1 <= r < n"};
        const long long cells = (long long)n * n;
        if (s < 0 || s > cells) throw Error{SORSVD_ERR_PARAMETER, "parameter: sparse cardinality s out of [0, n^2]"};
        if (!dX) throw Error{SORSVD_ERR_PARAMETER, "parameter: null buffer"};
        std::vector<double> hu((size_t)n * r), hv((size_t)n * r), ones((size_t)r, 1.0), val;
        std::vector<long long> pos;
        sorsvd_host::gaussian_fill(hu.data(), hu.size(), sorsvd_host::sub_seed(seed, 1), 0);
        sorsvd_host::gaussian_fill(hv.data(), hv.size(), sorsvd_host::sub_seed(seed, 2), 0);
        sorsvd_host::rpca_support(cells, s, seed, pos, val);
        double* U = dbuf(c, "gen_X", (size_t)n * r);
        double* V = dbuf(c, "gen_Y", (size_t)n * r);
        double* S1 = dbuf(c, "gen_S", (size_t)r);
        auto* dpos = reinterpret_cast<long long*>(dbuf(c, "gen_pos", std::max<size_t>(pos.size(), 1)));
        double* dval = dbuf(c, "gen_val", std::max<size_t>(val.size(), 1));
        CK(cudaMemcpyAsync(U, hu.data(), hu.size() * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(V, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(S1, ones.data(), (size_t)r * 8, cudaMemcpyHostToDevice, c->stream));
        if (!pos.empty()) {
            CK(cudaMemcpyAsync(dpos, pos.data(), pos.size() * 8, cudaMemcpyHostToDevice, c->stream));
            CK(cudaMemcpyAsync(dval, val.data(), val.size() * 8, cudaMemcpyHostToDevice, c->stream));
        }
        const dim3 grid((unsigned)cdiv(n, 64), (unsigned)cdiv(n, 64));
        gen_lowrank_kernel<double><<<grid, kRpcaThreads, 0, c->stream>>>(dX, n, n, n, U, r, S1, V, r, r, 0.0, 0, 0);
        check_launch(c);
        if (dL) CK(cudaMemcpyAsync(dL, dX, (size_t)cells * 8, cudaMemcpyDeviceToDevice, c->stream));
        if (dS) CK(cudaMemsetAsync(dS, 0, (size_t)cells * 8, c->stream));
        if (!pos.empty()) {
            const unsigned blocks = (unsigned)std::min<int64_t>(cdiv((int64_t)pos.size(), 256), (int64_t)c->num_sms * 8);
            scatter_add_kernel<<<blocks, 256, 0, c->stream>>>(dX, n, n, dpos, dval, (int64_t)pos.size());
            check_launch(c);
            if (dS) {
                scatter_add_kernel<<<blocks, 256, 0, c->stream>>>(dS, n, n, dpos, dval, (int64_t)pos.size());
                check_launch(c);
            }
        }
        CK(cudaStreamSynchronize(c->stream));
    });
}

// Per-iteration telemetry of the context's last rpca_alm (iter, mu, rel_error,
// rank_l, nnz_s): up to cap_rows rows of 5 doubles into out, *rows = iterations available.
int sorsvd_rpca_telemetry(sorsvd_ctx* c, int32_t cap_rows, double* out, int32_t* rows) {
    if (!c || !rows) return SORSVD_ERR_PARAMETER;
    const int32_t n = (int32_t)(c->rpca_tele.size() / 4);
    *rows = n;
    if (out)
        for (int32_t i = 0; i < n && i < cap_rows; ++i) {
            out[5 * i] = (double)(i + 1);
            for (int q = 0; q < 4; ++q) out[5 * i + 1 + q] = c->rpca_tele[(size_t)4 * i + q];
        }
    return SORSVD_OK;
}

int sorsvd_measure_peaks(sorsvd_ctx* c, double* fp64_tflops, double* hbm_read_gbs) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        double* out = dbuf(c, "peak_out", 8);
        float best = 1e30f;
        const int iters = 4000, tpb = 256, grid = c->num_sms * 4;
        for (int r = 0; r < 4; ++r) {
            CK(cudaEventRecord(c->ev_a, c->stream));
            peak_dmma_kernel<<<grid, tpb, 0, c->stream>>>(out, iters);
            check_launch(c);
            CK(cudaEventRecord(c->ev_b, c->stream));
            CK(cudaEventSynchronize(c->ev_b));
            float ms;
            CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
            if (r > 0) best = std::min(best, ms);
        }
        const double flops = 2.0 * 8 * 8 * 4 * 4.0 * iters * (grid * tpb / 32);
        if (fp64_tflops) *fp64_tflops = flops / (best * 1e-3) / 1e12;
        const size_t bytes = (size_t)4 << 30;
        double* buf = dbuf(c, "peak_buf", bytes / 8);
        best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaEventRecord(c->ev_a, c->stream));
            peak_read_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(reinterpret_cast<const double2*>(buf), bytes / 16, out);
            check_launch(c);
            CK(cudaEventRecord(c->ev_b, c->stream));
            CK(cudaEventSynchronize(c->ev_b));
            float ms;
            CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
            if (r > 0) best = std::min(best, ms);
        }
        if (hbm_read_gbs) *hbm_read_gbs = bytes / (best * 1e-3) / 1e9;
        // release the 4 GiB probe buffer
        Buf& b = c->bufs["peak_buf"];
        CK(cudaFree(b.p));
        b.p = nullptr;
        b.bytes = 0;
    });
}

// One A-streaming pass (T = A X or T = A^T X) launched `reps` times between
// CUDA events on the context stream; X/T are padded (ldx = ldt = npad(ell)).
static int pass_device_impl(sorsvd_ctx* c, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell,
                            const double* dA, const float* dAf, const double* dX, double* dT, int32_t reps,
                            double* ms_avg, int32_t* launches_per_pass) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        const int Np = npad(ell);
        GemmCall g;
        g.ta = ta != 0;
        g.A = dA;
        g.Af = dAf;
        g.lda = lda;
        g.M = ta ? n : m;
        g.K = ta ? m : n;
        g.B = dX;
        g.ldb = Np;
        g.N = Np;
        g.C = dT;
        g.ldc = Np;
        g.sk_bias = Np <= 128 ? 1.0 : 0.95;  // as the sketch passes of enqueue_sor
        run_gemm(c, g, c->stream);  // warm-up (sizes the split workspace)
        const int l0 = c->launches;
        CK(cudaEventRecord(c->ev_a, c->stream));
        for (int r = 0; r < reps; ++r) run_gemm(c, g, c->stream);
        CK(cudaEventRecord(c->ev_b, c->stream));
        CK(cudaEventSynchronize(c->ev_b));
        float ms;
        CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
        if (ms_avg) *ms_avg = ms / std::max(reps, 1);
        if (launches_per_pass) *launches_per_pass = (c->launches - l0) / std::max(reps, 1);
    });
}

// Test hook: copy `count` doubles of the context workspace buffer `name` (e.g. "T1",
// "T2", "Q1", "Q2", "Mk") to dst, after the stream's work so far.
int sorsvd_debug_buffer(sorsvd_ctx* c, const char* name, double* dst, int64_t count) {
    if (!c || !name || !dst) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        auto it = c->bufs.find(name);
        if (it == c->bufs.end() || it->second.bytes < (size_t)count * 8)
            throw Error{SORSVD_ERR_PARAMETER, std::string("parameter: no workspace buffer ") + name};
        CK(cudaMemcpyAsync(dst, it->second.p, (size_t)count * 8, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

// The Ozaki scale exponents of A (tests): row_e[m] and col_e[n], e with max|.| < 2^e.
int sorsvd_ozaki_scales_device(sorsvd_ctx* c, int64_t m, int64_t n, int64_t lda, int32_t dtype, const void* dA,
                               int32_t* row_e, int32_t* col_e) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        SorProblem P{};
        P.dtype = dtype;
        P.A = dtype == SORSVD_F64 ? static_cast<const double*>(dA) : nullptr;
        P.Af = dtype == SORSVD_F32 ? static_cast<const float*>(dA) : nullptr;
        P.m = m;
        P.n = n;
        P.lda = lda;
        OzScales oz = oz_prepare_a(c, P, c->stream);
        CK(cudaMemcpyAsync(row_e, oz.row_e, (size_t)m * 4, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(col_e, oz.col_e, (size_t)n * 4, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

// One Ozaki (int8 tensor-core) pass C = op(A) X (kernel tests and the bench's
// roofline line): ms_avg = the pass (X digits + GEMM), ms_scales = the per-call
// scale read of A that the 2q+3 passes of a call share.
int sorsvd_pass_ozaki_device(sorsvd_ctx* c, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell, int32_t dtype,
                             const void* dA, const double* dX, double* dT, int32_t reps, double* ms_avg,
                             double* ms_scales) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        const int dbg = (dtype >> 8) & 15;  // kernel timing experiments (tools/oz_pass.py): bits 8-11 of dtype
        dtype &= 0xff;
        (void)dbg;
        if (dtype != SORSVD_F64 && dtype != SORSVD_F32) throw Error{SORSVD_ERR_PARAMETER, "parameter: unknown dtype"};
        SorProblem P{};
        P.dtype = dtype;
        P.A = dtype == SORSVD_F64 ? static_cast<const double*>(dA) : nullptr;
        P.Af = dtype == SORSVD_F32 ? static_cast<const float*>(dA) : nullptr;
        P.m = m;
        P.n = n;
        P.lda = lda;
        P.ell = ell;
        P.k = ell;
        P.Np = npad(ell);
        P.ozaki = true;
        P.oz_pm = oz_planes_rows(c, P);
        P.oz_planes = P.oz_pm > 0;
        CK(cudaEventRecord(c->ev_h[0], c->stream));
        OzScales oz = oz_prepare_a(c, P, c->stream);
        CK(cudaEventRecord(c->ev_h[1], c->stream));
        run_ozaki(c, P, ta != 0, oz, dX, dT, c->stream);  // warm-up
        CK(cudaEventRecord(c->ev_a, c->stream));
        for (int r = 0; r < reps; ++r)
            run_ozaki(c, P, ta != 0, oz, dX, dT, c->stream, dbg);
        CK(cudaEventRecord(c->ev_b, c->stream));
        CK(cudaEventSynchronize(c->ev_b));
        float ms = 0.f, msc = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
        CK(cudaEventElapsedTime(&msc, c->ev_h[0], c->ev_h[1]));
        if (ms_avg) *ms_avg = ms / std::max(reps, 1);
        if (ms_scales) *ms_scales = msc;
    });
}

int sorsvd_pass_device(sorsvd_ctx* c, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell, const double* dA,
                       const double* dX, double* dT, int32_t reps, double* ms_avg, int32_t* launches_per_pass) {
    return pass_device_impl(c, ta, m, n, lda, ell, dA, nullptr, dX, dT, reps, ms_avg, launches_per_pass);
}

int sorsvd_pass_f32a_device(sorsvd_ctx* c, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell,
                            const float* dA, const double* dX, double* dT, int32_t reps, double* ms_avg,
                            int32_t* launches_per_pass) {
    return pass_device_impl(c, ta, m, n, lda, ell, nullptr, dA, dX, dT, reps, ms_avg, launches_per_pass);
}

int sorsvd_matmul_f32_device(sorsvd_ctx* c, int32_t ta, int64_t M, int64_t K, int32_t N, const float* dA, int64_t lda,
                             const float* dB, int64_t ldb, float* dC, int64_t ldc) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        if (M < 1 || K < 1 || N < 1) throw Error{SORSVD_ERR_SHAPE, "shape: matmul dims must be positive"};
        const int Np = npad32(N);
        float* Bp = reinterpret_cast<float*>(dbuf(c, "mmBf", (size_t)K * Np / 2 + 1, true));
        float* Cp = reinterpret_cast<float*>(dbuf(c, "mmCf", (size_t)M * Np / 2 + 1));
        CK(cudaMemcpy2DAsync(Bp, (size_t)Np * 4, dB, (size_t)ldb * 4, (size_t)N * 4, (size_t)K,
                             cudaMemcpyDeviceToDevice, c->stream));
        run_tc_gemm(c, ta != 0, dA, lda, M, K, Bp, Np, Np, Cp, Np, c->stream);
        CK(cudaMemcpy2DAsync(dC, (size_t)ldc * 4, Cp, (size_t)Np * 4, (size_t)N * 4, (size_t)M,
                             cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sorsvd_pass_f32_device(sorsvd_ctx* c, int32_t ta, int64_t m, int64_t n, int64_t lda, int32_t ell, const float* dA,
                           const float* dX, float* dT, int32_t reps, double* ms_avg, int32_t* launches_per_pass) {
    if (!c) return SORSVD_ERR_PARAMETER;
    return guarded(c, [&] {
        const int Np = npad32(ell);
        const int64_t M = ta ? n : m, K = ta ? m : n;
        run_tc_gemm(c, ta != 0, dA, lda, M, K, dX, Np, Np, dT, Np, c->stream);  // warm-up
        const int l0 = c->launches;
        CK(cudaEventRecord(c->ev_a, c->stream));
        for (int r = 0; r < reps; ++r) run_tc_gemm(c, ta != 0, dA, lda, M, K, dX, Np, Np, dT, Np, c->stream);
        CK(cudaEventRecord(c->ev_b, c->stream));
        CK(cudaEventSynchronize(c->ev_b));
        float ms;
        CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
        if (ms_avg) *ms_avg = ms / std::max(reps, 1);
        if (launches_per_pass) *launches_per_pass = (c->launches - l0) / std::max(reps, 1);
    });
}

uint64_t sorsvd_sub_seed(uint64_t seed, uint64_t stream) { return sorsvd_host::sub_seed(seed, stream); }

int sorsvd_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out, int nthreads) {
    if (rows < 1 || cols < 1 || !out) {
        g_global_err = "shape: matrix dimensions must be positive";
        return SORSVD_ERR_SHAPE;
    }
    sorsvd_host::gaussian_fill(out, (uint64_t)rows * cols, seed, nthreads);
    return SORSVD_OK;
}

// Rows [row0, row0 + rows) of gaussian_matrix(., cols, seed): the stream is counter based, so a
// row block of a larger draw (a rank's rows of a sharded factor) needs no prefix.
int sorsvd_gaussian_rows(int64_t cols, int64_t row0, int64_t rows, uint64_t seed, double* out, int nthreads) {
    if (rows < 1 || cols < 1 || row0 < 0 || !out) {
        g_global_err = "shape: matrix dimensions must be positive";
        return SORSVD_ERR_SHAPE;
    }
    sorsvd_host::gaussian_fill_range(out, (uint64_t)row0 * cols, (uint64_t)(row0 + rows) * cols, seed, nthreads);
    return SORSVD_OK;
}

long long sorsvd_flop_estimate(long long m, long long n, long long ell, long long k, long long q, int variant) {
    const long long v = sorsvd_host::flop_estimate(m, n, ell, k, q, variant);
    if (v < 0) g_global_err = "parameter: flop_estimate requires positive dimensions and q >= 0";
    return v;
}

int sorsvd_validate_sketch(int64_t m, int64_t n, int32_t k, int32_t ell, int32_t q) {
    if (const char* e = sorsvd_host::validate_sketch(m, n, k, ell, q)) {
        g_global_err = e;
        return SORSVD_ERR_PARAMETER;
    }
    return SORSVD_OK;
}

}  // extern "C"
