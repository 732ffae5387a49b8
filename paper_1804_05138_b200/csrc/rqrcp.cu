// rqrcp.cu -- the C ABI (include/rqrcp.h) and the host driver of the RQRCP
// hot path (Alg. 2).  The driver only enqueues kernels on the
// context's stream (no host synchronisation inside the panel loop; pivots
// stay on the device) and synchronises once at the end for the status.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rqrcp.h"
#include "common.cuh"
#include "gemm_dmma.cuh"
#include "gemm_tma.cuh"
#include "misc.cuh"
#include "panel.cuh"
#include "panel_cl.cuh"
#include "philox.cuh"
#include "sample_qrcp.cuh"
#include "sample_qrcp_cl.cuh"
#include "sample_qrcp_reg.cuh"
#include "tri.cuh"
#include "cqr.cuh"
#include "dist.cuh"
#include "srqr.cuh"
#include "lowrank.cuh"

using namespace rq;

static inline int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

enum Phase { PH_OMEGA, PH_SKETCH, PH_SQRCP, PH_SWAP, PH_PANEL, PH_TRAIL, PH_SUPD, PH_COMM, PH_N };

struct rqrcp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // concurrent small kernels (tri_kernel)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // overlap of the bulk trailing update (rows i+bb..m) with the next panel's
    // sample QRCP: the update runs on `upd` (lowest priority), the main stream
    // (highest priority when ctx-owned) joins it before the next swap
    cudaStream_t upd = nullptr;
    cudaEvent_t ev_r12 = nullptr, ev_upd = nullptr;
    int grid_cap = 0;  // > 0: persistent GEMM grids use at most this many CTAs
    int *tctr = nullptr;  // per-panel tile counters of the dynamically scheduled bulk update
    bool own_stream = false;
    int nranks = 1, rank = 0;
    int64_t max_m = 0, max_n = 0;
    int max_b = 0, max_p = 0;
    int lpad_max = 0, bpad_max = 0;
    int64_t ldo = 0;  // leading dim of Omega^T and Vfull (= round8(max_m))
    int num_sms = 0;
    std::string err;
    // workspace
    double *omt = nullptr;     // Omega^T  ldo x lpad_max
    double *bs[2] = {nullptr, nullptr};  // samples lpad_max x max_n
    double *vfull = nullptr;   // ldo x bpad_max
    double *vt = nullptr;      // bpad_max x max_m
    double *w = nullptr, *w2 = nullptr;  // bpad_max x max_n
    double *tneg = nullptr, *rhat11 = nullptr, *omhat = nullptr, *ybuf = nullptr;  // bpad_max^2
    double *vhat = nullptr;    // lpad_max x bpad_max
    double *tauhat = nullptr;
    double *splitk = nullptr;
    int64_t splitk_elems = 0;
    SqHdr *slot_hdr = nullptr;
    int *slot_col = nullptr;
    unsigned launch_seq = 0;  // tags of the sample-QRCP candidate headers
    double *slot_v2 = nullptr, *slot_data = nullptr;
    uint4 *sq_ll = nullptr;  // tagged exchange slots of the register grid sample QRCP
    double *sq_spill = nullptr;  // transposed sample columns beyond shared memory (lpad_max x max_n)
    double *pn_part = nullptr, *pn_rowj = nullptr;
    // CholeskyQR2 + reconstruction panel (cqr.cuh): Gram, R factors, inverses
    double *cq_g = nullptr, *cq_rc = nullptr, *cq_rinv = nullptr, *cq_uinv = nullptr, *cq_lu = nullptr;
    int *cqr_status = nullptr;  // 0: the CholeskyQR2 path factored the panel; 1: Householder fallback
    bool cqr_enabled = true;
    double *swap_stage = nullptr;
    int64_t *swap_dst = nullptr, *swap_src = nullptr, *swap_jstage = nullptr;
    int *swap_np = nullptr;
    int64_t *perm = nullptr, *piv = nullptr;
    double *sumsq_part = nullptr;
    // device scalars: [0] status [1] bb_eff [2] done [3] rank
    int *iscal = nullptr;
    double *stop_tol2 = nullptr;
    unsigned *bars = nullptr;  // one grid-barrier counter per cooperative launch
    // updating formula 2 (Eq. (5)): the pre-QRCP sample, Omega-bar_1 R12, W for Q^T Omega^T
    int update_rule = 1;
    double *bpre = nullptr, *c5 = nullptr, *wom = nullptr, *w2om = nullptr;
    int64_t nbars = 0;
    // host-path buffer (lazily allocated)
    double *a_dev = nullptr;
    int64_t a_dev_elems = 0;
    int64_t *jpvt_dev = nullptr;
    double *tau_dev = nullptr;
    // cooperative limits
    int sq_max_grid = 0, pn_max_grid = 0;
    int sqc_max = 0;  // largest cluster the register-resident sample QRCP can use (0: none)
    int pnc_max = 0;  // ... and the register-resident cluster panel kernel
    // multi-GPU (nranks > 1): NCCL communicator + exchange buffers
    ncclComm_t comm = nullptr;
    double *gsend = nullptr, *gbuf = nullptr, *pack = nullptr, *r11 = nullptr;
    int64_t gbuf_elems = 0;
    int64_t *dl_cols = nullptr;  // device lists for the cross-rank column moves
    int *dl_slots = nullptr;
    int64_t *h_pairs = nullptr;  // pinned host copy of (dst, src) pairs + count
    // timing
    bool timing = true;
    cudaEvent_t ev[2 * 4096 + 8];
    int nev = 0;
    int open_phase = -1, open_ev = -1;
    std::vector<int> rec_phase, rec_s, rec_e;
    rqrcp_timings last{};
    int lt_t0 = -1, lt_t1 = -1;  // total-time events of the last factorization (read lazily)
    int *hstatus = nullptr;      // pinned host copy of the device status words
    int64_t launches = 0;
    bool debug_sync = false;  // RQRCP_DEBUG_SYNC=1: synchronise after every launch
    unsigned long long *trace = nullptr;  // RQRCP_TRACE=1: per-step phase stamps of the sample QRCP
    unsigned long long *ptrace = nullptr; // ... and of the panel kernel
    int ptrace_kind = 0;                  // 0: grid panel kernel, 1: cluster panel kernel
};

static const char *g_static_err = "no context";

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);            \
            return RQRCP_E_CUDA;                                                      \
        }                                                                             \
    } while (0)

#define CKL()                                                                         \
    do {                                                                              \
        cudaError_t e_ = cudaGetLastError();                                          \
        if (e_ == cudaSuccess && ctx->debug_sync) e_ = cudaStreamSynchronize(ctx->stream); \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string("kernel launch #") + std::to_string(ctx->launches) + \
                       " (line " + std::to_string(__LINE__) + "): " + cudaGetErrorString(e_); \
            return RQRCP_E_CUDA;                                                      \
        }                                                                             \
        ctx->launches++;                                                              \
    } while (0)

static constexpr int kDynSmemMax = 200 * 1024;
static constexpr int64_t kCqrMinRows = 8192;  // auto panel path: CholeskyQR2 from this many rows  // dynamic shared memory cap for cached kernels

static int grid_for(int64_t total, int threads, int num_sms) {
    int64_t g = (total + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms * 8));
}

// ---------------------------------------------------------------------------
// GEMM dispatch: C = X^T Y (see gemm_dmma.cuh), M small (skinny) or large.
// ---------------------------------------------------------------------------
template <int MT, int NT, int WM, int WN, int BK, int ST, int EPI>
static int launch_tn_cfg(rqrcp_ctx *ctx, GemmArgs g, int splits) {
    constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
    const size_t smem = (size_t)ST * BK * (BM + BN) * sizeof(double);
    auto kern = gemm_tn_kernel<MT, NT, WM, WN, BK, ST, EPI>;
    static bool attr_set = false;
    if (!attr_set) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
    }
    dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM), (unsigned)splits);
    kern<<<grid, WM * WN * 32, smem, ctx->stream>>>(g);
    CKL();
    return 0;
}

template <int MT, int NT, int WM, int WN>
static int launch_skinny(rqrcp_ctx *ctx, int64_t M, int64_t N, int64_t K, const double *X, int64_t ldx,
                         const double *Y, int64_t ldy, double *C, int64_t ldc) {
    constexpr int BK = 32, ST = 3;
    constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
    const int64_t tiles = ((N + BN - 1) / BN) * ((M + BM - 1) / BM);
    int64_t splits = std::max<int64_t>(1, (2 * (int64_t)ctx->num_sms + tiles - 1) / tiles);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / 256));
    while (splits > 1 && splits * M * N > ctx->splitk_elems) --splits;
    int64_t kps = rup((K + splits - 1) / splits, BK);
    splits = (K + kps - 1) / kps;
    GemmArgs g{M, N, K, X, ldx, Y, ldy, C, ldc, kps, M * N};
    if (splits <= 1) {
        g.k_per_split = rup(std::max<int64_t>(K, 1), BK);
        return launch_tn_cfg<MT, NT, WM, WN, BK, ST, EPI_STORE>(ctx, g, 1);
    }
    g.C = ctx->splitk;
    int rc = launch_tn_cfg<MT, NT, WM, WN, BK, ST, EPI_PARTIAL>(ctx, g, (int)splits);
    if (rc) return rc;
    splitk_reduce_kernel<<<grid_for(M * N, 256, ctx->num_sms), 256, 0, ctx->stream>>>(ctx->splitk, M, N, (int)splits,
                                                                                      M * N, C, ldc);
    CKL();
    return 0;
}

// C (M x N) = X^T Y with M <= 144 rows (sample rows l_pad or panel width).
static int gemm_skinny(rqrcp_ctx *ctx, int64_t M, int64_t N, int64_t K, const double *X, int64_t ldx,
                       const double *Y, int64_t ldy, double *C, int64_t ldc) {
    if (M <= 32) return launch_skinny<4, 2, 1, 4>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc);
    if (M <= 40) return launch_skinny<5, 2, 1, 4>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc);
    if (M <= 64) return launch_skinny<4, 4, 2, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc);
    if (M <= 80) return launch_skinny<5, 4, 2, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc);
    if (M <= 128) return launch_skinny<4, 4, 4, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc);
    if (M <= 144) return launch_skinny<6, 4, 3, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc);
    return launch_skinny<4, 4, 4, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc);  // grid.y tiles M
}

// A22 (rows x cols, lda) += V W2 as (A22^T)(cols x rows) += W2^T Vt.
static int gemm_update(rqrcp_ctx *ctx, int64_t rows, int64_t cols, int64_t K, const double *w2, int64_t ldw,
                       const double *vt, int64_t ldvt, double *A22, int64_t lda) {
    if (rows <= 0 || cols <= 0) return 0;
    GemmArgs g{cols, rows, K, w2, ldw, vt, ldvt, A22, lda, rup(K, 32), 0};
    return launch_tn_cfg<4, 4, 2, 4, 32, 2, EPI_ACCUM_T>(ctx, g, 1);
}

// ---------------------------------------------------------------------------
// TMA-fed persistent DMMA kernels (gemm_tma.cuh).  Used when every operand's
// row stride is a multiple of 16 bytes (TMA requirement); otherwise the
// cp.async kernels above.
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 2-D map over a column-major matrix (dim0 = rows = K direction, contiguous),
// box {8 doubles, box1 columns}; out-of-range elements read as zero.
static bool make_tmap(CUtensorMap *m, const double *base, int64_t dim0, int64_t dim1, int64_t ld, int box1) {
    auto enc = tma_encode_fn();
    if (!enc && getenv("RQRCP_DEBUG_TMA")) fprintf(stderr, "[rqrcp] no cuTensorMapEncodeTiled entry point\n");
    if (!enc || ((uintptr_t)base & 15) || ((ld * 8) & 15) || dim0 < 1 || dim1 < 1) return false;
    cuuint64_t dims[2] = {(cuuint64_t)dim0, (cuuint64_t)dim1};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {8, (cuuint32_t)box1};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    static bool warned = false;
    if (r != CUDA_SUCCESS && !warned && getenv("RQRCP_DEBUG_TMA")) {
        fprintf(stderr, "[rqrcp] cuTensorMapEncodeTiled failed (%d): cp.async GEMM path\n", (int)r);
        warned = true;
    }
    return r == CUDA_SUCCESS;
}

// splits minimising ceil(T*S / grid) / S (persistent-grid wave quantisation)
static int choose_splits(int64_t tiles, int64_t K, int grid, int64_t max_elems_per_split, int64_t partial_cap,
                         int64_t kmin = 512) {
    int64_t smax = std::max<int64_t>(1, K / kmin);
    if (max_elems_per_split > 0) smax = std::min<int64_t>(smax, std::max<int64_t>(1, partial_cap / max_elems_per_split));
    int best = 1;
    double best_t = 1e30;
    for (int64_t s = 1; s <= std::min<int64_t>(smax, 64); ++s) {
        const double t = (double)((tiles * s + grid - 1) / grid) / (double)s + 0.002 * s;  // small per-split cost
        if (t < best_t - 1e-12) { best_t = t; best = (int)s; }
    }
    return best;
}

template <int MT, int NT, int WM, int WN, int EPI, bool DYN = false>
static int launch_tma_cfg(rqrcp_ctx *ctx, const double *X, int64_t xdim0, int64_t xdim1, int64_t ldx, const double *Y,
                          int64_t ydim0, int64_t ydim1, int64_t ldy, TmaGemmArgs g, bool *done) {
    constexpr int BK = 32;
    constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
    constexpr int ST = (4 * BK * (BM + BN) * 8 <= 216 * 1024) ? 4 : 3;
    *done = false;
    // TMA needs the box's inner (K) start offset 16-byte aligned: even
    // element coordinates for fp64 (an odd panel offset i falls back)
    if ((g.xk0 | g.yk0) & 1) return 0;
    CUtensorMap tx, ty;
    if (!make_tmap(&tx, X, xdim0, xdim1, ldx, BM) || !make_tmap(&ty, Y, ydim0, ydim1, ldy, BN)) return 0;
    const size_t smem = tma_gemm_smem<MT, NT, WM, WN, BK, ST>();
    auto kern = gemm_tma_kernel<MT, NT, WM, WN, BK, ST, EPI, DYN>;
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int64_t tiles = ((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM) * g.splits;
    const int grid = (int)std::min<int64_t>(tiles, ctx->grid_cap > 0 ? ctx->grid_cap : ctx->num_sms);
    kern<<<grid, WM * WN * 32, smem, ctx->stream>>>(tx, ty, g);
    CKL();
    *done = true;
    return 0;
}

// C (M x N, ldc) = X^T Y, X = tensor (xdim0 x xdim1, ldx) from coords (xk0, xm0),
// Y likewise; skinny M <= 144.  Returns 0 and sets *done when launched.
template <int MT, int NT, int WM, int WN>
static int tma_skinny_cfg(rqrcp_ctx *ctx, int64_t M, int64_t N, int64_t K, const double *X, int64_t xdim0,
                          int64_t xdim1, int64_t ldx, int64_t xk0, int64_t xm0, const double *Y, int64_t ydim0,
                          int64_t ydim1, int64_t ldy, int64_t yk0, int64_t yn0, double *C, int64_t ldc, bool *done,
                          int64_t kmin) {
    constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
    const int64_t tiles = ((N + BN - 1) / BN) * ((M + BM - 1) / BM);
    int splits = choose_splits(tiles, K, ctx->num_sms, M * N, ctx->splitk_elems, kmin);
    int64_t kps = rup((K + splits - 1) / splits, 32);
    splits = (int)((K + kps - 1) / kps);
    TmaGemmArgs g{M, N, K, xk0, xm0, yk0, yn0, C, ldc, kps, splits, M * N, 0};
    if (splits <= 1) return launch_tma_cfg<MT, NT, WM, WN, EPI_STORE>(ctx, X, xdim0, xdim1, ldx, Y, ydim0, ydim1, ldy, g, done);
    g.C = ctx->splitk;
    int rc = launch_tma_cfg<MT, NT, WM, WN, EPI_PARTIAL>(ctx, X, xdim0, xdim1, ldx, Y, ydim0, ydim1, ldy, g, done);
    if (rc || !*done) return rc;
    splitk_reduce_kernel<<<grid_for(M * N, 256, ctx->num_sms), 256, 0, ctx->stream>>>(ctx->splitk, M, N, splits, M * N,
                                                                                      C, ldc);
    CKL();
    return 0;
}

static int tma_skinny(rqrcp_ctx *ctx, int64_t M, int64_t N, int64_t K, const double *X, int64_t xdim0, int64_t xdim1,
                      int64_t ldx, int64_t xk0, int64_t xm0, const double *Y, int64_t ydim0, int64_t ydim1, int64_t ldy,
                      int64_t yk0, int64_t yn0, double *C, int64_t ldc, bool *done, int64_t kmin = 512) {
    *done = false;
    if (M <= 32) return tma_skinny_cfg<4, 4, 1, 8>(ctx, M, N, K, X, xdim0, xdim1, ldx, xk0, xm0, Y, ydim0, ydim1, ldy, yk0, yn0, C, ldc, done, kmin);
    if (M <= 40) return tma_skinny_cfg<5, 4, 1, 8>(ctx, M, N, K, X, xdim0, xdim1, ldx, xk0, xm0, Y, ydim0, ydim1, ldy, yk0, yn0, C, ldc, done, kmin);
    if (M <= 64) return tma_skinny_cfg<4, 4, 2, 4>(ctx, M, N, K, X, xdim0, xdim1, ldx, xk0, xm0, Y, ydim0, ydim1, ldy, yk0, yn0, C, ldc, done, kmin);
    if (M <= 80) return tma_skinny_cfg<5, 4, 2, 4>(ctx, M, N, K, X, xdim0, xdim1, ldx, xk0, xm0, Y, ydim0, ydim1, ldy, yk0, yn0, C, ldc, done, kmin);
    if (M <= 128) return tma_skinny_cfg<4, 4, 4, 2>(ctx, M, N, K, X, xdim0, xdim1, ldx, xk0, xm0, Y, ydim0, ydim1, ldy, yk0, yn0, C, ldc, done, kmin);
    if (M <= 144) return tma_skinny_cfg<6, 4, 3, 2>(ctx, M, N, K, X, xdim0, xdim1, ldx, xk0, xm0, Y, ydim0, ydim1, ldy, yk0, yn0, C, ldc, done, kmin);
    return 0;
}

// A22 (rows x cols, lda) += V W2  as  A22^T += W2^T Vt  (TMA operands W2, Vt).
// For K > 64 the C tile is moved by TMA as well (gemm_upd_tma_kernel; needs a
// 16-byte aligned A22 with an even lda); else the register-epilogue kernel.
static int tma_update(rqrcp_ctx *ctx, int64_t rows, int64_t cols, int64_t K, const double *w2, int64_t ldw,
                      const double *vt, int64_t ldvt, double *A22, int64_t lda, bool *done, int *tile_ctr = nullptr) {
    *done = false;
    if (rows <= 0 || cols <= 0) { *done = true; return 0; }
    // (measured: faster for K = 128, slower for K = 64 where the two-stage
    // operand ring is too shallow)
    if (K > 64 && !tile_ctr && (((uintptr_t)A22 & 15) == 0) && ((lda & 1) == 0)) {
        constexpr int MT = 4, NT = 4, WM = 2, WN = 4, BK = 32, ST = 2;
        constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
        CUtensorMap tx, ty, tc;
        if (make_tmap(&tx, w2, K, cols, ldw, BM) && make_tmap(&ty, vt, K, rows, ldvt, BN) &&
            make_tmap(&tc, A22, rows, cols, lda, BM)) {
            const size_t smem = tma_upd_smem<MT, NT, WM, WN, BK, ST>();
            auto kern = gemm_upd_tma_kernel<MT, NT, WM, WN, BK, ST>;
            static bool attr = false;
            if (!attr) {
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                attr = true;
            }
            TmaGemmArgs g{cols, rows, K, 0, 0, 0, 0, A22, lda, rup(K, 32), 1, 0, 0};
            const int64_t tiles = ((rows + BN - 1) / BN) * ((cols + BM - 1) / BM);
            const int grid = (int)std::min<int64_t>(tiles, ctx->grid_cap > 0 ? ctx->grid_cap : ctx->num_sms);
            kern<<<grid, WM * WN * 32, smem, ctx->stream>>>(tx, ty, tc, g);
            CKL();
            *done = true;
            return 0;
        }
    }
    if ((lda & 1) || ((uintptr_t)A22 & 7)) return 0;
    TmaGemmArgs g{cols, rows, K, 0, 0, 0, 0, A22, lda, rup(K, 32), 1, 0,
                  (((uintptr_t)A22 & 15) == 0 && (lda & 1) == 0) ? 1 : 0};
    // a short update (the R12 rows of the overlapped schedule): 32 x 64 tiles,
    // twice as many CTAs; same per-element DMMA sequence (same bits)
    if (rows <= 64) return launch_tma_cfg<2, 4, 2, 2, EPI_ACCUM_T_PRE>(ctx, w2, K, cols, ldw, vt, K, rows, ldvt, g, done);
    if (tile_ctr) {  // dynamic tile claiming (the GPU is shared with a concurrent kernel)
        g.tile_ctr = tile_ctr;
        return launch_tma_cfg<4, 4, 2, 4, EPI_ACCUM_T_PRE, true>(ctx, w2, K, cols, ldw, vt, K, rows, ldvt, g, done);
    }
    return launch_tma_cfg<4, 4, 2, 4, EPI_ACCUM_T_PRE>(ctx, w2, K, cols, ldw, vt, K, rows, ldvt, g, done);
}

// ---------------------------------------------------------------------------
// timing helpers
// ---------------------------------------------------------------------------
static constexpr int kMaxEv = 2 * 4096 + 8;
static void ph_begin(rqrcp_ctx *ctx, int phase) {
    ctx->open_phase = -1;
    // phase events are always recorded (measured: the schedule runs faster with
    // them than without, 4.31 vs 4.58 ms at C2); rqrcp_set_timing(ctx, 0) only
    // turns their reading off
    if (ctx->nev + 3 > kMaxEv) return;
    ctx->open_phase = phase;
    ctx->open_ev = ctx->nev;
    cudaEventRecord(ctx->ev[ctx->nev++], ctx->stream);
}
static void ph_end(rqrcp_ctx *ctx) {
    if (ctx->open_phase < 0) return;
    ctx->rec_phase.push_back(ctx->open_phase);
    ctx->rec_s.push_back(ctx->open_ev);
    ctx->rec_e.push_back(ctx->nev);
    cudaEventRecord(ctx->ev[ctx->nev++], ctx->stream);
    ctx->open_phase = -1;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" const char *rqrcp_version(void) { return "rqrcp-b200 0.1 (sm_100a, fp64 DMMA)"; }

extern "C" const char *rqrcp_last_error(const rqrcp_ctx *ctx) { return ctx ? ctx->err.c_str() : g_static_err; }

extern "C" int rqrcp_flops(int64_t m, int64_t n, int64_t k, int b, int p, double out[4]) {
    if (m < 1) return -1;
    if (n < 1) return -2;
    if (k < 1 || k > std::min(m, n)) return -3;
    if (b < 1) return -4;
    if (p < 0 || (int64_t)b + p > m) return -5;
    if (!out) return -6;
    const double l = (double)b + p;
    out[0] = 2.0 * l * (double)m * (double)n;
    double qr = 0.0, sq = 0.0, su = 0.0;
    for (int64_t j = 0; j < k; ++j) qr += 4.0 * (double)(m - j) * (double)(n - j);
    for (int64_t i = 0; i < k; i += b) {
        const int64_t bb = std::min<int64_t>(b, k - i);
        for (int64_t j = 0; j < bb; ++j) sq += 4.0 * (l - j) * (double)(n - i - j);
        su += 2.0 * (double)bb * bb * (double)(n - i - bb);
    }
    out[1] = qr;
    out[2] = sq;
    out[3] = su;
    return 0;
}

static int free_all(rqrcp_ctx *ctx) {
    if (ctx->comm && nccl().ok) nccl().CommDestroy(ctx->comm);
    ctx->comm = nullptr;
    for (void *q : {(void *)ctx->gsend, (void *)ctx->gbuf, (void *)ctx->pack, (void *)ctx->r11, (void *)ctx->dl_cols,
                    (void *)ctx->dl_slots})
        if (q) cudaFree(q);
    if (ctx->h_pairs) cudaFreeHost(ctx->h_pairs);
    if (ctx->hstatus) cudaFreeHost(ctx->hstatus);
    ctx->hstatus = nullptr;
    if (ctx->tctr) cudaFree(ctx->tctr);
    ctx->tctr = nullptr;
    void *ptrs[] = {ctx->omt,     ctx->bs[0],   ctx->bs[1],     ctx->vfull,     ctx->vt,        ctx->w,
                    ctx->w2,      ctx->tneg, ctx->ybuf,   ctx->rhat11,    ctx->omhat,     ctx->vhat,      ctx->tauhat,
                    ctx->splitk,  ctx->slot_hdr, ctx->slot_col, ctx->slot_v2,
                    ctx->slot_data, ctx->sq_ll, ctx->sq_spill, ctx->pn_part, ctx->pn_rowj, ctx->cq_g, ctx->cq_rc, ctx->cq_rinv, ctx->cq_uinv, ctx->cq_lu, ctx->cqr_status, ctx->bpre, ctx->c5, ctx->wom, ctx->w2om,   ctx->swap_stage,
                    ctx->swap_dst, ctx->swap_src, ctx->swap_jstage, ctx->swap_np, ctx->perm,     ctx->piv,       ctx->sumsq_part,
                    ctx->iscal,   ctx->stop_tol2, ctx->bars,  ctx->trace, ctx->ptrace,    ctx->a_dev,     ctx->jpvt_dev,  ctx->tau_dev};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    return 0;
}

extern "C" int rqrcp_create(rqrcp_ctx **out, const rqrcp_config *cfg) {
    if (!out) return -1;
    *out = nullptr;
    if (!cfg || cfg->max_m < 1 || cfg->max_n < 1 || cfg->max_b < 1 || cfg->max_b > 128 || cfg->max_p < 0 ||
        cfg->max_b + cfg->max_p > SQ_MAXL || cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks)
        return -2;
    if (cfg->nranks > 1 && !nccl().ok) return RQRCP_E_UNSUPPORTED;
    rqrcp_ctx *ctx = new rqrcp_ctx();
    ctx->device = cfg->device;
    ctx->nranks = cfg->nranks;
    ctx->rank = cfg->rank;
    ctx->max_m = cfg->max_m;
    ctx->max_n = cfg->max_n;
    ctx->max_b = cfg->max_b;
    ctx->max_p = cfg->max_p;
    {
        const char *d = getenv("RQRCP_DEBUG_SYNC");
        ctx->debug_sync = d && d[0] == '1';
    }
    const char *tr = getenv("RQRCP_TRACE");
    const bool want_trace = tr && tr[0] == '1';
    auto fail = [&](int code) {
        free_all(ctx);
        int rc = code;
        delete ctx;
        return rc;
    };
#define CKC(call)                                                                 \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            fprintf(stderr, "rqrcp_create: %s: %s\n", #call, cudaGetErrorString(e_)); \
            return fail(e_ == cudaErrorMemoryAllocation ? RQRCP_E_WORKSPACE : RQRCP_E_CUDA); \
        }                                                                         \
    } while (0)
    CKC(cudaSetDevice(ctx->device));
    CKC(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    if (cfg->stream) {
        ctx->stream = (cudaStream_t)cfg->stream;
    } else {
        int prio_lo = 0, prio_hi = 0;
        CKC(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        CKC(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, prio_hi));
        ctx->own_stream = true;
    }
    ctx->lpad_max = (int)rup(cfg->max_b + cfg->max_p, 8);
    ctx->bpad_max = (int)rup(cfg->max_b, 8);
    ctx->ldo = rup(cfg->max_m, 8);
    const int64_t lp = ctx->lpad_max, bp = ctx->bpad_max, mm = cfg->max_m, nn = cfg->max_n;
    const int G = ctx->num_sms;
    auto dalloc = [&](double **p, int64_t n) { return cudaMalloc((void **)p, sizeof(double) * std::max<int64_t>(n, 1)); };
    CKC(dalloc(&ctx->omt, ctx->ldo * lp));
    CKC(dalloc(&ctx->bs[0], lp * nn));
    CKC(dalloc(&ctx->bs[1], lp * nn));
    CKC(dalloc(&ctx->vfull, ctx->ldo * bp));
    CKC(dalloc(&ctx->vt, bp * mm));
    CKC(dalloc(&ctx->w, bp * nn));
    CKC(dalloc(&ctx->w2, bp * nn));
    CKC(dalloc(&ctx->tneg, bp * bp));
    CKC(dalloc(&ctx->rhat11, bp * bp));
    CKC(dalloc(&ctx->ybuf, bp * bp));
    CKC(dalloc(&ctx->omhat, bp * bp));
    CKC(dalloc(&ctx->vhat, lp * bp));
    CKC(dalloc(&ctx->tauhat, bp));
    ctx->splitk_elems = std::max<int64_t>(4 << 20, 0);
    CKC(dalloc(&ctx->splitk, ctx->splitk_elems));
    CKC(cudaMalloc((void **)&ctx->slot_hdr, sizeof(SqHdr) * 2 * SQ_MAXG * 8));
    CKC(cudaMemset(ctx->slot_hdr, 0, sizeof(SqHdr) * 2 * SQ_MAXG * 8));
    CKC(cudaMalloc((void **)&ctx->slot_col, sizeof(int) * 2 * G));
    CKC(dalloc(&ctx->slot_v2, 2 * G));
    CKC(dalloc(&ctx->slot_data, 2 * G * lp));
    CKC(cudaMalloc((void **)&ctx->sq_ll, sizeof(uint4) * 2 * SQ_MAXG * (SQ_MAXL + 2)));
    CKC(cudaMemset(ctx->sq_ll, 0, sizeof(uint4) * 2 * SQ_MAXG * (SQ_MAXL + 2)));
    CKC(dalloc(&ctx->sq_spill, lp * nn));
    CKC(dalloc(&ctx->bpre, lp * nn));
    CKC(dalloc(&ctx->c5, lp * nn));
    CKC(dalloc(&ctx->wom, bp * lp));
    CKC(dalloc(&ctx->w2om, bp * lp));
    CKC(dalloc(&ctx->pn_part, 2 * G * bp));
    CKC(dalloc(&ctx->pn_rowj, 2 * bp));
    for (double **q : {&ctx->cq_g, &ctx->cq_rc, &ctx->cq_rinv, &ctx->cq_uinv, &ctx->cq_lu}) CKC(dalloc(q, bp * bp));
    CKC(cudaMalloc((void **)&ctx->cqr_status, sizeof(int)));
    CKC(cudaMemset(ctx->cqr_status, 0xff, sizeof(int)));
    CKC(cudaFuncSetAttribute(cqr_chol_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (128 * 128 + 64 * 64) * 8));
    CKC(cudaFuncSetAttribute(cqr_chol_kernel<CQR_EPT_U>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (128 * 128 + 64 * 64) * 8));
    CKC(cudaFuncSetAttribute(cqr_recon_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (128 * 128 + 64 * 64) * 8));
    CKC(cudaFuncSetAttribute(cqr_recon_kernel<CQR_EPT_F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (128 * 128 + 64 * 64) * 8));
    CKC(cudaFuncSetAttribute(cqr_rowmul_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 132 * 8));
    CKC(dalloc(&ctx->swap_stage, 2 * bp * mm));
    CKC(cudaMalloc((void **)&ctx->swap_dst, sizeof(int64_t) * 2 * bp));
    CKC(cudaMalloc((void **)&ctx->swap_src, sizeof(int64_t) * 2 * bp));
    CKC(cudaMalloc((void **)&ctx->swap_jstage, sizeof(int64_t) * 2 * bp));
    CKC(cudaMalloc((void **)&ctx->swap_np, sizeof(int)));
    CKC(cudaMalloc((void **)&ctx->perm, sizeof(int64_t) * nn));
    CKC(cudaMalloc((void **)&ctx->piv, sizeof(int64_t) * bp));
    CKC(dalloc(&ctx->sumsq_part, 4 * G));
    CKC(cudaMalloc((void **)&ctx->iscal, sizeof(int) * 8));
    CKC(dalloc(&ctx->stop_tol2, 1));
    ctx->nbars = 2 * std::min(cfg->max_m, cfg->max_n) + 16;
    CKC(cudaMalloc((void **)&ctx->bars, sizeof(unsigned) * ctx->nbars));
    CKC(cudaMemset(ctx->bars, 0, sizeof(unsigned) * ctx->nbars));
    CKC(cudaMemset(ctx->tneg, 0, sizeof(double) * bp * bp));
    CKC(cudaFuncSetAttribute(sample_qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemMax));
    CKC(cudaFuncSetAttribute(panel_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemMax));
    CKC(cudaFuncSetAttribute(sample_qrcp_reg_kernel<40, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 40 * 8));
    CKC(cudaFuncSetAttribute(sample_qrcp_reg_kernel<74, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 74 * 8));
    CKC(cudaFuncSetAttribute(sample_qrcp_reg_kernel<72, 72>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 144 * 8));
    CKC(cudaFuncSetAttribute(sample_qrcp_cluster_kernel<40>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CKC(cudaFuncSetAttribute(sample_qrcp_cluster_kernel<40>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 40 * 8));
    CKC(cudaFuncSetAttribute(sample_qrcp_cluster_kernel<74>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CKC(cudaFuncSetAttribute(sample_qrcp_cluster_kernel<74>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 74 * 8));
    CKC(cudaFuncSetAttribute(sample_qrcp_cluster_kernel<80>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CKC(cudaFuncSetAttribute(sample_qrcp_cluster_kernel<80>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 80 * 8));
    {
        ctx->sqc_max = 0;
        for (int cs = SQC_MAXG; cs >= 1 && !ctx->sqc_max; --cs) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(cs);
            lc.blockDim = dim3(SQC_THREADS);
            lc.dynamicSmemBytes = 64 * 80 * 8;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, (void *)sample_qrcp_cluster_kernel<80>, &lc) == cudaSuccess &&
                ncl >= 1)
                ctx->sqc_max = cs;
        }
        cudaGetLastError();
    }
    CKC(cudaFuncSetAttribute(panel_qr_cluster_kernel<32, 64>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CKC(cudaFuncSetAttribute(panel_qr_cluster_kernel<64, 64>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CKC(cudaFuncSetAttribute(panel_qr_cluster_kernel<64, 32, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CKC(cudaFuncSetAttribute(panel_qr_cluster_kernel<32, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 65 * 8));
    CKC(cudaFuncSetAttribute(panel_qr_cluster_kernel<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 65 * 8));
    CKC(cudaFuncSetAttribute(panel_qr_cluster_kernel<64, 32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 64 * 8));
    {
        ctx->pnc_max = 0;
        for (int cs = PNC_MAXG; cs >= 1 && !ctx->pnc_max; --cs) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(cs);
            lc.blockDim = dim3(PNC_THREADS);
            lc.dynamicSmemBytes = 64 * 65 * 8;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, (void *)panel_qr_cluster_kernel<64, 64>, &lc) == cudaSuccess &&
                ncl >= 1)
                ctx->pnc_max = cs;
        }
        cudaGetLastError();
    }
    CKC(cudaFuncSetAttribute(tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (128 * 128 + 64 * 64) * 8));
    CKC(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CKC(cudaMallocHost((void **)&ctx->hstatus, sizeof(int) * 8));
    CKC(cudaMalloc((void **)&ctx->tctr, sizeof(int) * 8192));
    {
        int prio_lo = 0, prio_hi = 0;
        CKC(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        CKC(cudaStreamCreateWithPriority(&ctx->upd, cudaStreamNonBlocking, prio_lo));
    }
    CKC(cudaEventCreateWithFlags(&ctx->ev_r12, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_upd, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    for (auto &e : ctx->ev) CKC(cudaEventCreate(&e));
    if (ctx->nranks > 1) {
        const int P = ctx->nranks;
        CKC(dalloc(&ctx->gsend, lp * (nn + bp)));
        ctx->gbuf_elems = lp * (nn + (int64_t)P * bp);
        CKC(dalloc(&ctx->gbuf, ctx->gbuf_elems));
        CKC(dalloc(&ctx->pack, bp + 3 * bp * bp + 1));
        CKC(cudaMalloc((void **)&ctx->dl_cols, sizeof(int64_t) * 4 * bp));
        CKC(cudaMalloc((void **)&ctx->dl_slots, sizeof(int) * 4 * bp));
        CKC(cudaMallocHost((void **)&ctx->h_pairs, sizeof(int64_t) * (4 * bp + 2 + 8 * bp)));
        ncclUniqueId uid;
        memcpy(uid.internal, cfg->nccl_uid, sizeof(uid.internal));
        if (nccl().CommInitRank(&ctx->comm, P, uid, ctx->rank) != 0) {
            fprintf(stderr, "rqrcp_create: ncclCommInitRank failed\n");
            return fail(RQRCP_E_NCCL);
        }
    }
    if (want_trace) {
        CKC(cudaMalloc((void **)&ctx->trace, sizeof(unsigned long long) * SQ_MAXG * 64 * 4));
        CKC(cudaMemset(ctx->trace, 0, sizeof(unsigned long long) * SQ_MAXG * 64 * 4));
        CKC(cudaMalloc((void **)&ctx->ptrace, sizeof(unsigned long long) * 2 * 64 * 8));
        CKC(cudaMemset(ctx->ptrace, 0, sizeof(unsigned long long) * 2 * 64 * 8));
    }
#undef CKC
    *out = ctx;
    return 0;
}

extern "C" int rqrcp_destroy(rqrcp_ctx *ctx) {
    if (!ctx) return 0;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    free_all(ctx);
    for (auto &e : ctx->ev) cudaEventDestroy(e);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->upd) cudaStreamDestroy(ctx->upd);
    if (ctx->ev_r12) cudaEventDestroy(ctx->ev_r12);
    if (ctx->ev_upd) cudaEventDestroy(ctx->ev_upd);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return 0;
}

extern "C" int64_t rqrcp_shard_columns(int64_t n, int b, int nranks, int rank) {
    if (n < 0) return -1;
    if (b < 1) return -2;
    if (nranks < 1) return -3;
    if (rank < 0 || rank >= nranks) return -4;
    return dist_count(n, b, nranks, rank);
}

extern "C" int64_t rqrcp_shard_global_index(int64_t local_index, int b, int nranks, int rank) {
    if (local_index < 0) return -1;
    if (b < 1) return -2;
    if (nranks < 1) return -3;
    if (rank < 0 || rank >= nranks) return -4;
    return dist_global(local_index, b, nranks, rank);
}

extern "C" int rqrcp_nccl_unique_id(uint8_t *out) {
    if (!out) return -1;
    if (!nccl().ok) return RQRCP_E_UNSUPPORTED;
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != 0) return RQRCP_E_NCCL;
    memcpy(out, id.internal, sizeof(id.internal));
    return 0;
}

extern "C" int rqrcp_set_update_rule(rqrcp_ctx *ctx, int rule) {
    if (!ctx) return -1;
    if (rule != 1 && rule != 2) return -2;
    ctx->update_rule = rule;
    return 0;
}

extern "C" int rqrcp_set_timing(rqrcp_ctx *ctx, int enabled) {
    if (!ctx) return -1;
    ctx->timing = enabled != 0;
    return 0;
}

extern "C" int rqrcp_get_timings(const rqrcp_ctx *ctx, rqrcp_timings *out) {
    if (!ctx) return -1;
    if (!out) return -2;
    rqrcp_timings t = ctx->last;
    if (ctx->lt_t0 >= 0 && ctx->lt_t1 >= 0) {  // the last factorization's events (complete: it synchronized)
        float ms = 0;
        cudaEventElapsedTime(&ms, ctx->ev[ctx->lt_t0], ctx->ev[ctx->lt_t1]);
        t.total_ms = ms;
        double acc[PH_N] = {0};
        for (size_t q = 0; q < ctx->rec_phase.size(); ++q) {
            float x = 0;
            cudaEventElapsedTime(&x, ctx->ev[ctx->rec_s[q]], ctx->ev[ctx->rec_e[q]]);
            acc[ctx->rec_phase[q]] += x;
        }
        t.omega_ms = acc[PH_OMEGA];
        t.sketch_ms = acc[PH_SKETCH];
        t.sample_qrcp_ms = acc[PH_SQRCP];
        t.swap_ms = acc[PH_SWAP];
        t.panel_ms = acc[PH_PANEL];
        t.trailing_ms = acc[PH_TRAIL];
        t.sample_update_ms = acc[PH_SUPD];
        t.comm_ms = acc[PH_COMM];
    }
    *out = t;
    return 0;
}

// RQRCP_TRACE_PANEL=n: the panel (1-based) whose steps the trace records
static int trace_panel() {
    static const int tp = [] {
        const char *e = getenv("RQRCP_TRACE_PANEL");
        return e ? std::max(1, atoi(e)) : 1;
    }();
    return tp;
}

static int coop_launch(rqrcp_ctx *ctx, const void *func, int grid, int threads, void **args, size_t smem) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, smem);
    if (e == cudaSuccess && grid > occ * ctx->num_sms) {
        ctx->err = "cooperative grid exceeds co-residency";
        return RQRCP_E_WORKSPACE;
    }
    e = cudaLaunchCooperativeKernel(func, dim3(grid), dim3(threads), args, smem, ctx->stream);
    if (e != cudaSuccess) {
        ctx->err = std::string("cooperative launch: ") + cudaGetErrorString(e);
        return RQRCP_E_CUDA;
    }
    ctx->launches++;
    return 0;
}

__global__ void iota_kernel(int64_t *x, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        x[e] = e;
}

// ---------------------------------------------------------------------------
// multi-GPU helpers; all enqueue on ctx->stream
// ---------------------------------------------------------------------------
#define CKN(call)                                                                     \
    do {                                                                              \
        ncclResult_t r_ = (call);                                                     \
        if (r_ != 0) {                                                                \
            ctx->err = std::string(#call) + ": " + nccl().GetErrorString(r_);         \
            return RQRCP_E_NCCL;                                                      \
        }                                                                             \
    } while (0)

// AllGather each rank's ncols_loc sample columns (global columns >= j0, local
// order) and reorder into global order: out(:, p) = column j0 + p.
static int gather_sample(rqrcp_ctx *ctx, int lpad, int64_t ncols_loc, int64_t j0, int64_t ncols, int b, double *out) {
    const int P = ctx->nranks;
    int64_t cmax = 0;
    for (int r = 0; r < P; ++r)
        cmax = std::max<int64_t>(cmax, dist_count(j0 + ncols, b, P, r) - dist_count(j0, b, P, r));
    if (cmax * P * lpad > ctx->gbuf_elems) {
        ctx->err = "gather buffer too small";
        return RQRCP_E_WORKSPACE;
    }
    (void)ncols_loc;
    ph_begin(ctx, PH_COMM);
    CKN(nccl().AllGather(ctx->gsend, ctx->gbuf, (size_t)(cmax * lpad), ncclFloat64, ctx->comm, ctx->stream));
    ph_end(ctx);
    if (ncols > 0) {
        dist_reorder_kernel<<<grid_for(ncols * lpad, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
            ctx->gbuf, cmax, lpad, lpad, j0, ncols, b, P, out, lpad);
        CKL();
    }
    return 0;
}

// The sample QRCP's (dst <- src) column moves (positions relative to i) on
// the block-cyclic shards: local copies through the staging buffer, grouped
// ncclSend/ncclRecv for pairs that cross ranks; jpvt (replicated) on every rank.
static int dist_swaps(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t i, int b, int64_t *jpvt) {
    const int P = ctx->nranks, me = ctx->rank;
    cudaStream_t st = ctx->stream;
    const int bp = ctx->bpad_max;
    int64_t *hp = ctx->h_pairs;  // [0] count, [1..2bp] dst, [..] src
    int hnp = 0;
    CK(cudaMemcpyAsync(&hp[0], ctx->swap_np, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hp[1], ctx->swap_dst, sizeof(int64_t) * 2 * bp, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hp[1 + 2 * bp], ctx->swap_src, sizeof(int64_t) * 2 * bp, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));  // the pivots decide who talks to whom
    memcpy(&hnp, &hp[0], sizeof(int));
    const int64_t *dst = &hp[1], *src = &hp[1 + 2 * bp];
    int64_t *lc = &hp[1 + 4 * bp];          // host lists: stage cols, place cols
    int *ls = reinterpret_cast<int *>(&hp[1 + 6 * bp]);
    int nst = 0, npl = 0;
    std::vector<int> send_q, send_peer, recv_q, recv_peer;
    for (int q = 0; q < hnp; ++q) {
        const int so = dist_owner(i + src[q], b, P), dn = dist_owner(i + dst[q], b, P);
        if (so == me) { lc[nst] = dist_local(i + src[q], b, P); ls[nst] = q; ++nst; }
        if (so == me && dn != me) { send_q.push_back(q); send_peer.push_back(dn); }
        if (dn == me && so != me) { recv_q.push_back(q); recv_peer.push_back(so); }
    }
    for (int q = 0; q < hnp; ++q) {
        const int dn = dist_owner(i + dst[q], b, P);
        if (dn == me) { lc[2 * bp + npl] = dist_local(i + dst[q], b, P); ls[2 * bp + npl] = q; ++npl; }
    }
    CK(cudaMemcpyAsync(ctx->dl_cols, lc, sizeof(int64_t) * 4 * bp, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->dl_slots, ls, sizeof(int) * 4 * bp, cudaMemcpyHostToDevice, st));
    const int64_t lds = ctx->max_m;
    if (nst) {
        dist_columns_kernel<<<grid_for(nst * m, 256, ctx->num_sms), 256, 0, st>>>(A, lda, m, ctx->dl_cols, ctx->dl_slots,
                                                                                  nst, ctx->swap_stage, lds, 0);
        CKL();
    }
    if (!send_q.empty() || !recv_q.empty()) {
        ph_begin(ctx, PH_COMM);
        CKN(nccl().GroupStart());
        for (size_t e = 0; e < send_q.size(); ++e)
            CKN(nccl().Send(ctx->swap_stage + (int64_t)send_q[e] * lds, (size_t)m, ncclFloat64, send_peer[e], ctx->comm, st));
        for (size_t e = 0; e < recv_q.size(); ++e)
            CKN(nccl().Recv(ctx->swap_stage + (int64_t)recv_q[e] * lds, (size_t)m, ncclFloat64, recv_peer[e], ctx->comm, st));
        CKN(nccl().GroupEnd());
        ph_end(ctx);
    }
    if (npl) {
        dist_columns_kernel<<<grid_for(npl * m, 256, ctx->num_sms), 256, 0, st>>>(
            A, lda, m, ctx->dl_cols + 2 * bp, ctx->dl_slots + 2 * bp, npl, ctx->swap_stage, lds, 1);
        CKL();
    }
    dist_jpvt_kernel<<<1, 256, 0, st>>>(jpvt + i, ctx->swap_dst, ctx->swap_src, ctx->swap_np);
    CKL();
    return 0;
}

// Owner of the panel broadcasts Vfull (ldo x bbpad), and [tau | V^T V | R11];
// the others unpack and build V^T.
static int dist_panel_bcast(rqrcp_ctx *ctx, int owner, const double *panel, int64_t lda, int64_t mp, int bb,
                            int bbpad, double *tau_i) {
    cudaStream_t st = ctx->stream;
    const int me = ctx->rank;
    const int npk = bbpad + 3 * bbpad * bbpad + 1;
    if (me == owner) {
        dist_pack_kernel<<<grid_for(npk, 256, ctx->num_sms), 256, 0, st>>>(tau_i, ctx->ybuf, panel, lda, bb, bbpad,
                                                                           ctx->tneg, ctx->cqr_status, ctx->pack);
        CKL();
    }
    ph_begin(ctx, PH_COMM);
    CKN(nccl().GroupStart());
    CKN(nccl().Broadcast(ctx->vfull, ctx->vfull, (size_t)(ctx->ldo * bbpad), ncclFloat64, owner, ctx->comm, st));
    CKN(nccl().Broadcast(ctx->pack, ctx->pack, (size_t)npk, ncclFloat64, owner, ctx->comm, st));
    CKN(nccl().GroupEnd());
    ph_end(ctx);
    if (me != owner) {
        dist_unpack_kernel<<<grid_for(npk, 256, ctx->num_sms), 256, 0, st>>>(ctx->pack, bb, bbpad, tau_i, ctx->ybuf,
                                                                             ctx->tneg, ctx->cqr_status);
        CKL();
        dist_transpose_kernel<<<grid_for(mp * bbpad, 256, ctx->num_sms), 256, 0, st>>>(ctx->vfull, ctx->ldo, mp, bbpad,
                                                                                      ctx->vt);
        CKL();
    }
    return 0;
}

// S4 via CholeskyQR2 + Householder reconstruction (cqr.cuh).  Enqueues the
// whole sequence; every kernel is a no-op once *cqr_status = 1.
static int panel_cqr(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n_loc, int64_t i, int64_t ljp,
                     int64_t mp, int bb, int bbpad, const int *bb_eff, double *tau_i) {
    cudaStream_t st = ctx->stream;
    if (!ctx->cqr_enabled) {
        CK(cudaMemsetAsync(ctx->cqr_status, 0x01, sizeof(int), st));  // != 0: fallback
        return 0;
    }
    int nb = 8;
    while (nb < bbpad) nb *= 2;
    const size_t csm = ((size_t)nb * nb + (size_t)(nb / 2) * (nb / 2)) * sizeof(double);
    const size_t rsm = (size_t)bbpad * (bbpad + 4) * sizeof(double);
    double *P = A + i + ljp * lda;
    const int rows_per_cta = RM_ROWS * (CQR_THREADS / 32);
    const int rgrid = (int)std::max<int64_t>(1, (mp + rows_per_cta - 1) / rows_per_cta);
    bool done = false;
    int rc = 0;
    // G1 = P^T P (the panel: columns ljp.. of the local A, rows i..m)
    rc = tma_skinny(ctx, bb, bb, mp, A, m, n_loc, lda, i, ljp, A, m, n_loc, lda, i, ljp, ctx->cq_g, bbpad, &done, 128);
    if (rc) return rc;
    if (!done) rc = gemm_skinny(ctx, bb, bb, mp, P, lda, P, lda, ctx->cq_g, bbpad);
    if (rc) return rc;
    if (bb <= 64) cqr_chol_kernel<9><<<1, CQR_THREADS, csm, st>>>(ctx->cq_g, bb, bbpad, nb, 1, bb_eff, ctx->cqr_status,
                                                               ctx->cq_rc, ctx->cq_rinv);
    else cqr_chol_kernel<CQR_EPT_U><<<1, CQR_THREADS, csm, st>>>(ctx->cq_g, bb, bbpad, nb, 1, bb_eff, ctx->cqr_status,
                                                                ctx->cq_rc, ctx->cq_rinv);
    CKL();
    // Q1 = P R1^{-1} -> Vfull
    cqr_rowmul_kernel<<<rgrid, CQR_THREADS, rsm, st>>>(P, lda, 0, mp, bb, bbpad, ctx->cq_rinv, 1.0, ctx->vfull, ctx->ldo,
                                                       ctx->cqr_status, 0, nullptr, 0, nullptr);
    CKL();
    // G2 = Q1^T Q1, R2, Rc = R2 R1; Q = Q1 R2^{-1} (in place)
    rc = tma_skinny(ctx, bb, bb, mp, ctx->vfull, mp, bbpad, ctx->ldo, 0, 0, ctx->vfull, mp, bbpad, ctx->ldo, 0, 0,
                    ctx->cq_g, bbpad, &done, 128);
    if (rc) return rc;
    if (!done) rc = gemm_skinny(ctx, bb, bb, mp, ctx->vfull, ctx->ldo, ctx->vfull, ctx->ldo, ctx->cq_g, bbpad);
    if (rc) return rc;
    if (bb <= 64) cqr_chol_kernel<9><<<1, CQR_THREADS, csm, st>>>(ctx->cq_g, bb, bbpad, nb, 2, bb_eff, ctx->cqr_status,
                                                               ctx->cq_rc, ctx->cq_rinv);
    else cqr_chol_kernel<CQR_EPT_U><<<1, CQR_THREADS, csm, st>>>(ctx->cq_g, bb, bbpad, nb, 2, bb_eff, ctx->cqr_status,
                                                                ctx->cq_rc, ctx->cq_rinv);
    CKL();
    cqr_rowmul_kernel<<<rgrid, CQR_THREADS, rsm, st>>>(ctx->vfull, ctx->ldo, 0, mp, bb, bbpad, ctx->cq_rinv, 1.0,
                                                       ctx->vfull, ctx->ldo, ctx->cqr_status, 0, nullptr, 0, nullptr);
    CKL();
    // reconstruction: top block (L, R, T, tau), then V2 = -Q2 U^{-1} with the outputs
    if (bb <= 64)
        cqr_recon_kernel<16><<<1, CQR_THREADS, csm, st>>>(ctx->vfull, ctx->ldo, bb, bbpad, nb, ctx->cq_rc,
                                                          ctx->cqr_status, P, lda, tau_i, ctx->tneg, ctx->cq_uinv, ctx->vt);
    else
        cqr_recon_kernel<CQR_EPT_F><<<1, CQR_THREADS, csm, st>>>(ctx->vfull, ctx->ldo, bb, bbpad, nb, ctx->cq_rc,
                                                                 ctx->cqr_status, P, lda, tau_i, ctx->tneg,
                                                                 ctx->cq_uinv, ctx->vt);
    CKL();
    if (mp > bb) {
        const int vgrid = (int)std::max<int64_t>(1, (mp - bb + rows_per_cta - 1) / rows_per_cta);
        cqr_rowmul_kernel<<<vgrid, CQR_THREADS, rsm, st>>>(ctx->vfull, ctx->ldo, bb, mp, bb, bbpad, ctx->cq_uinv, -1.0,
                                                           ctx->vfull, ctx->ldo, ctx->cqr_status, 1, P, lda, ctx->vt);
        CKL();
    }
    return 0;
}

static int factor_impl(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                       uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out, const double *omega_in,
                       double *omega_out, double *gaps_out, bool keep_last = false, int *final_sample = nullptr) {
    if (!ctx) return -1;
    if (!A) return -2;
    if (lda < std::max<int64_t>(1, m)) return -3;
    if (m < 1) return -4;
    if (n < 1) return -5;
    if (k < 1 || k > std::min(m, n)) return -6;
    if (b < 1) return -7;
    if (p < 0 || (int64_t)b + p > m) return -8;
    if (!jpvt) return -10;
    if (!tau) return -11;
    if (!rank_out) return -12;
    if (m > ctx->max_m || n > ctx->max_n || b > ctx->max_b || p > ctx->max_p) {
        ctx->err = "problem exceeds the create-time workspace maxima";
        return RQRCP_E_WORKSPACE;
    }
    CK(cudaSetDevice(ctx->device));
    // panel path: RQRCP_PANEL=hh (column-by-column Householder, default),
    // =cqr (CholeskyQR2 + reconstruction wherever it is accurate), =auto
    // (CholeskyQR2 for panels of >= kCqrMinRows rows)
    int panel_mode = 0;  // measured (C2-C5): the column-by-column kernel is as fast or faster
    if (const char *e = getenv("RQRCP_PANEL")) panel_mode = (e[0] == 'h' || e[0] == 'H') ? 0 : (e[0] == 'a' ? 2 : 1);
    const int P = ctx->nranks, me = ctx->rank;
    const int64_t n_loc = dist_count(n, b, P, me);  // this rank's columns (n when P = 1)
    ctx->launches = 0;
    ctx->nev = 0;
    ctx->lt_t0 = ctx->lt_t1 = -1;
    ctx->rec_phase.clear();
    ctx->rec_s.clear();
    ctx->rec_e.clear();
    ctx->open_phase = -1;
    const int l = b + p;
    const int lpad = (int)rup(l, 8);
    const int G = ctx->num_sms;
    cudaStream_t st = ctx->stream;
    const int ev_t0 = ctx->nev;
    cudaEventRecord(ctx->ev[ctx->nev++], st);
    ph_begin(ctx, PH_OMEGA);
    CK(cudaMemsetAsync(ctx->iscal, 0, sizeof(int) * 8, st));
    const int64_t npanels = (k + b - 1) / b;
    CK(cudaMemsetAsync(ctx->bars, 0, sizeof(unsigned) * 2 * npanels, st));
    CK(cudaMemsetAsync(ctx->tctr, 0, sizeof(int) * std::min<int64_t>(npanels, 8192), st));
    // ---- S0: Omega^T -----------------------------------------------------
    if (omega_in) {
        omega_t_from_kernel<<<grid_for((int64_t)lpad * m, 256, G), 256, 0, st>>>(omega_in, l, lpad, m, ctx->omt,
                                                                                 ctx->ldo);
    } else {
        omega_t_kernel<<<grid_for((int64_t)lpad / 2 * m, 256, G), 256, 0, st>>>(seed, l, lpad, m, ctx->omt, ctx->ldo);
    }
    CKL();
    if (omega_out) {
        omega_from_t_kernel<<<grid_for((int64_t)l * m, 256, G), 256, 0, st>>>(ctx->omt, ctx->ldo, l, m, omega_out);
        CKL();
    }
    ph_end(ctx);
    // ---- S1: sketch B = Omega A -------------------------------------------
    ph_begin(ctx, PH_SKETCH);
    int cur = 0;
    bool tdone = false;
    // this rank's columns: all of them (P = 1) or its block-cyclic shard
    double *bdst = (P == 1) ? ctx->bs[cur] : ctx->gsend;
    int rc = tma_skinny(ctx, lpad, n_loc, m, ctx->omt, m, lpad, ctx->ldo, 0, 0, A, m, n_loc, lda, 0, 0, bdst, lpad,
                        &tdone);
    if (rc) return rc;
    if (!tdone) rc = gemm_skinny(ctx, lpad, n_loc, m, ctx->omt, ctx->ldo, A, lda, bdst, lpad);
    if (rc) return rc;
    if (P > 1) {  // replicate the sample in global column order (AllGather)
        rc = gather_sample(ctx, lpad, n_loc, 0, n, b, ctx->bs[cur]);
        if (rc) return rc;
    }
    sumsq_partial_kernel<<<4 * G, 256, 0, st>>>(ctx->bs[cur], lpad, n, lpad, ctx->sumsq_part);
    CKL();
    sumsq_final_kernel<<<1, 32, 0, st>>>(ctx->sumsq_part, 4 * G, ctx->stop_tol2, ctx->iscal + 0);
    CKL();
    ph_end(ctx);

    int *status = ctx->iscal + 0, *bb_eff = ctx->iscal + 1, *done = ctx->iscal + 2, *rankd = ctx->iscal + 3;
    // Pi = I_n
    iota_kernel<<<grid_for(n, 256, G), 256, 0, st>>>(jpvt, n);
    CKL();
    CK(cudaMemsetAsync(tau, 0, sizeof(double) * k, st));

    int panels = 0;
    bool upd_pending = false;
    double *bulk_A22 = nullptr;  // deferred bulk trailing update of this panel (overlap)
    int64_t bulk_cols = 0;
    int bulk_cs = 0;
    // the deferred update waiting for launch (after the next sample QRCP is queued)
    bool bulk_ready = false;
    double *bulk_A22_saved = nullptr;
    int64_t bulk_rows = 0;
    int bulk_bb = 0, bulk_bbpad = 0;
    int *bulk_dyn = nullptr;  // non-null: dynamically scheduled bulk update (its tile counter)
    auto launch_bulk = [&]() -> int {
        bulk_ready = false;
        CK(cudaStreamWaitEvent(ctx->upd, ctx->ev_r12, 0));
        cudaStream_t keep = ctx->stream;
        ctx->stream = ctx->upd;
        ctx->grid_cap = bulk_dyn ? 0 : G - bulk_cs;
        // timed on its own stream: trailing_ms adds the bulk update's duration
        // (concurrent with S2, so the phases sum to more than total_ms)
        ph_begin(ctx, PH_TRAIL);
        bool dn = false;
        const double *vt_b = ctx->vt + (int64_t)bulk_bb * bulk_bbpad;
        int r = tma_update(ctx, bulk_rows, bulk_cols, bulk_bbpad, ctx->w2, bulk_bbpad, vt_b, bulk_bbpad,
                           bulk_A22_saved + bulk_bb, lda, &dn, bulk_dyn);
        if (!r && !dn)
            r = gemm_update(ctx, bulk_rows, bulk_cols, bulk_bbpad, ctx->w2, bulk_bbpad, vt_b, bulk_bbpad,
                            bulk_A22_saved + bulk_bb, lda);
        ph_end(ctx);
        ctx->stream = keep;
        ctx->grid_cap = 0;
        if (r) return r;
        CK(cudaEventRecord(ctx->ev_upd, ctx->upd));
        upd_pending = true;
        return 0;
    };
    for (int64_t i = 0; i < k; i += b) {
        const int bb = (int)std::min<int64_t>(b, k - i);
        const int bbpad = (int)rup(bb, 8);
        const int64_t mp = m - i, np = n - i, npp = np - bb;
        ++panels;
        const bool more = (i + bb < k) || keep_last;  // a sample update follows this panel
        const bool rule5 = ctx->update_rule == 2 && more && npp > 0;
        if (rule5)  // Eq. (5) needs B2 = the pre-QRCP sample
            CK(cudaMemcpyAsync(ctx->bpre, ctx->bs[cur], sizeof(double) * (size_t)lpad * (size_t)np,
                               cudaMemcpyDeviceToDevice, st));
        // ---- S2: sample QRCP ---------------------------------------------
        ph_begin(ctx, PH_SQRCP);
        {
            SqArgs a{};
            a.B = ctx->bs[cur];
            a.ldb = lpad;
            a.l = l;
            a.lpad = lpad;
            a.nn = np;
            a.bb = bb;
            a.stop_tol2 = ctx->stop_tol2;
            a.slot_hdr = ctx->slot_hdr;
            a.slot_col = ctx->slot_col;
            a.tag0 = (++ctx->launch_seq) << 8;
            a.slot_v2 = ctx->slot_v2;
            a.slot_data = ctx->slot_data;
            a.ll = ctx->sq_ll;
            a.piv = ctx->piv;
            a.tauhat = ctx->tauhat;
            a.vhat = ctx->vhat;
            a.rhat11 = ctx->rhat11;
            a.bbpad = bbpad;
            a.perm = ctx->perm;
            a.bb_eff = bb_eff;
            a.done = done;
            a.rank = rankd;
            a.status = status;
            a.gaps = gaps_out ? gaps_out + i : nullptr;
            a.swap_dst = ctx->swap_dst;
            a.swap_src = ctx->swap_src;
            a.swap_np = ctx->swap_np;
            a.trace = (panels == trace_panel()) ? ctx->trace : nullptr;
            a.spill = ctx->sq_spill;
            bool sq_done = false;
            {
                // one column per thread in registers, one cluster (sample_qrcp_cl.cuh)
                const char *e = getenv("RQRCP_SQ_CLUSTER");
                const bool allow = !(e && e[0] == '0');
                const int64_t need = (np + SQC_THREADS - 1) / SQC_THREADS;
                void (*kfn)(SqArgs) = nullptr;
                if (l == 40) kfn = sample_qrcp_cluster_kernel<40>;
                else if (l == 74) kfn = sample_qrcp_cluster_kernel<74>;
                else if (l == 80) kfn = sample_qrcp_cluster_kernel<80>;
                if (allow && kfn && need <= ctx->sqc_max && !a.gaps) {
                    const int cs = (int)std::max<int64_t>(1, need);
                    cudaLaunchConfig_t lc = {};
                    lc.gridDim = dim3(cs);
                    lc.blockDim = dim3(SQC_THREADS);
                    lc.dynamicSmemBytes = (size_t)bb * l * sizeof(double);
                    lc.stream = st;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = cs;
                    at[0].val.clusterDim.y = 1;
                    at[0].val.clusterDim.z = 1;
                    lc.attrs = at;
                    lc.numAttrs = 1;
                    CK(cudaLaunchKernelEx(&lc, kfn, a));
                    CKL();
                    sq_done = true;
                }
            }
            if (!sq_done) {
                // one column per thread in registers (+ shared memory), a grid of
                // 1 + ceil(n'/256) CTAs (sample_qrcp_reg.cuh)
                const char *e = getenv("RQRCP_SQ_REG");
                const bool allow = !(e && e[0] == '0');
                const int grid = 1 + (int)((np + SQR_THREADS - 1) / SQR_THREADS);
                void (*kfn)(SqArgs) = nullptr;
                if (l == 40) kfn = sample_qrcp_reg_kernel<40, 0>;
                else if (l == 74) kfn = sample_qrcp_reg_kernel<74, 0>;
                else if (l == 144) kfn = sample_qrcp_reg_kernel<72, 72>;
                if (allow && kfn && !a.gaps && grid <= std::min(G, SQ_MAXG)) {
                    const int ls = (l == 144) ? 72 : 0;
                    const size_t smem = (size_t)std::max(ls * SQR_THREADS, bb * l) * sizeof(double);
                    a.hstride = 8;
                    void *args[] = {&a};
                    rc = coop_launch(ctx, (const void *)kfn, grid, SQR_THREADS, args, smem);
                    if (rc) return rc;
                    sq_done = true;
                }
            }
            if (!sq_done) {
            a.hstride = 8;
            a.poll_mode = 1;
            if (const char *e = getenv("RQRCP_SQ_HSTRIDE")) a.hstride = std::max(1, std::min(8, atoi(e)));
            if (const char *e = getenv("RQRCP_SQ_POLL")) a.poll_mode = std::max(0, std::min(2, atoi(e)));
            int gcap = std::min(G, SQ_MAXG);
            if (const char *e = getenv("RQRCP_SQ_GRID")) gcap = std::max(1, std::min(gcap, atoi(e)));
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(gcap, (np + 7) / 8));
            const int64_t cpb = (np + grid - 1) / grid;
            // threads per column: fill the CTA (columns x tpc <= 256)
            int tpc = 32;
            while (tpc > 1 && cpb * tpc > SQ_THREADS) tpc >>= 1;
            a.tpc = tpc;
            const int cpw = 32 / tpc;
            // as many columns in shared memory as the budget allows (row stride
            // ncs = cpw mod 16 keeps the group's accesses conflict-free), the
            // rest transposed in the L2-resident spill buffer
            auto pad_ncs = [&](int64_t x) -> int64_t {
                if (cpw >= 16 || x <= 0) return std::max<int64_t>(x, 1);
                return x + (((cpw - x) % 16) + 16) % 16;
            };
            const int64_t state = cpb * (2 * (int64_t)sizeof(double) + 2 * (int64_t)sizeof(int));
            int64_t nsm = cpb;
            if (const char *e = getenv("RQRCP_SQ_NSM")) nsm = std::max<int64_t>(0, std::min<int64_t>(nsm, atoi(e)));
            while (nsm > 0 && (int64_t)l * pad_ncs(nsm) * 8 + state > kDynSmemMax) --nsm;
            a.nsm = (int)nsm;
            a.ncs = (int)pad_ncs(nsm);
            const size_t smem = sq_smem_bytes(a.ncs, cpb, l);
            void *args[] = {&a};
            rc = coop_launch(ctx, (const void *)sample_qrcp_kernel, grid, SQ_THREADS, args, smem);
            if (rc) return rc;
            }
        }
        ph_end(ctx);
        if (bulk_ready) {  // the previous panel's bulk update, now that S2 is queued
            rc = launch_bulk();
            if (rc) return rc;
        }
        // ---- S3: swaps on A and Pi -----------------------------------------
        ph_begin(ctx, PH_SWAP);
        if (upd_pending) {  // the previous panel's bulk trailing update (overlapped with S2)
            CK(cudaStreamWaitEvent(st, ctx->ev_upd, 0));
            upd_pending = false;
        }
        if (P > 1) {
            rc = dist_swaps(ctx, A, lda, m, i, b, jpvt);
            if (rc) return rc;
        } else {
            if (2 * bb <= SW_MAXP) {  // one launch: rows are independent
                swap_fused_kernel<<<(unsigned)((m + SW_ROWS - 1) / SW_ROWS), 256, 0, st>>>(
                    A + i * lda, lda, m, jpvt + i, ctx->swap_src, ctx->swap_dst, ctx->swap_np);
                CKL();
            } else {
                const int64_t lds = ctx->max_m;
                const int gg = grid_for(2 * (int64_t)bb * m, 256, G);
                swap_gather_kernel<<<gg, 256, 0, st>>>(A + i * lda, lda, m, jpvt + i, ctx->swap_src, ctx->swap_np,
                                                        ctx->swap_stage, lds, ctx->swap_jstage);
                CKL();
                swap_scatter_kernel<<<gg, 256, 0, st>>>(A + i * lda, lda, m, jpvt + i, ctx->swap_dst, ctx->swap_np,
                                                         ctx->swap_stage, lds, ctx->swap_jstage);
                CKL();
            }
        }
        ph_end(ctx);
        // ---- S4: panel QR + T ----------------------------------------------
        ph_begin(ctx, PH_PANEL);
        const int owner = dist_owner(i, b, P);
        const int64_t ljp = dist_local(i, b, P);  // owner's local column of the panel
        if (me == owner) {
            // CholeskyQR2 + Householder reconstruction (cqr.cuh); on failure
            // (*cqr_status = 1) the column-by-column kernel below factors it
            ctx->cqr_enabled = (panel_mode == 1) || (panel_mode == 2 && mp >= kCqrMinRows);
            rc = panel_cqr(ctx, A, lda, m, n_loc, i, ljp, mp, bb, bbpad, bb_eff, tau + i);
            if (rc) return rc;
            PanelArgs a{};
            a.skip = ctx->cqr_status;
            a.count = ctx->iscal + 4;
            a.A = A + i + ljp * lda;
            a.lda = lda;
            a.mp = mp;
            a.bb = bb;
            a.bbpad = bbpad;
            a.bb_eff = bb_eff;
            a.tau = tau + i;
            a.vfull = ctx->vfull;
            a.ldv = ctx->ldo;
            a.vt = ctx->vt;
            a.ybuf = ctx->ybuf;
            a.part = ctx->pn_part;
            a.rowj = ctx->pn_rowj;
            a.bar = ctx->bars + 2 * (panels - 1) + 1;
            a.trace = (panels == trace_panel()) ? ctx->ptrace : nullptr;
            // register-resident cluster kernel (panel_cl.cuh) when the panel fits
            // one cluster: bb <= 64 and m' <= clusters x rows per CTA
            bool pn_done = false;
            {
                const char *e = getenv("RQRCP_PN_CLUSTER");
                const bool allow = !(e && e[0] == '0');
                void (*kfn)(PanelArgs) = nullptr;
                int64_t rc_rows = 0;
                size_t psm = 0;
                const char *ec = getenv("RQRCP_PN_CPT");
                const bool cpt2 = !(ec && ec[0] == '1');
                if (bb <= 32) { kfn = panel_qr_cluster_kernel<32, 64>; rc_rows = 8 * 64; psm = 32 * 65 * 8; }
                else if (bb <= 64 && cpt2) {  // two columns x 32 rows per thread
                    kfn = panel_qr_cluster_kernel<64, 32, 2>; rc_rows = 8 * 32; psm = 64 * 64 * 8;
                } else if (bb <= 64) { kfn = panel_qr_cluster_kernel<64, 64>; rc_rows = 4 * 64; psm = 64 * 65 * 8; }
                const int64_t cs = kfn ? (mp + rc_rows - 1) / rc_rows : 0;
                if (allow && kfn && cs <= ctx->pnc_max) {
                    cudaLaunchConfig_t lc = {};
                    lc.gridDim = dim3((unsigned)cs);
                    lc.blockDim = dim3(PNC_THREADS);
                    lc.dynamicSmemBytes = psm;
                    lc.stream = st;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = (unsigned)cs;
                    at[0].val.clusterDim.y = 1;
                    at[0].val.clusterDim.z = 1;
                    lc.attrs = at;
                    lc.numAttrs = 1;
                    CK(cudaLaunchKernelEx(&lc, kfn, a));
                    CKL();
                    pn_done = true;
                    if (a.trace) ctx->ptrace_kind = 1;
                }
            }
            int pcap = G;
            if (const char *e = getenv("RQRCP_PN_GRID")) pcap = std::max(1, std::min(G, atoi(e)));
            // ~128 rows per CTA: fewer CTAs shrink the per-column all-to-all of
            // partial Gram rows (G x bb doubles read by every CTA), more rows
            // per CTA lengthen the local pass (measured best at C3: 64 / 96 /
            // 128 / 192 / 256 rows -> 8.17 / 8.16 / 7.76 / 8.32 / 9.18 ms)
            int64_t prows = 128;
            if (const char *e = getenv("RQRCP_PN_ROWS")) prows = std::max(1, atoi(e));
            const int grid = (int)std::max<int64_t>((mp + PN_MAXROWS - 1) / PN_MAXROWS,
                                                    std::min<int64_t>(pcap, (mp + prows - 1) / prows));
            const int64_t rpb = (mp + grid - 1) / grid;
            if (rpb > PN_MAXROWS) {
                ctx->err = "panel too tall for the cooperative grid";
                return RQRCP_E_WORKSPACE;
            }
            // as many of each CTA's rows in shared memory as fit, the rest via L2
            a.nsm = (int)std::min<int64_t>(rpb, kDynSmemMax / ((int64_t)bb * sizeof(double)));
            const size_t smem = (size_t)a.nsm * bb * sizeof(double);
            void *args[] = {&a};
            if (!pn_done) {
                rc = coop_launch(ctx, (const void *)panel_qr_kernel, grid, PN_THREADS, args, smem);
                if (a.trace) ctx->ptrace_kind = 0;
            }
            if (rc) return rc;
        }
        const double *R11p = A + i + ljp * lda;
        int64_t ldr11 = lda;
        if (P > 1) {  // owner broadcasts V, tau, V^T V and R11
            rc = dist_panel_bcast(ctx, owner, A + i + ljp * lda, lda, mp, bb, bbpad, tau + i);
            if (rc) return rc;
            R11p = ctx->pack + bbpad + (int64_t)bbpad * bbpad;
            ldr11 = bbpad;
        }
        // T and Omega-hat11 on the side stream, overlapping W = V^T A22
        {
            int nb = 8;
            while (nb < bbpad) nb *= 2;
            const size_t smem = ((size_t)nb * nb + (size_t)(nb / 2) * (nb / 2)) * sizeof(double);
            CK(cudaEventRecord(ctx->ev_fork, st));
            CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            const int do_om = (more && npp > 0 && !rule5) ? 1 : 0;
            tri_kernel<<<2, TRI_THREADS, smem, ctx->side>>>(ctx->ybuf, tau + i, ctx->rhat11, R11p, ldr11, bb, bbpad,
                                                          nb, bb_eff, ctx->tneg, ctx->omhat, do_om, ctx->cqr_status);
            CKL();
            CK(cudaEventRecord(ctx->ev_join, ctx->side));
        }
        ph_end(ctx);
        // ---- S5: trailing update A22 -= V T^T V^T A22 ------------------------
        ph_begin(ctx, PH_TRAIL);
        // this rank's trailing columns: local [lj0, n_loc) = global columns >= i + bb
        const int64_t lj0 = dist_count(i + bb, b, P, me);
        const int64_t npl = n_loc - lj0;
        if (npl > 0) {
            double *A22 = A + i + lj0 * lda;
            // W = V^T A22: V = Vfull(0:m', 0:bbpad); A22 = A(i:m, lj0:n_loc) by TMA coordinates
            rc = tma_skinny(ctx, bbpad, npl, mp, ctx->vfull, mp, bbpad, ctx->ldo, 0, 0, A, m, n_loc, lda, i, lj0,
                            ctx->w, bbpad, &tdone);
            if (rc) return rc;
            if (!tdone) rc = gemm_skinny(ctx, bbpad, npl, mp, ctx->vfull, ctx->ldo, A22, lda, ctx->w, bbpad);
            if (rc) return rc;
            CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
            rc = gemm_skinny(ctx, bbpad, npl, bbpad, ctx->tneg, bbpad, ctx->w, bbpad, ctx->w2, bbpad);
            if (rc) return rc;
            // Overlap: when the next panel's sample QRCP runs on one cluster, only
            // the R12 rows (all Eq. (4) needs) are updated here; the bulk A22 rows
            // i+bb..m go to the low-priority `upd` stream on G - (cluster) CTAs and
            // run concurrently with S6 and the next sample QRCP (the next swap
            // waits for them).  P = 1, Eq. (4) only.
            bool ovl = false;
            int next_cs = 0;
            if (P == 1 && !rule5 && more && npp > 0 && mp > bb && (bb % 2) == 0 && !gaps_out &&
                (l == 40 || l == 74 || l == 80)) {
                const char *e1 = getenv("RQRCP_OVERLAP"), *e2 = getenv("RQRCP_SQ_CLUSTER");
                next_cs = (int)std::max<int64_t>(1, (npp + SQC_THREADS - 1) / SQC_THREADS);
                ovl = !(e1 && e1[0] == '0') && !(e2 && e2[0] == '0') && next_cs <= ctx->sqc_max;
            }
            // the next sample QRCP on the register grid (C3-sized samples): the bulk
            // update runs on the whole GPU with dynamically claimed tiles, so the
            // CTAs that find their SM taken by the sample QRCP start late and take
            // fewer tiles (bb <= 64: the K <= 64 update kernel)
            bool dyn = false;
            if (!ovl && P == 1 && !rule5 && more && npp > 0 && mp > bb && (bb % 2) == 0 && bbpad <= 64 &&
                !gaps_out && (l == 40 || l == 74)) {
                const char *e1 = getenv("RQRCP_OVERLAP"), *e2 = getenv("RQRCP_SQ_REG"),
                           *e3 = getenv("RQRCP_OVERLAP_GRID");
                const int64_t ngrid = 1 + (npp + SQR_THREADS - 1) / SQR_THREADS;
                dyn = !(e1 && e1[0] == '0') && !(e2 && e2[0] == '0') && !(e3 && e3[0] == '0') &&
                      ngrid <= std::min(G, SQ_MAXG) && panels <= 8192;
                ovl = dyn;
                next_cs = 0;
            }
            if (ovl) {
                rc = tma_update(ctx, bb, npl, bbpad, ctx->w2, bbpad, ctx->vt, bbpad, A22, lda, &tdone);
                if (rc) return rc;
                if (!tdone) rc = gemm_update(ctx, bb, npl, bbpad, ctx->w2, bbpad, ctx->vt, bbpad, A22, lda);
                if (rc) return rc;
                bulk_A22 = A22;
                bulk_cols = npl;
                bulk_cs = next_cs;
                bulk_dyn = dyn ? ctx->tctr + (panels - 1) : nullptr;
            } else {
                rc = tma_update(ctx, mp, npl, bbpad, ctx->w2, bbpad, ctx->vt, bbpad, A22, lda, &tdone);
                if (rc) return rc;
                if (!tdone) rc = gemm_update(ctx, mp, npl, bbpad, ctx->w2, bbpad, ctx->vt, bbpad, A22, lda);
                if (rc) return rc;
            }
        } else {
            CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
        }
        ph_end(ctx);
        // ---- S6: sample update (Eq. (4) or (5)); skipped after the last panel (R-G9)
        if (more && npp > 0) {
            ph_begin(ctx, PH_SUPD);
            double *udst = (P == 1) ? ctx->bs[cur ^ 1] : ctx->gsend;
            if (rule5) {
                // Omega-bar^T = Q_panel^T Omega_cur^T on rows i..m of Omega^T (same
                // three contractions as the trailing update), then
                // C = Omega-bar_1 R12 and B_next = B2 - C
                bool dn = false;
                rc = tma_skinny(ctx, bbpad, lpad, mp, ctx->vfull, mp, bbpad, ctx->ldo, 0, 0, ctx->omt, m, lpad,
                                ctx->ldo, i, 0, ctx->wom, bbpad, &dn);
                if (rc) return rc;
                if (!dn) rc = gemm_skinny(ctx, bbpad, lpad, mp, ctx->vfull, ctx->ldo, ctx->omt + i, ctx->ldo, ctx->wom,
                                          bbpad);
                if (rc) return rc;
                rc = gemm_skinny(ctx, bbpad, lpad, bbpad, ctx->tneg, bbpad, ctx->wom, bbpad, ctx->w2om, bbpad);
                if (rc) return rc;
                rc = tma_update(ctx, mp, lpad, bbpad, ctx->w2om, bbpad, ctx->vt, bbpad, ctx->omt + i, ctx->ldo, &dn);
                if (rc) return rc;
                if (!dn) rc = gemm_update(ctx, mp, lpad, bbpad, ctx->w2om, bbpad, ctx->vt, bbpad, ctx->omt + i, ctx->ldo);
                if (rc) return rc;
                if (npl > 0) {
                    rc = gemm_skinny(ctx, lpad, npl, bb, ctx->omt + i, ctx->ldo, A + i + lj0 * lda, lda, ctx->c5, lpad);
                    if (rc) return rc;
                    sample_update5_kernel<<<grid_for((int64_t)lpad * npl, 256, G), 256, 0, st>>>(
                        ctx->bpre, lpad, ctx->perm, ctx->c5, lpad, bb, l, lpad, npl, bb_eff, udst, lpad, i, lj0, b, P,
                        me);
                    CKL();
                }
            } else if (npl > 0) {
                // C = Omega-hat11 R12 (DMMA; omhat holds Omega-hat11^T), then the
                // gather B_next = [R-hat12 - C; R-hat22] (Eq. (4))
                rc = gemm_skinny(ctx, bbpad, npl, bb, ctx->omhat, bbpad, A + i + lj0 * lda, lda, ctx->c5, lpad);
                if (rc) return rc;
                sample_update4_kernel<<<grid_for((int64_t)lpad * npl, 256, G), 256, 0, st>>>(
                    ctx->bs[cur], lpad, ctx->perm, ctx->c5, lpad, bb, l, lpad, npl, bb_eff, udst, lpad, i, lj0, b, P,
                    me);
                CKL();
            }
            if (P > 1) {
                rc = gather_sample(ctx, lpad, npl, i + bb, n - i - bb, b, ctx->bs[cur ^ 1]);
                if (rc) return rc;
            }
            ph_end(ctx);
            cur ^= 1;
        }
        if (bulk_A22) {
            // the bulk rows i+bb..m of this panel's trailing update may start once
            // S6 is done; they are launched after the next sample QRCP has been
            // queued (below), so that kernel is dispatched onto its cluster first
            CK(cudaEventRecord(ctx->ev_r12, st));
            bulk_rows = mp - bb;
            bulk_bb = bb;
            bulk_bbpad = bbpad;
            bulk_ready = true;
            bulk_A22_saved = bulk_A22;
            bulk_A22 = nullptr;
        }
    }
    if (bulk_ready) {
        rc = launch_bulk();
        if (rc) return rc;
    }
    if (upd_pending) CK(cudaStreamWaitEvent(st, ctx->ev_upd, 0));
    if (final_sample) *final_sample = cur;
    // ---- status (pinned host words) ----------------------------------------
    int *hs = ctx->hstatus;
    CK(cudaMemcpyAsync(hs, ctx->iscal, sizeof(int) * 5, cudaMemcpyDeviceToHost, st));
    const int ev_t1 = ctx->nev;
    cudaEventRecord(ctx->ev[ctx->nev++], st);
    CK(cudaStreamSynchronize(st));
    // timings: the events are read lazily by rqrcp_get_timings (the elapsed-time
    // queries stay off the caller's critical path between factorizations)
    rqrcp_timings t{};
    ctx->lt_t0 = ctx->timing ? ev_t0 : -1;
    ctx->lt_t1 = ctx->timing ? ev_t1 : -1;
    if (ctx->trace) {
        std::vector<unsigned long long> H((size_t)SQ_MAXG * 64 * 4);
        cudaMemcpy(H.data(), ctx->trace, sizeof(unsigned long long) * H.size(), cudaMemcpyDeviceToHost);
        cudaMemset(ctx->trace, 0, sizeof(unsigned long long) * H.size());
        const char *names[4] = {"wait/poll+winner+householder", "apply", "publish", "->next"};
        double all[4] = {0}, worst_apply = 0;
        int ncta = 0, worst = -1;
        for (int c = 0; c < SQ_MAXG; ++c) {
            double acc[4] = {0};
            int cnt = 0;
            for (int jj = 1; jj < 63; ++jj) {
                const unsigned long long *r = H.data() + ((size_t)c * 64 + jj) * 4;
                const unsigned long long *nx = H.data() + ((size_t)c * 64 + jj + 1) * 4;
                if (!r[0] || !r[3] || !nx[0]) continue;
                for (int q = 0; q < 3; ++q) acc[q] += (double)(r[q + 1] - r[q]);
                acc[3] += (double)(nx[0] - r[3]);
                ++cnt;
            }
            if (!cnt) continue;
            for (int q = 0; q < 4; ++q) acc[q] /= cnt;
            if (c == 0) {
                fprintf(stderr, "[rqrcp trace] sample QRCP CTA 0, %d steps, mean cycles:", cnt);
                for (int q = 0; q < 4; ++q) fprintf(stderr, " %s=%.0f", names[q], acc[q]);
                fprintf(stderr, "\n");
            }
            for (int q = 0; q < 4; ++q) all[q] += acc[q];
            if (acc[1] + acc[2] > worst_apply) { worst_apply = acc[1] + acc[2]; worst = c; }
            ++ncta;
        }
        if (ncta) {
            fprintf(stderr, "[rqrcp trace] sample QRCP mean over %d CTAs:", ncta);
            for (int q = 0; q < 4; ++q) fprintf(stderr, " %s=%.0f", names[q], all[q] / ncta);
            fprintf(stderr, "; slowest apply+publish: CTA %d (%.0f cycles)\n", worst, worst_apply);
        }
        unsigned long long h[2 * 64 * 8];
        cudaMemcpy(h, ctx->ptrace, sizeof(h), cudaMemcpyDeviceToHost);
        const char *pn0[5] = {"gram", "barrier", "reduce", "tau+w+x", "update"};
        const char *pn1[5] = {"gram", "push", "mbar-wait", "sum", "update+publish"};
        const char **pn = ctx->ptrace_kind ? pn1 : pn0;
        for (int c = 0; c < 2; ++c) {
            double acc[5] = {0};
            int cnt = 0;
            for (int jj = 1; jj < 63; ++jj) {
                const unsigned long long *r = h + ((size_t)c * 64 + jj) * 8;
                if (!r[0] || !r[5]) continue;
                for (int q = 0; q < 5; ++q) acc[q] += (double)(r[q + 1] - r[q]);
                ++cnt;
            }
            fprintf(stderr, "[rqrcp trace] panel CTA %s, %d steps, mean cycles:", c ? "last" : "0", cnt);
            for (int q = 0; q < 5; ++q) fprintf(stderr, " %s=%.0f", pn[q], cnt ? acc[q] / cnt : 0.0);
            if (ctx->ptrace_kind == 1) {  // update+publish split: dlarfg+w | update loop | publish
                double d6 = 0, d7 = 0, d5 = 0;
                for (int jj = 1; jj < 63; ++jj) {
                    const unsigned long long *r = h + ((size_t)c * 64 + jj) * 8;
                    if (!r[0] || !r[5]) continue;
                    d6 += (double)(r[6] - r[4]);
                    d7 += (double)(r[7] - r[6]);
                    d5 += (double)(r[5] - r[7]);
                }
                if (cnt) fprintf(stderr, " [dlarfg+w=%.0f loop=%.0f publish=%.0f]", d6 / cnt, d7 / cnt, d5 / cnt);
            }
            fprintf(stderr, "\n");
        }
    }
    t.panels = panels;
    t.panels_householder = hs[4];
    t.kernel_launches = ctx->launches;
    ctx->last = t;
    *rank_out = hs[3];
    if (hs[0] == 4) {
        ctx->err = "non-finite values in the sample (A contains NaN/Inf)";
        return RQRCP_E_NONFINITE;
    }
    if (hs[3] < k) {
        ctx->err = "rank-deficient: early stop";
        return RQRCP_W_RANK_DEFICIENT;
    }
    return 0;
}

extern "C" int rqrcp_factor(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                            uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out) {
    return factor_impl(ctx, A, lda, m, n, k, b, p, seed, jpvt, tau, rank_out, nullptr, nullptr, nullptr);
}

extern "C" int rqrcp_factor_ex(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                               uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out, const double *omega_in,
                               double *omega_out, double *gaps_out) {
    return factor_impl(ctx, A, lda, m, n, k, b, p, seed, jpvt, tau, rank_out, omega_in, omega_out, gaps_out);
}

extern "C" int rqrcp_srqr_verify(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b,
                                 int p, uint64_t seed, int d, int64_t *jpvt, double *tau, int64_t *rank_out,
                                 double *diag) {
    if (ctx && (d < 1 || d > 64)) return -13;
    if (ctx && ctx->nranks > 1) {
        ctx->err = "rqrcp_srqr_verify is single-GPU only";
        return RQRCP_E_UNSUPPORTED;
    }
    if (ctx && m >= 1 && n >= 1 && k >= std::min(m, n)) {
        ctx->err = "SRQR verification needs k < min(m, n)";
        return RQRCP_E_UNSUPPORTED;
    }
    int fin = 0;
    int rc = factor_impl(ctx, A, lda, m, n, k, b, p, seed, jpvt, tau, rank_out, nullptr, nullptr, nullptr, true, &fin);
    if (rc != 0) return rc;  // including the rank-deficient early stop: nothing to verify
    if (!diag) return -14;
    cudaStream_t st = ctx->stream;
    const int l = b + p;
    const int lpad = (int)rup(l, 8);
    const int64_t nt = n - k;
    int *iota = ctx->iscal + 5;
    srqr_pick_kernel<<<1, SRQR_THREADS, 0, st>>>(ctx->bs[fin], lpad, l, nt, iota);
    CKL();
    srqr_swaplist_kernel<<<1, 1, 0, st>>>(iota, ctx->swap_dst, ctx->swap_src, ctx->swap_np);
    CKL();
    const int64_t lds = ctx->max_m;
    swap_gather_kernel<<<grid_for(2 * m, 256, ctx->num_sms), 256, 0, st>>>(A + k * lda, lda, m, jpvt + k, ctx->swap_src,
                                                                            ctx->swap_np, ctx->swap_stage, lds,
                                                                            ctx->swap_jstage);
    CKL();
    swap_scatter_kernel<<<grid_for(2 * m, 256, ctx->num_sms), 256, 0, st>>>(A + k * lda, lda, m, jpvt + k,
                                                                             ctx->swap_dst, ctx->swap_np,
                                                                             ctx->swap_stage, lds, ctx->swap_jstage);
    CKL();
    unsigned long long *maxbits = reinterpret_cast<unsigned long long *>(ctx->sumsq_part);
    double *alpha = ctx->sumsq_part + 1;
    CK(cudaMemsetAsync(ctx->sumsq_part, 0, 2 * sizeof(double), st));
    srqr_norms_kernel<<<grid_for(nt * 32, 256, ctx->num_sms), 256, 0, st>>>(A + k + k * lda, lda, m - k, nt, maxbits,
                                                                            alpha);
    CKL();
    const size_t ssm = sizeof(double) * (size_t)(k + 1);
    if (ssm > 200 * 1024) {
        ctx->err = "SRQR verification: k too large for the shared-memory solve";
        return RQRCP_E_WORKSPACE;
    }
    CK(cudaFuncSetAttribute(srqr_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    double *Y = ctx->splitk;  // (k+1) x d <= 4 M doubles
    if ((k + 1) * (int64_t)d > ctx->splitk_elems) {
        ctx->err = "SRQR verification: workspace";
        return RQRCP_E_WORKSPACE;
    }
    srqr_solve_kernel<<<d, SRQR_THREADS, ssm, st>>>(A, lda, k, alpha, seed, Y);
    CKL();
    double *dout = ctx->sumsq_part + 2;
    srqr_g2_kernel<<<1, SRQR_THREADS, 0, st>>>(Y, k, d, maxbits, alpha, iota, n, dout);
    CKL();
    CK(cudaMemcpyAsync(diag, dout, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int rqrcp_form_q1(rqrcp_ctx *ctx, const double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b,
                             const double *tau, double *Q1, int64_t ldq) {
    if (!ctx) return -1;
    if (!A) return -2;
    if (lda < std::max<int64_t>(1, m)) return -3;
    if (m < 1) return -4;
    if (n < 1) return -5;
    if (k < 1 || k > std::min(m, n)) return -6;
    if (b < 1) return -7;
    if (!tau) return -8;
    if (!Q1) return -9;
    if (ldq < m) return -10;
    if (m > ctx->max_m || b > ctx->max_b || k > ctx->max_n) {
        ctx->err = "problem exceeds the create-time workspace maxima";
        return RQRCP_E_WORKSPACE;
    }
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int G = ctx->num_sms;
    int rc = 0;
    lr_eye_kernel<<<grid_for(m * k, 256, G), 256, 0, st>>>(Q1, ldq, m, k);
    CKL();
    int *bbd = ctx->iscal + 6;
    const int64_t npanels = (k + b - 1) / b;
    for (int64_t t = npanels - 1; t >= 0; --t) {
        const int64_t i = t * b;
        const int bb = (int)std::min<int64_t>(b, k - i);
        const int bbpad = (int)rup(bb, 8);
        const int64_t mp = m - i, ncols = k - i;
        lr_extract_v_kernel<<<grid_for(mp * bbpad, 256, G), 256, 0, st>>>(A + i + i * lda, lda, mp, bb, bbpad,
                                                                          ctx->vfull, ctx->ldo, ctx->vt);
        CKL();
        rc = gemm_skinny(ctx, bbpad, bbpad, mp, ctx->vfull, ctx->ldo, ctx->vfull, ctx->ldo, ctx->ybuf, bbpad);
        if (rc) return rc;
        lr_set_int_kernel<<<1, 1, 0, st>>>(bbd, bb);
        CKL();
        int nb = 8;
        while (nb < bbpad) nb *= 2;
        const size_t tsm = ((size_t)nb * nb + (size_t)(nb / 2) * (nb / 2)) * sizeof(double);
        tri_kernel<<<1, TRI_THREADS, tsm, st>>>(ctx->ybuf, tau + i, nullptr, nullptr, 0, bb, bbpad, nb, bbd, ctx->tneg,
                                                ctx->omhat, 0, nullptr);
        CKL();
        lr_transpose_kernel<<<grid_for((int64_t)bbpad * bbpad, 256, G), 256, 0, st>>>(ctx->tneg, bbpad, ctx->omhat);
        CKL();
        double *X = Q1 + i + i * ldq;
        // X <- (I - V T V^T) X:  W = V^T X,  W2 = -T W,  X += V W2
        rc = gemm_skinny(ctx, bbpad, ncols, mp, ctx->vfull, ctx->ldo, X, ldq, ctx->w, bbpad);
        if (rc) return rc;
        rc = gemm_skinny(ctx, bbpad, ncols, bbpad, ctx->omhat, bbpad, ctx->w, bbpad, ctx->w2, bbpad);
        if (rc) return rc;
        rc = gemm_update(ctx, mp, ncols, bbpad, ctx->w2, bbpad, ctx->vt, bbpad, X, ldq);
        if (rc) return rc;
    }
    CK(cudaStreamSynchronize(st));
    return 0;
}

extern "C" int rqrcp_cx(rqrcp_ctx *ctx, const double *A, int64_t lda, int64_t m, int64_t n, int64_t k,
                        const int64_t *jpvt, double *X, int64_t ldx) {
    if (!ctx) return -1;
    if (!A) return -2;
    if (lda < std::max<int64_t>(1, m)) return -3;
    if (m < 1) return -4;
    if (n < 1) return -5;
    if (k < 1 || k > std::min(m, n)) return -6;
    if (!jpvt) return -7;
    if (!X) return -8;
    if (ldx < k) return -9;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int G = ctx->num_sms;
    const int64_t n2 = n - k;
    double *RT = nullptr, *Z = nullptr, *C = nullptr;
    auto cleanup = [&]() {
        cudaStreamSynchronize(st);
        if (RT) cudaFree(RT);
        if (Z) cudaFree(Z);
        if (C) cudaFree(C);
    };
    if (n2 > 0) {
        if (cudaMalloc((void **)&RT, sizeof(double) * (size_t)(k * k)) != cudaSuccess ||
            cudaMalloc((void **)&Z, sizeof(double) * (size_t)(k * n2)) != cudaSuccess ||
            cudaMalloc((void **)&C, sizeof(double) * (size_t)(64 * n2)) != cudaSuccess) {
            cleanup();
            ctx->err = "rqrcp_cx: temporary allocation failed";
            return RQRCP_E_WORKSPACE;
        }
        lr_r11t_kernel<<<grid_for(k * k, 256, G), 256, 0, st>>>(A, lda, k, RT);
        CKL();
        // Z = R11^{-1} R12, 64-row blocks from the bottom
        const int64_t nblk = (k + 63) / 64;
        for (int64_t bi = nblk - 1; bi >= 0; --bi) {
            const int64_t r0 = bi * 64, r1 = std::min<int64_t>(k, r0 + 64);
            const int bs = (int)(r1 - r0);
            const double *Cp = nullptr;
            if (r1 < k) {  // C = R11(r0:r1, r1:k) Z(r1:k, :) = RT(r1:k, r0:r1)^T Z(r1:k, :)
                int rc = gemm_skinny(ctx, bs, n2, k - r1, RT + r1 + r0 * k, k, Z + r1, k, C, 64);
                if (rc) { cleanup(); return rc; }
                Cp = C;
            }
            lr_block_solve_kernel<<<(unsigned)((n2 + 127) / 128), 128, 0, st>>>(A, lda, k, n2, r0, bs, Cp, 64, Z, k);
            CKL();
        }
    }
    lr_cx_scatter_kernel<<<grid_for(k * n, 256, G), 256, 0, st>>>(Z, k, jpvt, k, n, X, ldx);
    CKL();
    cleanup();
    return 0;
}

extern "C" int rqrcp_factor_host(rqrcp_ctx *ctx, const double *A_host, int64_t lda, int64_t m, int64_t n, int64_t k,
                                 int b, int p, uint64_t seed, double *A_out_host, int64_t *jpvt_host,
                                 double *tau_host, int64_t *rank_out) {
    if (!ctx) return -1;
    if (!A_host) return -2;
    if (lda < std::max<int64_t>(1, m)) return -3;
    if (m < 1) return -4;
    if (n < 1) return -5;
    if (k < 1 || k > std::min(m, n)) return -6;
    if (!A_out_host) return -10;
    if (!jpvt_host) return -11;
    if (!tau_host) return -12;
    if (!rank_out) return -13;
    if (m > ctx->max_m || n > ctx->max_n) {
        ctx->err = "problem exceeds the create-time workspace maxima";
        return RQRCP_E_WORKSPACE;
    }
    if (ctx->nranks > 1) {
        ctx->err = "rqrcp_factor_host is single-GPU only";
        return RQRCP_E_UNSUPPORTED;
    }
    CK(cudaSetDevice(ctx->device));
    const int64_t need = m * n;
    if (ctx->a_dev_elems < need) {
        if (ctx->a_dev) cudaFree(ctx->a_dev);
        if (ctx->jpvt_dev) cudaFree(ctx->jpvt_dev);
        if (ctx->tau_dev) cudaFree(ctx->tau_dev);
        ctx->a_dev = nullptr;
        ctx->a_dev_elems = 0;
        CK(cudaMalloc((void **)&ctx->a_dev, sizeof(double) * need));
        CK(cudaMalloc((void **)&ctx->jpvt_dev, sizeof(int64_t) * ctx->max_n));
        CK(cudaMalloc((void **)&ctx->tau_dev, sizeof(double) * std::min(ctx->max_m, ctx->max_n)));
        ctx->a_dev_elems = need;
    }
    CK(cudaMemcpy2DAsync(ctx->a_dev, sizeof(double) * m, A_host, sizeof(double) * lda, sizeof(double) * m, n,
                         cudaMemcpyHostToDevice, ctx->stream));
    int64_t rk = 0;
    int rc = factor_impl(ctx, ctx->a_dev, m, m, n, k, b, p, seed, ctx->jpvt_dev, ctx->tau_dev, &rk, nullptr, nullptr,
                         nullptr);
    *rank_out = rk;
    if (rc != 0 && rc != RQRCP_W_RANK_DEFICIENT) return rc;
    CK(cudaMemcpy2DAsync(A_out_host, sizeof(double) * lda, ctx->a_dev, sizeof(double) * m, sizeof(double) * m, n,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(jpvt_host, ctx->jpvt_dev, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(tau_host, ctx->tau_dev, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return rc;
}

extern "C" int rqrcp_fill_gaussian(rqrcp_ctx *ctx, uint64_t seed, uint32_t stream, int64_t rows, int64_t cols,
                                   int64_t row0, int64_t col0, double *out, int64_t ld) {
    if (!ctx) return -1;
    if (rows < 0) return -4;
    if (cols < 0) return -5;
    if (row0 < 0) return -6;
    if (col0 < 0) return -7;
    if (!out && rows * cols > 0) return -8;
    if (ld < std::max<int64_t>(1, rows)) return -9;
    if (rows * cols == 0) return 0;
    CK(cudaSetDevice(ctx->device));
    const int64_t npairs = ((row0 + rows - 1) >> 1) - (row0 >> 1) + 1;
    gaussian_fill_kernel<<<grid_for(npairs * cols, 256, ctx->num_sms), 256, 0, ctx->stream>>>(seed, stream, rows, cols,
                                                                                               row0, col0, out, ld);
    CKL();
    CK(cudaStreamSynchronize(ctx->stream));
    return 0;
}

extern "C" int rqrcp_philox_words(rqrcp_ctx *ctx, const uint32_t *ctr, const uint32_t *key, uint32_t *out,
                                  int64_t count) {
    if (!ctx) return -1;
    if (!ctr) return -2;
    if (!key) return -3;
    if (!out) return -4;
    if (count < 0) return -5;
    if (count == 0) return 0;
    CK(cudaSetDevice(ctx->device));
    philox_words_kernel<<<(unsigned)((count + 255) / 256), 256, 0, ctx->stream>>>(ctr, make_uint2(key[0], key[1]), out,
                                                                                  count);
    CKL();
    CK(cudaStreamSynchronize(ctx->stream));
    return 0;
}
