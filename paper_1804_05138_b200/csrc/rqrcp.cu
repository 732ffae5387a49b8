// rqrcp.cu -- the C ABI (include/rqrcp.h) and the host driver of the RQRCP
// hot path (Alg. 2).  The driver only enqueues kernels and
// collectives on the context's streams (no host synchronisation inside the
// panel loop: pivots, swap lists and rank-stop state stay on the device) and
// synchronises once at the end for the status.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "rqrcp.h"
#include "common.cuh"
#include "gemm_dmma.cuh"
#include "gemm_tma.cuh"
#include "misc.cuh"
#include "moves.cuh"
#include "panel.cuh"
#include "panel_cl.cuh"
#include "philox.cuh"
#include "sample_qrcp.cuh"
#include "sample_qrcp_cl.cuh"
#include "sample_qrcp_reg.cuh"
#include "sample_qrcp_reg2.cuh"
#include "tri.cuh"
#include "cqr.cuh"
#include "dist.cuh"
#include "transport.cuh"
#include "tournament.cuh"
#include "srqr.cuh"
#include "lowrank.cuh"
#include "cqr_rg.cuh"

using namespace rq;

static inline int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

enum Phase { PH_OMEGA, PH_SKETCH, PH_SQRCP, PH_SWAP, PH_PANEL, PH_TRAIL, PH_SUPD, PH_COMM, PH_N };

// Launch-path options (rqrcp_set_option; environment RQRCP_<NAME> at create).
struct Opts {
    int schedule = -1;       // -1 auto, 0 serial, 1 bulk || next sample QRCP, 2 bulk || next panel (look-ahead)
    int panel = 2;           // 0 Householder columns, 1 CholeskyQR2 + reconstruction, 2 CholeskyQR2 from 8192 rows (measured: C3-C5)
    int pn_cluster = 1, pn_cpt = 2, pn_grid = 0, pn_rows = 128, la_panel_ctas = 48;
    int gemm_ws = 1;         // skinny TMA GEMMs (sketch, W): 1 warp-specialised, 0 CTA-barrier ring
    int tournament = 0;      // > 1: tournament pivoting on the sample over this many column groups (reading R-TP)
    int pn_blocked = 1;      // grid panel on 32-column sub-panels + in-panel DMMA updates: 0 never, 1 when
                             // a CTA's rows do not fit shared memory, 2 always
    int upd_kernel = 2;      // update GEMM: 0 CTA-wide TMA epilogue, 1 / 2 warp-specialised (BK 32 x 2 / 16 x 4 stages)
    int sq_cluster = 1, sq_reg = 1, sq_grid = 0, sq_nsm = -1, sq_hstride = 8, sq_poll = 3;
    int debug_sync = 0, trace = 0, trace_panel = 1;
    int sq_wide = 1;         // register-grid sample QRCP on every SM for wide samples (0: the fewest CTAs; 2: always)
    int sq_smtop = 1;        // register-grid sample QRCP: shared-memory rows above the register rows (they drop out
                             // of the per-step traffic as the panel advances); 0: below
    int sq_spec = 0;         // register-grid sample QRCP: 1 fetch the best arrived candidate's column while the
                             // last headers arrive (measured slower: C4 S2 51.0 vs 46.8 ms), 0 after every header
    int cqr_rg = 1;          // CholeskyQR2 panel: 1 register-grid one-CTA factorizations (cqr_rg.cuh), 0 shared-memory
    int host_out = 0;        // rqrcp_factor_host output: 0 the whole factored A, 1 the factors only (columns
                             // 0..k-1 full height = V and R11, rows 0..k-1 of columns k..n-1 = R12; R22 not copied)
    int64_t nccl_timeout_ms = 600000;
};
struct OptDesc {
    const char *name;
    int64_t lo, hi;
};
static const OptDesc kOpts[] = {{"schedule", -1, 2},     {"panel", 0, 2},     {"pn_cluster", 0, 1},
                                {"pn_cpt", 1, 2},        {"pn_grid", 0, 4096}, {"pn_rows", 1, 1 << 20},
                                {"la_panel_ctas", 1, 4096}, {"sq_cluster", 0, 1}, {"sq_reg", 0, 2},
                                {"sq_grid", 0, 4096},    {"sq_nsm", -1, 1 << 20}, {"sq_hstride", 1, 8},
                                {"sq_poll", 0, 3},       {"debug_sync", 0, 1}, {"trace", 0, 1},
                                {"trace_panel", 1, 1 << 30}, {"nccl_timeout_ms", 1, (int64_t)1 << 40},
                                {"upd_kernel", 0, 2}, {"pn_blocked", 0, 2},
                                {"tournament", 0, 64}, {"gemm_ws", 0, 1}, {"host_out", 0, 1}, {"cqr_rg", 0, 1}, {"sq_wide", 0, 2},
                                {"sq_smtop", 0, 1}, {"sq_spec", 0, 1}};
static bool opt_set(Opts &o, const std::string &n, int64_t v) {
#define OPT(field)                    \
    if (n == #field) {                \
        o.field = (decltype(o.field))v; \
        return true;                  \
    }
    OPT(schedule) OPT(panel) OPT(pn_cluster) OPT(pn_cpt) OPT(pn_grid) OPT(pn_rows) OPT(la_panel_ctas)
    OPT(sq_cluster) OPT(sq_reg) OPT(sq_grid) OPT(sq_nsm) OPT(sq_hstride) OPT(sq_poll) OPT(debug_sync) OPT(trace)
    OPT(trace_panel) OPT(nccl_timeout_ms) OPT(upd_kernel) OPT(pn_blocked) OPT(tournament) OPT(gemm_ws) OPT(host_out) OPT(cqr_rg) OPT(sq_wide) OPT(sq_smtop) OPT(sq_spec)
#undef OPT
    return false;
}

struct rqrcp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // concurrent small kernels (tri_kernel)
    cudaStream_t upd = nullptr;   // the bulk trailing update (lowest priority)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_r12 = nullptr, ev_upd = nullptr, ev_pack = nullptr,
                ev_h2d = nullptr;
    cudaStream_t cps = nullptr;   // host <-> device copies of the end-to-end path
    int grid_cap = 0;  // > 0: persistent GEMM grids use at most this many CTAs
    int *tctr = nullptr;  // per-panel tile counters of the dynamically scheduled bulk update
    bool own_stream = false;
    int nranks = 1, rank = 0;
    std::unique_ptr<Transport> tr;
    int64_t max_m = 0, max_n = 0;
    int max_b = 0, max_p = 0;
    int lpad_max = 0, bpad_max = 0;
    int64_t ldo = 0;  // leading dim of Omega^T, V and the panel buffers (= round8(max_m))
    int num_sms = 0;
    Opts opt;
    std::string err;
    // workspace
    double *omt = nullptr;                 // Omega^T  ldo x lpad_max
    double *bs[2] = {nullptr, nullptr};    // samples lpad_max x max_n
    double *vfull_b[2] = {nullptr, nullptr};  // V (ldv x bpad), double buffered for the look-ahead
    double *vt_b[2] = {nullptr, nullptr};     // V^T (bpad x max_m)
    double *w = nullptr, *w2 = nullptr;    // bpad_max x max_n
    double *w2g = nullptr;                 // bpad x bpad: W2 columns of the next panel's pivots
    double *tneg = nullptr, *rhat11 = nullptr, *omhat = nullptr, *ybuf = nullptr;  // bpad_max^2
    double *vhat = nullptr;    // lpad_max x bpad_max
    double *tauhat = nullptr;
    double *splitk = nullptr;
    int64_t splitk_elems = 0;
    double *pbuf = nullptr;    // the panel's columns, full height (ldo x bpad)
    double *packbuf = nullptr; // P > 1: this rank's contribution to pbuf (ldo x bpad)
    double *dispbuf = nullptr; // P > 1: the owner's displaced slot columns (ldo x bpad)
    double *colss = nullptr, *ptol2 = nullptr;  // R11-diagonal stop scale
    double *ybs = nullptr, *tns = nullptr, *wsub = nullptr, *w2sub = nullptr;  // blocked panel scratch
    int *subeff = nullptr;
    // tournament pivoting scratch (tournament.cuh)
    int64_t *tp_cand = nullptr, *tp_perm = nullptr, *tp_idx = nullptr, *tp_piv = nullptr, *tp_sd = nullptr,
            *tp_ss = nullptr;
    int *tp_cnt = nullptr, *tp_ints = nullptr;
    double *tp_w = nullptr, *tp_w2 = nullptr;  // W / W2 of the Q-hat^T application (S5's W2 may still be in use)
    double *tp_u = nullptr, *tp_tau = nullptr, *tp_vhat = nullptr, *tp_r11 = nullptr, *tp_vt = nullptr, *tp_y = nullptr,
           *tp_tn = nullptr;
    int *stopc = nullptr;      // panel kernels: the R11-diagonal stop column (-1: none)
    SqHdr *slot_hdr = nullptr;
    int *slot_col = nullptr;
    unsigned launch_seq = 0;
    double *slot_v2 = nullptr, *slot_data = nullptr;
    uint4 *sq_ll = nullptr;
    double *sq_spill = nullptr;
    int64_t spill_cap = 0;  // doubles in sq_spill
    double *pn_part = nullptr, *pn_rowj = nullptr;
    double *cq_g = nullptr, *cq_rc = nullptr, *cq_rinv = nullptr, *cq_uinv = nullptr, *cq_lu = nullptr,
           *cq_c = nullptr, *cq_q = nullptr;
    int *cqr_status = nullptr;
    bool cqr_enabled = true;
    double *swap_stage = nullptr;
    int64_t *swap_dst = nullptr, *swap_src = nullptr, *swap_jstage = nullptr;
    int *swap_np = nullptr;
    int64_t *perm = nullptr, *piv = nullptr;
    double *sumsq_part = nullptr;
    // device scalars: [0] status [1] bb_eff [2] done [3] rank [4] householder panels [5] srqr iota [6] form_q1
    int *iscal = nullptr;
    double *stop_tol2 = nullptr;
    unsigned *bars = nullptr;
    int update_rule = 1;
    double *bpre = nullptr, *c5 = nullptr, *wom = nullptr, *w2om = nullptr;
    int64_t nbars = 0;
    // host-path buffer (lazily allocated)
    double *a_dev = nullptr;
    int64_t a_dev_elems = 0;
    int64_t *jpvt_dev = nullptr;
    double *tau_dev = nullptr;
    int sqc_max = 0, pnc_max = 0;
    // multi-GPU exchange buffers
    double *gsend = nullptr, *gbuf = nullptr, *pack = nullptr;
    int64_t gbuf_elems = 0;
    // timing
    bool timing = true;
    cudaEvent_t ev[2 * 4096 + 8];
    int nev = 0;
    int open_phase = -1, open_ev = -1;
    std::vector<int> rec_phase, rec_s, rec_e;
    rqrcp_timings last{};
    int lt_t0 = -1, lt_t1 = -1;
    int *hstatus = nullptr;
    int64_t launches = 0;
    unsigned long long *trace = nullptr;
    unsigned long long *ptrace = nullptr;
    int ptrace_kind = 0;
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
        if (e_ == cudaSuccess && ctx->opt.debug_sync) e_ = cudaDeviceSynchronize();   \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string("kernel launch #") + std::to_string(ctx->launches) + \
                       " (line " + std::to_string(__LINE__) + "): " + cudaGetErrorString(e_); \
            return RQRCP_E_CUDA;                                                      \
        }                                                                             \
        ctx->launches++;                                                              \
    } while (0)

#define CKT(call)                                 \
    do {                                          \
        int r_ = (call);                          \
        if (r_) return r_;                        \
    } while (0)

static constexpr int kDynSmemMax = 200 * 1024;
static constexpr int kPanelSub = 32;
static constexpr int kTpMaxGroups = 64;  // tournament pivoting: column groups  // blocked grid panel: sub-panel width (columns factored per kernel)
static constexpr int64_t kCqrMinRows = 8192;

static int grid_for(int64_t total, int threads, int num_sms) {
    int64_t g = (total + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms * 8));
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, so a context on another GPU of the same process
// sets it again.
static std::mutex g_attr_mu;
static std::set<std::tuple<const void *, int, int>> g_attr_done;
static cudaError_t smem_attr(const void *kern, int bytes, int device) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto key = std::make_tuple(kern, device, bytes);
    if (g_attr_done.count(key)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) g_attr_done.insert(key);
    return e;
}

// ---------------------------------------------------------------------------
// GEMM dispatch: C = X^T Y (see gemm_dmma.cuh), M small (skinny) or large.
// Split-K is CANONICAL: the number of K slices depends only on (M, K, the
// global N), never on a rank's column count, so every contraction's
// per-element summation order -- hence every bit of the result -- is the same
// for any number of ranks (SURVEY.md §8(e) "Determinism across P").
// ---------------------------------------------------------------------------
template <int MT, int NT, int WM, int WN, int BK, int ST, int EPI>
static int launch_tn_cfg(rqrcp_ctx *ctx, GemmArgs g, int splits) {
    constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
    const size_t smem = (size_t)ST * BK * (BM + BN) * sizeof(double);
    auto kern = gemm_tn_kernel<MT, NT, WM, WN, BK, ST, EPI>;
    CK(smem_attr((const void *)kern, (int)smem, ctx->device));
    dim3 grid((unsigned)((g.N + BN - 1) / BN), (unsigned)((g.M + BM - 1) / BM), (unsigned)splits);
    kern<<<grid, WM * WN * 32, smem, ctx->stream>>>(g);
    CKL();
    return 0;
}

// splits minimising ceil(T*S / grid) / S (persistent-grid wave quantisation);
// T = tiles of the GLOBAL problem (canonical, see above)
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

template <int MT, int NT, int WM, int WN>
static int launch_skinny(rqrcp_ctx *ctx, int64_t M, int64_t N, int64_t K, const double *X, int64_t ldx,
                         const double *Y, int64_t ldy, double *C, int64_t ldc, int64_t Ncanon) {
    constexpr int BK = 32, ST = 3;
    constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
    const int64_t tiles = ((Ncanon + BN - 1) / BN) * ((M + BM - 1) / BM);
    int64_t splits = std::max<int64_t>(1, (2 * (int64_t)ctx->num_sms + tiles - 1) / tiles);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / 256));
    while (splits > 1 && splits * M * Ncanon > ctx->splitk_elems) --splits;
    int64_t kps = rup((K + splits - 1) / splits, BK);
    splits = (K + kps - 1) / kps;
    GemmArgs g{M, N, K, X, ldx, Y, ldy, C, ldc, kps, M * N};
    if (splits <= 1) {
        g.k_per_split = rup(std::max<int64_t>(K, 1), BK);
        return launch_tn_cfg<MT, NT, WM, WN, BK, ST, EPI_STORE>(ctx, g, 1);
    }
    g.C = ctx->splitk;
    CKT((launch_tn_cfg<MT, NT, WM, WN, BK, ST, EPI_PARTIAL>(ctx, g, (int)splits)));
    splitk_reduce_kernel<<<grid_for(M * N, 256, ctx->num_sms), 256, 0, ctx->stream>>>(ctx->splitk, M, N, (int)splits,
                                                                                      M * N, C, ldc);
    CKL();
    return 0;
}

// C (M x N) = X^T Y with M <= 144 rows (sample rows l_pad or panel width).
static int gemm_skinny(rqrcp_ctx *ctx, int64_t M, int64_t N, int64_t K, const double *X, int64_t ldx,
                       const double *Y, int64_t ldy, double *C, int64_t ldc, int64_t Ncanon = -1) {
    if (N <= 0) return 0;
    if (Ncanon < 0) Ncanon = N;
    if (M <= 32) return launch_skinny<4, 2, 1, 4>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc, Ncanon);
    if (M <= 40) return launch_skinny<5, 2, 1, 4>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc, Ncanon);
    if (M <= 64) return launch_skinny<4, 4, 2, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc, Ncanon);
    if (M <= 80) return launch_skinny<5, 4, 2, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc, Ncanon);
    if (M <= 128) return launch_skinny<4, 4, 4, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc, Ncanon);
    if (M <= 144) return launch_skinny<6, 4, 3, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc, Ncanon);
    return launch_skinny<4, 4, 4, 2>(ctx, M, N, K, X, ldx, Y, ldy, C, ldc, Ncanon);  // grid.y tiles M
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
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    return fn;
}

// 2-D map over a column-major matrix (dim0 = rows = K direction, contiguous),
// box {8 doubles, box1 columns}; out-of-range elements read as zero.
static bool make_tmap(CUtensorMap *m, const double *base, int64_t dim0, int64_t dim1, int64_t ld, int box1) {
    auto enc = tma_encode_fn();
    if (!enc || ((uintptr_t)base & 15) || ((ld * 8) & 15) || dim0 < 1 || dim1 < 1) return false;
    cuuint64_t dims[2] = {(cuuint64_t)dim0, (cuuint64_t)dim1};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {8, (cuuint32_t)box1};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
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
    const int64_t tiles = ((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM) * g.splits;
    const int grid = (int)std::min<int64_t>(tiles, ctx->grid_cap > 0 ? ctx->grid_cap : ctx->num_sms);
    if (!DYN && (EPI == EPI_STORE || EPI == EPI_PARTIAL) && ctx->opt.gemm_ws) {
        // warp-specialised variant (producer warp, no CTA-wide barrier): same bits
        constexpr int WST = (4 * BK * (BM + BN) * 8 <= 200 * 1024) ? 4 : 3;
        const size_t smem = ws_gemm_smem<MT, NT, WM, WN, BK, WST>();
        auto kern = gemm_ws_kernel<MT, NT, WM, WN, BK, WST, EPI>;
        CK(smem_attr((const void *)kern, (int)smem, ctx->device));
        kern<<<grid, (WM * WN + 1) * 32, smem, ctx->stream>>>(tx, ty, g);
        CKL();
        *done = true;
        return 0;
    }
    const size_t smem = tma_gemm_smem<MT, NT, WM, WN, BK, ST>();
    auto kern = gemm_tma_kernel<MT, NT, WM, WN, BK, ST, EPI, DYN>;
    CK(smem_attr((const void *)kern, (int)smem, ctx->device));
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
                          int64_t kmin, int64_t Ncanon) {
    constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
    const int64_t tiles = ((Ncanon + BN - 1) / BN) * ((M + BM - 1) / BM);
    int splits = choose_splits(tiles, K, ctx->num_sms, M * Ncanon, ctx->splitk_elems, kmin);
    // a product with a few output tiles (the blocked panel's W_s and V^T V):
    // spread K over the whole GPU (the partials are small; the K-loop of a few
    // CTAs was latency-bound: 114 us for 32 x 96 x 32768 on 22 CTAs)
    if (tiles * 4 < ctx->num_sms) {
        const int64_t s2 = std::min<int64_t>(std::max<int64_t>(1, K / 128), ctx->num_sms / tiles);
        if (s2 > splits && s2 * M * Ncanon <= ctx->splitk_elems) splits = (int)s2;
    }
    int64_t kps = rup((K + splits - 1) / splits, 32);
    splits = (int)((K + kps - 1) / kps);
    TmaGemmArgs g{M, N, K, xk0, xm0, yk0, yn0, C, ldc, kps, splits, M * N, 0};
    if (splits <= 1) return launch_tma_cfg<MT, NT, WM, WN, EPI_STORE>(ctx, X, xdim0, xdim1, ldx, Y, ydim0, ydim1, ldy, g, done);
    g.C = ctx->splitk;
    CKT((launch_tma_cfg<MT, NT, WM, WN, EPI_PARTIAL>(ctx, X, xdim0, xdim1, ldx, Y, ydim0, ydim1, ldy, g, done)));
    if (!*done) return 0;
    splitk_reduce_kernel<<<grid_for(M * N, 256, ctx->num_sms), 256, 0, ctx->stream>>>(ctx->splitk, M, N, splits, M * N,
                                                                                      C, ldc);
    CKL();
    return 0;
}

static int tma_skinny(rqrcp_ctx *ctx, int64_t M, int64_t N, int64_t K, const double *X, int64_t xdim0, int64_t xdim1,
                      int64_t ldx, int64_t xk0, int64_t xm0, const double *Y, int64_t ydim0, int64_t ydim1, int64_t ldy,
                      int64_t yk0, int64_t yn0, double *C, int64_t ldc, bool *done, int64_t kmin = 512,
                      int64_t Ncanon = -1) {
    *done = false;
    if (N <= 0) { *done = true; return 0; }
    if (Ncanon < 0) Ncanon = N;
#define TS(a, b, c, d) \
    tma_skinny_cfg<a, b, c, d>(ctx, M, N, K, X, xdim0, xdim1, ldx, xk0, xm0, Y, ydim0, ydim1, ldy, yk0, yn0, C, ldc, done, kmin, Ncanon)
    if (M <= 32) return TS(4, 4, 1, 8);
    if (M <= 40) return TS(5, 4, 1, 8);
    if (M <= 64) return TS(4, 4, 2, 4);
    if (M <= 80) return TS(5, 4, 2, 4);
    if (M <= 128) return TS(4, 4, 4, 2);
    if (M <= 144) return TS(9, 2, 2, 4);  // 8 consumer warps (2 per sub-partition)
#undef TS
    return 0;
}

// A22 (rows x cols, lda) += V W2  as  A22^T += W2^T Vt  (TMA operands W2, Vt).
// For K > 64 the C tile is moved by TMA as well (gemm_upd_tma_kernel; needs a
// 16-byte aligned A22 with an even lda); else the register-epilogue kernel.
// Every variant computes each element as A + (sum over k, DMMA order): the
// same bits whichever rows / columns one launch covers.
static int tma_update(rqrcp_ctx *ctx, int64_t rows, int64_t cols, int64_t K, const double *w2, int64_t ldw,
                      const double *vt, int64_t ldvt, double *A22, int64_t lda, bool *done, int *tile_ctr = nullptr) {
    *done = false;
    if (rows <= 0 || cols <= 0) { *done = true; return 0; }
    // warp-specialised kernel (per-warp TMA epilogue, mbarrier ring): rows > 64
    const int uk = ctx->opt.upd_kernel;
    if (uk > 0 && rows > 64 && !tile_ctr && (((uintptr_t)A22 & 15) == 0) && ((lda & 1) == 0)) {
        CUtensorMap tx, ty, tc;
        if (make_tmap(&tx, w2, K, cols, ldw, 64) && make_tmap(&ty, vt, K, rows, ldvt, 128) &&
            make_tmap(&tc, A22, rows, cols, lda, 32)) {
            TmaGemmArgs g{cols, rows, K, 0, 0, 0, 0, A22, lda, rup(K, 32), 1, 0, 0};
            const int64_t tiles = ((rows + 127) / 128) * ((cols + 63) / 64);
            const int grid = (int)std::min<int64_t>(tiles, ctx->grid_cap > 0 ? ctx->grid_cap : ctx->num_sms);
            if (uk == 1) {
                const size_t smem = upd_ws_smem<2, 4, 32, 2>();
                auto kern = gemm_upd_ws_kernel<2, 4, 32, 2>;
                CK(smem_attr((const void *)kern, (int)smem, ctx->device));
                kern<<<grid, 9 * 32, smem, ctx->stream>>>(tx, ty, tc, g);
            } else {
                const size_t smem = upd_ws_smem<2, 4, 16, 4>();
                auto kern = gemm_upd_ws_kernel<2, 4, 16, 4>;
                CK(smem_attr((const void *)kern, (int)smem, ctx->device));
                kern<<<grid, 9 * 32, smem, ctx->stream>>>(tx, ty, tc, g);
            }
            CKL();
            *done = true;
            return 0;
        }
    }
    if (K > 64 && !tile_ctr && (((uintptr_t)A22 & 15) == 0) && ((lda & 1) == 0)) {
        constexpr int MT = 4, NT = 4, WM = 2, WN = 4, BK = 32, ST = 2;
        constexpr int BM = 8 * MT * WM, BN = 8 * NT * WN;
        CUtensorMap tx, ty, tc;
        if (make_tmap(&tx, w2, K, cols, ldw, BM) && make_tmap(&ty, vt, K, rows, ldvt, BN) &&
            make_tmap(&tc, A22, rows, cols, lda, BM)) {
            const size_t smem = tma_upd_smem<MT, NT, WM, WN, BK, ST>();
            auto kern = gemm_upd_tma_kernel<MT, NT, WM, WN, BK, ST>;
            CK(smem_attr((const void *)kern, (int)smem, ctx->device));
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
    // a short update (the R12 rows of the overlapped schedules): 32 x 64 tiles
    if (rows <= 64) return launch_tma_cfg<2, 4, 2, 2, EPI_ACCUM_T_PRE>(ctx, w2, K, cols, ldw, vt, K, rows, ldvt, g, done);
    if (tile_ctr) {  // dynamic tile claiming (the GPU is shared with a concurrent kernel)
        g.tile_ctr = tile_ctr;
        return launch_tma_cfg<4, 4, 2, 4, EPI_ACCUM_T_PRE, true>(ctx, w2, K, cols, ldw, vt, K, rows, ldvt, g, done);
    }
    return launch_tma_cfg<4, 4, 2, 4, EPI_ACCUM_T_PRE>(ctx, w2, K, cols, ldw, vt, K, rows, ldvt, g, done);
}

static int update_any(rqrcp_ctx *ctx, int64_t rows, int64_t cols, int64_t K, const double *w2, int64_t ldw,
                      const double *vt, int64_t ldvt, double *A22, int64_t lda, int *tile_ctr = nullptr) {
    bool dn = false;
    CKT(tma_update(ctx, rows, cols, K, w2, ldw, vt, ldvt, A22, lda, &dn, tile_ctr));
    if (!dn) CKT(gemm_update(ctx, rows, cols, K, w2, ldw, vt, ldvt, A22, lda));
    return 0;
}

// ---------------------------------------------------------------------------
// timing helpers: events recorded on the stream that runs the phase
// ---------------------------------------------------------------------------
static constexpr int kMaxEv = 2 * 4096 + 8;
static void ph_begin(rqrcp_ctx *ctx, int phase) {
    ctx->open_phase = -1;
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
// run f on stream s as the context stream (launch helpers use ctx->stream)
template <class F>
static int on_stream(rqrcp_ctx *ctx, cudaStream_t s, F f) {
    cudaStream_t keep = ctx->stream;
    ctx->stream = s;
    int rc = f();
    ctx->stream = keep;
    return rc;
}

// ---------------------------------------------------------------------------
// C ABI: small entry points
// ---------------------------------------------------------------------------
extern "C" const char *rqrcp_version(void) { return "rqrcp-b200 0.2 (sm_100a, fp64 DMMA, look-ahead)"; }

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

extern "C" int rqrcp_set_option(rqrcp_ctx *ctx, const char *name, int64_t value) {
    if (!ctx) return -1;
    if (!name) return -2;
    for (const OptDesc &d : kOpts)
        if (std::string(d.name) == name) {
            if (value < d.lo || value > d.hi) return -3;
            opt_set(ctx->opt, name, value);
            return 0;
        }
    return -2;
}

static void opts_from_env(Opts &o) {
    for (const OptDesc &d : kOpts) {
        std::string env = "RQRCP_";
        for (const char *c = d.name; *c; ++c) env += (char)toupper(*c);
        const char *v = getenv(env.c_str());
        if (!v || !*v) continue;
        int64_t x = 0;
        if (!strcmp(d.name, "panel")) x = (v[0] == 'h' || v[0] == 'H' || v[0] == '0') ? 0 : (v[0] == 'a' || v[0] == '2' ? 2 : 1);
        else x = atoll(v);
        if (x >= d.lo && x <= d.hi) opt_set(o, d.name, x);
    }
}

static int free_all(rqrcp_ctx *ctx) {
    ctx->tr.reset();
    if (ctx->hstatus) cudaFreeHost(ctx->hstatus);
    ctx->hstatus = nullptr;
    void *ptrs[] = {ctx->omt,       ctx->bs[0],     ctx->bs[1],      ctx->vfull_b[0], ctx->vfull_b[1], ctx->vt_b[0],
                    ctx->vt_b[1],   ctx->w,         ctx->w2,         ctx->w2g,        ctx->tneg,       ctx->ybuf,
                    ctx->rhat11,    ctx->omhat,     ctx->vhat,       ctx->tauhat,     ctx->splitk,     ctx->pbuf,
                    ctx->packbuf,   ctx->dispbuf,   ctx->colss,      ctx->ptol2,      ctx->stopc,      ctx->slot_hdr,
                    ctx->ybs,       ctx->tns,       ctx->wsub,       ctx->w2sub,      ctx->subeff,
                    ctx->tp_cand,   ctx->tp_perm,   ctx->tp_idx,     ctx->tp_piv,     ctx->tp_sd,      ctx->tp_ss,
                    ctx->tp_cnt,    ctx->tp_ints,   ctx->tp_u,       ctx->tp_tau,     ctx->tp_vhat,    ctx->tp_r11,
                    ctx->tp_vt,     ctx->tp_y,      ctx->tp_tn,      ctx->tp_w,       ctx->tp_w2,
                    ctx->slot_col,  ctx->slot_v2,   ctx->slot_data,  ctx->sq_ll,      ctx->sq_spill,   ctx->pn_part,
                    ctx->pn_rowj,   ctx->cq_g,      ctx->cq_rc,      ctx->cq_rinv,    ctx->cq_uinv,    ctx->cq_lu,    ctx->cq_c,    ctx->cq_q,
                    ctx->cqr_status, ctx->bpre,     ctx->c5,         ctx->wom,        ctx->w2om,       ctx->swap_stage,
                    ctx->swap_dst,  ctx->swap_src,  ctx->swap_jstage, ctx->swap_np,   ctx->perm,       ctx->piv,
                    ctx->sumsq_part, ctx->iscal,    ctx->stop_tol2,  ctx->bars,       ctx->trace,      ctx->ptrace,
                    ctx->a_dev,     ctx->jpvt_dev,  ctx->tau_dev,    ctx->tctr,       ctx->gsend,      ctx->gbuf,
                    ctx->pack};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    return 0;
}

static void destroy_events(rqrcp_ctx *ctx) {
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_join, ctx->ev_r12, ctx->ev_upd, ctx->ev_pack, ctx->ev_h2d})
        if (e) cudaEventDestroy(e);
    if (ctx->cps) cudaStreamDestroy(ctx->cps);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->upd) cudaStreamDestroy(ctx->upd);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
}

// Allocates every buffer; the transport is attached by the caller.
static int create_impl(rqrcp_ctx **out, const rqrcp_config *cfg, int nranks, int rank, bool own_stream_forced) {
    if (!out) return -1;
    *out = nullptr;
    if (!cfg || cfg->max_m < 1 || cfg->max_n < 1 || cfg->max_b < 1 || cfg->max_b > 128 || cfg->max_p < 0 ||
        cfg->max_b + cfg->max_p > SQ_MAXL || nranks < 1 || rank < 0 || rank >= nranks)
        return -2;
    rqrcp_ctx *ctx = new rqrcp_ctx();
    for (auto &e : ctx->ev) e = nullptr;
    ctx->device = cfg->device;
    ctx->nranks = nranks;
    ctx->rank = rank;
    ctx->max_m = cfg->max_m;
    ctx->max_n = cfg->max_n;
    ctx->max_b = cfg->max_b;
    ctx->max_p = cfg->max_p;
    opts_from_env(ctx->opt);
    const bool want_trace = ctx->opt.trace != 0;
    auto fail = [&](int code) {
        free_all(ctx);
        destroy_events(ctx);
        delete ctx;
        return code;
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
    int prio_lo = 0, prio_hi = 0;
    CKC(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    if (cfg->stream && !own_stream_forced) {
        ctx->stream = (cudaStream_t)cfg->stream;
    } else {
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
    for (int q = 0; q < 2; ++q) {
        CKC(dalloc(&ctx->vfull_b[q], ctx->ldo * bp));
        CKC(dalloc(&ctx->vt_b[q], bp * mm));
    }
    CKC(dalloc(&ctx->w, bp * nn));
    CKC(dalloc(&ctx->w2, bp * nn));
    CKC(dalloc(&ctx->w2g, bp * bp));
    CKC(dalloc(&ctx->tneg, bp * bp));
    CKC(dalloc(&ctx->rhat11, bp * bp));
    CKC(dalloc(&ctx->ybuf, bp * bp));
    CKC(dalloc(&ctx->omhat, bp * bp));
    CKC(dalloc(&ctx->vhat, lp * bp));
    CKC(dalloc(&ctx->tauhat, bp));
    // split-K partials: up to 8 slices of the widest skinny product (W = V^T A22,
    // the sketch) so the wave-quantisation choice is never capped by space
    ctx->splitk_elems = std::max<int64_t>(4 << 20, 8 * std::max<int64_t>(bp, lp) * nn);
    CKC(dalloc(&ctx->splitk, ctx->splitk_elems));
    CKC(dalloc(&ctx->pbuf, ctx->ldo * bp));
    if (nranks > 1) {
        CKC(dalloc(&ctx->packbuf, ctx->ldo * bp));
        CKC(dalloc(&ctx->dispbuf, ctx->ldo * bp));
    }
    CKC(dalloc(&ctx->colss, bp));
    CKC(dalloc(&ctx->ptol2, 1));
    CKC(cudaMalloc((void **)&ctx->stopc, sizeof(int)));
    CKC(dalloc(&ctx->ybs, kPanelSub * kPanelSub));
    CKC(dalloc(&ctx->tns, kPanelSub * kPanelSub));
    CKC(cudaMemset(ctx->tns, 0, sizeof(double) * kPanelSub * kPanelSub));
    CKC(dalloc(&ctx->wsub, kPanelSub * bp));
    CKC(dalloc(&ctx->w2sub, kPanelSub * bp));
    CKC(cudaMalloc((void **)&ctx->subeff, sizeof(int)));
    CKC(cudaMalloc((void **)&ctx->tp_cand, sizeof(int64_t) * kTpMaxGroups * bp));
    CKC(cudaMalloc((void **)&ctx->tp_perm, sizeof(int64_t) * std::max<int64_t>(nn, 2 * bp)));
    CKC(cudaMalloc((void **)&ctx->tp_idx, sizeof(int64_t) * std::max<int64_t>(nn, 2 * bp)));
    CKC(cudaMalloc((void **)&ctx->tp_piv, sizeof(int64_t) * bp));
    CKC(cudaMalloc((void **)&ctx->tp_sd, sizeof(int64_t) * 4 * bp));
    CKC(cudaMalloc((void **)&ctx->tp_ss, sizeof(int64_t) * 4 * bp));
    CKC(cudaMalloc((void **)&ctx->tp_cnt, sizeof(int) * kTpMaxGroups));
    CKC(cudaMalloc((void **)&ctx->tp_ints, sizeof(int) * 8));
    CKC(dalloc(&ctx->tp_u, lp * 2 * bp));
    CKC(dalloc(&ctx->tp_w, bp * nn));
    CKC(dalloc(&ctx->tp_w2, bp * nn));
    CKC(dalloc(&ctx->tp_tau, bp));
    CKC(dalloc(&ctx->tp_vhat, lp * bp));
    CKC(dalloc(&ctx->tp_r11, bp * bp));
    CKC(dalloc(&ctx->tp_vt, bp * lp));
    CKC(dalloc(&ctx->tp_y, bp * bp));
    CKC(dalloc(&ctx->tp_tn, bp * bp));
    CKC(cudaMalloc((void **)&ctx->slot_hdr, sizeof(SqHdr) * 2 * SQ_MAXG * 8));
    CKC(cudaMemset(ctx->slot_hdr, 0, sizeof(SqHdr) * 2 * SQ_MAXG * 8));
    CKC(cudaMalloc((void **)&ctx->slot_col, sizeof(int) * 2 * G));
    CKC(dalloc(&ctx->slot_v2, 2 * G));
    CKC(dalloc(&ctx->slot_data, 2 * G * lp));
    CKC(cudaMalloc((void **)&ctx->sq_ll, sizeof(uint4) * 2 * SQ_MAXG * SQS_UNITS));
    CKC(cudaMemset(ctx->sq_ll, 0, sizeof(uint4) * 2 * SQ_MAXG * SQS_UNITS));
    CKC(dalloc(&ctx->sq_spill, lp * nn));
    ctx->spill_cap = lp * nn;
    CKC(dalloc(&ctx->bpre, lp * nn));
    CKC(dalloc(&ctx->c5, lp * nn));
    CKC(dalloc(&ctx->wom, bp * lp));
    CKC(dalloc(&ctx->w2om, bp * lp));
    CKC(dalloc(&ctx->pn_part, 2 * G * bp));
    CKC(dalloc(&ctx->pn_rowj, 2 * bp));
    for (double **q : {&ctx->cq_g, &ctx->cq_rc, &ctx->cq_rinv, &ctx->cq_uinv, &ctx->cq_lu, &ctx->cq_c, &ctx->cq_q})
        CKC(dalloc(q, bp * bp));
    CKC(cudaMalloc((void **)&ctx->cqr_status, sizeof(int)));
    CKC(cudaMemset(ctx->cqr_status, 0xff, sizeof(int)));
    CKC(dalloc(&ctx->swap_stage, 2 * bp * mm));
    CKC(cudaMalloc((void **)&ctx->swap_dst, sizeof(int64_t) * 2 * bp));
    CKC(cudaMalloc((void **)&ctx->swap_src, sizeof(int64_t) * 2 * bp));
    CKC(cudaMalloc((void **)&ctx->swap_jstage, sizeof(int64_t) * 2 * bp));
    CKC(cudaMalloc((void **)&ctx->swap_np, sizeof(int)));
    CKC(cudaMemset(ctx->swap_np, 0, sizeof(int)));
    CKC(cudaMalloc((void **)&ctx->perm, sizeof(int64_t) * nn));
    CKC(cudaMalloc((void **)&ctx->piv, sizeof(int64_t) * bp));
    CKC(dalloc(&ctx->sumsq_part, 4 * G));
    CKC(cudaMalloc((void **)&ctx->iscal, sizeof(int) * 8));
    CKC(dalloc(&ctx->stop_tol2, 1));
    ctx->nbars = 2 * std::min(cfg->max_m, cfg->max_n) + 16;
    CKC(cudaMalloc((void **)&ctx->bars, sizeof(unsigned) * ctx->nbars));
    CKC(cudaMemset(ctx->bars, 0, sizeof(unsigned) * ctx->nbars));
    CKC(cudaMemset(ctx->tneg, 0, sizeof(double) * bp * bp));
    const int dev = ctx->device;
    CKC(smem_attr((const void *)sample_qrcp_kernel, kDynSmemMax, dev));
    CKC(smem_attr((const void *)panel_qr_kernel<4>, kDynSmemMax, dev));
    CKC(smem_attr((const void *)panel_qr_kernel<8>, kDynSmemMax, dev));
    CKC(smem_attr((const void *)sample_qrcp_reg_kernel<40, 0>, 128 * 40 * 8, dev));
    CKC(smem_attr((const void *)sample_qrcp_reg_kernel<74, 0>, 128 * 74 * 8, dev));
    CKC(smem_attr((const void *)sample_qrcp_reg_kernel<72, 72>, 128 * 144 * 8, dev));
    CKC(smem_attr((const void *)sample_qrcp_reg_kernel<72, 72, true>, 128 * 144 * 8, dev));
    CKC(smem_attr((const void *)sample_qrcp_reg2_kernel<60, 32, 52>, 52 * SQR2_THREADS * 8, dev));
    CKC(smem_attr((const void *)sample_qrcp_reg2_kernel<60, 32, 52, true>, 52 * SQR2_THREADS * 8, dev));
    for (const void *k : {(const void *)sample_qrcp_cluster_kernel<40>, (const void *)sample_qrcp_cluster_kernel<74>,
                          (const void *)sample_qrcp_cluster_kernel<80>}) {
        CKC(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    CKC(smem_attr((const void *)sample_qrcp_cluster_kernel<40>, 128 * 40 * 8, dev));
    CKC(smem_attr((const void *)sample_qrcp_cluster_kernel<74>, 128 * 74 * 8, dev));
    CKC(smem_attr((const void *)sample_qrcp_cluster_kernel<80>, 128 * 80 * 8, dev));
    CKC(smem_attr((const void *)cqr_chol_kernel, (int)cqr_smem_bytes(128), dev));
    CKC(smem_attr((const void *)cqr_recon_kernel, (int)cqr_smem_bytes(128), dev));
    CKC(smem_attr((const void *)cqr_chol_rg_kernel<128>, (int)cqr_rg_smem_bytes(128), dev));
    CKC(smem_attr((const void *)cqr_chol_rg_kernel<64>, (int)cqr_rg_smem_bytes(64), dev));
    CKC(smem_attr((const void *)cqr_recon_rg_kernel<128>, (int)cqr_rg_smem_bytes(128), dev));
    CKC(smem_attr((const void *)cqr_recon_rg_kernel<64>, (int)cqr_rg_smem_bytes(64), dev));
    CKC(smem_attr((const void *)cqr_rowmul_kernel, 128 * 132 * 8, dev));
    CKC(smem_attr((const void *)cqr_rowmul2_kernel, 128 * 132 * 8, dev));
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
    for (const void *k : {(const void *)panel_qr_cluster_kernel<32, 64>, (const void *)panel_qr_cluster_kernel<64, 64>,
                          (const void *)panel_qr_cluster_kernel<64, 32, 2>})
        CKC(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CKC(smem_attr((const void *)panel_qr_cluster_kernel<32, 64>, 32 * 65 * 8, dev));
    CKC(smem_attr((const void *)panel_qr_cluster_kernel<64, 64>, 64 * 65 * 8, dev));
    CKC(smem_attr((const void *)panel_qr_cluster_kernel<64, 32, 2>, 64 * 64 * 8, dev));
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
    CKC(smem_attr((const void *)tri_kernel, (int)tri_smem_bytes(128), dev));
    CKC(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithPriority(&ctx->upd, cudaStreamNonBlocking, prio_lo));
    CKC(cudaMallocHost((void **)&ctx->hstatus, sizeof(int) * 8));
    CKC(cudaMalloc((void **)&ctx->tctr, sizeof(int) * 8192));
    for (cudaEvent_t *e : {&ctx->ev_r12, &ctx->ev_upd, &ctx->ev_fork, &ctx->ev_join, &ctx->ev_pack, &ctx->ev_h2d})
        CKC(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CKC(cudaStreamCreateWithFlags(&ctx->cps, cudaStreamNonBlocking));
    for (auto &e : ctx->ev) CKC(cudaEventCreate(&e));
    if (nranks > 1) {
        CKC(dalloc(&ctx->gsend, lp * (nn + bp)));
        ctx->gbuf_elems = lp * (nn + (int64_t)nranks * bp);
        CKC(dalloc(&ctx->gbuf, ctx->gbuf_elems));
        CKC(dalloc(&ctx->pack, bp + 3 * bp * bp + 4));
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

extern "C" int rqrcp_create(rqrcp_ctx **out, const rqrcp_config *cfg) {
    if (!out) return -1;
    if (!cfg) return -2;
    if (cfg->nranks > 1 && !nccl().ok) return RQRCP_E_UNSUPPORTED;
    int rc = create_impl(out, cfg, cfg->nranks, cfg->rank, false);
    if (rc) return rc;
    rqrcp_ctx *ctx = *out;
    if (cfg->nranks > 1) {
        auto t = std::make_unique<NcclTransport>();
        t->nranks = cfg->nranks;
        t->rank = cfg->rank;
        ncclUniqueId uid;
        memcpy(uid.internal, cfg->nccl_uid, sizeof(uid.internal));
        if (nccl().CommInitRank(&t->comm, cfg->nranks, uid, cfg->rank) != 0) {
            fprintf(stderr, "rqrcp_create: ncclCommInitRank failed\n");
            t->comm = nullptr;
            rqrcp_destroy(ctx);
            *out = nullptr;
            return RQRCP_E_NCCL;
        }
        ctx->tr = std::move(t);
    }
    return 0;
}

extern "C" int rqrcp_create_loopback_group(rqrcp_ctx **ctxs, int nranks, const rqrcp_config *cfg) {
    if (!ctxs) return -1;
    if (!cfg || nranks < 2 || nranks > LOOP_MAXP) return -2;
    for (int r = 0; r < nranks; ++r) ctxs[r] = nullptr;
    if (cudaSetDevice(cfg->device) != cudaSuccess) return RQRCP_E_CUDA;
    auto grp = std::make_shared<LoopGroup>(nranks);
    for (int r = 0; r < nranks; ++r) {
        int rc = create_impl(&ctxs[r], cfg, nranks, r, true);
        if (rc) {
            for (int q = 0; q < r; ++q) {
                rqrcp_destroy(ctxs[q]);
                ctxs[q] = nullptr;
            }
            return rc;
        }
        auto t = std::make_unique<LoopTransport>();
        t->nranks = nranks;
        t->rank = r;
        t->grp = grp;
        ctxs[r]->tr = std::move(t);
    }
    return 0;
}

extern "C" int rqrcp_destroy(rqrcp_ctx *ctx) {
    if (!ctx) return 0;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    free_all(ctx);
    destroy_events(ctx);
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
    if (ctx->opt.debug_sync) {
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            ctx->err = std::string("cooperative kernel: ") + cudaGetErrorString(e);
            return RQRCP_E_CUDA;
        }
    }
    ctx->launches++;
    return 0;
}

static int cluster_launch(rqrcp_ctx *ctx, void (*kfn)(SqArgs), int cs, int threads, size_t smem, SqArgs a) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(cs);
    lc.blockDim = dim3(threads);
    lc.dynamicSmemBytes = smem;
    lc.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, kfn, a));
    CKL();
    return 0;
}

__global__ void iota_kernel(int64_t *x, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        x[e] = e;
}

// ---------------------------------------------------------------------------
// The instantiated sample-QRCP kernels (one table: dispatch and schedule
// choice read the same entries).  Samples of other heights run on the generic
// cooperative kernel (sample_qrcp.cuh), measured 2-4x slower per pivot.
// ---------------------------------------------------------------------------
struct SqKernels {
    void (*cluster)(SqArgs);
    void (*reg)(SqArgs);
    int reg_ls;  // rows of the register-grid kernel kept in shared memory
    void (*reg2)(SqArgs);  // 512-thread register grid with the top rows in global memory
    int reg2_lt, reg2_ls;
};
static SqKernels sq_kernels(int l, bool smtop = true) {
    if (l == 40) return {sample_qrcp_cluster_kernel<40>, sample_qrcp_reg_kernel<40, 0>, 0, nullptr, 0, 0};
    if (l == 74) return {sample_qrcp_cluster_kernel<74>, sample_qrcp_reg_kernel<74, 0>, 0, nullptr, 0, 0};
    if (l == 80) return {sample_qrcp_cluster_kernel<80>, nullptr, 0, nullptr, 0, 0};
    if (l == 144) {
        if (smtop)
            return {nullptr, sample_qrcp_reg_kernel<72, 72, true>, 72, sample_qrcp_reg2_kernel<60, 32, 52, true>, 60,
                    52};
        return {nullptr, sample_qrcp_reg_kernel<72, 72>, 72, sample_qrcp_reg2_kernel<60, 32, 52>, 60, 52};
    }
    return {nullptr, nullptr, 0, nullptr, 0, 0};
}
enum SqKind { SQK_CLUSTER = 0, SQK_REG = 1, SQK_GRID = 2, SQK_REG2 = 3 };
static int sq_reg2_grid(int64_t np) { return 1 + (int)((np + SQR2_THREADS - 1) / SQR2_THREADS); }
// Launch grid of the register-grid kernels: the fewest CTAs that hold the
// sample (one column per thread) -- or, for wide samples that fit, every SM
// (fewer columns per CTA: less per-step apply work on each SM; the exchange
// polls one header per CTA either way).  Decided from (np, SM count) only.
static int sq_reg_launch_grid(const rqrcp_ctx *ctx, int64_t np, int threads) {
    const int base = 1 + (int)((np + threads - 1) / threads);
    const int cap = std::min(ctx->num_sms, SQR_MAXG);
    if (ctx->opt.sq_wide && base <= cap && (np >= (int64_t)64 * cap || ctx->opt.sq_wide == 2)) return cap;
    return base;
}
static SqKind sq_kind(const rqrcp_ctx *ctx, int l, int64_t np) {
    const SqKernels k = sq_kernels(l);
    const int64_t need = (np + SQC_THREADS - 1) / SQC_THREADS;
    if (ctx->opt.sq_cluster && k.cluster && need <= ctx->sqc_max) return SQK_CLUSTER;
    const int grid = 1 + (int)((np + SQR_THREADS - 1) / SQR_THREADS);
    const int cap = std::min(ctx->num_sms, SQR_MAXG);  // (register grids; the generic kernel takes SQ_MAXG)
    if (ctx->opt.sq_reg == 1 && k.reg && grid <= cap) return SQK_REG;
    // wider samples: the 512-thread register grid (top rows in the spill scratch)
    if (ctx->opt.sq_reg && k.reg2 && sq_reg2_grid(np) <= cap &&
        (int64_t)sq_reg_launch_grid(ctx, np, SQR2_THREADS) * k.reg2_lt * SQR2_THREADS <= ctx->spill_cap)
        return SQK_REG2;
    return SQK_GRID;
}
static int sq_ctas(const rqrcp_ctx *ctx, int l, int64_t np) {
    switch (sq_kind(ctx, l, np)) {
        case SQK_CLUSTER: return (int)std::max<int64_t>(1, (np + SQC_THREADS - 1) / SQC_THREADS);
        case SQK_REG: return sq_reg_launch_grid(ctx, np, SQR_THREADS);
        case SQK_REG2: return sq_reg_launch_grid(ctx, np, SQR2_THREADS);
        default: return std::min(ctx->num_sms, SQ_MAXG);
    }
}

// ---------------------------------------------------------------------------
// One factorization
// ---------------------------------------------------------------------------
struct Run {
    rqrcp_ctx *ctx;
    double *A;
    int64_t lda, m, n, k;
    int b, p, l, lpad, P, me, G;
    int64_t n_loc;
    uint64_t seed;
    int64_t *jpvt;
    double *tau;
    const double *omega_in;
    double *omega_out;
    rqrcp_trace *trace;
    bool keep_last;
    int panel_mode;
    int sched;
    int cur = 0;         // sample buffer of the current panel
    int vb = 0;          // V buffer of the current panel
    int panels = 0;
    // the bulk trailing update of the previous panel, not yet launched / joined
    struct Bulk {
        bool ready = false, launched = false;
        double *A22 = nullptr;  // rows i+bb.. of the trailing local columns
        int64_t rows = 0, cols = 0, lj0 = 0;
        int bb = 0, bbpad = 0, vbuf = 0;
        int *dyn = nullptr;
        int cap = 0;
    } bulk;
    int *status, *bb_eff, *done, *rankd;
    cudaStream_t st;
    // end-to-end path (rqrcp_factor_host): A streamed in by column chunks that
    // feed the sketch, finished panels streamed out while later panels run
    const double *h_in = nullptr;
    double *h_out = nullptr;
    int64_t h_ld = 0;
    cudaStream_t cps = nullptr;  // copy stream

    int64_t ldv_for(int64_t mp) const { return P > 1 ? rup(mp, 8) : ctx->ldo; }
    bool more_after(int64_t i, int bb) const { return (i + bb < k) || keep_last; }

    // ---- S2 -------------------------------------------------------------
    SqArgs sq_args(double *B, int64_t nn, int bb) {
        SqArgs a{};
        a.B = B;
        a.ldb = lpad;
        a.l = l;
        a.lpad = lpad;
        a.nn = nn;
        a.bb = bb;
        a.stop_tol2 = ctx->stop_tol2;
        a.slot_hdr = ctx->slot_hdr;
        a.slot_col = ctx->slot_col;
        a.slot_v2 = ctx->slot_v2;
        a.slot_data = ctx->slot_data;
        a.ll = ctx->sq_ll;
        a.piv = ctx->piv;
        a.tauhat = ctx->tauhat;
        a.vhat = ctx->vhat;
        a.rhat11 = ctx->rhat11;
        a.bbpad = (int)rup(bb, 8);
        a.perm = ctx->perm;
        a.bb_eff = bb_eff;
        a.done = done;
        a.rank = rankd;
        a.status = status;
        a.gaps = nullptr;
        a.swap_dst = ctx->swap_dst;
        a.swap_src = ctx->swap_src;
        a.swap_np = ctx->swap_np;
        a.trace = nullptr;
        a.spill = ctx->sq_spill;
        a.spec = ctx->opt.sq_spec;
        return a;
    }
    // one sample QRCP launch (bb steps of Alg. 1 on the nn columns of a.B),
    // the kernel chosen from the table by (l, nn)
    int launch_sq(SqArgs a) {
        const int64_t np = a.nn;
        const int bb = a.bb;
        a.tag0 = (++ctx->launch_seq) << 8;
        const SqKind kind = sq_kind(ctx, l, np);
        const SqKernels kt = sq_kernels(l, ctx->opt.sq_smtop != 0);
        if (kind == SQK_CLUSTER) {
            const int cs = (int)std::max<int64_t>(1, (np + SQC_THREADS - 1) / SQC_THREADS);
            return cluster_launch(ctx, kt.cluster, cs, SQC_THREADS, (size_t)bb * l * sizeof(double), a);
        }
        if (kind == SQK_REG2) {
            const int grid = sq_reg_launch_grid(ctx, np, SQR2_THREADS);
            const size_t smem = (size_t)std::max(kt.reg2_ls * SQR2_THREADS, bb * l) * sizeof(double);
            void *args[] = {&a};
            return coop_launch(ctx, (const void *)kt.reg2, grid, SQR2_THREADS, args, smem);
        }
        if (kind == SQK_REG) {
            const int grid = sq_reg_launch_grid(ctx, np, SQR_THREADS);
            const size_t smem = (size_t)std::max(kt.reg_ls * SQR_THREADS, bb * l) * sizeof(double);
            a.hstride = 8;
            void *args[] = {&a};
            return coop_launch(ctx, (const void *)kt.reg, grid, SQR_THREADS, args, smem);
        }
        a.hstride = ctx->opt.sq_hstride;
        a.poll_mode = ctx->opt.sq_poll;
        int gcap = std::min(G, SQ_MAXG);
        if (ctx->opt.sq_grid > 0) gcap = std::max(1, std::min(gcap, ctx->opt.sq_grid));
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(gcap, (np + 7) / 8));
        const int64_t cpb = (np + grid - 1) / grid;
        int tpc = 32;
        while (tpc > 1 && cpb * tpc > SQ_THREADS) tpc >>= 1;
        a.tpc = tpc;
        const int cpw = 32 / tpc;
        auto pad_ncs = [&](int64_t x) -> int64_t {
            if (cpw >= 16 || x <= 0) return std::max<int64_t>(x, 1);
            return x + (((cpw - x) % 16) + 16) % 16;
        };
        const int64_t state = cpb * (2 * (int64_t)sizeof(double) + 2 * (int64_t)sizeof(int));
        int64_t nsm = cpb;
        if (ctx->opt.sq_nsm >= 0) nsm = std::max<int64_t>(0, std::min<int64_t>(nsm, ctx->opt.sq_nsm));
        while (nsm > 0 && (int64_t)l * pad_ncs(nsm) * 8 + state > kDynSmemMax) --nsm;
        a.nsm = (int)nsm;
        a.ncs = (int)pad_ncs(nsm);
        const size_t smem = sq_smem_bytes(a.ncs, cpb, l);
        void *args[] = {&a};
        return coop_launch(ctx, (const void *)sample_qrcp_kernel, grid, SQ_THREADS, args, smem);
    }

    int sample_qrcp(int64_t i) {
        const int bb = (int)std::min<int64_t>(b, k - i);
        const int bbpad = (int)rup(bb, 8);
        const int64_t np = n - i;
        const bool rule5 = ctx->update_rule == 2 && more_after(i, bb) && np - bb > 0;
        if (rule5)  // Eq. (5) needs B2 = the pre-QRCP sample
            CK(cudaMemcpyAsync(ctx->bpre, ctx->bs[cur], sizeof(double) * (size_t)lpad * (size_t)np,
                               cudaMemcpyDeviceToDevice, st));
        ph_begin(ctx, PH_SQRCP);
        if (ctx->opt.tournament > 1) {
            CKT(tournament(i, bb, np));
        } else {
            SqArgs a = sq_args(ctx->bs[cur], np, bb);
            a.trace = (panels + 1 == ctx->opt.trace_panel) ? ctx->trace : nullptr;
            CKT(launch_sq(a));
        }
        ph_end(ctx);
        // trace: R-hat in pivoted order
        const int64_t t = i / b;
        if (trace && trace->rhat && t >= trace->first_panel && t < trace->first_panel + trace->npanels) {
            double *out = trace->rhat + (t - trace->first_panel) * (int64_t)l * n;
            trace_rhat_kernel<<<grid_for((int64_t)l * np, 256, G), 256, 0, st>>>(ctx->bs[cur], lpad, ctx->perm,
                                                                               ctx->rhat11, bbpad, l, np, bb_eff, out);
            CKL();
        }
        return 0;
    }

    // Tournament pivoting on the sample (reading R-TP; tournament.cuh)
    int tournament(int64_t i, int bb, int64_t np) {
        const int Gt = ctx->opt.tournament;
        const int bbpad = (int)rup(bb, 8);
        double *B = ctx->bs[cur];
        int *ti = ctx->tp_ints;  // [0] bb_eff [1] done [2] rank of a scratch QRCP
        // local selections: group g's columns gathered into the scratch sample
        std::vector<int64_t> maxc(Gt, 0);
        for (int g = 0; g < Gt; ++g) {
            const int64_t lq0 = dist_count(i, b, Gt, g);
            const int64_t ng = dist_count(n, b, Gt, g) - lq0;
            int *cnt = ctx->tp_cnt + g;
            int64_t *cand = ctx->tp_cand + (int64_t)g * bbpad;
            if (ng <= 0) {
                CK(cudaMemsetAsync(cnt, 0, sizeof(int), st));
                continue;
            }
            const int bg = (int)std::min<int64_t>(bb, ng);
            maxc[g] = bg;
            tp_gather_group_kernel<<<grid_for(ng * lpad, 256, G), 256, 0, st>>>(B, lpad, lpad, i, b, Gt, g, lq0, ng,
                                                                              ctx->c5, ctx->tp_idx);
            CKL();
            CK(cudaMemsetAsync(ti, 0, sizeof(int) * 3, st));
            SqArgs a = sq_args(ctx->c5, ng, bg);
            a.perm = ctx->tp_perm;
            a.piv = ctx->tp_piv;
            a.tauhat = ctx->tp_tau;
            a.vhat = ctx->tp_vhat;
            a.rhat11 = ctx->tp_r11;
            a.bb_eff = ti;
            a.done = ti + 1;
            a.rank = ti + 2;
            a.swap_dst = ctx->tp_sd;
            a.swap_src = ctx->tp_ss;
            a.swap_np = ti + 3;
            CKT(launch_sq(a));
            tp_collect_kernel<<<1, 128, 0, st>>>(ctx->tp_perm, ti, ctx->tp_idx, cand, cnt);
            CKL();
        }
        // merges up the tree; the last one (into group 0) is the root.  The
        // root's reflector buffer is cleared first: columns beyond its pivot
        // count are multiplied by zero rows of W2 below and must be finite.
        CK(cudaMemsetAsync(ctx->vhat, 0, sizeof(double) * (size_t)lpad * bbpad, st));
        for (int span = 1; span < Gt; span *= 2)
            for (int g = 0; g + span < Gt; g += 2 * span) {
                const int h = g + span;
                const bool root = (2 * span >= Gt);
                const int nu = (int)(maxc[g] + maxc[h]);
                const int bu = std::min(bb, std::max(nu, 1));
                const int ncols = std::max(nu, 1);
                tp_union_kernel<<<grid_for((int64_t)ncols * lpad, 256, G), 256, 0, st>>>(
                    B, lpad, lpad, ctx->tp_cand + (int64_t)g * bbpad, ctx->tp_cnt + g, ctx->tp_cand + (int64_t)h * bbpad,
                    ctx->tp_cnt + h, ncols, ctx->tp_u, ctx->tp_idx);
                CKL();
                CK(cudaMemsetAsync(ti, 0, sizeof(int) * 3, st));
                SqArgs a = sq_args(ctx->tp_u, ncols, bu);
                a.perm = ctx->tp_perm;
                a.piv = ctx->tp_piv;
                a.bb_eff = ti;
                a.done = ti + 1;
                a.rank = ti + 2;
                a.swap_dst = ctx->tp_sd;
                a.swap_src = ctx->tp_ss;
                a.swap_np = ti + 3;
                if (!root) {  // the root's reflectors / R-hat11 go to the panel's buffers
                    a.tauhat = ctx->tp_tau;
                    a.vhat = ctx->tp_vhat;
                    a.rhat11 = ctx->tp_r11;
                }
                a.bbpad = bbpad;
                CKT(launch_sq(a));
                tp_collect_kernel<<<1, 128, 0, st>>>(ctx->tp_perm, ti, ctx->tp_idx, ctx->tp_cand + (int64_t)g * bbpad,
                                                     ctx->tp_cnt + g);
                CKL();
                maxc[g] = std::min<int64_t>(bb, nu);
            }
        // R-hat = Q-hat^T B for every sample column: W = V-hat^T B, W2 = -T-hat^T W,
        // B += V-hat W2 (V-hat, tau-hat: the root's reflectors = the QR of the
        // chosen columns in pivot order)
        tp_transpose_kernel<<<grid_for((int64_t)lpad * bbpad, 256, G), 256, 0, st>>>(ctx->vhat, lpad, bbpad, ctx->tp_vt);
        CKL();
        CKT(gemm_skinny(ctx, bbpad, bbpad, lpad, ctx->vhat, lpad, ctx->vhat, lpad, ctx->tp_y, bbpad));
        {
            int nb = 8;
            while (nb < bbpad) nb *= 2;
            const size_t smem = tri_smem_bytes(nb);
            tri_kernel<<<1, TRI_THREADS, smem, st>>>(ctx->tp_y, ctx->tauhat, nullptr, nullptr, 0, bb, bbpad, nb,
                                                     ctx->tp_cnt, ctx->tp_tn, nullptr, 0, nullptr);
            CKL();
        }
        CKT(gemm_skinny(ctx, bbpad, np, lpad, ctx->vhat, lpad, B, lpad, ctx->tp_w, bbpad));
        CKT(gemm_skinny(ctx, bbpad, np, bbpad, ctx->tp_tn, bbpad, ctx->tp_w, bbpad, ctx->tp_w2, bbpad));
        CKT(update_any(ctx, lpad, np, bbpad, ctx->tp_w2, bbpad, ctx->tp_vt, bbpad, B, lpad));
        // perm, moves and the panel state, as the S2 kernels leave them
        tp_iota_kernel<<<grid_for(np, 256, G), 256, 0, st>>>(ctx->perm, np);
        CKL();
        tp_finish_kernel<<<1, 32, 0, st>>>(ctx->tp_cand, ctx->tp_cnt, bb, status, done, bb_eff, rankd, ctx->perm,
                                           ctx->swap_dst, ctx->swap_src, ctx->swap_np);
        CKL();
        return 0;
    }

    // ---- the bulk rows of a deferred trailing update ------------------------
    int launch_bulk() {
        Bulk &u = bulk;
        if (!u.ready || u.launched) return 0;
        u.launched = true;
        CK(cudaStreamWaitEvent(ctx->upd, ctx->ev_pack, 0));
        ctx->grid_cap = u.dyn ? 0 : u.cap;
        int rc = on_stream(ctx, ctx->upd, [&]() -> int {
            ph_begin(ctx, PH_TRAIL);
            const double *vtb = ctx->vt_b[u.vbuf] + (int64_t)u.bb * u.bbpad;
            int r = update_any(ctx, u.rows, u.cols, u.bbpad, ctx->w2, u.bbpad, vtb, u.bbpad, u.A22, lda, u.dyn);
            ph_end(ctx);
            return r;
        });
        ctx->grid_cap = 0;
        if (rc) return rc;
        CK(cudaEventRecord(ctx->ev_upd, ctx->upd));
        return 0;
    }
    int join_bulk() {
        if (!bulk.ready) return 0;
        if (!bulk.launched) CKT(launch_bulk());
        CK(cudaStreamWaitEvent(st, ctx->ev_upd, 0));
        bulk = Bulk();
        return 0;
    }

    // ---- S3 pack + S4 panel + S3 unpack -----------------------------------
    int panel(int64_t i) {
        const int bb = (int)std::min<int64_t>(b, k - i);
        const int bbpad = (int)rup(bb, 8);
        const int64_t mp = m - i;
        const int owner = dist_owner(i, b, P);
        const int64_t ljs = dist_local(i, b, P);  // owner's local column of slot 0
        const int64_t ldp = ctx->ldo;
        const int nvb = (bulk.ready && sched == 2) ? (vb ^ 1) : vb;  // this panel's V buffer
        double *vfull = ctx->vfull_b[nvb], *vt = ctx->vt_b[nvb];
        const int64_t ldv = ldv_for(mp);
        const bool narrow = bulk.ready && sched == 2;
        ph_begin(ctx, PH_SWAP);
        // schedule 1: the bulk update ran beside the sample QRCP; the pivot
        // columns are read only after it finished
        if (bulk.ready && sched != 2) CKT(join_bulk());
        // (1) pack the pivot columns (full height) into this rank's buffer
        double *pk = (P > 1) ? ctx->packbuf : ctx->pbuf;
        {
            dim3 grid((unsigned)std::min<int64_t>(64, (m + 2047) / 2048), (unsigned)bb);
            pack_pivots_kernel<<<grid, 256, 0, st>>>(A, lda, m, i, ctx->perm, bb, bb_eff, b, P, me, pk, ldp,
                                                    narrow ? ctx->w2 : nullptr, bulk.bbpad, bulk.bbpad, bulk.lj0,
                                                    ctx->w2g);
            CKL();
        }
        // (2) look-ahead: the previous panel's update on these columns (same
        //     arithmetic per element as the bulk update), then the bulk itself
        if (narrow) {
            const double *vtb = ctx->vt_b[bulk.vbuf] + (int64_t)bulk.bb * bulk.bbpad;
            CKT(update_any(ctx, mp, bb, bulk.bbpad, ctx->w2g, bulk.bbpad, vtb, bulk.bbpad, pk + i, ldp));
        }
        CK(cudaEventRecord(ctx->ev_pack, st));
        if (bulk.ready && sched == 2) CKT(launch_bulk());
        // (3) P > 1: the owner receives the exact bits (integer sum, one contributor)
        if (P > 1) {
            ph_begin(ctx, PH_COMM);
            CKT(ctx->tr->reduce_u64((const uint64_t *)ctx->packbuf, (uint64_t *)ctx->pbuf, (size_t)(ldp * bb), owner,
                                    st, ctx->err));
            ph_end(ctx);
        }
        ph_end(ctx);
        // (4) the panel QR on the owner
        ph_begin(ctx, PH_PANEL);
        double *Pp = ctx->pbuf + i;
        if (me == owner) {
            ctx->cqr_enabled = (panel_mode == 1) || (panel_mode == 2 && mp >= kCqrMinRows);
            // the stop scale: from the CholeskyQR2 Gram diagonal (register-grid path), else
            // one pass of column sums of squares
            if (!(ctx->cqr_enabled && ctx->opt.cqr_rg)) {
                colsumsq_kernel<<<bb, 256, 0, st>>>(Pp, ldp, mp, bb, bb_eff, ctx->colss);
                CKL();
                panel_tol_kernel<<<1, 32, 0, st>>>(ctx->colss, bb, bb_eff, ctx->ptol2);
                CKL();
            }
            CK(cudaMemsetAsync(ctx->stopc, 0xff, sizeof(int), st));
            CKT(panel_cqr(i, mp, bb, bbpad, Pp, ldp, vfull, ldv, vt));
            PanelArgs a{};
            a.skip = ctx->cqr_status;
            a.count = ctx->iscal + 4;
            a.A = Pp;
            a.lda = ldp;
            a.mp = mp;
            a.bb = bb;
            a.bbpad = bbpad;
            a.bb_eff = bb_eff;
            a.tau = tau + i;
            a.vfull = vfull;
            a.ldv = ldv;
            a.vt = vt;
            a.ybuf = ctx->ybuf;
            a.part = ctx->pn_part;
            a.rowj = ctx->pn_rowj;
            a.bar = ctx->bars + 2 * panels + 1;
            a.tol2 = ctx->ptol2;
            a.stop_col = ctx->stopc;
            a.trace = (panels + 1 == ctx->opt.trace_panel) ? ctx->ptrace : nullptr;
            bool pn_done = false;
            if (ctx->opt.pn_cluster) {
                void (*kfn)(PanelArgs) = nullptr;
                int64_t rc_rows = 0;
                size_t psm = 0;
                const bool cpt2 = ctx->opt.pn_cpt != 1;
                if (bb <= 32) { kfn = panel_qr_cluster_kernel<32, 64>; rc_rows = 8 * 64; psm = 32 * 65 * 8; }
                else if (bb <= 64 && cpt2) { kfn = panel_qr_cluster_kernel<64, 32, 2>; rc_rows = 8 * 32; psm = 64 * 64 * 8; }
                else if (bb <= 64) { kfn = panel_qr_cluster_kernel<64, 64>; rc_rows = 4 * 64; psm = 64 * 65 * 8; }
                const int64_t cs = kfn ? (mp + rc_rows - 1) / rc_rows : 0;
                if (kfn && cs <= ctx->pnc_max) {
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
            // blocked when the panel's rows of one CTA do not fit its shared memory
            // (C4 / C5; measured slower at C3 where they fit: 10.0 vs 7.7 ms)
            const int64_t rows_cta = (mp + G - 1) / G;
            const bool blk = ctx->opt.pn_blocked == 2 ||
                             (ctx->opt.pn_blocked == 1 && rows_cta * bb * (int64_t)sizeof(double) > kDynSmemMax);
            if (!pn_done && blk && bb > kPanelSub && !ctx->cqr_enabled) {
                CKT(panel_blocked(a, i, mp, bb, bbpad, Pp, ldp, vfull, ldv, vt));  // applies its own stops
            } else {
                if (!pn_done) {
                    CKT(launch_grid_panel(a, mp, bb));
                    if (a.trace) ctx->ptrace_kind = 0;
                }
                panel_stop_apply_kernel<<<1, 32, 0, st>>>(ctx->stopc, 0, bb_eff, rankd, done);
                CKL();
            }
        }
        // (5) P > 1: the owner broadcasts V, tau, V^T V, R11 (and T), the state
        const double *R11p = Pp;
        int64_t ldr11 = ldp;
        if (P > 1) {
            const int npk = bbpad + 3 * bbpad * bbpad + 4;
            if (me == owner) {
                dist_pack_kernel<<<grid_for(npk, 256, G), 256, 0, st>>>(tau + i, ctx->ybuf, Pp, ldp, bb, bbpad,
                                                                      ctx->tneg, ctx->cqr_status, bb_eff, ctx->pack);  // state = iscal[1..3]
                CKL();
            }
            ph_begin(ctx, PH_COMM);
            CKT(ctx->tr->bcast(vfull, sizeof(double) * (size_t)(ldv * bbpad), owner, st, ctx->err));
            CKT(ctx->tr->bcast(ctx->pack, sizeof(double) * (size_t)npk, owner, st, ctx->err));
            ph_end(ctx);
            if (me != owner) {
                dist_unpack_kernel<<<grid_for(npk, 256, G), 256, 0, st>>>(ctx->pack, bb, bbpad, tau + i, ctx->ybuf,
                                                                        ctx->tneg, ctx->cqr_status, bb_eff);  // state = iscal[1..3]
                CKL();
                dist_transpose_kernel<<<grid_for(mp * bbpad, 256, G), 256, 0, st>>>(vfull, ldv, mp, bbpad, vt);
                CKL();
            }
            R11p = ctx->pack + bbpad + (int64_t)bbpad * bbpad;
            ldr11 = bbpad;
        }
        // T (and Omega-hat11 for Eq. (4)) on the side stream, overlapping W = V^T A22
        {
            const bool rule5 = ctx->update_rule == 2 && more_after(i, bb) && n - i - bb > 0;
            int nb = 8;
            while (nb < bbpad) nb *= 2;
            const size_t smem = tri_smem_bytes(nb);
            CK(cudaEventRecord(ctx->ev_fork, st));
            CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            const int do_om = (more_after(i, bb) && n - i - bb > 0 && !rule5) ? 1 : 0;
            tri_kernel<<<2, TRI_THREADS, smem, ctx->side>>>(ctx->ybuf, tau + i, ctx->rhat11, R11p, ldr11, bb, bbpad,
                                                          nb, bb_eff, ctx->tneg, ctx->omhat, do_om, ctx->cqr_status);
            CKL();
            CK(cudaEventRecord(ctx->ev_join, ctx->side));
        }
        ph_end(ctx);
        // (6) the previous panel's bulk update must be complete before the
        //     displaced columns move and the panel is written back
        ph_begin(ctx, PH_SWAP);
        CKT(join_bulk());
        const dim3 g1((unsigned)std::min<int64_t>(64, (m + 2047) / 2048), (unsigned)(2 * bb));
        if (P > 1) {
            if (me == owner) {
                pack_slots_kernel<<<dim3(g1.x, bb), 256, 0, st>>>(A, lda, m, ljs, bb, bb_eff, ctx->dispbuf, ldp);
                CKL();
            }
            ph_begin(ctx, PH_COMM);
            CKT(ctx->tr->bcast(ctx->dispbuf, sizeof(double) * (size_t)(ldp * bb), owner, st, ctx->err));
            ph_end(ctx);
            place_displaced_kernel<<<g1, 256, 0, st>>>(A, lda, m, i, ctx->swap_dst, ctx->swap_src, ctx->swap_np, bb,
                                                      bb_eff, b, P, me, ctx->dispbuf, ldp);
            CKL();
        } else {
            place_displaced_kernel<<<g1, 256, 0, st>>>(A, lda, m, i, ctx->swap_dst, ctx->swap_src, ctx->swap_np, bb,
                                                      bb_eff, b, P, me, A + i * lda, lda);
            CKL();
        }
        if (me == owner) {
            copy_back_kernel<<<dim3(g1.x, bb), 256, 0, st>>>(A, lda, m, ljs, bb, bb_eff, ctx->pbuf, ldp);
            CKL();
        }
        {
            const int64_t t = i / b;
            int64_t *pv = nullptr;
            if (trace && trace->pivots && t >= trace->first_panel && t < trace->first_panel + trace->npanels)
                pv = trace->pivots + (t - trace->first_panel) * b;
            jpvt_moves_kernel<<<1, 256, 0, st>>>(jpvt + i, ctx->swap_dst, ctx->swap_src, ctx->swap_np, bb_eff, bb, pv);
            CKL();
        }
        ph_end(ctx);
        vb = nvb;
        return 0;
    }

    int launch_grid_panel(PanelArgs &a, int64_t mp, int bb) {
        int pcap = G;
        if (ctx->opt.pn_grid > 0) pcap = std::max(1, std::min(G, ctx->opt.pn_grid));
        if (bulk.ready && bulk.launched) pcap = std::min(pcap, ctx->opt.la_panel_ctas);  // share with the bulk
        const int64_t prows = ctx->opt.pn_rows;
        const int grid = (int)std::max<int64_t>((mp + PN_MAXROWS - 1) / PN_MAXROWS,
                                                std::min<int64_t>(pcap, (mp + prows - 1) / prows));
        const int64_t rpb = (mp + grid - 1) / grid;
        if (rpb > PN_MAXROWS) {
            ctx->err = "panel too tall for the cooperative grid";
            return RQRCP_E_WORKSPACE;
        }
        if (grid > PN_MAXG) {
            ctx->err = "panel grid exceeds PN_MAXG";
            return RQRCP_E_WORKSPACE;
        }
        a.nsm = (int)std::min<int64_t>(rpb, kDynSmemMax / ((int64_t)bb * sizeof(double)));
        const size_t smem = (size_t)a.nsm * bb * sizeof(double);
        void *args[] = {&a};
        const void *kern = (bb <= 32) ? (const void *)panel_qr_kernel<4> : (const void *)panel_qr_kernel<8>;
        return coop_launch(ctx, kern, grid, PN_THREADS, args, smem);
    }

    // S4, blocked (dgeqrf-style): the grid kernel factors 32-column
    // sub-panels (the whole sub-panel then stays in shared memory: one on-chip
    // pass per column instead of L2 round trips for the rows that do not fit),
    // and after each sub-panel s the panel columns to its right receive its
    // reflectors as three DMMA contractions W = V_s^T P, W2 = -T_s^T W,
    // P += V_s W2 (T_s by tri_kernel).  Same reflectors as the column-by-column
    // kernel in exact arithmetic; T of the whole panel from Y = V^T V (DMMA).
    int panel_blocked(PanelArgs a0, int64_t i, int64_t mp, int bb, int bbpad, double *Pp, int64_t ldp, double *vfull,
                      int64_t ldv, double *vt) {
        const int w = kPanelSub;
        zero_top_kernel<<<grid_for((int64_t)bbpad * bbpad, 256, G), 256, 0, st>>>(vfull, ldv, vt, bbpad, bbpad);
        CKL();
        for (int c0 = 0; c0 < bb; c0 += w) {
            const int c1 = std::min(bb, c0 + w), ws = c1 - c0;
            const int wpad = (int)rup(ws, 8);
            sub_eff_kernel<<<1, 32, 0, st>>>(bb_eff, c0, ws, ctx->subeff);
            CKL();
            CK(cudaMemsetAsync(ctx->stopc, 0xff, sizeof(int), st));
            PanelArgs a = a0;
            a.A = Pp + c0 + (int64_t)c0 * ldp;
            a.mp = mp - c0;
            a.bb = ws;
            a.bbpad = wpad;
            a.col0 = c0;
            a.tau = tau + i + c0;
            a.vfull = vfull + c0 + (int64_t)c0 * ldv;
            a.ldv = ldv;
            a.vt = vt + c0 + (int64_t)c0 * bbpad;
            a.ldvt = bbpad;
            a.ybuf = ctx->ybs;
            a.ldy = w;
            a.count = (c0 == 0) ? a0.count : nullptr;
            a.bar = ctx->bars + 2 * panels + 1;
            CK(cudaMemsetAsync(a.bar, 0, sizeof(unsigned), st));
            CKT(launch_grid_panel(a, mp - c0, ws));
            panel_stop_apply_kernel<<<1, 32, 0, st>>>(ctx->stopc, c0, bb_eff, rankd, done);
            CKL();
            if (c1 < bb) {
                // T_s, then the in-panel update of columns c1..bb (rows c0..m')
                tri_kernel<<<1, TRI_THREADS, tri_smem_bytes(w), st>>>(
                    ctx->ybs, tau + i + c0, nullptr, nullptr, 0, ws, w, w, ctx->subeff, ctx->tns, nullptr, 0, nullptr);
                CKL();
                const int64_t nr = bb - c1, K = mp - c0;
                bool dn = false;
                CKT(tma_skinny(ctx, wpad, nr, K, vfull, mp, bbpad, ldv, c0, c0, ctx->pbuf, m, bb, ldp, i + c0, c1,
                               ctx->wsub, w, &dn, 512));
                if (!dn) CKT(gemm_skinny(ctx, wpad, nr, K, vfull + c0 + (int64_t)c0 * ldv, ldv, Pp + c0 + c1 * ldp, ldp,
                                         ctx->wsub, w));
                CKT(gemm_skinny(ctx, wpad, nr, wpad, ctx->tns, w, ctx->wsub, w, ctx->w2sub, w));
                CKT(update_any(ctx, K, nr, wpad, ctx->w2sub, w, vt + c0 + (int64_t)c0 * bbpad, bbpad,
                               Pp + c0 + c1 * ldp, ldp));
            }
        }
        // Y = V^T V for the compact-WY T of the whole panel (tri_kernel, strict upper part)
        bool dn = false;
        CKT(tma_skinny(ctx, bbpad, bbpad, mp, vfull, mp, bbpad, ldv, 0, 0, vfull, mp, bbpad, ldv, 0, 0, ctx->ybuf,
                       bbpad, &dn, 512));
        if (!dn) CKT(gemm_skinny(ctx, bbpad, bbpad, mp, vfull, ldv, vfull, ldv, ctx->ybuf, bbpad));
        return 0;
    }

    // S4 via CholeskyQR2 + Householder reconstruction (cqr.cuh) on the panel
    // buffer.  Every kernel is a no-op once *cqr_status = 1.
    int panel_cqr(int64_t i, int64_t mp, int bb, int bbpad, double *Pp, int64_t ldp, double *vfull, int64_t ldv,
                  double *vt) {
        if (!ctx->cqr_enabled) {
            CK(cudaMemsetAsync(ctx->cqr_status, 0x01, sizeof(int), st));  // != 0: fallback
            return 0;
        }
        int nb = 8;
        while (nb < bbpad) nb *= 2;
        const size_t csm = cqr_smem_bytes(nb);
        const size_t rsm = (size_t)bbpad * (bbpad + 4) * sizeof(double);
        // DMMA row products: grid-strided 8-row tiles, at most one CTA per SM
        auto rgrid = [&](int64_t rows) {
            return (int)std::max<int64_t>(1, std::min<int64_t>(G, (rows + 8 * (CQR_THREADS / 32) - 1) / (8 * (CQR_THREADS / 32))));
        };
        // small (bb-row) products: 8-row warp tiles x 4 column slices
        auto sgrid = [&](int64_t rows) {
            return dim3((unsigned)std::max<int64_t>(1, (rows + 8 * (CQR_THREADS / 32) - 1) / (8 * (CQR_THREADS / 32))), 4);
        };
        bool dn = false;
        // G1 = P^T P
        CKT(tma_skinny(ctx, bb, bb, mp, ctx->pbuf, m, bb, ldp, i, 0, ctx->pbuf, m, bb, ldp, i, 0, ctx->cq_g, bbpad, &dn, 128));
        if (!dn) CKT(gemm_skinny(ctx, bb, bb, mp, Pp, ldp, Pp, ldp, ctx->cq_g, bbpad));
        const bool rg = ctx->opt.cqr_rg != 0;
        const int nbr = std::max(16, nb);
        auto chol = [&](int pass, double *tol) -> int {
            if (!rg) {
                cqr_chol_kernel<<<1, CQR_THREADS, csm, st>>>(ctx->cq_g, bb, bbpad, nb, pass, bb_eff, ctx->cqr_status,
                                                            ctx->cq_rc, ctx->cq_rinv, tol);
                CKL();
                return 0;
            }
            const size_t sm = cqr_rg_smem_bytes(nbr);
            switch (nbr) {
#define RGC(NBV)                                                                                                  \
    case NBV:                                                                                                     \
        cqr_chol_rg_kernel<NBV><<<1, RG_THREADS, sm, st>>>(ctx->cq_g, bb, bbpad, pass, bb_eff, ctx->cqr_status, \
                                                            ctx->cq_rc, ctx->cq_rinv, tol, pass == 1 ? 1 : 0);    \
        break;
                RGC(16) RGC(32) RGC(64) RGC(128)
#undef RGC
                default: ctx->err = "cqr: unsupported panel width"; return RQRCP_E_UNSUPPORTED;
            }
            CKL();
            return 0;
        };
        CKT(chol(1, ctx->ptol2));
        // Q1 = P R1^{-1}
        // (rg path: the 512-thread variant, bitwise the same products)
        auto bigmul = rg ? cqr_rowmul2_kernel : cqr_rowmul_kernel;
        const int bthreads = rg ? RM2_THREADS : CQR_THREADS;
        bigmul<<<rgrid(mp), bthreads, rsm, st>>>(Pp, ldp, 0, mp, bb, bbpad, ctx->cq_rinv, 1.0, vfull, ldv,
                                                               ctx->cqr_status, 0, nullptr, 0, nullptr);
        CKL();
        // G2 = Q1^T Q1, R2, Rc = R2 R1
        CKT(tma_skinny(ctx, bb, bb, mp, vfull, mp, bbpad, ldv, 0, 0, vfull, mp, bbpad, ldv, 0, 0, ctx->cq_g, bbpad, &dn, 128));
        if (!dn) CKT(gemm_skinny(ctx, bb, bb, mp, vfull, ldv, vfull, ldv, ctx->cq_g, bbpad));
        CKT(chol(2, nullptr));
        // Q = Q1 R2^{-1}: only its top bb rows are formed (in place); the rows below
        // go straight to V2 = -Qbottom U^{-1} = -Q1bottom (R2^{-1} U^{-1}) below
        // (rg path: one pass over the panel fewer)
        // (rg path: Q_top into its own bbpad x bbpad buffer, read by both CTAs of the
        // reconstruction while CTA 0 writes the top rows of V)
        cqr_rowmul_kernel<<<rg ? sgrid(std::min<int64_t>(mp, bb)) : dim3(rgrid(mp)), CQR_THREADS, rsm, st>>>(
                                                                         vfull, ldv, 0, rg ? std::min<int64_t>(mp, bb) : mp,
                                                                         bb, bbpad, ctx->cq_rinv, 1.0, rg ? ctx->cq_q : vfull,
                                                                         rg ? (int64_t)bbpad : ldv,
                                                                         ctx->cqr_status, 0, nullptr, 0, nullptr);
        CKL();
        // reconstruction of the top block: L, U S, U^{-1}, L^{-T} (L^{-T} into cq_g: G2 is consumed)
        if (!rg) {
            cqr_recon_kernel<<<1, CQR_THREADS, csm, st>>>(vfull, ldv, bb, bbpad, nb, ctx->cq_rc, ctx->cqr_status, Pp, ldp,
                                                         tau + i, ctx->cq_lu, ctx->cq_uinv, ctx->cq_g, vt);
        } else {
            switch (nbr) {
#define RGR(NBV)                                                                                                      \
    case NBV:                                                                                                         \
        cqr_recon_rg_kernel<NBV><<<2, RG_THREADS, cqr_rg_smem_bytes(NBV), st>>>(ctx->cq_q, bbpad, vfull, ldv, bb, bbpad, ctx->cq_rc, ctx->cqr_status, Pp, ldp, \
                                                           tau + i, ctx->cq_lu, ctx->cq_uinv, ctx->cq_g, vt,          \
                                                           ctx->cq_rinv, ctx->cq_c);                                  \
        break;
                RGR(16) RGR(32) RGR(64) RGR(128)
#undef RGR
                default: ctx->err = "cqr: unsupported panel width"; return RQRCP_E_UNSUPPORTED;
            }
        }
        CKL();
        // -T = -(U S) L^{-T}: first needed by W2 = -T^T W after W = V^T A22, so on one
        // GPU it runs on the side stream (ahead of tri_kernel there, which skips T when
        // this path succeeded; the main stream joins before W2).  P > 1: the owner
        // broadcasts T right after the panel, so it stays on the main stream.
        cudaStream_t tst = st;
        if (P == 1) {
            CK(cudaEventRecord(ctx->ev_fork, st));
            CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            tst = ctx->side;
        }
        cqr_rowmul_kernel<<<sgrid(bbpad), CQR_THREADS, rsm, tst>>>(ctx->cq_lu, bbpad, 0, bbpad, bb, bbpad, ctx->cq_g, -1.0,
                                                                ctx->tneg, bbpad, ctx->cqr_status, 0, nullptr, 0, nullptr);
        CKL();
        // V2 = -Qbottom U^{-1} (into Vfull, the panel and Vt); rg path: C = R2^{-1} U^{-1}
        // (bb x bb, one CTA) then V2 = -Q1bottom C
        if (mp > bb) {
            const double *cm = ctx->cq_uinv;
            if (rg) cm = ctx->cq_c;  // formed by the reconstruction's second CTA
            bigmul<<<rgrid(mp - bb), bthreads, rsm, st>>>(vfull, ldv, bb, mp, bb, bbpad, cm, -1.0,
                                                                        vfull, ldv, ctx->cqr_status, 1, Pp, ldp, vt);
            CKL();
        }
        return 0;
    }

    // ---- S5 trailing update (+ S6 sample update) and the next S2 ------------
    int trailing_and_sample(int64_t i) {
        const int bb = (int)std::min<int64_t>(b, k - i);
        const int bbpad = (int)rup(bb, 8);
        const int64_t mp = m - i, np = n - i, npp = np - bb;
        const bool more = more_after(i, bb);
        const bool rule5 = ctx->update_rule == 2 && more && npp > 0;
        const int64_t lj0 = dist_count(i + bb, b, P, me);
        const int64_t npl = n_loc - lj0;
        const double *vfull = ctx->vfull_b[vb];
        const double *vt = ctx->vt_b[vb];
        const int64_t ldv = ldv_for(mp);
        // the next sample QRCP decides the schedule of this panel's bulk rows
        const int64_t inext = i + bb;
        const bool next_panel = (i + bb < k);
        // (decided from global sizes only: every rank takes the same schedule,
        // so kernel shapes -- and bits -- do not depend on the rank count)
        int s = sched;
        if (!next_panel || npp <= 0 || mp <= bb) s = 0;
        ph_begin(ctx, PH_TRAIL);
        if (npl > 0) {
            double *A22 = A + i + lj0 * lda;
            bool dn = false;
            // W = V^T A22 (canonical split-K over the GLOBAL trailing width)
            CKT(tma_skinny(ctx, bbpad, npl, mp, vfull, mp, bbpad, ldv, 0, 0, A, m, n_loc, lda, i, lj0, ctx->w, bbpad,
                           &dn, 512, npp));
            if (!dn) CKT(gemm_skinny(ctx, bbpad, npl, mp, vfull, ldv, A22, lda, ctx->w, bbpad, npp));
            CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
            // W2 = -T^T W (K = bbpad: no split; the persistent TMA kernel when the
            // operands allow it -- decided by pointers and sizes only, never by P)
            CKT(tma_skinny(ctx, bbpad, npl, bbpad, ctx->tneg, bbpad, bbpad, bbpad, 0, 0, ctx->w, bbpad, npl, bbpad, 0,
                           0, ctx->w2, bbpad, &dn, 512, npp));
            if (!dn) CKT(gemm_skinny(ctx, bbpad, npl, bbpad, ctx->tneg, bbpad, ctx->w, bbpad, ctx->w2, bbpad, npp));
            if (s == 0) {
                CKT(update_any(ctx, mp, npl, bbpad, ctx->w2, bbpad, vt, bbpad, A22, lda));
            } else {
                // the R12 rows (all Eq. (4) / (5) need) now; the bulk rows later
                CKT(update_any(ctx, bb, npl, bbpad, ctx->w2, bbpad, vt, bbpad, A22, lda));
                bulk = Bulk();
                bulk.ready = true;
                bulk.A22 = A22 + bb;
                bulk.rows = mp - bb;
                bulk.cols = npl;
                bulk.lj0 = lj0;
                bulk.bb = bb;
                bulk.bbpad = bbpad;
                bulk.vbuf = vb;
            }
        } else {
            CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
            if (s != 0) {  // no local trailing columns: an empty bulk keeps the schedule uniform
                bulk = Bulk();
                bulk.ready = true;
                bulk.A22 = A + i + bb + lj0 * lda;
                bulk.lj0 = lj0;
                bulk.bb = bb;
                bulk.bbpad = bbpad;
                bulk.vbuf = vb;
            }
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
                CKT(tma_skinny(ctx, bbpad, lpad, mp, vfull, mp, bbpad, ldv, 0, 0, ctx->omt, m, lpad, ctx->ldo, i, 0,
                               ctx->wom, bbpad, &dn));
                if (!dn) CKT(gemm_skinny(ctx, bbpad, lpad, mp, vfull, ldv, ctx->omt + i, ctx->ldo, ctx->wom, bbpad));
                CKT(gemm_skinny(ctx, bbpad, lpad, bbpad, ctx->tneg, bbpad, ctx->wom, bbpad, ctx->w2om, bbpad));
                CKT(update_any(ctx, mp, lpad, bbpad, ctx->w2om, bbpad, vt, bbpad, ctx->omt + i, ctx->ldo));
                if (npl > 0) {
                    CKT(gemm_skinny(ctx, lpad, npl, bb, ctx->omt + i, ctx->ldo, A + i + lj0 * lda, lda, ctx->c5, lpad, npp));
                    sample_update5_kernel<<<grid_for((int64_t)lpad * npl, 256, G), 256, 0, st>>>(
                        ctx->bpre, lpad, ctx->perm, ctx->c5, lpad, bb, l, lpad, npl, bb_eff, udst, lpad, i, lj0, b, P, me);
                    CKL();
                }
            } else if (npl > 0) {
                // C = Omega-hat11 R12 (DMMA; omhat holds Omega-hat11^T), then the
                // gather B_next = [R-hat12 - C; R-hat22] (Eq. (4))
                {
                    bool dn4 = false;  // persistent TMA kernel (rows i.. of A as the K operand), else cp.async
                    CKT(tma_skinny(ctx, bbpad, npl, bb, ctx->omhat, bbpad, bbpad, bbpad, 0, 0, A, m, n_loc, lda, i, lj0,
                                   ctx->c5, lpad, &dn4, 512, npp));
                    if (!dn4)
                        CKT(gemm_skinny(ctx, bbpad, npl, bb, ctx->omhat, bbpad, A + i + lj0 * lda, lda, ctx->c5, lpad,
                                        npp));
                }
                sample_update4_kernel<<<grid_for((int64_t)lpad * npl, 256, G), 256, 0, st>>>(
                    ctx->bs[cur], lpad, ctx->perm, ctx->c5, lpad, bb, l, lpad, npl, bb_eff, udst, lpad, i, lj0, b, P, me);
                CKL();
            }
            if (P > 1) CKT(gather_sample(npl, i + bb, n - i - bb, ctx->bs[cur ^ 1]));
            ph_end(ctx);
            cur ^= 1;
            const int64_t t = i / b;
            if (trace && trace->bnext && t >= trace->first_panel && t < trace->first_panel + trace->npanels) {
                double *out = trace->bnext + (t - trace->first_panel) * (int64_t)l * n;
                trace_copy_kernel<<<grid_for((int64_t)l * npp, 256, G), 256, 0, st>>>(ctx->bs[cur], lpad, l, npp, out);
                CKL();
            }
        }
        if (!next_panel) return 0;
        // ---- the next panel's S2; schedule 1 launches the bulk rows behind it
        if (s == 1) CK(cudaEventRecord(ctx->ev_pack, st));  // the bulk may start once S6 is done
        CKT(sample_qrcp(inext));
        if (s == 1) {
            // the bulk rows on the SMs the sample QRCP leaves free (cluster), or on
            // the whole GPU with dynamically claimed tiles (register grid)
            const SqKind kind = sq_kind(ctx, l, n - inext);
            if (kind == SQK_CLUSTER) bulk.cap = G - sq_ctas(ctx, l, n - inext);
            else if (kind == SQK_REG && bulk.bbpad <= 64 && panels < 8192) bulk.dyn = ctx->tctr + panels;
            else bulk.cap = 0;
            CKT(launch_bulk());
        } else if (s == 2) {
            bulk.cap = std::max(1, G - ctx->opt.la_panel_ctas);
        }
        return 0;
    }

    // AllGather each rank's ncols_loc sample columns (global columns >= j0, local
    // order) and reorder into global order: out(:, p) = column j0 + p.
    int gather_sample(int64_t ncols_loc, int64_t j0, int64_t ncols, double *out) {
        int64_t cmax = 0;
        for (int r = 0; r < P; ++r)
            cmax = std::max<int64_t>(cmax, dist_count(j0 + ncols, b, P, r) - dist_count(j0, b, P, r));
        if (cmax * P * lpad > ctx->gbuf_elems) {
            ctx->err = "gather buffer too small";
            return RQRCP_E_WORKSPACE;
        }
        (void)ncols_loc;
        ph_begin(ctx, PH_COMM);
        CKT(ctx->tr->allgather(ctx->gsend, ctx->gbuf, sizeof(double) * (size_t)(cmax * lpad), st, ctx->err));
        ph_end(ctx);
        if (ncols > 0) {
            dist_reorder_kernel<<<grid_for(ncols * lpad, 256, G), 256, 0, st>>>(ctx->gbuf, cmax, lpad, lpad, j0, ncols, b,
                                                                               P, out, lpad);
            CKL();
        }
        return 0;
    }

    int setup() {
        ph_begin(ctx, PH_OMEGA);
        CK(cudaMemsetAsync(ctx->iscal, 0, sizeof(int) * 8, st));
        const int64_t npanels = (k + b - 1) / b;
        CK(cudaMemsetAsync(ctx->bars, 0, sizeof(unsigned) * std::min<int64_t>(ctx->nbars, 2 * npanels + 2), st));
        CK(cudaMemsetAsync(ctx->tctr, 0, sizeof(int) * std::min<int64_t>(npanels, 8192), st));
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
        // ---- S1: sketch B = Omega A (canonical split-K over the global n) ----
        ph_begin(ctx, PH_SKETCH);
        bool tdone = false;
        double *bdst = (P == 1) ? ctx->bs[cur] : ctx->gsend;
        if (h_in) {
            // column chunks: H2D on the copy stream, each chunk's sketch on the
            // main stream as soon as it has landed (same K slices: same bits)
            const int64_t CH = 2048;
            for (int64_t c0 = 0; c0 < n_loc; c0 += CH) {
                const int64_t nc = std::min(CH, n_loc - c0);
                CK(cudaMemcpy2DAsync(A + c0 * lda, sizeof(double) * lda, h_in + c0 * h_ld, sizeof(double) * h_ld,
                                     sizeof(double) * m, nc, cudaMemcpyHostToDevice, cps));
                CK(cudaEventRecord(ctx->ev_h2d, cps));
                CK(cudaStreamWaitEvent(st, ctx->ev_h2d, 0));
                CKT(tma_skinny(ctx, lpad, nc, m, ctx->omt, m, lpad, ctx->ldo, 0, 0, A, m, n_loc, lda, 0, c0,
                               bdst + c0 * lpad, lpad, &tdone, 512, n));
                if (!tdone)
                    CKT(gemm_skinny(ctx, lpad, nc, m, ctx->omt, ctx->ldo, A + c0 * lda, lda, bdst + c0 * lpad, lpad, n));
            }
        } else {
            CKT(tma_skinny(ctx, lpad, n_loc, m, ctx->omt, m, lpad, ctx->ldo, 0, 0, A, m, n_loc, lda, 0, 0, bdst, lpad,
                           &tdone, 512, n));
            if (!tdone) CKT(gemm_skinny(ctx, lpad, n_loc, m, ctx->omt, ctx->ldo, A, lda, bdst, lpad, n));
        }
        ph_end(ctx);
        if (P > 1) CKT(gather_sample(n_loc, 0, n, ctx->bs[cur]));
        sumsq_partial_kernel<<<4 * G, 256, 0, st>>>(ctx->bs[cur], lpad, n, lpad, ctx->sumsq_part);
        CKL();
        sumsq_final_kernel<<<1, 32, 0, st>>>(ctx->sumsq_part, 4 * G, ctx->stop_tol2, ctx->iscal + 0);
        CKL();
        // Pi = I_n
        iota_kernel<<<grid_for(n, 256, G), 256, 0, st>>>(jpvt, n);
        CKL();
        CK(cudaMemsetAsync(tau, 0, sizeof(double) * k, st));
        return 0;
    }

    int run() {
        CKT(setup());
        CKT(sample_qrcp(0));
        for (int64_t i = 0; i < k; i += b) {
            CKT(panel(i));
            if (h_out) {  // the panel's columns are final: stream them out behind the next panels
                const int64_t bb = std::min<int64_t>(b, k - i);
                CK(cudaEventRecord(ctx->ev_h2d, st));
                CK(cudaStreamWaitEvent(cps, ctx->ev_h2d, 0));
                CK(cudaMemcpy2DAsync(h_out + i * h_ld, sizeof(double) * h_ld, A + i * lda, sizeof(double) * lda,
                                     sizeof(double) * m, bb, cudaMemcpyDeviceToHost, cps));
            }
            CKT(trailing_and_sample(i));
            ++panels;
        }
        CKT(join_bulk());
        if (h_out && k < n) {  // the trailing columns (R12 rows, R22) are final now
            CK(cudaEventRecord(ctx->ev_h2d, st));
            CK(cudaStreamWaitEvent(cps, ctx->ev_h2d, 0));
            // host_out 1: only the R12 rows (later panels' swaps move whole trailing
            // columns, so they are final only here); R22 stays on the device
            const int64_t rows = ctx->opt.host_out ? k : m;
            CK(cudaMemcpy2DAsync(h_out + k * h_ld, sizeof(double) * h_ld, A + k * lda, sizeof(double) * lda,
                                 sizeof(double) * rows, n - k, cudaMemcpyDeviceToHost, cps));
        }
        if (h_out) {
            CK(cudaEventRecord(ctx->ev_h2d, cps));
            CK(cudaStreamWaitEvent(st, ctx->ev_h2d, 0));
        }
        return 0;
    }
};

// Status words through pinned memory; multi-GPU: poll the communicator while
// waiting (asynchronous NCCL errors, timeout -> abort).
static int finish_wait(rqrcp_ctx *ctx, cudaStream_t st) {
    if (!ctx->tr || ctx->nranks == 1 || !strcmp(ctx->tr->kind(), "loopback")) {
        CK(cudaStreamSynchronize(st));
        return 0;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) return 0;
        if (q != cudaErrorNotReady) CK(q);
        if (ctx->tr->poll(ctx->err)) {
            ctx->tr->abort();
            return RQRCP_E_NCCL;
        }
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > (double)ctx->opt.nccl_timeout_ms) {
            ctx->err = "multi-GPU factorization exceeded nccl_timeout_ms: communicator aborted";
            ctx->tr->abort();
            return RQRCP_E_NCCL;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
}

static void print_traces(rqrcp_ctx *ctx);

static int factor_impl(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                       uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out, const double *omega_in,
                       double *omega_out, rqrcp_trace *trace, bool keep_last = false, int *final_sample = nullptr,
                       const double *h_in = nullptr, double *h_out = nullptr, int64_t h_ld = 0) {
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
    ctx->launches = 0;
    ctx->nev = 0;
    ctx->lt_t0 = ctx->lt_t1 = -1;
    ctx->rec_phase.clear();
    ctx->rec_s.clear();
    ctx->rec_e.clear();
    ctx->open_phase = -1;
    if (trace) trace->recorded = 0;
    Run R{};
    R.ctx = ctx;
    R.A = A;
    R.lda = lda;
    R.m = m;
    R.n = n;
    R.k = k;
    R.b = b;
    R.p = p;
    R.l = b + p;
    R.lpad = (int)rup(R.l, 8);
    R.P = ctx->nranks;
    R.me = ctx->rank;
    R.G = ctx->num_sms;
    R.n_loc = dist_count(n, b, R.P, R.me);
    R.seed = seed;
    R.jpvt = jpvt;
    R.tau = tau;
    R.omega_in = omega_in;
    R.omega_out = omega_out;
    R.trace = trace;
    R.keep_last = keep_last;
    R.panel_mode = ctx->opt.panel;
    R.st = ctx->stream;
    R.status = ctx->iscal + 0;
    R.bb_eff = ctx->iscal + 1;
    R.done = ctx->iscal + 2;
    R.rankd = ctx->iscal + 3;
    R.h_in = h_in;
    R.h_out = h_out;
    R.h_ld = h_ld;
    R.cps = ctx->cps;
    // schedule: the bulk rows of each trailing update overlap the next sample
    // QRCP when that sample QRCP is one cluster (C2: 4.34 vs 4.78 ms serial);
    // the register grids fill the GPU and the update kernels run at their best
    // alone: serial (C3 43.9 vs 46.6 ms, C4 / C5 likewise).  The panel
    // look-ahead (schedule 2) loses everywhere: its panel kernel slows down
    // when it shares the GPU with the update.
    int sched = ctx->opt.schedule;
    if (sched < 0) {
        const SqKind kind = sq_kind(ctx, R.l, n);
        sched = (kind == SQK_CLUSTER) ? 1 : 0;
    }
    R.sched = sched;
    const int ev_t0 = ctx->nev;
    cudaEventRecord(ctx->ev[ctx->nev++], ctx->stream);
    int rc = R.run();
    if (rc) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->upd);
        return rc;
    }
    if (final_sample) *final_sample = R.cur;
    int *hs = ctx->hstatus;
    CK(cudaMemcpyAsync(hs, ctx->iscal, sizeof(int) * 5, cudaMemcpyDeviceToHost, ctx->stream));
    const int ev_t1 = ctx->nev;
    cudaEventRecord(ctx->ev[ctx->nev++], ctx->stream);
    rc = finish_wait(ctx, ctx->stream);
    if (rc) return rc;
    ctx->lt_t0 = ctx->timing ? ev_t0 : -1;
    ctx->lt_t1 = ctx->timing ? ev_t1 : -1;
    if (ctx->trace) print_traces(ctx);
    rqrcp_timings t{};
    t.panels = R.panels;
    t.panels_householder = hs[4];
    t.kernel_launches = ctx->launches;
    ctx->last = t;
    if (trace) trace->recorded = std::max<int64_t>(0, std::min<int64_t>(trace->npanels, R.panels - trace->first_panel));
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

// RQRCP_TRACE=1: per-step clock64 phase traces of the latency-bound kernels
static void print_traces(rqrcp_ctx *ctx) {
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
        fprintf(stderr, "\n");
    }
}

extern "C" int rqrcp_factor(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                            uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out) {
    return factor_impl(ctx, A, lda, m, n, k, b, p, seed, jpvt, tau, rank_out, nullptr, nullptr, nullptr);
}

extern "C" int rqrcp_factor_ex(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                               uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out, const double *omega_in,
                               double *omega_out, rqrcp_trace *trace) {
    if (trace && (trace->first_panel < 0 || trace->npanels < 0)) return -15;
    return factor_impl(ctx, A, lda, m, n, k, b, p, seed, jpvt, tau, rank_out, omega_in, omega_out, trace);
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
    CK(smem_attr((const void *)srqr_solve_kernel, (int)ssm, ctx->device));
    double *Y = ctx->splitk;  // (k+1) x d
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
    double *vfull = ctx->vfull_b[0], *vt = ctx->vt_b[0];
    lr_eye_kernel<<<grid_for(m * k, 256, G), 256, 0, st>>>(Q1, ldq, m, k);
    CKL();
    int *bbd = ctx->iscal + 6;
    const int64_t npanels = (k + b - 1) / b;
    for (int64_t t = npanels - 1; t >= 0; --t) {
        const int64_t i = t * b;
        const int bb = (int)std::min<int64_t>(b, k - i);
        const int bbpad = (int)rup(bb, 8);
        const int64_t mp = m - i, ncols = k - i;
        lr_extract_v_kernel<<<grid_for(mp * bbpad, 256, G), 256, 0, st>>>(A + i + i * lda, lda, mp, bb, bbpad, vfull,
                                                                          ctx->ldo, vt);
        CKL();
        CKT(gemm_skinny(ctx, bbpad, bbpad, mp, vfull, ctx->ldo, vfull, ctx->ldo, ctx->ybuf, bbpad));
        lr_set_int_kernel<<<1, 1, 0, st>>>(bbd, bb);
        CKL();
        int nb = 8;
        while (nb < bbpad) nb *= 2;
        const size_t tsm = tri_smem_bytes(nb);
        tri_kernel<<<1, TRI_THREADS, tsm, st>>>(ctx->ybuf, tau + i, nullptr, nullptr, 0, bb, bbpad, nb, bbd, ctx->tneg,
                                                ctx->omhat, 0, nullptr);
        CKL();
        lr_transpose_kernel<<<grid_for((int64_t)bbpad * bbpad, 256, G), 256, 0, st>>>(ctx->tneg, bbpad, ctx->omhat);
        CKL();
        double *X = Q1 + i + i * ldq;
        // X <- (I - V T V^T) X:  W = V^T X,  W2 = -T W,  X += V W2
        CKT(gemm_skinny(ctx, bbpad, ncols, mp, vfull, ctx->ldo, X, ldq, ctx->w, bbpad));
        CKT(gemm_skinny(ctx, bbpad, ncols, bbpad, ctx->omhat, bbpad, ctx->w, bbpad, ctx->w2, bbpad));
        CKT(gemm_update(ctx, mp, ncols, bbpad, ctx->w2, bbpad, vt, bbpad, X, ldq));
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
    // A streams in by column chunks that feed the sketch, and the finished
    // panels stream out while later panels run (copy stream); A_out_host may
    // equal A_host: every input chunk has landed before the first output copy
    int64_t rk = 0;
    int rc = factor_impl(ctx, ctx->a_dev, m, m, n, k, b, p, seed, ctx->jpvt_dev, ctx->tau_dev, &rk, nullptr, nullptr,
                         nullptr, false, nullptr, A_host, A_out_host, lda);
    *rank_out = rk;
    if (rc != 0 && rc != RQRCP_W_RANK_DEFICIENT) return rc;
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
