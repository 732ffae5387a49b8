/*
 * rqrcp.h -- C ABI of the B200-native randomized QR with column pivoting
 * (RQRCP) hot path.  Xiao, Gu, Langou, "Fast Parallel Randomized QR with
 * Column Pivoting Algorithms for Reliable Low-rank Matrix Approximations",
 * HiPC 2017 (arXiv 1804.05138).  Citations: P:n = line n of the paper text
 * (PAPER.md), S:n = line n of the desk-scale SPEC.md.
 *
 * What rqrcp_factor computes: the partial QRCP
 *       A Pi = Q [R11 R12; 0 R22] ~= Q1 [R11 R12]
 * by Alg. 2: Omega ~ N(0,1)^{(b+p) x m}, B = Omega A
 * (P:144); per panel of width bb = min(b, k-i): partial QRCP of
 * the sample B(:, i:n) for bb pivots, the same swaps on A and Pi
 * (P:148), Householder QR of the panel A(i:m, i:i+bb) with compact-WY
 * T, the trailing update A22 <- Q~^T A22 = A22 - V T^T V^T A22, and the
 * sample update of Eq. (4): B <- [R^12 - R^11 R11^{-1} R12; R^22].
 *
 * Conventions (all identical to LAPACK dgeqp3's):
 *   - matrices are column-major fp64; every pointer to matrix data is a
 *     DEVICE pointer on the context's device unless the name says _host;
 *   - on return A holds V below the diagonal of its first rank columns
 *     (unit diagonal implicit), R11 (upper triangle of A(0:k,0:k)) and R12
 *     (A(0:k, k:n)) in pivoted column order, and the trailing R22 by-product;
 *   - jpvt (int64, 0-based): column j of A Pi is column jpvt[j] of
 *     the input;  tau[k]: Householder scalars, H_j = I - tau_j v_j v_j^T,
 *     Q = H_0 H_1 ... H_{k-1};
 *   - Householder sign convention = LAPACK dlarfg (reading R-G7);
 *   - Omega is drawn from Philox4x32-10 (key = seed) + Box-Muller with the
 *     counter mapping of DESIGN.md "Generator mapping" (reading R-G8).
 *
 * Ownership: the caller owns A, jpvt, tau (and every buffer it passes); the
 * context owns its workspace (sized at create time) and, for nranks > 1, its
 * NCCL communicator.  No allocation happens inside rqrcp_factor.  A context
 * is not thread-safe; use one per (device, rank).
 *
 * Errors: every function returns 0 on success, a negative value -i when its
 * i-th argument is invalid (LAPACK "info" style), or a positive RQRCP_E_*
 * code; rqrcp_last_error(ctx) gives a human-readable message.  A positive
 * RQRCP_W_* code is a warning: outputs are valid.
 */
#ifndef RQRCP_H
#define RQRCP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RQRCP_OK 0
#define RQRCP_E_CUDA 1          /* a CUDA runtime call failed */
#define RQRCP_E_NCCL 2          /* an NCCL call failed */
#define RQRCP_E_WORKSPACE 3     /* size exceeds the create-time maxima, or out of memory */
#define RQRCP_E_NONFINITE 4     /* NaN/Inf in the sample (hence in A) */
#define RQRCP_E_UNSUPPORTED 5   /* feature not built (e.g. nranks > 1 without NCCL) */
#define RQRCP_W_RANK_DEFICIENT 16 /* early stop (reading R-G12): *rank_out < k */

typedef struct rqrcp_ctx rqrcp_ctx;

typedef struct rqrcp_config {
    int device;            /* CUDA device ordinal */
    void *stream;          /* cudaStream_t to run on; NULL -> a context-owned stream */
    int nranks;            /* GPUs in the 1D column-block-cyclic layout (1 = single GPU) */
    int rank;              /* this process's rank in [0, nranks) */
    uint8_t nccl_uid[128]; /* ncclUniqueId bytes from rank 0 (ignored if nranks == 1) */
    int64_t max_m;         /* workspace maxima: rqrcp_factor fails with RQRCP_E_WORKSPACE */
    int64_t max_n;         /*   when m > max_m, n > max_n, b > max_b or p > max_p     */
    int max_b;
    int max_p;
} rqrcp_config;

/* Per-phase device times of the last rqrcp_factor (CUDA events, ms).
 * total_ms is the wall time of the call on the device.  The phases are
 * timed on the stream that runs them; when the bulk rows of a panel's
 * trailing update run concurrently with the next panel's sample QRCP
 * (single GPU, Eq. (4), sample QRCP on one cluster), trailing_ms includes
 * that concurrent update, so the phases may sum to more than total_ms. */
typedef struct rqrcp_timings {
    double total_ms;
    double omega_ms;        /* S0: Philox Omega */
    double sketch_ms;       /* S1: B = Omega A */
    double sample_qrcp_ms;  /* S2 */
    double swap_ms;         /* S3 */
    double panel_ms;        /* S4 (panel QR + T) */
    double trailing_ms;     /* S5 (W = V^T A22, W2 = -T^T W, A22 += V W2) */
    double sample_update_ms;/* S6 */
    double comm_ms;         /* NCCL collectives (nranks > 1) */
    int64_t panels;
    int64_t kernel_launches;/* kernels this library launched in the call */
    int64_t panels_householder; /* panels factored column by column (the
                                   CholeskyQR2 path declined: ill-conditioned
                                   or rank-stopped panel, or RQRCP_PANEL=hh);
                                   on this rank's owned panels */
} rqrcp_timings;

/* Create a context: allocates every workspace buffer for the maxima in cfg
 * (and the NCCL communicator when nranks > 1).  *ctx is NULL on failure.
 * Returns 0, -1 (ctx null), -2 (cfg null or invalid field), or RQRCP_E_*. */
int rqrcp_create(rqrcp_ctx **ctx, const rqrcp_config *cfg);

/* Factor A in place (Alg. 2).
 *   A      device, column-major m x n (single GPU) or this rank's shard of the
 *          global columns {j : floor(j/b) mod nranks == rank}, m x n_loc with
 *          n_loc = rqrcp_shard_columns(n, b, nranks, rank) (multi-GPU: every
 *          rank calls rqrcp_factor with the same m, n, k, b, p, seed; jpvt and
 *          tau come back identical on every rank), lda >= max(1, m); overwritten.
 *   m, n   global sizes, 1 <= m, n;  k target rank, 1 <= k <= min(m, n)
 *   b      panel width >= 1;  p oversampling >= 0 with b + p <= m
 *   seed   Philox key for Omega (never invalid)
 *   jpvt   device int64[n] (output);  tau device double[k] (output)
 *   rank_out host int64 (output): achieved rank (== k unless the warning)
 * Synchronous: returns after the work on the context's stream completed.
 * Argument codes: -1 ctx, -2 A, -3 lda, -4 m, -5 n, -6 k, -7 b, -8 p,
 * -10 jpvt, -11 tau, -12 rank_out.  Returns RQRCP_W_RANK_DEFICIENT when the
 * factorization stopped before k columns (reading R-G12): either every
 * candidate sample column norm fell below 1e3*eps*||Omega A||_F, or a
 * panel's R11 diagonal entry |R(j,j)| fell below 1e3*eps*||A(i:m, i:i+bb)||_F
 * (the panel after its swaps).  Outputs are valid for the first
 * *rank_out columns (tau = 0 beyond; A(rank:m, rank:n) is the trailing matrix
 * after rank reflectors).  Multi-GPU: NCCL errors are polled while the call
 * waits and the communicator is aborted after nccl_timeout_ms (RQRCP_E_NCCL). */
int rqrcp_factor(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                 uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out);

/* Same computation with HOST buffers (the end-to-end path): copies A_host
 * (m x n, lda) to a context-owned device buffer, factors, and copies the
 * factored A, jpvt and tau back (A_out_host may equal A_host).  Single GPU
 * only.  Pinned host memory gives full PCIe bandwidth.  Codes as
 * rqrcp_factor, plus RQRCP_E_WORKSPACE if m*n exceeds max_m*max_n. */
int rqrcp_factor_host(rqrcp_ctx *ctx, const double *A_host, int64_t lda, int64_t m, int64_t n, int64_t k,
                      int b, int p, uint64_t seed, double *A_out_host, int64_t *jpvt_host, double *tau_host,
                      int64_t *rank_out);

/* Testing API: per-panel trace of the factorization.
 * Panels t in [first_panel, first_panel + npanels) are recorded; each output
 * pointer may be NULL.  Panel t starts at column i = t*b with width
 * bb = min(b, k - i); l = b + p.
 *   pivots  device int64[npanels * b]: entry [(t - first_panel) b + q], q < bb:
 *           the input column placed at position i + q by this panel's swaps
 *           (= the final jpvt[i + q]) -- the pivots the sample QRCP chose;
 *   rhat    device double[npanels * l * n]: block t - first_panel (stride l n)
 *           holds the l x (n - i) sample right after the panel's sample QRCP
 *           (Alg. 2 line P:147), column-major ld l, in PIVOTED column order:
 *           R-hat = [R-hat11 R-hat12; 0 R-hat22] with zeros below
 *           the diagonal of the first bb columns;
 *   bnext   device double[npanels * l * n]: block t - first_panel holds the
 *           l x (n - i - bb) sample after the update of Eq. (4) or
 *           Eq. (5), ld l (untouched when no update follows: the
 *           last panel, reading R-G9, or an early stop);
 *   recorded  (out) number of panels recorded.
 * With nranks > 1 every rank records the replicated sample. */
typedef struct rqrcp_trace {
    int64_t first_panel;
    int64_t npanels;
    int64_t *pivots;
    double *rhat;
    double *bnext;
    int64_t recorded;
} rqrcp_trace;

/* Testing API: rqrcp_factor with optional hooks (every one may be NULL).
 *   omega_in   device l x m (ld = l) sketch to use instead of the Philox draw
 *   omega_out  device l x m (ld = l) receives the Omega used
 *   trace      per-panel pivots and sample snapshots (rqrcp_trace above)
 * Same kernels and schedule as rqrcp_factor (the hooks only add copies). */
int rqrcp_factor_ex(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                    uint64_t seed, int64_t *jpvt, double *tau, int64_t *rank_out, const double *omega_in,
                    double *omega_out, rqrcp_trace *trace);

/* Testing / diagnosis API: a launch-path option of ctx, applied to
 * subsequent calls (defaults are the measured best; every variant computes
 * the same factorization).  Returns 0, -1 (ctx null), -2 (unknown name) or
 * -3 (value out of range).  Names (initial values from the environment
 * variable RQRCP_<NAME upper-cased> at create time):
 *   schedule      -1 auto, 0 serial, 1 the bulk trailing update overlaps the
 *                 next sample QRCP, 2 ... overlaps the next panel QR (look-ahead)
 *   panel         0 column-by-column Householder, 1 CholeskyQR2 + reconstruction,
 *                 2 CholeskyQR2 from 8192 rows
 *   pn_cluster, pn_cpt, pn_grid, pn_rows, la_panel_ctas   panel kernel choice / shape
 *   tournament    > 1: the panel pivots come from tournament pivoting on the sample over this
 *                 many block-cyclic column groups (the paper's future work; DESIGN.md
 *                 reading R-TP) instead of Alg. 1 on the whole sample; 0 / 1: Alg. 1
 *   upd_kernel    trailing-update GEMM: 0 CTA-wide TMA epilogue, 1 / 2 warp-specialised
 *                 (per-warp TMA epilogue; 32 x 2 / 16 x 4 k-stages)
 *   sq_cluster, sq_grid, sq_nsm, sq_hstride   sample QRCP kernel choice / shape
 *   sq_reg        register-resident grid sample QRCP: 1 the 256-thread kernel when the sample
 *                 fits, else the 512-thread kernel with the top rows in global memory (l = 144);
 *                 2 always the 512-thread kernel when it exists for l; 0 neither
 *   sq_poll       grid sample QRCP exchange: 3 tagged 16-byte units (no fences), 0 acquire
 *                 polls, 1 relaxed polls + one fence, 2 as 1 with backoff
 *   sq_wide       register-grid sample QRCP launch: 1 (default) every SM for wide samples
 *                 (n' >= 64 x SMs), 2 always every SM, 0 the fewest CTAs that hold the sample
 *   sq_smtop      register-grid sample QRCP row layout (l = 144): 1 (default) the shared-memory
 *                 rows above the register rows (step j touches rows >= j only, so they drop out
 *                 of the per-step shared-memory traffic), 0 below them
 *   sq_spec       register-grid sample QRCP exchange: 0 (default) fetch the winner's column after
 *                 every header has arrived; 1 fetch the column of the best candidate seen so far
 *                 while the last headers arrive (the same winner; measured slower: the per-poll
 *                 warp reduction delays the last header more than the column round trip saves)
 *   cqr_rg        CholeskyQR2 panel one-CTA factorizations: 1 (default) register grid, 0 shared
 *                 memory
 *   debug_sync    synchronise after every launch
 *   host_out      rqrcp_factor_host output: 0 (default) the whole factored A; 1 the factors
 *                 only -- columns 0..k-1 full height (V below, R11 on / above the diagonal) and
 *                 rows 0..k-1 of columns k..n-1 (R12); the R22 block of A_out_host is left
 *                 as it was (the partial factorization's outputs are Pi, V + tau, R11, R12:
 *                 P:79-83)
 *   nccl_timeout_ms   multi-GPU: abort the communicator when a call exceeds it */
int rqrcp_set_option(rqrcp_ctx *ctx, const char *name, int64_t value);

/* Testing API (multi-rank logic on ONE GPU): create nranks contexts on
 * cfg->device that form one in-process group; their collectives are host
 * rendezvous + device copies (no kernel waits on another rank's kernel).
 * Each context must be driven by its own host thread, all calling the same
 * rqrcp_factor concurrently with their shards (layout as for NCCL ranks).
 * cfg->nranks / rank / nccl_uid / stream are ignored (each context owns a
 * stream).  ctxs: host array of nranks pointers (out).  Returns 0, -1, -2
 * (cfg invalid or nranks < 2 or > 16) or RQRCP_E_*. */
int rqrcp_create_loopback_group(rqrcp_ctx **ctxs, int nranks, const rqrcp_config *cfg);

/* Testing/bench API: rows [row0, row0+rows) x cols [col0, col0+cols) of the
 * N(0,1) matrix (seed, stream) with the Omega generator, into out (device,
 * column-major, ld >= rows).  Stream 0 is Omega itself. */
int rqrcp_fill_gaussian(rqrcp_ctx *ctx, uint64_t seed, uint32_t stream, int64_t rows, int64_t cols, int64_t row0,
                        int64_t col0, double *out, int64_t ld);

/* Testing API: raw Philox4x32-10 words.  ctr (device uint32[4*count]),
 * key (host, 2 words), out (device uint32[4*count]). */
int rqrcp_philox_words(rqrcp_ctx *ctx, const uint32_t *ctr, const uint32_t *key, uint32_t *out, int64_t count);

/* Algorithmic flop counts: out[0] sketch 2lmn, out[1]
 * Householder QR sum_j 4(m-j)(n-j), out[2] sample QRCP, out[3] sample
 * update.  Host only; needs no context.  Returns 0 or a negative code. */
int rqrcp_flops(int64_t m, int64_t n, int64_t k, int b, int p, double out[4]);

/* Multi-GPU layout (1D column-block-cyclic, block = b):
 * global column j lives on rank (j / b) mod nranks at local index
 * (j / (b nranks)) b + j mod b; a rank's shard keeps global column order.
 * Host-only, no context needed.
 *   rqrcp_shard_columns: number of columns of `rank` (its n_loc); negative on
 *     invalid arguments (-1 n, -2 b, -3 nranks, -4 rank).
 *   rqrcp_shard_global_index: global column of local column `local_index`
 *     of `rank` (negative on invalid arguments). */
int64_t rqrcp_shard_columns(int64_t n, int b, int nranks, int rank);
int64_t rqrcp_shard_global_index(int64_t local_index, int b, int nranks, int rank);

/* Fresh ncclUniqueId bytes for rqrcp_config.nccl_uid (call on rank 0 and
 * broadcast with torch.distributed).  Returns 0, or RQRCP_E_UNSUPPORTED when
 * libnccl.so.2 cannot be loaded, or RQRCP_E_NCCL.  out: host, 128 bytes. */
int rqrcp_nccl_unique_id(uint8_t *out);

/* Per-phase timings of the last rqrcp_factor on ctx. */
int rqrcp_get_timings(const rqrcp_ctx *ctx, rqrcp_timings *out);

/* SRQR verification (Alg. 3 first half): RQRCP to rank k exactly
 * as rqrcp_factor (same arguments and outputs), keeping the sample after the
 * last panel (reading G9), then
 *   r_i = ||B(:, i)||^2 / (b+p) for the trailing columns, iota = argmax
 *   (P:635-637); columns k and k + iota of A and jpvt are swapped;
 *   |alpha| = ||A(k:m, k)|| (one QR step; its reflector is not
 *   applied); g1 = ||A(k:m, k:n)||_{1,2} / |alpha| (Eq. 8);
 *   g2 ~= |alpha|/sqrt(d) ||Omega_d R-hat^{-T}||_{1,2}, Omega_d the d x (k+1)
 *   N(0,1) matrix of (seed, Philox stream 7), R-hat = [[R11, a], [0, |alpha|]]
 *   (P:505-511).
 * Requires k < min(m, n) and 1 <= d <= 64; single GPU (nranks = 1).
 * diag (host, 6 doubles): {g1, g2 estimate, |alpha|, the tau cap
 * g1 g2 sqrt((k+1)(n-k)) of Eq. (10), the tau-hat cap g1 g2 sqrt(k(n-k)) of
 * Eq. (12), iota}.  Returns as rqrcp_factor, -13 for an invalid d, or
 * RQRCP_E_UNSUPPORTED (nranks > 1 or k = min(m, n)). */
int rqrcp_srqr_verify(rqrcp_ctx *ctx, double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b, int p,
                      uint64_t seed, int d, int64_t *jpvt, double *tau, int64_t *rank_out, double *diag);

/* Low-rank outputs of a factorization (SURVEY.md
 * §8(f) N4), from the outputs of rqrcp_factor (single GPU):
 *
 * rqrcp_form_q1: Q1 (device, m x k, ld ldq >= m, caller-owned, overwritten) =
 *   the first k columns of Q = H_1 ... H_k, from the reflectors below the
 *   diagonal of the factored A (device, ld lda) and tau (device, k); b is
 *   the panel width the factorization used (T is rebuilt per panel).
 *   A Pi ~= Q1 [R11 R12].  Returns 0, -1 ctx null, -2 A null, -3 lda,
 *   -4 m, -5 n, -6 k, -7 b, -8 tau null, -9 Q1 null, -10 ldq, or RQRCP_E_*.
 *
 * rqrcp_cx: X (device, k x n, ld ldx >= k, caller-owned) = C^+ A with
 *   C = A Pi(:, 0:k) the first k pivot columns (the CX decomposition of
 *   P:813-815; exact for full-rank R11: X Pi = [I, R11^{-1} R12]), from the
 *   factored A and jpvt (device, n).  Allocates and frees k*k + (k+64)(n-k)
 *   doubles of temporary device memory.  ||A - C X||_F = ||R22||_F.
 *   Returns 0, -1 ctx null, -2 A null, -3 lda, -4 m, -5 n, -6 k, -7 jpvt
 *   null, -8 X null, -9 ldx, or RQRCP_E_*. */
int rqrcp_form_q1(rqrcp_ctx *ctx, const double *A, int64_t lda, int64_t m, int64_t n, int64_t k, int b,
                  const double *tau, double *Q1, int64_t ldq);
int rqrcp_cx(rqrcp_ctx *ctx, const double *A, int64_t lda, int64_t m, int64_t n, int64_t k, const int64_t *jpvt,
             double *X, int64_t ldx);

/* Sample updating formula for subsequent rqrcp_factor calls on ctx (Alg. 2
 * line P:151): 1 = Eq. (4) (default: reuse the sample's triangular
 * factor, O(nkb) flops), 2 = Eq. (5) (keep Omega-bar = Omega Q
 * up to date and form B2 - Omega-bar_1 R12, O((b+p)(m+n)k) flops).  Both give
 * the same pivots in exact arithmetic.  Returns 0, -1 (ctx null) or
 * -2 (rule not 1 or 2). */
int rqrcp_set_update_rule(rqrcp_ctx *ctx, int rule);

/* Enable (1) / disable (0) reading the per-phase CUDA-event times in
 * rqrcp_get_timings (default 1).  The events themselves are always recorded
 * (they are cheap, and the overlapped schedule measured faster with them). */
int rqrcp_set_timing(rqrcp_ctx *ctx, int enabled);

/* Destroy: frees workspace and the communicator.  NULL is a no-op. */
int rqrcp_destroy(rqrcp_ctx *ctx);

/* Message for the last non-zero return on ctx (static string if ctx NULL). */
const char *rqrcp_last_error(const rqrcp_ctx *ctx);

/* Library version string. */
const char *rqrcp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RQRCP_H */
