/*
 * oracle/rqrcp_oracle.c -- plain, slow, unblocked CPU fp64 RQRCP.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's
 * library.  It shares no code, header, helper or constant generator with the
 * CUDA path in paper_1804_05138_b200/ and neither includes the other.
 *
 * What it computes, step by step in the paper's order (PAPER.md = P:line):
 *   Alg. 2 (RQRCP) with the updating formula Eq. (4)
 *   (P:206-221), or Eq. (5) in cross-check mode; the partial
 *   QRCP on the sample is Alg. 1 (Businger-Golub) run for bb
 *   steps; the panel QR + trailing update of P:149-150 is done as
 *   unblocked Householder (LAPACK dgeqr2 order), which equals the blocked
 *   "Q~^T A22" of P:150 in exact arithmetic.
 *   Readings of ambiguous passages (DESIGN.md
 *   "Readings") are cited where they are taken.
 *
 * No BLAS, no blocking, no fusion.  Every sum runs over ascending index.
 * Multi-threading (OpenMP) is only across independent columns, so results
 * are bitwise independent of the thread count.  Compiled with
 * -ffp-contract=off so that no FMA contraction changes a rounding.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define COL(M, ld, r, c) ((M)[(size_t)(r) + (size_t)(c) * (size_t)(ld)])

/* ------------------------------------------------------------------------
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
 * easy as 1, 2, 3", SC'11): 10 rounds of the 4x32 Philox S-box with the
 * Weyl key schedule.  The paper only says "i.i.d Gaussian"; the
 * generator choice is reading G8.
 * ---------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t y0 = hi1 ^ x1 ^ k0;
        uint32_t y1 = lo1;
        uint32_t y2 = hi0 ^ x3 ^ k1;
        uint32_t y3 = lo0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* Element (r, c) of the N(0,1) matrix (seed, stream): counter
 * (c mod 2^32, floor(r/2), stream, c >> 32), key (seed lo, seed hi);
 * 53-bit uniforms in (0,1); Box-Muller (reading G8). */
static double oracle_normal_at(uint64_t seed, uint32_t stream, int64_t r, int64_t c)
{
    uint32_t ctr[4] = {(uint32_t)((uint64_t)c & 0xFFFFFFFFu), (uint32_t)((uint64_t)r >> 1), stream,
                       (uint32_t)((uint64_t)c >> 32)};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    uint64_t a1 = (((uint64_t)w[0] << 32) | w[1]) >> 11;
    uint64_t a2 = (((uint64_t)w[2] << 32) | w[3]) >> 11;
    double u1 = ((double)a1 + 0.5) * 0x1p-53;
    double u2 = ((double)a2 + 0.5) * 0x1p-53;
    double rho = sqrt(-2.0 * log(u1));
    double ang = 2.0 * M_PI * u2;
    return (r & 1) ? rho * sin(ang) : rho * cos(ang);
}

/* Fill out(0:rows, 0:cols) (column-major, ld) with rows [row0, row0+rows) and
 * columns [col0, col0+cols) of the N(0,1) matrix (seed, stream). */
void oracle_normal_fill(uint64_t seed, uint32_t stream, int64_t row0, int64_t rows, int64_t col0,
                        int64_t cols, double *out, int64_t ld)
{
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < cols; ++c)
        for (int64_t r = 0; r < rows; ++r)
            COL(out, ld, r, c) = oracle_normal_at(seed, stream, row0 + r, col0 + c);
}

/* ------------------------------------------------------------------------
 * Householder reflector, LAPACK dlarfg convention (reading G7; the paper
 * only says "Form Householder reflection H_i"):
 *   H = I - tau v v^T, v(0) = 1, H x = beta e1,
 *   beta = -sign(alpha) ||x||, tau = (beta - alpha)/beta,
 *   v(1:) = x(1:) / (alpha - beta);  tau = 0 (H = I) when ||x(1:)|| = 0.
 * x has n elements at stride 1; on return x(0) = beta, x(1:) = v(1:).
 * The norm is the plain ascending sum of squares (no dnrm2 scaling). */
static double oracle_dlarfg(int64_t n, double *x)
{
    if (n <= 1) return 0.0;
    double alpha = x[0];
    double xnorm2 = 0.0;
    for (int64_t t = 1; t < n; ++t) xnorm2 += x[t] * x[t];
    if (xnorm2 == 0.0) return 0.0;
    double norm = sqrt(alpha * alpha + xnorm2);
    double beta = (alpha >= 0.0) ? -norm : norm;
    double tau = (beta - alpha) / beta;
    double scal = 1.0 / (alpha - beta);
    for (int64_t t = 1; t < n; ++t) x[t] *= scal;
    x[0] = beta;
    return tau;
}

/* y <- (I - tau v v^T) y for a vector y of n elements, v(0)=1 implicit,
 * v(1:) = vtail.  w = v.y summed in ascending order. */
static void oracle_apply_reflector(int64_t n, const double *vtail, double tau, double *y)
{
    if (tau == 0.0 || n <= 0) return;
    double w = y[0];
    for (int64_t t = 1; t < n; ++t) w += vtail[t - 1] * y[t];
    double tw = tau * w;
    y[0] -= tw;
    for (int64_t t = 1; t < n; ++t) y[t] -= tw * vtail[t - 1];
}

/* ------------------------------------------------------------------------
 * Step O1: sketch B = Omega A.  Omega l x m (ld = ldo), A m x n,
 * B l x n (ld = ldb).  B(r,c) = sum_t Omega(r,t) A(t,c), t ascending.
 * ---------------------------------------------------------------------- */
void oracle_sketch(int64_t l, int64_t m, int64_t n, const double *Omega, int64_t ldo,
                   const double *A, int64_t lda, double *B, int64_t ldb)
{
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c)
        for (int64_t r = 0; r < l; ++r) {
            double s = 0.0;
            for (int64_t t = 0; t < m; ++t) s += COL(Omega, ldo, r, t) * COL(A, lda, t, c);
            COL(B, ldb, r, c) = s;
        }
}

static void swap_cols(int64_t rows, double *M, int64_t ld, int64_t a, int64_t b)
{
    if (a == b) return;
    for (int64_t r = 0; r < rows; ++r) {
        double t = COL(M, ld, r, a);
        COL(M, ld, r, a) = COL(M, ld, r, b);
        COL(M, ld, r, b) = t;
    }
}

/* ------------------------------------------------------------------------
 * Step O3: partial QRCP (Alg. 1) for bb steps on the l x nn
 * sample Bw.  Squared column norms r_s with the downdate
 * r_s -= B(j,s)^2 and recompute when r_s < 1e-6 r0_s (reading G6);
 * argmax with the lowest current position on exact ties (reading G5).
 * Returns the number of pivots taken (< bb when every candidate norm is
 * <= stop_tol2, reading G12, or -1 on a non-finite norm).
 * On return: piv[j] = chosen position (transposition j <-> piv[j]);
 * R-hat in the upper triangle of Bw(:, 0:steps) and in Bw(:, steps:);
 * reflector tails below the diagonal, tauhat[j]; gaps[j] = relative gap
 * (best - runner-up)/best of the squared norms at step j (diagnostic, H3).
 * ---------------------------------------------------------------------- */
int64_t oracle_sample_qrcp(int64_t l, int64_t nn, int64_t bb, double *Bw, int64_t ldb, int64_t *piv,
                           double *tauhat, double stop_tol2, double *gaps)
{
    double *r = (double *)malloc(sizeof(double) * (size_t)(nn > 0 ? nn : 1));
    double *r0 = (double *)malloc(sizeof(double) * (size_t)(nn > 0 ? nn : 1));
    int64_t steps = 0;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < nn; ++s) {
        double acc = 0.0;
        for (int64_t t = 0; t < l; ++t) acc += COL(Bw, ldb, t, s) * COL(Bw, ldb, t, s);
        r[s] = acc;
        r0[s] = acc;
    }
    for (int64_t j = 0; j < bb && j < nn; ++j) {
        /* (a) argmax_{s >= j} r_s, lowest index on exact ties */
        int64_t best = j;
        for (int64_t s = j + 1; s < nn; ++s)
            if (r[s] > r[best]) best = s;
        for (int64_t s = j; s < nn; ++s)
            if (!isfinite(r[s])) { steps = -1; goto done; }
        if (gaps) {
            double second = -1.0;
            for (int64_t s = j; s < nn; ++s)
                if (s != best && r[s] > second) second = r[s];
            gaps[j] = (second < 0.0 || r[best] == 0.0) ? 1.0 : (r[best] - second) / r[best];
        }
        if (!(r[best] > stop_tol2)) break; /* reading G12: rank exhausted */
        /* (b) swap columns j <-> best of B and of the norm arrays */
        piv[j] = best;
        if (best != j) {
            swap_cols(l, Bw, ldb, j, best);
            double t = r[j]; r[j] = r[best]; r[best] = t;
            t = r0[j]; r0[j] = r0[best]; r0[best] = t;
        }
        /* (c) Householder on B(j:l, j) */
        double *x = &COL(Bw, ldb, j, j);
        double tau = oracle_dlarfg(l - j, x);
        tauhat[j] = tau;
        /* (d) apply H_j to every remaining column */
#pragma omp parallel for schedule(static)
        for (int64_t s = j + 1; s < nn; ++s) {
            oracle_apply_reflector(l - j, x + 1, tau, &COL(Bw, ldb, j, s));
            /* (e) norm downdate with the cancellation guard (G6) */
            double bjs = COL(Bw, ldb, j, s);
            r[s] -= bjs * bjs;
            if (r[s] < 1e-6 * r0[s]) {
                double acc = 0.0;
                for (int64_t t = j + 1; t < l; ++t) acc += COL(Bw, ldb, t, s) * COL(Bw, ldb, t, s);
                r[s] = acc;
            }
        }
        steps = j + 1;
    }
done:
    free(r);
    free(r0);
    return steps;
}

/* ------------------------------------------------------------------------
 * Tournament pivoting on the sample (the paper's future work: "the
 * partial QRCP on B ... tournament pivoting"; reading R-TP of DESIGN.md).
 * The np trailing positions of the panel are split into `groups` groups by
 * the 1D block-cyclic layout (position c belongs to group ((i + c) / b) mod
 * groups: the columns a rank of that layout owns).  Each group selects up to
 * bb candidates by Alg. 1 (the function above: same norm rules, tie rule and
 * stop rule) on ITS columns of the sample; the candidate lists are then merged
 * pairwise up a binary tree (group g with g + span, span = 1, 2, 4, ...): the
 * union (left list, then right list) of original sample columns is reduced
 * to bb candidates by Alg. 1 again.  The root's pivot order is the panel's
 * pivot order.  F (out): the chosen positions; returns their number (or -1
 * on a non-finite norm).  With groups = 1 this is exactly Alg. 1's pivots.
 * ---------------------------------------------------------------------- */
static int64_t oracle_tournament(int64_t l, int64_t np, int64_t bb, const double *B, int64_t ldb, int64_t i, int b,
                                 int groups, double stop_tol2, int64_t *F)
{
    int64_t **cand = (int64_t **)calloc((size_t)groups, sizeof(int64_t *));
    int64_t *nc = (int64_t *)calloc((size_t)groups, sizeof(int64_t));
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(np > 2 * bb ? np : 2 * bb));
    double *W = (double *)malloc(sizeof(double) * (size_t)(l * (np > 2 * bb ? np : 2 * bb)));
    int64_t *pv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bb > 0 ? bb : 1));
    double *th = (double *)malloc(sizeof(double) * (size_t)(bb > 0 ? bb : 1));
    int64_t ret = 0;
    /* local selections */
    for (int g = 0; g < groups; ++g) {
        int64_t n_g = 0;
        for (int64_t c = 0; c < np; ++c)
            if (((i + c) / b) % groups == g) {
                idx[n_g] = c;
                memcpy(&W[n_g * l], &B[c * ldb], sizeof(double) * (size_t)l);
                ++n_g;
            }
        cand[g] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bb > 0 ? bb : 1));
        const int64_t want = bb < n_g ? bb : n_g;
        const int64_t got = want > 0 ? oracle_sample_qrcp(l, n_g, want, W, l, pv, th, stop_tol2, NULL) : 0;
        if (got < 0) { ret = -1; goto out; }
        for (int64_t j = 0; j < got; ++j) {  /* the transpositions, in order, on the index list */
            const int64_t s_ = pv[j], t = idx[j];
            idx[j] = idx[s_];
            idx[s_] = t;
        }
        for (int64_t j = 0; j < got; ++j) cand[g][j] = idx[j];
        nc[g] = got;
    }
    /* the merge tree */
    for (int span = 1; span < groups; span *= 2)
        for (int g = 0; g + span < groups; g += 2 * span) {
            const int h = g + span;
            int64_t nu = 0;
            for (int64_t q = 0; q < nc[g]; ++q) idx[nu++] = cand[g][q];
            for (int64_t q = 0; q < nc[h]; ++q) idx[nu++] = cand[h][q];
            for (int64_t q = 0; q < nu; ++q) memcpy(&W[q * l], &B[idx[q] * ldb], sizeof(double) * (size_t)l);
            const int64_t want = bb < nu ? bb : nu;
            const int64_t got = want > 0 ? oracle_sample_qrcp(l, nu, want, W, l, pv, th, stop_tol2, NULL) : 0;
            if (got < 0) { ret = -1; goto out; }
            for (int64_t j = 0; j < got; ++j) {
                const int64_t s_ = pv[j], t = idx[j];
                idx[j] = idx[s_];
                idx[s_] = t;
            }
            for (int64_t j = 0; j < got; ++j) cand[g][j] = idx[j];
            nc[g] = got;
        }
    for (int64_t j = 0; j < nc[0]; ++j) F[j] = cand[0][j];
    ret = nc[0];
out:
    for (int g = 0; g < groups; ++g) free(cand[g]);
    free(cand); free(nc); free(idx); free(W); free(pv); free(th);
    return ret;
}

/* The sample with given pivots (positions F[0..nsel), in order): the
 * transpositions j <-> current position of F[j] applied to Bw (piv[j] records
 * them, as Alg. 1 does), then the Householder QR of the first nsel columns,
 * each H_j applied to every column right of j: R-hat = Q-hat^T B Pi. */
static void oracle_sample_qr_given(int64_t l, int64_t nn, int64_t nsel, double *Bw, int64_t ldb, const int64_t *F,
                                   int64_t *piv, double *tauhat)
{
    int64_t *where = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nn > 0 ? nn : 1));
    int64_t *arr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nn > 0 ? nn : 1));
    for (int64_t c = 0; c < nn; ++c) { where[c] = c; arr[c] = c; }
    for (int64_t j = 0; j < nsel; ++j) {
        const int64_t s_ = where[F[j]];
        piv[j] = s_;
        if (s_ != j) {
            swap_cols(l, Bw, ldb, j, s_);
            const int64_t a_ = arr[j], b_ = arr[s_];
            arr[j] = b_; arr[s_] = a_;
            where[b_] = j; where[a_] = s_;
        }
    }
    for (int64_t j = 0; j < nsel; ++j) {
        double *x = &COL(Bw, ldb, j, j);
        const double t = oracle_dlarfg(l - j, x);
        tauhat[j] = t;
#pragma omp parallel for schedule(static)
        for (int64_t s_ = j + 1; s_ < nn; ++s_) oracle_apply_reflector(l - j, x + 1, t, &COL(Bw, ldb, j, s_));
    }
    free(where);
    free(arr);
}

/* Optional per-panel snapshot callback (tests only).  Pointers are valid only
 * during the call.  Rhat: l x n' (ld l), the sample after the bb-step QRCP in
 * pivoted column order, zero below the diagonal of its first bb columns.
 * Bnext: l x n'' (ld l) next sample or NULL.  OmegaCur: l x m' (ld l) the
 * effective Gaussian of this panel (B_cur = OmegaCur * A_cur) or NULL;
 * OmegaNew: l x m' (ld l), Omega-hat = Qhat^T OmegaCur Q (rule 1) or
 * Omega-bar = OmegaCur Q (rule 2), or NULL. */
typedef void (*oracle_panel_cb)(void *user, int64_t i, int64_t bb, int64_t l, int64_t mp, int64_t np,
                                const double *Rhat, const double *Bnext, const double *OmegaCur,
                                const double *OmegaNew, const double *A, int64_t lda);

#define ORACLE_INVARIANT 1 /* track Omega_cur, always run the sample update */

/* ------------------------------------------------------------------------
 * Alg. 2: returns 0, or a negative argument index (LAPACK info
 * style, same codes as include/rqrcp.h), or 4 (non-finite sample).
 *   Omega: l x m (ld l) explicit sketch, or NULL to draw it from (seed,
 *          stream 0) with the generator above.  l = b + p.
 *   update_rule: 1 = Eq. (4) (default), 2 = Eq. (5).
 *   A: m x n column-major, overwritten with V (below diag), R11/R12 (top k
 *      rows), R22 (trailing by-product) -- LAPACK dgeqp3 layout (G11).
 *   jpvt[n]: A Pi(:, j) = A(:, jpvt[j]), 0-based.  tau[k].  *rank_out.
 *   gaps[k] (optional): per-step relative pivot gap.
 * ---------------------------------------------------------------------- */
int oracle_rqrcp_tp(int64_t m, int64_t n, int64_t k, int b, int p, uint64_t seed, const double *Omega_in,
                    int update_rule, int flags, int tp_groups, double *A, int64_t lda, int64_t *jpvt, double *tau,
                    int64_t *rank_out, double *gaps, oracle_panel_cb cb, void *user);

int oracle_rqrcp(int64_t m, int64_t n, int64_t k, int b, int p, uint64_t seed, const double *Omega_in,
                 int update_rule, int flags, double *A, int64_t lda, int64_t *jpvt, double *tau,
                 int64_t *rank_out, double *gaps, oracle_panel_cb cb, void *user)
{
    return oracle_rqrcp_tp(m, n, k, b, p, seed, Omega_in, update_rule, flags, 0, A, lda, jpvt, tau, rank_out, gaps,
                           cb, user);
}

/* tp_groups > 1: the panel pivots come from tournament pivoting on the sample
 * (oracle_tournament above) instead of Alg. 1; everything else is Alg. 2. */
int oracle_rqrcp_tp(int64_t m, int64_t n, int64_t k, int b, int p, uint64_t seed, const double *Omega_in,
                    int update_rule, int flags, int tp_groups, double *A, int64_t lda, int64_t *jpvt, double *tau,
                    int64_t *rank_out, double *gaps, oracle_panel_cb cb, void *user)
{
    if (!A) return -2;
    if (lda < (m > 1 ? m : 1)) return -3;
    if (m < 1) return -4;
    if (n < 1) return -5;
    if (k < 1 || k > (m < n ? m : n)) return -6;
    if (b < 1) return -7;
    if (p < 0 || (int64_t)b + p > m) return -8;
    if (!jpvt) return -10;
    if (!tau) return -11;
    if (!rank_out) return -12;
    if (update_rule != 1 && update_rule != 2) return -13;

    const int64_t l = (int64_t)b + p;
    const int invariant = (flags & ORACLE_INVARIANT) != 0;
    const int track_omega = invariant || update_rule == 2;

    for (int64_t j = 0; j < n; ++j) jpvt[j] = j; /* Pi = I */
    for (int64_t j = 0; j < k; ++j) tau[j] = 0.0;
    *rank_out = 0;

    /* Omega */
    double *Om = (double *)malloc(sizeof(double) * (size_t)(l * m));
    if (Omega_in) memcpy(Om, Omega_in, sizeof(double) * (size_t)(l * m));
    else oracle_normal_fill(seed, 0u, 0, l, 0, m, Om, l);

    /* O1: B = Omega A */
    double *B = (double *)malloc(sizeof(double) * (size_t)(l * n));
    oracle_sketch(l, m, n, Om, l, A, lda, B, l);
    double bf2 = 0.0;
    for (int64_t t = 0; t < l * n; ++t) bf2 += B[t] * B[t];
    if (!isfinite(bf2)) { free(Om); free(B); return 4; }
    /* reading G12: stop when every candidate sample norm is
     * <= 1e3 eps ||B||_F; compared on squares */
    const double eps = 0x1p-52;
    const double stop_tol2 = (1e3 * eps) * (1e3 * eps) * bf2;

    /* Omega_cur (l x m'), only when tracking (invariant / Eq. (5) modes) */
    double *OmCur = NULL, *OmBar = NULL, *OmNew = NULL, *Bpre = NULL;
    if (track_omega) {
        OmCur = (double *)malloc(sizeof(double) * (size_t)(l * m));
        OmBar = (double *)malloc(sizeof(double) * (size_t)(l * m));
        OmNew = (double *)malloc(sizeof(double) * (size_t)(l * m));
        memcpy(OmCur, Om, sizeof(double) * (size_t)(l * m));
        Bpre = (double *)malloc(sizeof(double) * (size_t)(l * n));
    }
    double *Bnext = (double *)malloc(sizeof(double) * (size_t)(l * n));
    int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(b));
    double *tauhat = (double *)malloc(sizeof(double) * (size_t)(b));
    double *Vhat = (double *)malloc(sizeof(double) * (size_t)(l * b));

    int status = 0;
    int64_t i = 0;
    /* O2: for i = 1:b:k */
    while (i < k) {
        const int64_t planned = (int64_t)b < k - i ? (int64_t)b : k - i;
        int64_t bb = planned;
        const int64_t mp = m - i, np = n - i;
        double *Bcur = B; /* l x np sample of the trailing columns, ld l */
        if (update_rule == 2) memcpy(Bpre, Bcur, sizeof(double) * (size_t)(l * np));

        /* O3: partial QRCP on B(:, i:n), or tournament pivoting */
        int64_t got;
        if (tp_groups > 1) {
            int64_t *F = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bb > 0 ? bb : 1));
            got = oracle_tournament(l, np, bb, Bcur, l, i, b, tp_groups, stop_tol2, F);
            if (got > 0) oracle_sample_qr_given(l, np, got, Bcur, l, F, piv, tauhat);
            free(F);
        } else {
            got = oracle_sample_qrcp(l, np, bb, Bcur, l, piv, tauhat, stop_tol2, gaps ? gaps + i : NULL);
        }
        if (got < 0) { status = 4; break; }
        if (got == 0) break; /* rank exhausted before this panel */
        bb = got;

        /* O4: the same transpositions, in order, on A, Pi */
        for (int64_t j = 0; j < bb; ++j) {
            int64_t s = piv[j];
            if (s != j) {
                swap_cols(m, A, lda, i + j, i + s);
                int64_t t = jpvt[i + j]; jpvt[i + j] = jpvt[i + s]; jpvt[i + s] = t;
                if (update_rule == 2) swap_cols(l, Bpre, l, j, s);
            }
        }
        /* keep the sample reflectors, zero them out of R-hat */
        for (int64_t j = 0; j < bb; ++j)
            for (int64_t t = 0; t < l; ++t) {
                COL(Vhat, l, t, j) = (t > j) ? COL(Bcur, l, t, j) : (t == j ? 1.0 : 0.0);
                if (t > j) COL(Bcur, l, t, j) = 0.0;
            }

        /* O5: unblocked Householder QR of the panel A(i:m, i:i+bb) (P:149,
         * LAPACK dgeqr2: each H_j applied to the panel columns right of j),
         * then the trailing update A(i:m, i+bb:n) <- Q~^T A(i:m, i+bb:n)
         * column by column: H_i, ..., H_{i+bb-1} in order on each
         * trailing column.  Each column sees exactly the same sequence of
         * reflector applications as in the all-columns dgeqr2 order (columns
         * are independent), so the bits are those of dgeqr2 on A(i:m, i:n).
         * R11-diagonal rank stop (reading R-G12b, "singular R11 panel
         * (diagonal entry below 1e3 eps ||panel||)"): before column j is
         * transformed, |R(j,j)| = |beta_j| is compared with
         * 1e3 eps ||A(i:m, i:i+bb)||_F (the panel after its swaps); below it,
         * the factorization stops with rank j: column j and the rest of the
         * panel keep the reflectors < j (tau = 0 from j on), the trailing
         * columns get the reflectors < j. */
        double pan2 = 0.0;
        for (int64_t c = i; c < i + bb; ++c)
            for (int64_t r = i; r < m; ++r) pan2 += COL(A, lda, r, c) * COL(A, lda, r, c);
        const double ptol2 = (1e3 * eps) * (1e3 * eps) * pan2;
        int64_t diag_stop = -1;
        int64_t jend = i + bb;  /* reflectors i..jend-1 were formed */
        for (int64_t j = i; j < i + bb; ++j) {
            double *x = &COL(A, lda, j, j);
            double xn2 = 0.0;
            for (int64_t t = 1; t < m - j; ++t) xn2 += x[t] * x[t];
            const double alpha = x[0];
            const double beta = (xn2 == 0.0) ? alpha : ((alpha >= 0.0) ? -sqrt(alpha * alpha + xn2)
                                                                         : sqrt(alpha * alpha + xn2));
            if (beta * beta < ptol2) { diag_stop = j; jend = j; break; }
            double tj = oracle_dlarfg(m - j, x);
            tau[j] = tj;
            for (int64_t c = j + 1; c < i + bb; ++c) oracle_apply_reflector(m - j, x + 1, tj, &COL(A, lda, j, c));
        }
#pragma omp parallel for schedule(static)
        for (int64_t c = i + bb; c < n; ++c)
            for (int64_t j = i; j < jend; ++j)
                oracle_apply_reflector(m - j, &COL(A, lda, j + 1, j), tau[j], &COL(A, lda, j, c));
        if (diag_stop >= 0) {
            if (cb) cb(user, i, bb, l, mp, np, Bcur, NULL, NULL, NULL, A, lda);
            *rank_out = diag_stop;
            break;
        }

        const int64_t npp = np - bb; /* n'' */
        int last = (i + bb >= k);
        int do_update = (!last || invariant) && npp > 0;

        /* Omega tracking: OmBar = OmegaCur Q_panel (Omega-bar,
         * P:225), the panel reflectors applied to each row from the right;
         * OmNew = Omega-bar (rule 2) or Omega-hat = Qhat^T Omega-bar (rule 1,
         * P:183). */
        if (track_omega) {
            memcpy(OmBar, OmCur, sizeof(double) * (size_t)(l * mp));
#pragma omp parallel for schedule(static)
            for (int64_t r = 0; r < l; ++r) {
                for (int64_t j = 0; j < bb; ++j) {
                    const double *v = &COL(A, lda, i + j + 1, i + j); /* tail of v_j */
                    double tj = tau[i + j];
                    if (tj == 0.0) continue;
                    double w = COL(OmBar, l, r, j);
                    for (int64_t t = j + 1; t < mp; ++t) w += COL(OmBar, l, r, t) * v[t - j - 1];
                    double tw = tj * w;
                    COL(OmBar, l, r, j) -= tw;
                    for (int64_t t = j + 1; t < mp; ++t) COL(OmBar, l, r, t) -= tw * v[t - j - 1];
                }
            }
            memcpy(OmNew, OmBar, sizeof(double) * (size_t)(l * mp));
            if (update_rule == 1) {
#pragma omp parallel for schedule(static)
                for (int64_t c = 0; c < mp; ++c)
                    for (int64_t j = 0; j < bb; ++j)
                        oracle_apply_reflector(l - j, &COL(Vhat, l, j + 1, j), tauhat[j], &COL(OmNew, l, j, c));
            }
        }

        if (do_update) {
            if (update_rule == 1) {
                /* O6: Eq. (4): top rows R-hat12 - R-hat11 R11^-1 R12, bottom R-hat22
                 * (readings G1-G3, G20) */
#pragma omp parallel for schedule(static)
                for (int64_t c = 0; c < npp; ++c) {
                    double xs[1024];
                    double *x = xs;
                    if (bb > 1024) x = (double *)malloc(sizeof(double) * (size_t)bb);
                    /* X = R11^-1 R12(:, c): back substitution */
                    for (int64_t r = bb - 1; r >= 0; --r) {
                        double s = COL(A, lda, i + r, i + bb + c);
                        for (int64_t q = r + 1; q < bb; ++q) s -= COL(A, lda, i + r, i + q) * x[q];
                        x[r] = s / COL(A, lda, i + r, i + r);
                    }
                    /* top: R-hat12 - R-hat11 X */
                    for (int64_t r = 0; r < bb; ++r) {
                        double y = 0.0;
                        for (int64_t q = r; q < bb; ++q) y += COL(Bcur, l, r, q) * x[q];
                        COL(Bnext, l, r, c) = COL(Bcur, l, r, bb + c) - y;
                    }
                    for (int64_t r = bb; r < l; ++r) COL(Bnext, l, r, c) = COL(Bcur, l, r, bb + c);
                    if (x != xs) free(x);
                }
            } else {
                /* O8: Eq. (5): B2 - Omega-bar_1 R12 */
#pragma omp parallel for schedule(static)
                for (int64_t c = 0; c < npp; ++c)
                    for (int64_t r = 0; r < l; ++r) {
                        double y = 0.0;
                        for (int64_t q = 0; q < bb; ++q) y += COL(OmBar, l, r, q) * COL(A, lda, i + q, i + bb + c);
                        COL(Bnext, l, r, c) = COL(Bpre, l, r, bb + c) - y;
                    }
            }
        }
        if (cb) cb(user, i, bb, l, mp, np, Bcur, do_update ? Bnext : NULL, track_omega ? OmCur : NULL,
                   track_omega ? OmNew : NULL, A, lda);
        i += bb;
        *rank_out = i;
        if (bb < planned) break; /* rank exhausted inside this panel (G12) */
        if (!do_update) break;
        /* next panel: sample <- Bnext, OmegaCur <- OmNew(:, bb:) */
        memcpy(B, Bnext, sizeof(double) * (size_t)(l * npp));
        if (track_omega)
            for (int64_t c = 0; c < mp - bb; ++c)
                memcpy(&COL(OmCur, l, 0, c), &COL(OmNew, l, 0, bb + c), sizeof(double) * (size_t)l);
    }

    free(Om); free(B); free(Bnext); free(piv); free(tauhat); free(Vhat);
    if (OmCur) { free(OmCur); free(OmBar); free(OmNew); free(Bpre); }
    return status;
}

/* Thread count for the column-parallel loops (tests check that results are
 * bitwise independent of it).  Returns the previous maximum. */
int oracle_set_threads(int nthreads)
{
#ifdef _OPENMP
    int prev = omp_get_max_threads();
    if (nthreads > 0) omp_set_num_threads(nthreads);
    return prev;
#else
    (void)nthreads;
    return 1;
#endif
}
