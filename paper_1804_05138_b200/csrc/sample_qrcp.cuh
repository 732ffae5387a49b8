// sample_qrcp.cuh -- S2 (kernels K3+K4): bb steps of Businger-Golub QRCP
// (Alg. 1) on the l x n' sample B(:, i:n) (Alg. 2 line P:147).
//
// One persistent cooperative kernel; CTA g owns a contiguous range of the
// sample's PHYSICAL columns and keeps them in place for the whole panel
// (pivoting is bookkept, not performed: a transposition j <-> s* only
// relabels logical positions).  Warp per column: lanes over the l <= 160
// rows, deterministic butterfly sums.  Per step j, one grid barrier:
//   1. every CTA scans the G candidate slots (value, logical position,
//      physical column) and picks the global argmax of the squared norms,
//      lowest logical position on exact ties (reading R-G5);
//   2. every CTA loads the winner's column (written to its slot by the
//      owner before the barrier) and computes the same dlarfg (R-G7)
//      redundantly (identical bits: same code, same data, fixed order);
//   3. each CTA applies H_j to its active columns and downdates the squared
//      norms, r_s -= B(j,s)^2, recomputing when r_s < 1e-6 r0_s (R-G6);
//   4. each CTA writes its best (and second best) candidate + column data
//      into the slot buffer of parity (j+1)&1, then the grid barrier.
// Stops early (bb_eff < bb) when the winning squared norm is <= stop_tol2
// = (1e3 eps)^2 ||Omega A||_F^2 (reading R-G12).
// Outputs: piv[j] (transposition j <-> piv[j], relative to column i),
// tauhat, Vhat (l x bb reflectors), Rhat11 (bb x bb), perm (logical ->
// physical column of the transformed sample, consumed by S6), bb_eff.
#pragma once
#include "common.cuh"

namespace rq {

constexpr int SQ_THREADS = 256;
constexpr int SQ_WARPS = SQ_THREADS / 32;
constexpr int SQ_MAXL = 160;   // l = b + p <= 160 rows (5 per lane)
constexpr int SQ_MAXB = 128;   // panel width
constexpr int SQ_TBL = 2 * SQ_MAXB + 2;

struct SqArgs {
    double *B;            // sample, physical columns, lpad x nn, ld ldb
    int64_t ldb;
    int l, lpad;
    int64_t nn;           // n' = trailing columns of this panel
    int bb;               // planned panel width
    const double *stop_tol2;
    double *r, *r0;       // per physical column
    int *lpos;            // logical position per physical column
    unsigned char *active;
    double *slot_val;     // [2][G][2] best, second best
    int64_t *slot_pos;    // [2][G]
    int64_t *slot_col;    // [2][G]
    double *slot_data;    // [2][G][lpad]
    int64_t *piv;         // [bb]
    double *tauhat;       // [bb]
    double *vhat;         // lpad x bbpad (ld lpad)
    double *rhat11;       // bbpad x bbpad (ld bbpad)
    int bbpad;
    int64_t *perm;        // [nn] logical -> physical
    int *bb_eff;          // out
    int *done;            // in/out: set when the factorization stopped early
    int *rank;            // in/out: accumulated rank
    const int *status;    // non-zero -> no-op
    double *gaps;         // [bb] or nullptr
    unsigned *bar;
};

struct SqCand {
    double v, v2;
    int64_t pos, col;
};

RQ_DEV bool sq_better(double v, int64_t pos, double bv, int64_t bpos) {
    return (v > bv) || (v == bv && pos < bpos);
}

__global__ void __launch_bounds__(SQ_THREADS) sample_qrcp_kernel(SqArgs a) {
    __shared__ double xs[SQ_MAXL];
    __shared__ double wv[SQ_WARPS], wv2[SQ_WARPS];
    __shared__ int64_t wpos[SQ_WARPS], wcol[SQ_WARPS];
    __shared__ int tbl_pos[SQ_TBL];
    __shared__ int64_t tbl_phys[SQ_TBL];
    __shared__ int tbl_n;
    __shared__ double s_tau, s_beta;
    __shared__ int64_t s_wpos, s_wcol;
    __shared__ int s_stop;

    const int G = gridDim.x;
    const int g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = a.l;
    const int64_t nn = a.nn;
    const int64_t cpb = (nn + G - 1) / G;
    const int64_t c_lo = min(nn, (int64_t)g * cpb), c_hi = min(nn, c_lo + cpb);

    if (*a.status != 0 || *a.done) {
        if (g == 0 && tid == 0) *a.bb_eff = 0;
        return;
    }
    const double stop2 = *a.stop_tol2;
    if (tid == 0) tbl_n = 0;

    // ---- initial squared norms (K3) and the first candidates -------------
    auto local_argmax = [&](int parity) {
        double bv = -1.0, bv2 = -1.0;
        int64_t bpos = INT64_MAX, bcol = -1;
        for (int64_t c = c_lo + warp; c < c_hi; c += SQ_WARPS) {
            if (!a.active[c]) continue;
            const double v = a.r[c];
            const int64_t p = a.lpos[c];
            if (sq_better(v, p, bv, bpos)) {
                bv2 = fmax(bv2, bv);
                bv = v; bpos = p; bcol = c;
            } else {
                bv2 = fmax(bv2, v);
            }
        }
        if (lane == 0) { wv[warp] = bv; wv2[warp] = bv2; wpos[warp] = bpos; wcol[warp] = bcol; }
        __syncthreads();
        if (tid == 0) {
            double v = -1.0, v2 = -1.0;
            int64_t p = INT64_MAX, c = -1;
            for (int w = 0; w < SQ_WARPS; ++w) {
                if (wcol[w] < 0) continue;
                if (sq_better(wv[w], wpos[w], v, p)) {
                    v2 = fmax(v2, v);
                    v = wv[w]; p = wpos[w]; c = wcol[w];
                } else {
                    v2 = fmax(v2, wv[w]);
                }
                v2 = fmax(v2, wv2[w]);
            }
            const int si = parity * G + g;
            a.slot_val[2 * si] = v;
            a.slot_val[2 * si + 1] = v2;
            a.slot_pos[si] = p;
            a.slot_col[si] = c;
            s_wcol = c;
        }
        __syncthreads();
        const int64_t c = s_wcol;
        double *dst = a.slot_data + (int64_t)(parity * G + g) * a.lpad;
        if (c >= 0)
            for (int t = tid; t < l; t += SQ_THREADS) dst[t] = a.B[t + c * a.ldb];
    };

    for (int64_t c = c_lo + warp; c < c_hi; c += SQ_WARPS) {
        const double *col = a.B + c * a.ldb;
        double s = 0.0;
        for (int t = lane; t < l; t += 32) s += col[t] * col[t];
        s = warp_sum(s);
        if (lane == 0) { a.r[c] = s; a.r0[c] = s; a.lpos[c] = (int)c; a.active[c] = 1; }
    }
    __syncthreads();
    local_argmax(0);
    grid_barrier(a.bar, G);

    int j = 0;
    for (; j < a.bb; ++j) {
        const int par = j & 1;
        // ---- 1. global winner --------------------------------------------
        if (tid == 0) {
            double v = -1.0, v2 = -1.0;
            int64_t p = INT64_MAX, c = -1;
            int ws = -1;
            for (int q = 0; q < G; ++q) {
                const int si = par * G + q;
                const int64_t cq = *(volatile int64_t *)(a.slot_col + si);
                if (cq < 0) continue;
                const double vq = *(volatile double *)(a.slot_val + 2 * si);
                const double vq2 = *(volatile double *)(a.slot_val + 2 * si + 1);
                const int64_t pq = *(volatile int64_t *)(a.slot_pos + si);
                if (sq_better(vq, pq, v, p)) {
                    v2 = fmax(v2, v);
                    v = vq; p = pq; c = cq; ws = q;
                } else {
                    v2 = fmax(v2, vq);
                }
                v2 = fmax(v2, vq2);
            }
            s_wpos = p; s_wcol = c;
            s_stop = (c < 0) || !(v > stop2);
            if (g == 0 && a.gaps && !s_stop) a.gaps[j] = (v2 < 0.0 || v == 0.0) ? 1.0 : (v - v2) / v;
            xs[0] = (double)ws;  // stash slot index
        }
        __syncthreads();
        if (s_stop) break;
        const int ws = (int)xs[0];
        __syncthreads();
        // ---- 2. winner column -> Householder (identical in every CTA) -----
        {
            const double *src = a.slot_data + (int64_t)(par * G + ws) * a.lpad;
            for (int t = tid; t < l; t += SQ_THREADS) xs[t] = ld_cg(src + t);
        }
        __syncthreads();
        if (warp == 0) {
            double s = 0.0;
            for (int t = j + 1 + lane; t < l; t += 32) s += xs[t] * xs[t];
            s = warp_sum(s);
            const double alpha = xs[j];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (s != 0.0) {
                const double nrm = sqrt(alpha * alpha + s);
                beta = (alpha >= 0.0) ? -nrm : nrm;
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            __syncwarp();
            for (int t = j + 1 + lane; t < l; t += 32) xs[t] *= scal;
            if (lane == 0) { s_tau = tau; s_beta = beta; }
        }
        __syncthreads();
        const double tau = s_tau;
        // ---- outputs + transposition bookkeeping (identical in all CTAs) --
        if (g == 0) {
            for (int t = tid; t < a.lpad; t += SQ_THREADS)
                a.vhat[t + (int64_t)j * a.lpad] = (t < j) ? 0.0 : (t == j ? 1.0 : (t < l ? xs[t] : 0.0));
            for (int t = tid; t < a.bbpad; t += SQ_THREADS)
                a.rhat11[t + (int64_t)j * a.bbpad] = (t < j) ? xs[t] : (t == j ? s_beta : 0.0);
            if (tid == 0) { a.piv[j] = s_wpos; a.tauhat[j] = tau; }
        }
        if (tid == 0) {
            // q = physical column at logical position j
            int64_t q = j;
            for (int e = 0; e < tbl_n; ++e)
                if (tbl_pos[e] == j) q = tbl_phys[e];
            const int64_t wp = s_wpos, wc = s_wcol;
            // position j <- winner, position wp <- q
            auto assign = [&](int pos, int64_t phys) {
                for (int e = 0; e < tbl_n; ++e)
                    if (tbl_pos[e] == pos) { tbl_phys[e] = phys; return; }
                tbl_pos[tbl_n] = pos; tbl_phys[tbl_n] = phys; ++tbl_n;
            };
            assign(j, wc);
            if (wp != j) {
                assign((int)wp, q);
                if (q >= c_lo && q < c_hi) a.lpos[q] = (int)wp;
            }
            if (wc >= c_lo && wc < c_hi) a.active[wc] = 0;
        }
        __syncthreads();
        // ---- 3. apply H_j to own active columns, downdate norms -----------
        for (int64_t c = c_lo + warp; c < c_hi; c += SQ_WARPS) {
            if (!a.active[c]) continue;
            double *col = a.B + c * a.ldb;
            double wsum = 0.0;
            for (int t = j + lane; t < l; t += 32) wsum += ((t == j) ? 1.0 : xs[t]) * col[t];
            wsum = warp_sum(wsum);
            const double tw = tau * wsum;
            for (int t = j + lane; t < l; t += 32) col[t] -= tw * ((t == j) ? 1.0 : xs[t]);
            __syncwarp();
            const double bj = col[j];
            double rn = a.r[c] - bj * bj;
            if (rn < 1e-6 * a.r0[c]) {
                double s = 0.0;
                for (int t = j + 1 + lane; t < l; t += 32) s += col[t] * col[t];
                rn = warp_sum(s);
            }
            if (lane == 0) a.r[c] = rn;
        }
        __syncthreads();
        // ---- 4. candidates for step j+1 -----------------------------------
        local_argmax(par ^ 1);
        grid_barrier(a.bar, G);
    }

    // ---- results: perm (logical -> physical), bb_eff, rank ---------------
    for (int64_t x = c_lo + tid; x < c_hi; x += SQ_THREADS) a.perm[x] = x;
    __syncthreads();
    if (tid == 0)
        for (int e = 0; e < tbl_n; ++e)
            if (tbl_pos[e] >= c_lo && tbl_pos[e] < c_hi) a.perm[tbl_pos[e]] = tbl_phys[e];
    if (g == 0 && tid == 0) {
        *a.bb_eff = j;
        *a.rank += j;
        if (j < a.bb) *a.done = 1;
    }
}

}  // namespace rq
