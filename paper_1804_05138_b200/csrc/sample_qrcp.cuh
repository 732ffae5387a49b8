// sample_qrcp.cuh -- S2 (kernels K3+K4): bb steps of Businger-Golub QRCP
// (Alg. 1) on the l x n' sample B(:, i:n) (Alg. 2 line P:147).
//
// One persistent cooperative kernel; CTA g owns a contiguous range of the
// sample's PHYSICAL columns, caches them (and their norms) in shared memory
// when they fit, and keeps them in place for the whole panel: a
// transposition j <-> s* only relabels logical positions.  Warp per column,
// lanes over the l <= 160 rows, deterministic butterfly sums.  Per step j,
// exactly one grid barrier:
//   1. warp 0 of every CTA scans the G candidate slots in parallel and
//      reduces (value, logical position) -> the global argmax of the squared
//      norms, lowest logical position on exact ties (reading R-G5);
//   2. every CTA loads the winner's column (published in its slot by the
//      owner before the barrier) and computes the same dlarfg (R-G7)
//      redundantly -- identical bits everywhere (same code, same data);
//   3. each CTA applies H_j to its active columns and downdates the squared
//      norms, r_s -= B(j,s)^2, recomputing when r_s < 1e-6 r0_s (R-G6); the
//      column that sat at logical position j takes position s*;
//   4. each CTA publishes its best (and second best) candidate + column into
//      the slot buffer of parity (j+1)&1, then the grid barrier.
// Stops early (bb_eff < bb) when the winning squared norm is <= stop_tol2
// = (1e3 eps)^2 ||Omega A||_F^2 (reading R-G12).
// CTA 0 alone maintains pos2phys (logical position -> physical column) in
// global memory; at the end it emits the (dst, src) column moves that apply
// the same transpositions, in order, to A and Pi (S3) and pos2phys becomes
// `perm` for the sample update (S6).
// Other outputs: piv[j] (s* of step j, relative to column i), tauhat, Vhat
// (l x bb reflectors), Rhat11 (bb x bb), bb_eff, rank, gaps (diagnostic).
#pragma once
#include "common.cuh"

namespace rq {

constexpr int SQ_THREADS = 256;
constexpr int SQ_WARPS = SQ_THREADS / 32;
constexpr int SQ_MAXL = 160;   // l = b + p <= 160 rows (5 per lane)
constexpr int SQ_MAXB = 128;   // panel width

struct SqArgs {
    double *B;            // sample, physical columns, lpad x nn, ld ldb
    int64_t ldb;
    int l, lpad;
    int64_t nn;           // n' = trailing columns of this panel
    int bb;               // planned panel width
    int use_smem;         // cache own columns + state in dynamic shared memory
    const double *stop_tol2;
    double *r, *r0;       // per physical column (global mode)
    int *lpos;            // logical position per physical column (global mode)
    int *active;          // (global mode)
    double *slot_val;     // [2][G][2] best, second best
    int64_t *slot_pos;    // [2][G]
    int64_t *slot_col;    // [2][G]
    double *slot_data;    // [2][G][lpad]
    int64_t *piv;         // [bb]
    double *tauhat;       // [bb]
    double *vhat;         // lpad x bbpad (ld lpad)
    double *rhat11;       // bbpad x bbpad (ld bbpad)
    int bbpad;
    int64_t *perm;        // [nn] pos2phys: logical -> physical
    int64_t *swap_dst, *swap_src;  // [2 bb] column moves for S3
    int *swap_np;
    int *bb_eff;          // out
    int *done;            // in/out: set when the factorization stopped early
    int *rank;            // in/out: accumulated rank
    const int *status;    // non-zero -> no-op
    double *gaps;         // [bb] or nullptr
    unsigned *bar;        // per-launch barrier counter (zeroed by the host)
};

RQ_DEV bool sq_better(double v, int64_t pos, double bv, int64_t bpos) {
    return (v > bv) || (v == bv && pos < bpos);
}

// (best value, position, column, slot) + second-best value, reduced over a warp.
struct SqCand {
    double v, v2;
    int64_t pos, col;
    int slot;
};
RQ_DEV SqCand sq_combine(SqCand a, SqCand b) {
    SqCand r;
    if (sq_better(b.v, b.pos, a.v, a.pos)) {
        r = b;
        r.v2 = fmax(fmax(a.v2, b.v2), a.v);
    } else {
        r = a;
        r.v2 = fmax(fmax(a.v2, b.v2), b.v);
    }
    return r;
}
RQ_DEV SqCand sq_warp_reduce(SqCand c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        SqCand d;
        d.v = __shfl_xor_sync(0xffffffffu, c.v, o);
        d.v2 = __shfl_xor_sync(0xffffffffu, c.v2, o);
        d.pos = __shfl_xor_sync(0xffffffffu, c.pos, o);
        d.col = __shfl_xor_sync(0xffffffffu, c.col, o);
        d.slot = __shfl_xor_sync(0xffffffffu, c.slot, o);
        c = sq_combine(c, d);
    }
    return c;
}

// dynamic shared memory bytes needed to cache cpb columns
__host__ __device__ inline size_t sq_smem_bytes(int64_t cpb, int lpad) {
    return (size_t)cpb * ((size_t)lpad * sizeof(double) + 2 * sizeof(double) + 2 * sizeof(int));
}

__global__ void __launch_bounds__(SQ_THREADS) sample_qrcp_kernel(SqArgs a) {
    extern __shared__ __align__(16) double sq_dyn[];
    __shared__ double xs[SQ_MAXL];
    __shared__ SqCand wc[SQ_WARPS];
    __shared__ double s_tau, s_beta;
    __shared__ int64_t s_wpos, s_wcol;
    __shared__ int s_wslot, s_stop, s_np;

    const int G = gridDim.x;
    const int g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = a.l, lpad = a.lpad;
    const int64_t nn = a.nn;
    const int64_t cpb = (nn + G - 1) / G;
    const int64_t c_lo = min(nn, (int64_t)g * cpb), c_hi = min(nn, c_lo + cpb);
    const int ncol = (int)(c_hi - c_lo);

    if (*a.status != 0 || *a.done) {
        if (g == 0 && tid == 0) { *a.bb_eff = 0; *a.swap_np = 0; }
        return;
    }
    const double stop2 = *a.stop_tol2;
    unsigned epoch = 0;

    // column storage (local index cl = c - c_lo) and per-column state
    double *cols;
    int64_t ldc;
    double *r, *r0;
    int *lpos, *act;
    if (a.use_smem) {
        cols = sq_dyn;
        ldc = lpad;
        r = sq_dyn + (size_t)cpb * lpad;
        r0 = r + cpb;
        lpos = reinterpret_cast<int *>(r0 + cpb);
        act = lpos + cpb;
        for (int e = tid; e < ncol * l; e += SQ_THREADS) {
            const int t = e % l, cl = e / l;
            cols[t + (int64_t)cl * ldc] = a.B[t + (c_lo + cl) * a.ldb];
        }
        __syncthreads();
    } else {
        cols = a.B + c_lo * a.ldb;
        ldc = a.ldb;
        r = a.r + c_lo;
        r0 = a.r0 + c_lo;
        lpos = a.lpos + c_lo;
        act = a.active + c_lo;
    }
    for (int64_t x = c_lo + tid; x < c_hi; x += SQ_THREADS) a.perm[x] = x;

    // ---- initial squared norms (K3) ---------------------------------------
    for (int cl = warp; cl < ncol; cl += SQ_WARPS) {
        const double *col = cols + (int64_t)cl * ldc;
        double s = 0.0;
        for (int t = lane; t < l; t += 32) s += col[t] * col[t];
        s = warp_sum(s);
        if (lane == 0) { r[cl] = s; r0[cl] = s; lpos[cl] = (int)(c_lo + cl); act[cl] = 1; }
    }
    __syncthreads();

    // publish this CTA's best candidate into slot buffer `parity`
    auto publish = [&](int parity) {
        SqCand c{-1.0, -1.0, INT64_MAX, -1, g};
        for (int cl = warp; cl < ncol; cl += SQ_WARPS) {
            if (!act[cl]) continue;
            SqCand d{r[cl], -1.0, (int64_t)lpos[cl], c_lo + cl, g};
            c = sq_combine(c, d);
        }
        if (lane == 0) wc[warp] = c;
        __syncthreads();
        if (warp == 0) {
            SqCand d = (lane < SQ_WARPS) ? wc[lane] : SqCand{-1.0, -1.0, INT64_MAX, -1, g};
            d = sq_warp_reduce(d);
            if (lane == 0) {
                const int si = parity * G + g;
                a.slot_val[2 * si] = d.v;
                a.slot_val[2 * si + 1] = d.v2;
                a.slot_pos[si] = d.pos;
                a.slot_col[si] = d.col;
                s_wcol = d.col;
            }
        }
        __syncthreads();
        const int64_t c0 = s_wcol;
        if (c0 >= 0) {
            double *dst = a.slot_data + (int64_t)(parity * G + g) * lpad;
            const double *src = cols + (c0 - c_lo) * ldc;
            for (int t = tid; t < l; t += SQ_THREADS) dst[t] = src[t];
        }
    };

    publish(0);
    grid_barrier(a.bar, G, epoch);

    int j = 0;
    for (; j < a.bb; ++j) {
        const int par = j & 1;
        // ---- 1. global winner (warp 0, parallel over slots) ---------------
        if (warp == 0) {
            // all slot loads first (G <= 160: at most 5 per lane), then combine
            SqCand d[5];
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const int q = lane + 32 * u;
                d[u] = SqCand{-1.0, -1.0, INT64_MAX, -1, q};
                if (q < G) {
                    const int si = par * G + q;
                    d[u].col = __ldcg(a.slot_col + si);
                    d[u].v = __ldcg(a.slot_val + 2 * si);
                    d[u].v2 = __ldcg(a.slot_val + 2 * si + 1);
                    d[u].pos = __ldcg(a.slot_pos + si);
                }
            }
            SqCand c{-1.0, -1.0, INT64_MAX, -1, -1};
#pragma unroll
            for (int u = 0; u < 5; ++u)
                if (d[u].col >= 0) c = sq_combine(c, d[u]);
            c = sq_warp_reduce(c);
            if (lane == 0) {
                s_wpos = c.pos;
                s_wcol = c.col;
                s_wslot = c.slot;
                s_stop = (c.col < 0) || !(c.v > stop2);
                if (g == 0 && a.gaps && !s_stop) a.gaps[j] = (c.v2 < 0.0 || c.v == 0.0) ? 1.0 : (c.v - c.v2) / c.v;
            }
        }
        __syncthreads();
        if (s_stop) break;
        const int64_t wp = s_wpos, wcl = s_wcol;
        // ---- 2. winner column -> Householder (identical in every CTA) -----
        {
            const double *src = a.slot_data + (int64_t)(par * G + s_wslot) * lpad;
            for (int t = tid; t < l; t += SQ_THREADS) xs[t] = ld_cg(src + t);
        }
        if (wcl >= c_lo && wcl < c_hi && tid == 0) act[wcl - c_lo] = 0;  // retire the pivot
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
        // ---- outputs (CTA 0) ------------------------------------------------
        if (g == 0) {
            for (int t = tid; t < lpad; t += SQ_THREADS)
                a.vhat[t + (int64_t)j * lpad] = (t < j) ? 0.0 : (t == j ? 1.0 : (t < l ? xs[t] : 0.0));
            for (int t = tid; t < a.bbpad; t += SQ_THREADS)
                a.rhat11[t + (int64_t)j * a.bbpad] = (t < j) ? xs[t] : (t == j ? s_beta : 0.0);
            if (tid == 0) {
                a.piv[j] = wp;
                a.tauhat[j] = tau;
                // transposition j <-> wp on the logical -> physical map
                const int64_t q = a.perm[j];
                a.perm[j] = wcl;
                if (wp != j) a.perm[wp] = q;
            }
        }
        // ---- 3. apply H_j to own active columns, downdate norms -----------
        for (int cl = warp; cl < ncol; cl += SQ_WARPS) {
            if (!act[cl]) continue;
            double *col = cols + (int64_t)cl * ldc;
            double wsum = 0.0;
            for (int t = j + lane; t < l; t += 32) wsum += ((t == j) ? 1.0 : xs[t]) * col[t];
            wsum = warp_sum(wsum);
            const double tw = tau * wsum;
            for (int t = j + lane; t < l; t += 32) col[t] -= tw * ((t == j) ? 1.0 : xs[t]);
            __syncwarp();
            const double bj = col[j];
            double rn = r[cl] - bj * bj;
            if (rn < 1e-6 * r0[cl]) {
                double s = 0.0;
                for (int t = j + 1 + lane; t < l; t += 32) s += col[t] * col[t];
                rn = warp_sum(s);
            }
            if (lane == 0) {
                r[cl] = rn;
                if (lpos[cl] == j) lpos[cl] = (int)wp;  // the column at position j moves to s*
            }
        }
        __syncthreads();
        // ---- 4. candidates for step j+1 -----------------------------------
        publish(par ^ 1);
        grid_barrier(a.bar, G, epoch);
    }

    // ---- results ------------------------------------------------------------
    if (a.use_smem) {  // write the transformed columns back (S6 reads R-hat12/22)
        for (int e = tid; e < ncol * l; e += SQ_THREADS) {
            const int t = e % l, cl = e / l;
            a.B[t + (c_lo + cl) * a.ldb] = cols[t + (int64_t)cl * ldc];
        }
    }
    if (g == 0) {
        if (tid == 0) s_np = 0;
        __syncthreads();
        // column moves (dst <- src) for every touched position whose content changed
        for (int e = tid; e < 2 * j; e += SQ_THREADS) {
            int64_t x;
            bool take;
            if (e < j) {
                x = e;
                take = true;
            } else {
                const int jj = e - j;
                x = a.piv[jj];
                take = x >= j;  // positions < j are covered above
                for (int q = jj + 1; q < j && take; ++q)
                    if (a.piv[q] == x) take = false;  // keep only the last occurrence
            }
            if (take) {
                const int64_t src = a.perm[x];
                if (src != x) {
                    const int slot = atomicAdd(&s_np, 1);
                    a.swap_dst[slot] = x;
                    a.swap_src[slot] = src;
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            *a.swap_np = s_np;
            *a.bb_eff = j;
            *a.rank += j;
            if (j < a.bb) *a.done = 1;
        }
    }
}

}  // namespace rq
