// sample_qrcp.cuh -- S2 (kernels K3+K4): bb steps of Businger-Golub QRCP
// (Alg. 1) on the l x n' sample B(:, i:n) (Alg. 2 line P:147).
//
// One persistent cooperative kernel; CTA g owns a contiguous range of the
// sample's PHYSICAL columns and keeps them in place for the whole panel (a
// transposition j <-> s* only relabels logical positions).  As many of its
// columns as fit live in shared memory, the rest stay in global memory (L2);
// per-column state (squared norm, its panel-start value, logical position,
// active flag) always lives in shared memory.  Each warp processes SQ_CB
// columns at a time with all their loads in flight, lanes over the l <= 160
// rows, deterministic butterfly sums.  Per step j, exactly one grid barrier:
//   1. warp 0 of every CTA loads the G candidate headers (one 16-byte load
//      each; a step tag makes stale slots detectable) and reduces
//      (value, logical position) -> the global argmax of
//      the squared norms, lowest logical position on exact ties (R-G5);
//   2. warp 0 of every CTA loads the winner's column (published in its slot
//      by the owner before the barrier) and computes the same dlarfg (R-G7)
//      redundantly -- identical bits everywhere (same code, same data);
//   3. each CTA applies H_j to its active columns and downdates the squared
//      norms, r_s -= B(j,s)^2, recomputing when r_s < 1e-6 r0_s (R-G6); the
//      column that sat at logical position j takes position s*; each warp
//      tracks its best remaining column on the fly;
//   4. each CTA publishes its best candidate (header + column) into the slot
//      buffer of parity (j+1)&1, then the grid barrier.
// Stops early (bb_eff < bb) when the winning squared norm is <= stop_tol2
// = (1e3 eps)^2 ||Omega A||_F^2 (reading R-G12).
// CTA 0 tracks the logical -> physical map of the touched positions in
// shared memory (positions < bb direct-mapped, others in a short list); at the
// end it writes `perm` (consumed by S6) and the (dst, src) column moves that
// apply the same transpositions, in order, to A and Pi (S3).
// Other outputs: piv[j] (s* of step j, relative to column i), tauhat, Vhat
// (l x bb reflectors), Rhat11 (bb x bb), bb_eff, rank, gaps (diagnostic).
#pragma once
#include <climits>
#include "common.cuh"

namespace rq {

constexpr int SQ_THREADS = 256;
constexpr int SQ_WARPS = SQ_THREADS / 32;
constexpr int SQ_MAXL = 160;  // l = b + p <= 160 rows
constexpr int SQ_RPL = 5;     // rows per lane
constexpr int SQ_MAXB = 128;  // panel width
constexpr int SQ_CB = 4;      // columns per warp iteration (memory-level parallelism)

struct SqHdr {    // one candidate slot header (16 bytes, written as one vector store)
    double v;       // squared norm of the best active column (-1: none)
    unsigned tag;   // launch sequence * 256 + step: never repeats within a context
    int pos;        // logical position (INT_MAX: none)
};

struct SqArgs {
    double *B;            // sample, physical columns, lpad x nn, ld ldb
    int64_t ldb;
    int l, lpad;
    int64_t nn;           // n' = trailing columns of this panel
    int bb;               // planned panel width
    int nsm;              // columns per CTA cached in shared memory
    const double *stop_tol2;
    SqHdr *slot_hdr;      // [2][G]
    int *slot_col;        // [2][G] physical column of the candidate (written before the header)
    double *slot_v2;      // [2][G] second best (diagnostic, only with gaps)
    double *slot_data;    // [2][G][lpad]
    int64_t *piv;         // [bb]
    double *tauhat;       // [bb]
    double *vhat;         // lpad x bbpad (ld lpad)
    double *rhat11;       // bbpad x bbpad (ld bbpad)
    int bbpad;
    int64_t *perm;        // [nn] logical -> physical
    int64_t *swap_dst, *swap_src;  // [2 bb] column moves for S3
    int *swap_np;
    int *bb_eff;          // out
    int *done;            // in/out: set when the factorization stopped early
    int *rank;            // in/out: accumulated rank
    const int *status;    // non-zero -> no-op
    double *gaps;         // [bb] or nullptr
    unsigned *bar;        // per-launch barrier counter (zeroed by the host)
    unsigned tag0;        // launch sequence * 256 (distinct per launch)
    unsigned long long *trace;  // debug: [2 CTAs][64 steps][8 phases] clock64 stamps, or nullptr
};

RQ_DEV bool sq_better(double v, int pos, double bv, int bpos) { return (v > bv) || (v == bv && pos < bpos); }

// dynamic shared memory: nsm cached columns + state of cpb columns
__host__ __device__ inline size_t sq_smem_bytes(int64_t nsm, int64_t cpb, int lpad) {
    return (size_t)nsm * lpad * sizeof(double) + (size_t)cpb * (2 * sizeof(double) + 2 * sizeof(int));
}

__global__ void __launch_bounds__(SQ_THREADS) sample_qrcp_kernel(SqArgs a) {
    extern __shared__ __align__(16) double sq_dyn[];
    __shared__ double xs[SQ_MAXL];
    __shared__ double wv[SQ_WARPS], wv2[SQ_WARPS];
    __shared__ int wpos[SQ_WARPS], wcol[SQ_WARPS];
    __shared__ double s_tau, s_beta, s_hv;
    __shared__ int s_wpos, s_wcol, s_stop, s_np, s_hpos;
    __shared__ int64_t low[SQ_MAXB];  // CTA 0: phys column at positions < bb
    __shared__ int hi_pos[SQ_MAXB];   // CTA 0: touched positions >= bb ...
    __shared__ int64_t hi_phys[SQ_MAXB];  // ... and their phys columns
    __shared__ int hi_n;

    const int G = gridDim.x;
    const int g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = a.l, lpad = a.lpad;
    const int64_t nn = a.nn;
    const int64_t cpb = (nn + G - 1) / G;
    const int64_t c_lo = min(nn, (int64_t)g * cpb), c_hi = min(nn, c_lo + cpb);
    const int ncol = (int)(c_hi - c_lo);
    const int nsm = min(ncol, a.nsm);
    const bool want_v2 = a.gaps != nullptr;

    if (*a.status != 0 || *a.done) {
        if (g == 0 && tid == 0) { *a.bb_eff = 0; *a.swap_np = 0; }
        return;
    }
    const double stop2 = *a.stop_tol2;

    // shared layout: [nsm cached columns][r][r0][lpos][act]
    double *cols_s = sq_dyn;
    double *r = sq_dyn + (size_t)a.nsm * lpad;
    double *r0 = r + cpb;
    int *lpos = reinterpret_cast<int *>(r0 + cpb);
    int *act = lpos + cpb;
    auto colp = [&](int cl) -> const double * {
        return (cl < nsm) ? cols_s + (size_t)cl * lpad : a.B + (c_lo + cl) * a.ldb;
    };
    for (int e = tid; e < nsm * l; e += SQ_THREADS) {
        const int t = e % l, cl = e / l;
        cols_s[t + (size_t)cl * lpad] = a.B[t + (c_lo + cl) * a.ldb];
    }
    for (int64_t x = c_lo + tid; x < c_hi; x += SQ_THREADS) a.perm[x] = x;
    if (g == 0) {
        for (int x = tid; x < a.bb; x += SQ_THREADS) low[x] = x;
        if (tid == 0) hi_n = 0;
    }
    __syncthreads();

    // this warp's best active column (and second-best value)
    double bv = -1.0, bv2 = -1.0;
    int bpos = INT_MAX, bcol = -1;
    auto consider = [&](double v, int pos, int col) {
        if (sq_better(v, pos, bv, bpos)) {
            bv2 = fmax(bv2, bv);
            bv = v; bpos = pos; bcol = col;
        } else {
            bv2 = fmax(bv2, v);
        }
    };
    // ---- initial squared norms (K3) ---------------------------------------
    for (int cl0 = warp * SQ_CB; cl0 < ncol; cl0 += SQ_WARPS * SQ_CB) {
        double x[SQ_CB][SQ_RPL];
#pragma unroll
        for (int u = 0; u < SQ_CB; ++u) {
            const int cl = cl0 + u;
            const double *col = (cl < ncol) ? colp(cl) : nullptr;
#pragma unroll
            for (int q = 0; q < SQ_RPL; ++q) {
                const int t = lane + 32 * q;
                x[u][q] = (col && t < l) ? col[t] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < SQ_CB; ++u) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < SQ_RPL; ++q) s += x[u][q] * x[u][q];
            s = warp_sum(s);
            const int cl = cl0 + u;
            if (cl < ncol) {
                if (lane == 0) { r[cl] = s; r0[cl] = s; lpos[cl] = (int)(c_lo + cl); act[cl] = 1; }
                consider(s, (int)(c_lo + cl), (int)(c_lo + cl));
            }
        }
    }

    // publish this CTA's best candidate for step `step` (slot parity step & 1);
    // the grid barrier that follows makes it visible.
    auto publish = [&](int step) {
        const int parity = step & 1;
        if (lane == 0) { wv[warp] = bv; wv2[warp] = bv2; wpos[warp] = bpos; wcol[warp] = bcol; }
        __syncthreads();
        if (warp == 0) {
            double v = -1.0, v2 = -1.0;
            int p = INT_MAX, c = -1;
            if (lane < SQ_WARPS) { v = wv[lane]; v2 = wv2[lane]; p = wpos[lane]; c = wcol[lane]; }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {  // 8 warps
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const double ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                const int oc = __shfl_xor_sync(0xffffffffu, c, o);
                if (sq_better(ov, op, v, p)) {
                    v2 = fmax(fmax(v2, ov2), v);
                    v = ov; p = op; c = oc;
                } else {
                    v2 = fmax(fmax(v2, ov2), ov);
                }
            }
            if (lane == 0) {
                s_hv = v; s_hpos = p; s_wcol = c;
                if (want_v2) a.slot_v2[parity * G + g] = v2;
                a.slot_col[parity * G + g] = c;
            }
        }
        __syncthreads();
        const int c0 = s_wcol;
        if (c0 >= 0) {
            double *dst = a.slot_data + (int64_t)(parity * G + g) * lpad;
            const int cl = c0 - (int)c_lo;
            const double *src = (cl < nsm) ? cols_s + (size_t)cl * lpad : a.B + (int64_t)c0 * a.ldb;
            for (int t = tid; t < l; t += SQ_THREADS) dst[t] = src[t];
        }
        __syncthreads();
        if (tid == 0) {
            SqHdr h;
            h.v = s_hv;
            h.tag = a.tag0 + (unsigned)step;
            h.pos = s_hpos;
            st_cg_v2(reinterpret_cast<double2 *>(a.slot_hdr + parity * G + g), *reinterpret_cast<double2 *>(&h));
        }
    };

    publish(0);
    unsigned epoch = 0;
    grid_barrier(a.bar, G, epoch);

    int j = 0;
    const int tsel = (g == 0) ? 0 : (g == (int)gridDim.x - 1 ? 1 : -1);
    auto stamp = [&](int ph) {
        if (a.trace && tsel >= 0 && tid == 0 && j < 64) a.trace[((size_t)tsel * 64 + j) * 8 + ph] = clock64();
    };
    for (; j < a.bb; ++j) {
        const int par = j & 1;
        stamp(0);
        // ---- 1+2. global winner and its Householder reflector ----------------
        // warps 0..ceil(G/32)-1 each reduce 32 headers (one 16-byte load per
        // lane) and speculatively prefetch their local winner's column; the
        // warp holding the global winner then forms dlarfg (R-G7) from its
        // registers -- identical bits in every CTA (same data, same code).
        const int nsw = (G + 31) >> 5;  // scanning warps (<= 5)
        double xv[SQ_RPL];
        if (warp < nsw) {
            double v = -1.0, v2 = -1.0;
            int p = INT_MAX, sl = -1;
            const int q = lane + 32 * warp;
            if (q < G) {
                const double2 raw = __ldcg(reinterpret_cast<const double2 *>(a.slot_hdr + par * G + q));
                const int qp = __double2hiint(raw.y);
                if (qp != INT_MAX) { v = raw.x; p = qp; sl = q; }
                if (want_v2) v2 = __ldcg(a.slot_v2 + par * G + q);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                const int osl = __shfl_xor_sync(0xffffffffu, sl, o);
                const double ov2 = want_v2 ? __shfl_xor_sync(0xffffffffu, v2, o) : -1.0;
                if (sq_better(ov, op, v, p)) {
                    v2 = fmax(fmax(v2, ov2), v);
                    v = ov; p = op; sl = osl;
                } else {
                    v2 = fmax(fmax(v2, ov2), ov);
                }
            }
            const double *src = a.slot_data + (int64_t)(par * G + (sl >= 0 ? sl : 0)) * lpad;
#pragma unroll
            for (int qq = 0; qq < SQ_RPL; ++qq) {
                const int t = lane + 32 * qq;
                xv[qq] = (sl >= 0 && t < l) ? __ldcg(src + t) : 0.0;
            }
            if (lane == 0) { wv[warp] = v; wv2[warp] = v2; wpos[warp] = p; wcol[warp] = sl; }
        }
        __syncthreads();
        int ww = 0;  // warp holding the global winner (same choice in every thread)
        {
            double v = wv[0];
            int p = wpos[0];
            for (int w2 = 1; w2 < nsw; ++w2)
                if (wcol[w2] >= 0 && (wcol[ww] < 0 || sq_better(wv[w2], wpos[w2], v, p))) {
                    ww = w2; v = wv[w2]; p = wpos[w2];
                }
        }
        if (warp == ww) {
            const int sl = wcol[ww];
            const double vbest = wv[ww];
            double v2 = -1.0;
            for (int w2 = 0; w2 < nsw; ++w2) v2 = fmax(v2, (w2 == ww) ? wv2[w2] : wv[w2]);
            const bool stop = (sl < 0) || !(vbest > stop2);
            if (lane == 0) {
                s_stop = stop;
                s_wpos = wpos[ww];
                s_wcol = (sl >= 0) ? __ldcg(a.slot_col + par * G + sl) : -1;
                if (g == 0 && want_v2 && !stop) a.gaps[j] = (v2 < 0.0 || vbest == 0.0) ? 1.0 : (vbest - v2) / vbest;
            }
            if (!stop) {
                double sx = 0.0, mine = 0.0;
#pragma unroll
                for (int qq = 0; qq < SQ_RPL; ++qq) {
                    const int t = lane + 32 * qq;
                    if (t > j) sx += xv[qq] * xv[qq];
                    if (qq == (j >> 5)) mine = xv[qq];
                }
                sx = warp_sum(sx);
                const double alpha = __shfl_sync(0xffffffffu, mine, j & 31);
                double tau = 0.0, beta = alpha, scal = 0.0;
                if (sx != 0.0) {
                    const double nrm = sqrt(alpha * alpha + sx);
                    beta = (alpha >= 0.0) ? -nrm : nrm;
                    tau = (beta - alpha) / beta;
                    scal = 1.0 / (alpha - beta);
                }
#pragma unroll
                for (int qq = 0; qq < SQ_RPL; ++qq) {
                    const int t = lane + 32 * qq;
                    if (t < l) xs[t] = (t > j) ? xv[qq] * scal : (t == j ? 1.0 : xv[qq]);
                }
                if (lane == 0) { s_tau = tau; s_beta = beta; }
            }
        }
        __syncthreads();
        stamp(1);
        if (s_stop) break;
        const int wp = s_wpos, wcl = s_wcol;
        if (tid == 0 && wcl >= c_lo && wcl < c_hi) act[wcl - c_lo] = 0;  // retire the pivot
        __syncthreads();
        stamp(2);
        const double tau = s_tau;
        // ---- outputs + position map (CTA 0) ----------------------------------
        // step-j outputs written by CTA (j+1) mod G (spreads the extra work:
        // every CTA waits for the slowest at the barrier)
        if (g == (j + 1) % G) {
            for (int t = tid; t < lpad; t += SQ_THREADS)
                a.vhat[t + (int64_t)j * lpad] = (t < j) ? 0.0 : (t == j ? 1.0 : (t < l ? xs[t] : 0.0));
            for (int t = tid; t < a.bbpad; t += SQ_THREADS)
                a.rhat11[t + (int64_t)j * a.bbpad] = (t < j) ? xs[t] : (t == j ? s_beta : 0.0);
            if (tid == 0) { a.piv[j] = wp; a.tauhat[j] = tau; }
        }
        if (g == 0) {
            if (warp == SQ_WARPS - 1) {
                // transposition j <-> wp; q = phys column at position j (< bb)
                const int64_t q = low[j];
                __syncwarp();
                if (lane == 0) low[j] = wcl;
                if (wp != j) {
                    if (wp < a.bb) {
                        if (lane == 0) low[wp] = q;
                    } else {
                        // find wp in the short list (warp-parallel), else append
                        int found = -1;
                        for (int e0 = 0; e0 < hi_n; e0 += 32) {
                            const int e = e0 + lane;
                            const unsigned m = __ballot_sync(0xffffffffu, e < hi_n && hi_pos[e] == wp);
                            if (m) { found = e0 + __ffs(m) - 1; break; }
                        }
                        if (lane == 0) {
                            if (found >= 0) hi_phys[found] = q;
                            else { hi_pos[hi_n] = wp; hi_phys[hi_n] = q; ++hi_n; }
                        }
                    }
                }
                __syncwarp();
            }
        }
        // ---- 3. apply H_j to own active columns, downdate norms -----------
        bv = -1.0; bv2 = -1.0; bpos = INT_MAX; bcol = -1;
        auto apply_batch = [&](int cl0, int cend, auto colbase, int64_t ldcol) {
            double x[SQ_CB][SQ_RPL];
            bool live[SQ_CB];
            double rr[SQ_CB], rr0[SQ_CB];
            int lp[SQ_CB];
            // all loads of the batch first (column rows + per-column state)
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) {
                const int cl = cl0 + u;
                const int cs = (cl < cend) ? cl : cl0;
                live[u] = (cl < cend) && act[cs];
                rr[u] = r[cs];
                rr0[u] = r0[cs];
                lp[u] = lpos[cs];
                const double *col = colbase + (int64_t)cs * ldcol;
#pragma unroll
                for (int q = 0; q < SQ_RPL; ++q) {
                    const int t = lane + 32 * q;
                    x[u][q] = (live[u] && t < l) ? col[t] : 0.0;
                }
            }
            double w[SQ_CB];
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) {
                double sacc = 0.0;
#pragma unroll
                for (int q = 0; q < SQ_RPL; ++q) {
                    const int t = lane + 32 * q;
                    if (t >= j && t < l) sacc += xs[t] * x[u][q];
                }
                w[u] = sacc;
            }
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) w[u] = warp_sum(w[u]);
            double bj[SQ_CB], tail[SQ_CB];
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) {
                const double tw = tau * w[u];
                bj[u] = 0.0;
                tail[u] = 0.0;
#pragma unroll
                for (int q = 0; q < SQ_RPL; ++q) {
                    const int t = lane + 32 * q;
                    if (t >= j && t < l) x[u][q] -= tw * xs[t];
                    if (t == j) bj[u] = x[u][q];
                    if (t > j && t < l) tail[u] += x[u][q] * x[u][q];
                }
            }
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) bj[u] = __shfl_sync(0xffffffffu, bj[u], j & 31);
            // stores + norm downdates (recompute on cancellation, R-G6)
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) {
                if (!live[u]) continue;
                const int cl = cl0 + u;
                double *col = colbase + (int64_t)cl * ldcol;
#pragma unroll
                for (int q = 0; q < SQ_RPL; ++q) {
                    const int t = lane + 32 * q;
                    if (t >= j && t < l) col[t] = x[u][q];
                }
                double rn = rr[u] - bj[u] * bj[u];
                if (rn < 1e-6 * rr0[u]) rn = warp_sum(tail[u]);  // uniform per column
                const int pos = (lp[u] == j) ? wp : lp[u];         // position j moves to s*
                if (lane == 0) { r[cl] = rn; lpos[cl] = pos; }
                consider(rn, pos, (int)(c_lo + cl));
            }
        };
        // shared-memory columns (LDS/STS), then the L2-resident rest
        for (int cl0 = warp * SQ_CB; cl0 < nsm; cl0 += SQ_WARPS * SQ_CB) apply_batch(cl0, nsm, cols_s, (int64_t)lpad);
        for (int cl0 = nsm + warp * SQ_CB; cl0 < ncol; cl0 += SQ_WARPS * SQ_CB)
            apply_batch(cl0, ncol, a.B + c_lo * a.ldb, a.ldb);
        stamp(3);
        // ---- 4. candidates for step j+1, then the step barrier -------------
        publish(j + 1);
        stamp(4);
        grid_barrier(a.bar, G, epoch);
        stamp(5);
    }

    // ---- results ------------------------------------------------------------
    // transformed cached columns back to global (S6 reads R-hat12/22)
    for (int e = tid; e < nsm * l; e += SQ_THREADS) {
        const int t = e % l, cl = e / l;
        a.B[t + (c_lo + cl) * a.ldb] = cols_s[t + (size_t)cl * lpad];
    }
    if (g == 0) {
        if (tid == 0) s_np = 0;
        __syncthreads();
        // perm + column moves for every touched position whose content changed
        const int nlow = a.bb;
        for (int e = tid; e < nlow + hi_n; e += SQ_THREADS) {
            int64_t x, src;
            if (e < nlow) { x = e; src = low[e]; }
            else { x = hi_pos[e - nlow]; src = hi_phys[e - nlow]; }
            a.perm[x] = src;
            if (src != x) {
                const int slot = atomicAdd(&s_np, 1);
                a.swap_dst[slot] = x;
                a.swap_src[slot] = src;
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
