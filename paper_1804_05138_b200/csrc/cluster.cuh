// cluster.cuh -- S2 sample QRCP and S4 panel QR for problems whose sample /
// panel fits in the shared memory of one thread-block cluster (up to 16 SMs,
// ~3.2 MB): the per-step exchange goes through distributed shared memory
// (DSMEM) and the step barrier is the hardware cluster barrier, instead of L2
// round trips and a grid-wide barrier.  Same arithmetic, same order of
// operations and same outputs as the grid kernels in sample_qrcp.cuh /
// panel.cuh (the fixed-order partial sums run over the cluster's CTAs).
#pragma once
#include <climits>
#include <cooperative_groups.h>

#include "common.cuh"
#include "panel.cuh"
#include "sample_qrcp.cuh"

namespace rq {
namespace cg = cooperative_groups;

constexpr int CL_MAX = 16;

// ---------------------------------------------------------------------------
// Sample QRCP (Alg. 1 on the sample, P:100-123 / P:147), cluster version.
// Shared layout per CTA: [cpb columns x lpad][r][r0][lpos][act].
// ---------------------------------------------------------------------------
struct ClHdr {
    double v;
    int pos;
    int col;
};

__global__ void __launch_bounds__(SQ_THREADS) sample_qrcp_cluster_kernel(SqArgs a) {
    extern __shared__ __align__(16) double cq_dyn[];
    __shared__ double xs[SQ_MAXL];
    __shared__ double wv[SQ_WARPS], wv2[SQ_WARPS];
    __shared__ int wpos[SQ_WARPS], wcol[SQ_WARPS];
    __shared__ ClHdr hdr[2];
    __shared__ double hdr_v2[2];
    __shared__ double s_tau, s_beta;
    __shared__ int s_wpos, s_wcol, s_wrank, s_stop, s_np;
    __shared__ int64_t low[SQ_MAXB];
    __shared__ int hi_pos[SQ_MAXB];
    __shared__ int64_t hi_phys[SQ_MAXB];
    __shared__ int hi_n;

    cg::cluster_group cluster = cg::this_cluster();
    const int G = (int)cluster.num_blocks();
    const int g = (int)cluster.block_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = a.l, lpad = a.lpad;
    const int64_t nn = a.nn;
    const int64_t cpb = (nn + G - 1) / G;
    auto lo_of = [&](int rank) { return min(nn, (int64_t)rank * cpb); };
    const int64_t c_lo = lo_of(g), c_hi = min(nn, c_lo + cpb);
    const int ncol = (int)(c_hi - c_lo);
    const bool want_v2 = a.gaps != nullptr;

    if (*a.status != 0 || *a.done) {
        if (g == 0 && tid == 0) { *a.bb_eff = 0; *a.swap_np = 0; }
        return;
    }
    const double stop2 = *a.stop_tol2;
    double *cols = cq_dyn;
    double *r = cq_dyn + (size_t)cpb * lpad;
    double *r0 = r + cpb;
    int *lpos = reinterpret_cast<int *>(r0 + cpb);
    int *act = lpos + cpb;
    for (int e = tid; e < ncol * l; e += SQ_THREADS) {
        const int t = e % l, cl = e / l;
        cols[t + (size_t)cl * lpad] = a.B[t + (c_lo + cl) * a.ldb];
    }
    if (g == 0) {
        for (int x = tid; x < a.bb; x += SQ_THREADS) low[x] = x;
        if (tid == 0) hi_n = 0;
    }
    __syncthreads();

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
    for (int cl0 = warp * SQ_CB; cl0 < ncol; cl0 += SQ_WARPS * SQ_CB) {
        double x[SQ_CB][SQ_RPL];
#pragma unroll
        for (int u = 0; u < SQ_CB; ++u) {
            const int cl = min(cl0 + u, ncol - 1);
#pragma unroll
            for (int q = 0; q < SQ_RPL; ++q) {
                const int t = lane + 32 * q;
                x[u][q] = (t < l) ? cols[t + (size_t)cl * lpad] : 0.0;
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
    auto publish = [&](int parity) {
        if (lane == 0) { wv[warp] = bv; wv2[warp] = bv2; wpos[warp] = bpos; wcol[warp] = bcol; }
        __syncthreads();
        if (warp == 0) {
            double v = -1.0, v2 = -1.0;
            int p = INT_MAX, c = -1;
            if (lane < SQ_WARPS) { v = wv[lane]; v2 = wv2[lane]; p = wpos[lane]; c = wcol[lane]; }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
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
            if (lane == 0) { hdr[parity].v = v; hdr[parity].pos = p; hdr[parity].col = c; hdr_v2[parity] = v2; }
        }
    };
    publish(0);
    cluster.sync();

    int j = 0;
    for (; j < a.bb; ++j) {
        const int par = j & 1;
        // ---- 1. winner over the cluster's CTA headers (DSMEM) ---------------
        if (warp == 0) {
            double v = -1.0, v2 = -1.0;
            int p = INT_MAX, c = -1, rk = -1;
            if (lane < G) {
                const ClHdr *h = cluster.map_shared_rank(&hdr[par], lane);
                v = h->v; p = h->pos; c = h->col; rk = lane;
                if (want_v2) v2 = *cluster.map_shared_rank(&hdr_v2[par], lane);
                if (c < 0) { v = -1.0; p = INT_MAX; rk = -1; }
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {  // <= 16 CTAs
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const double ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                const int oc = __shfl_xor_sync(0xffffffffu, c, o);
                const int ork = __shfl_xor_sync(0xffffffffu, rk, o);
                if (ork >= 0 && (rk < 0 || sq_better(ov, op, v, p))) {
                    v2 = fmax(fmax(v2, ov2), v);
                    v = ov; p = op; c = oc; rk = ork;
                } else {
                    v2 = fmax(fmax(v2, ov2), ov);
                }
            }
            if (lane == 0) {
                s_wpos = p; s_wcol = c; s_wrank = rk;
                s_stop = (rk < 0) || !(v > stop2);
                if (g == 0 && want_v2 && !s_stop) a.gaps[j] = (v2 < 0.0 || v == 0.0) ? 1.0 : (v - v2) / v;
            }
        }
        __syncthreads();
        if (s_stop) break;
        const int wp = s_wpos, wcl = s_wcol, wrk = s_wrank;
        // ---- 2. winner column (DSMEM) -> Householder -------------------------
        if (warp == 0) {
            const double *src = cluster.map_shared_rank(cols, wrk) + (size_t)(wcl - lo_of(wrk)) * lpad;
            double xv[SQ_RPL];
#pragma unroll
            for (int q = 0; q < SQ_RPL; ++q) {
                const int t = lane + 32 * q;
                xv[q] = (t < l) ? src[t] : 0.0;
            }
            double s = 0.0, mine = 0.0;
#pragma unroll
            for (int q = 0; q < SQ_RPL; ++q) {
                const int t = lane + 32 * q;
                if (t > j) s += xv[q] * xv[q];
                if (q == (j >> 5)) mine = xv[q];
            }
            s = warp_sum(s);
            const double alpha = __shfl_sync(0xffffffffu, mine, j & 31);
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (s != 0.0) {
                const double nrm = sqrt(alpha * alpha + s);
                beta = (alpha >= 0.0) ? -nrm : nrm;
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
#pragma unroll
            for (int q = 0; q < SQ_RPL; ++q) {
                const int t = lane + 32 * q;
                if (t < l) xs[t] = (t > j) ? xv[q] * scal : (t == j ? 1.0 : xv[q]);
            }
            if (lane == 0) { s_tau = tau; s_beta = beta; }
        } else if (warp == 1 && lane == 0 && wrk == g) {
            act[wcl - c_lo] = 0;
        }
        __syncthreads();
        const double tau = s_tau;
        if (g == 0) {
            for (int t = tid; t < lpad; t += SQ_THREADS)
                a.vhat[t + (int64_t)j * lpad] = (t < j) ? 0.0 : (t == j ? 1.0 : (t < l ? xs[t] : 0.0));
            for (int t = tid; t < a.bbpad; t += SQ_THREADS)
                a.rhat11[t + (int64_t)j * a.bbpad] = (t < j) ? xs[t] : (t == j ? s_beta : 0.0);
            if (warp == SQ_WARPS - 1) {
                const int64_t q = low[j];
                __syncwarp();
                if (lane == 0) { a.piv[j] = wp; a.tauhat[j] = tau; low[j] = wcl; }
                if (wp != j) {
                    if (wp < a.bb) {
                        if (lane == 0) low[wp] = q;
                    } else {
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
        // ---- 3. apply H_j to own active columns --------------------------------
        bv = -1.0; bv2 = -1.0; bpos = INT_MAX; bcol = -1;
        for (int cl0 = warp * SQ_CB; cl0 < ncol; cl0 += SQ_WARPS * SQ_CB) {
            double x[SQ_CB][SQ_RPL];
            bool live[SQ_CB];
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) {
                const int cl = cl0 + u;
                live[u] = (cl < ncol) && act[cl];
                const int cs = live[u] ? cl : 0;
#pragma unroll
                for (int q = 0; q < SQ_RPL; ++q) {
                    const int t = lane + 32 * q;
                    x[u][q] = (live[u] && t < l) ? cols[t + (size_t)cs * lpad] : 0.0;
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
#pragma unroll
            for (int u = 0; u < SQ_CB; ++u) {
                if (!live[u]) continue;
                const int cl = cl0 + u;
                const double tw = tau * w[u];
                double bj = 0.0, tail = 0.0;
#pragma unroll
                for (int q = 0; q < SQ_RPL; ++q) {
                    const int t = lane + 32 * q;
                    if (t >= j && t < l) {
                        x[u][q] -= tw * xs[t];
                        cols[t + (size_t)cl * lpad] = x[u][q];
                    }
                    if (t == j) bj = x[u][q];
                    if (t > j && t < l) tail += x[u][q] * x[u][q];
                }
                bj = __shfl_sync(0xffffffffu, bj, j & 31);
                double rn = r[cl] - bj * bj;
                if (rn < 1e-6 * r0[cl]) rn = warp_sum(tail);
                int pos = lpos[cl];
                if (pos == j) pos = wp;
                __syncwarp();
                if (lane == 0) { r[cl] = rn; lpos[cl] = pos; }
                consider(rn, pos, (int)(c_lo + cl));
            }
        }
        publish(par ^ 1);
        cluster.sync();
    }
    // ---- results ------------------------------------------------------------
    for (int e = tid; e < ncol * l; e += SQ_THREADS) {
        const int t = e % l, cl = e / l;
        a.B[t + (c_lo + cl) * a.ldb] = cols[t + (size_t)cl * lpad];
    }
    // perm: identity for untouched positions (every CTA its own range), then
    // CTA 0 the touched ones -- ordered by the cluster barrier below
    for (int64_t x = c_lo + tid; x < c_hi; x += SQ_THREADS) a.perm[x] = x;
    cluster.sync();  // also: nobody still reads this CTA's shared memory
    if (g == 0) {
        if (tid == 0) s_np = 0;
        __syncthreads();
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

// ---------------------------------------------------------------------------
// Panel Householder QR (PDGEQRF P:760) + V^T V columns for T, cluster
// version: rows distributed over the cluster's CTAs, all in shared memory.
// Shared layout per CTA: [rpb x bb rows block][2][bbpad] partials [2][bbpad] row j.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PN_THREADS) panel_qr_cluster_kernel(PanelArgs a) {
    extern __shared__ __align__(16) double cp_dyn[];
    __shared__ double w[PN_MAXB];
    __shared__ double xs[PN_MAXROWS];
    __shared__ double s_scal, s_tau, s_beta;
    cg::cluster_group cluster = cg::this_cluster();
    const int G = (int)cluster.num_blocks(), g = (int)cluster.block_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bb = a.bb, bbpad = a.bbpad;
    const int bbe = *a.bb_eff;
    const int64_t mp = a.mp;
    const int64_t rpb = (mp + G - 1) / G;
    const int64_t r_lo = min(mp, (int64_t)g * rpb), r_hi = min(mp, r_lo + rpb);
    const int nrows = (int)(r_hi - r_lo);
    const int64_t lda = a.lda;
    double *P = cp_dyn;                           // nrows(max rpb) x bb, ld rpb
    const int64_t ldp = rpb;
    double *part = cp_dyn + (size_t)rpb * bb;     // [2][bbpad]
    double *rowj = part + 2 * bbpad;              // [2][bbpad]
    for (int c = warp; c < bb; c += PN_WARPS)
        for (int rr = lane; rr < nrows; rr += 32) P[rr + (int64_t)c * ldp] = a.A[r_lo + rr + c * lda];
    __syncthreads();
    const int owner_of_row = 0;
    (void)owner_of_row;
    for (int j = 0; j < bbe; ++j) {
        const int par = j & 1;
        const int rj = (int)(j - r_lo);
        const int rs = max(0, rj + 1);
        for (int c = warp; c < bb; c += PN_WARPS) {
            double s = 0.0;
            for (int rr = rs + lane; rr < nrows; rr += 32) s += P[rr + (int64_t)c * ldp] * P[rr + (int64_t)j * ldp];
            s = warp_sum(s);
            if (lane == 0) part[par * bbpad + c] = s;
        }
        if (rj >= 0 && rj < nrows)
            for (int c = tid; c < bb; c += PN_THREADS) rowj[par * bbpad + c] = P[rj + (int64_t)c * ldp];
        cluster.sync();
        // fixed-order reduction over the cluster's CTAs (lanes = CTA ranks)
        const int jown = (int)min((int64_t)(G - 1), (int64_t)j / rpb);
        const double *rj_remote = cluster.map_shared_rank(rowj, jown) + par * bbpad;
        for (int c = warp; c < bb; c += PN_WARPS) {
            double s = (lane < G) ? cluster.map_shared_rank(part, lane)[par * bbpad + c] : 0.0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) w[c] = s;
        }
        __syncthreads();
        if (tid == 0) {
            const double alpha = rj_remote[j];
            const double xn2 = w[j];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (xn2 != 0.0) {
                const double nrm = sqrt(alpha * alpha + xn2);
                beta = (alpha >= 0.0) ? -nrm : nrm;
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            s_tau = tau; s_beta = beta; s_scal = scal;
            if (g == 0) a.tau[j] = tau;
        }
        __syncthreads();
        const double tau = s_tau, scal = s_scal;
        if (g == 0)
            for (int c = tid; c < j; c += PN_THREADS) a.ybuf[c + (int64_t)j * bbpad] = rj_remote[c] + scal * w[c];
        for (int c = j + 1 + tid; c < bb; c += PN_THREADS) w[c] = tau * (rj_remote[c] + scal * w[c]);
        for (int rr = tid; rr < nrows; rr += PN_THREADS) xs[rr] = P[rr + (int64_t)j * ldp];
        __syncthreads();
        if (tau != 0.0) {
            for (int c = j + 1 + warp; c < bb; c += PN_WARPS) {
                const double wc = w[c];
                for (int rr = lane; rr < nrows; rr += 32) {
                    if (rr > rj) P[rr + (int64_t)c * ldp] -= wc * (scal * xs[rr]);
                    else if (rr == rj) P[rr + (int64_t)c * ldp] -= wc;
                }
            }
            for (int rr = tid; rr < nrows; rr += PN_THREADS) {
                if (rr > rj) P[rr + (int64_t)j * ldp] = scal * xs[rr];
                else if (rr == rj) P[rr + (int64_t)j * ldp] = s_beta;
            }
        }
        __syncthreads();
    }
    for (int c = warp; c < bb; c += PN_WARPS)
        for (int rr = lane; rr < nrows; rr += 32) a.A[r_lo + rr + c * lda] = P[rr + (int64_t)c * ldp];
    for (int rr = warp; rr < nrows; rr += PN_WARPS) {
        const int64_t gr = r_lo + rr;
        for (int c = lane; c < bbpad; c += 32) {
            double v = 0.0;
            if (c < bbe) v = (gr > c) ? P[rr + (int64_t)c * ldp] : (gr == c ? 1.0 : 0.0);
            a.vt[c + gr * bbpad] = v;
        }
    }
    for (int c = warp; c < bbpad; c += PN_WARPS)
        for (int rr = lane; rr < nrows; rr += 32) {
            const int64_t gr = r_lo + rr;
            double v = 0.0;
            if (c < bbe) v = (gr > c) ? P[rr + (int64_t)c * ldp] : (gr == c ? 1.0 : 0.0);
            a.vfull[gr + c * a.ldv] = v;
        }
    if (g == 0)
        for (int c = bbe + tid; c < bb; c += PN_THREADS) a.tau[c] = 0.0;
    cluster.sync();  // nobody still reads this CTA's shared memory
}

}  // namespace rq
