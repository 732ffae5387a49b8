// sample_qrcp_reg2.cuh -- S2 sample QRCP (Alg. 1, on the l x n'
// sample, Alg. 2 line P:147) for samples too wide for sample_qrcp_reg.cuh
// (C5: 65536 columns of 144 rows = 75.5 MB, more than the 148 SMs' registers
// and shared memory together).  Same exchange, arithmetic contract and
// outputs as sample_qrcp_reg_kernel (dlarfg R-G7, squared-norm downdates with
// the R-G6 recompute, lowest position on ties R-G5, stop rule R-G12; tagged
// 16-byte slot units, no fences), with two differences:
//   * TH = 512 threads per CTA, one column per thread (so the grid of
//     1 + n'/512 CTAs fits one CTA per SM for n' <= 75264);
//   * each column is split in three row ranges: rows [0, LT) in a global
//     scratch (transposed [row][thread] per CTA: coalesced), rows
//     [LT, LT + LR) in registers, rows [LT + LR, L) in shared memory
//     (the global rows are read with ld.global.cg: they stream past L1, which
//     keeps the few spilled registers of this 128-register kernel).
// Step j only touches rows >= j, so the global rows -- the TOP rows -- drop
// out of the traffic after step LT: summed over a 128-step panel the L2
// traffic is sum_{j < LT} (LT - j) rows instead of LT rows per step.
// (The spill kernel, sample_qrcp.cuh, keeps whole columns in L2 and streams
// all their rows twice per step: 31 us per pivot at C5.)
#pragma once
#include <climits>
#include "common.cuh"
#include "sample_qrcp.cuh"
#include "sample_qrcp_reg.cuh"

namespace rq {

constexpr int SQR2_THREADS = 512;

// SMT: the shared-memory rows directly below the global ones (rows
// [LT, LT + LS)) and the register rows at the bottom, so the shared-memory
// rows also drop out of the per-step traffic as the panel advances (as
// sample_qrcp_reg_kernel's SMT layout).
template <int LT, int LR, int LS, bool SMT = false>
__global__ void __launch_bounds__(SQR2_THREADS, 1) sample_qrcp_reg2_kernel(SqArgs a) {
    constexpr int TH = SQR2_THREADS;
    constexpr int NW = TH / 32;
    constexpr int L = LT + LR + LS;
    constexpr int R0 = SMT ? LT + LS : LT;  // first register row
    constexpr int S0 = SMT ? LT : LT + LR;  // first shared-memory row
    constexpr int SE = S0 + LS;             // end of the shared-memory rows
    extern __shared__ __align__(16) double sq_dyn[];  // max(LS x TH, bb x L) doubles
    __shared__ __align__(16) double xs[L + 1];
    __shared__ __align__(16) double xraw[L + (L & 1)];
    __shared__ double wv[NW];
    __shared__ int wpos[NW], wcol[NW];
    __shared__ double s_tau, s_beta, s_alpha;
    __shared__ int s_wpos, s_wcol, s_stop, s_np;
    __shared__ int64_t low[SQ_MAXB];
    __shared__ int hi_pos[SQ_MAXB];
    __shared__ int64_t hi_phys[SQ_MAXB];
    __shared__ int hi_n;
    __shared__ int s_piv[SQ_MAXB];
    __shared__ double s_tauh[SQ_MAXB];
    __shared__ unsigned long long s_trace[64 * 4];

    const int G = gridDim.x, g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = a.l;
    const int64_t nn = a.nn;
    // CTA 0 records the outputs (no columns); CTAs 1.. hold cpb <= TH columns each
    const int64_t cpb = (nn + G - 2) / (G - 1);
    const int64_t c_lo = (g == 0) ? 0 : min(nn, (int64_t)(g - 1) * cpb);
    const int64_t c_hi = (g == 0) ? 0 : min(nn, c_lo + cpb);
    const bool have = tid < (int)(c_hi - c_lo);
    const int64_t pc = c_lo + tid;
    double *xsm = sq_dyn;                                // CTAs >= 1: [LS][TH]
    double *comp = sq_dyn;                               // CTA 0: [bb][L]
    double *xt = a.spill + (int64_t)g * LT * TH + tid;   // this thread's top rows, stride TH
    if (*a.status != 0 || *a.done) {
        if (g == 0 && tid == 0) { *a.bb_eff = 0; *a.swap_np = 0; }
        return;
    }
    const double stop2 = *a.stop_tol2;

    double x[LR];
    {
        const double *src = a.B + pc * a.ldb;
#pragma unroll 4
        for (int t = 0; t < LT; ++t) xt[t * TH] = have ? src[t] : 0.0;
#pragma unroll
        for (int t = 0; t < LR; ++t) x[t] = have ? src[R0 + t] : 0.0;
#pragma unroll 4
        for (int t = 0; t < LS; ++t) xsm[t * TH + tid] = have ? src[S0 + t] : 0.0;
    }
    double r = 0.0;
    for (int t = 0; t < LT; ++t) r += xt[t * TH] * xt[t * TH];  // (just written: from L1)
    if (SMT)  // ascending rows
        for (int t = 0; t < LS; ++t) r += xsm[t * TH + tid] * xsm[t * TH + tid];
#pragma unroll
    for (int t = 0; t < LR; ++t) r += x[t] * x[t];
    if (!SMT)
        for (int t = 0; t < LS; ++t) r += xsm[t * TH + tid] * xsm[t * TH + tid];
    double r0 = r;
    int lpos = (int)pc;
    bool act = have;
    if (have) a.perm[pc] = pc;
    if (g == 0) {
        for (int q = tid; q < a.bb; q += TH) low[q] = q;
        if (tid == 0) hi_n = 0;
    }

    auto publish = [&](int step) {
        const int par = step & 1;
        double v = act ? r : -1.0;
        int p = act ? lpos : INT_MAX, c = act ? (int)pc : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            const int oc = __shfl_xor_sync(0xffffffffu, c, o);
            if (sq_better(ov, op, v, p)) { v = ov; p = op; c = oc; }
        }
        if (lane == 0) { wv[warp] = v; wpos[warp] = p; wcol[warp] = c; }
        __syncthreads();
        double bv = wv[0];
        int bp = wpos[0], bc = wcol[0];
        for (int w = 1; w < NW; ++w)
            if (sq_better(wv[w], wpos[w], bv, bp)) { bv = wv[w]; bp = wpos[w]; bc = wcol[w]; }
        // the owner stages its top and register rows in xraw (free until the next poll)
        if (act && (int)pc == bc) {
            for (int t = 0; t < LT; ++t) xraw[t] = __ldcg(&xt[t * TH]);
            if ((R0 & 1) == 0) {  // 16-byte stores (xraw is 16-byte aligned)
#pragma unroll
                for (int t = 0; t + 1 < LR; t += 2)
                    *reinterpret_cast<double2 *>(&xraw[R0 + t]) = make_double2(x[t], x[t + 1]);
                if (LR & 1) xraw[R0 + LR - 1] = x[LR - 1];
            } else {
#pragma unroll
                for (int t = 0; t < LR; ++t) xraw[R0 + t] = x[t];
            }
        }
        __syncthreads();
        if (warp == 0) {
            uint4 *dst = a.ll + (int64_t)(par * G + g) * SQR_UNITS;
            const unsigned tg = a.tag0 + (unsigned)step;
            if (bc >= 0) {
                const int oc = bc - (int)c_lo;
                for (int t = lane; t < l; t += 32) {
                    const double xv = (t >= S0 && t < SE) ? xsm[(t - S0) * TH + oc] : xraw[t];
                    ll_store(dst + 2 + t, (unsigned long long)__double_as_longlong(xv), tg);
                }
            }
            if (lane == 0) ll_store(dst, (unsigned long long)__double_as_longlong(bv), tg);
            if (lane == 1) ll_store(dst + 1, (unsigned long long)(unsigned)bp | ((unsigned long long)(unsigned)bc << 32), tg);
        }
    };

    if (a.trace)
        for (int e = tid; e < 64 * 4; e += TH) s_trace[e] = 0ull;
    publish(0);

    int j = 0;
    auto stamp = [&](int ph) {
        if (a.trace && tid == 0 && j < 64) s_trace[j * 4 + ph] = clock64();
    };
    for (; j < a.bb; ++j) {
        const int par = j & 1;
        stamp(0);
        // ---- 1. winner and its reflector (warp 0, redundantly per CTA) --------
        if (warp == 0) {
            const unsigned want = a.tag0 + (unsigned)j;
            const uint4 *slots = a.ll + (int64_t)(par * G) * SQR_UNITS;
            double xv[SQ_RPL];
            const SqWin win = sq_exchange(slots, G, want, l, stop2, a.spec, lane, xv);
            const bool stop = win.stop;
            const int p = win.p, wc = win.wc;
            if (lane == 0) { s_stop = stop; s_wpos = p; s_wcol = wc; }
            if (!stop) {
                double sx = 0.0;
#pragma unroll
                for (int qq = 0; qq < SQ_RPL; ++qq) {
                    const int t = lane + 32 * qq;
                    if (t > j && t < L) sx += xv[qq] * xv[qq];
                    if (t == j) s_alpha = xv[qq];
                }
                sx = warp_sum(sx);
                __syncwarp();
                const double alpha = s_alpha;
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
                    if (t < L) {
                        const double vt = (t > j) ? xv[qq] * scal : (t == j ? 1.0 : 0.0);
                        xs[t] = vt;
                        xraw[t] = xv[qq];
                    }
                }
                if (lane == 0) { s_tau = tau; s_beta = beta; }
            }
        }
        __syncthreads();
        stamp(1);
        if (s_stop) break;
        const int wp = s_wpos, wcl = s_wcol;
        const double tau = s_tau;
        if (g == 0) {
            for (int t = tid; t < L; t += TH) comp[j * L + t] = (t < j) ? xraw[t] : (t == j ? s_beta : xs[t]);
            if (tid == 0) { s_piv[j] = wp; s_tauh[j] = tau; }
        }
        if (g == 0 && warp == NW - 1) {
            const int64_t q = low[j];
            __syncwarp();
            if (lane == 0) low[j] = wcl;
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
        // ---- 2. apply H_j to this thread's column, downdate the norm ---------
        if (act && (int)pc == wcl) act = false;
        if (act) {
            // w = v^T x over rows >= j (xs is zero above row j): top rows (global,
            // only while j < LT; all loads of a batch in flight), register rows
            // (SQR_CH chunks entirely above row j skipped), shared-memory rows
            double d[4] = {0.0, 0.0, 0.0, 0.0};
            if (j < LT) {  // batches of 8 loads in flight (one L2 round trip each)
                int t = j;
                for (; t + 7 < LT; t += 8) {
                    double y[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) y[u] = __ldcg(&xt[(t + u) * TH]);
#pragma unroll
                    for (int u = 0; u < 8; ++u) d[u & 3] += xs[t + u] * y[u];
                }
                for (; t < LT; ++t) d[0] += xs[t] * __ldcg(&xt[t * TH]);
            }
            auto smem_dot = [&]() {
                int t = (j > S0 ? j : S0);
                const double *xc = xsm + tid - S0 * TH;
                if ((t & 1) && t < SE) { d[1] += xs[t] * xc[t * TH]; ++t; }  // (S0 is even)
                for (; t + 3 < SE; t += 4) {
                    const double2 v01 = *reinterpret_cast<const double2 *>(&xs[t]);
                    const double2 v23 = *reinterpret_cast<const double2 *>(&xs[t + 2]);
                    d[0] += v01.x * xc[t * TH];
                    d[1] += v01.y * xc[(t + 1) * TH];
                    d[2] += v23.x * xc[(t + 2) * TH];
                    d[3] += v23.y * xc[(t + 3) * TH];
                }
                for (; t < SE; ++t) d[0] += xs[t] * xc[t * TH];
            };
            if (SMT && LS > 0) smem_dot();
#pragma unroll
            for (int c0 = 0; c0 < LR; c0 += SQR_CH) {
                if (j < R0 + c0 + SQR_CH) {
#pragma unroll
                    for (int t = c0; t < c0 + SQR_CH && t + 1 < LR; t += 2) {
                        const double2 v2 = *reinterpret_cast<const double2 *>(&xs[R0 + t]);
                        d[(t >> 1) & 3] += v2.x * x[t] + v2.y * x[t + 1];
                    }
                    if ((LR & 1) && c0 + SQR_CH >= LR) d[0] += xs[R0 + LR - 1] * x[LR - 1];
                }
            }
            if (!SMT && LS > 0) smem_dot();
            const double tw = tau * ((d[0] + d[1]) + (d[2] + d[3]));
            // x -= tw v; bj = x(j) from the range that holds row j
            double bj = 0.0;
            if (j < LT) {
                int t = j;
                for (; t + 7 < LT; t += 8) {
                    double y[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) y[u] = __ldcg(&xt[(t + u) * TH]);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double nv = y[u] - tw * xs[t + u];
                        xt[(t + u) * TH] = nv;
                        if (t + u == j) bj = nv;
                    }
                }
                for (; t < LT; ++t) {
                    const double nv = __ldcg(&xt[t * TH]) - tw * xs[t];
                    xt[t * TH] = nv;
                    if (t == j) bj = nv;
                }
            }
#pragma unroll
            for (int c0 = 0; c0 < LR; c0 += SQR_CH) {
                if (j < R0 + c0 + SQR_CH) {
#pragma unroll
                    for (int t = c0; t < c0 + SQR_CH && t + 1 < LR; t += 2) {
                        const double2 v2 = *reinterpret_cast<const double2 *>(&xs[R0 + t]);
                        x[t] -= tw * v2.x;
                        x[t + 1] -= tw * v2.y;
                    }
                    if ((LR & 1) && c0 + SQR_CH >= LR) x[LR - 1] -= tw * xs[R0 + LR - 1];
                    if (j >= R0 + c0) {
#pragma unroll
                        for (int t = c0; t < c0 + SQR_CH && t < LR; ++t) bj = (R0 + t == j) ? x[t] : bj;
                    }
                }
            }
            if (LS > 0) {
                int t = (j > S0 ? j : S0);
                if ((t & 1) && t < SE) {
                    double *q = &xsm[(t - S0) * TH + tid];
                    const double nv = *q - tw * xs[t];
                    *q = nv;
                    ++t;
                }
#pragma unroll 2
                for (; t + 1 < SE; t += 2) {
                    const double2 v01 = *reinterpret_cast<const double2 *>(&xs[t]);
                    double *q = &xsm[(t - S0) * TH + tid];
                    const double n0 = q[0] - tw * v01.x;
                    const double n1 = q[TH] - tw * v01.y;
                    q[0] = n0;
                    q[TH] = n1;
                }
                for (; t < SE; ++t) {
                    double *q = &xsm[(t - S0) * TH + tid];
                    const double nv = *q - tw * xs[t];
                    *q = nv;
                }
                // the updated x(j), read back once instead of selected in the loop
                if (j >= S0 && j < SE) bj = xsm[(j - S0) * TH + tid];
            }
            double rn = r - bj * bj;
            if (rn < 1e-6 * r0) {  // recompute from the updated rows (R-G6)
                double s0 = 0.0;
                for (int t = j + 1; t < LT; ++t) s0 += __ldcg(&xt[t * TH]) * __ldcg(&xt[t * TH]);
                auto smem_ss = [&]() {
                    for (int t = (j + 1 > S0 ? j + 1 : S0); t < SE; ++t)
                        s0 += xsm[(t - S0) * TH + tid] * xsm[(t - S0) * TH + tid];
                };
                if (SMT) smem_ss();
#pragma unroll
                for (int t = 0; t < LR; ++t)
                    if (R0 + t > j) s0 += x[t] * x[t];
                if (!SMT) smem_ss();
                rn = s0;
            }
            r = rn;
            if (lpos == j) lpos = wp;
        }
        stamp(2);
        if (j + 1 < a.bb) publish(j + 1);
        stamp(3);
    }
    __syncthreads();

    // ---- results --------------------------------------------------------------
    if (a.trace)
        for (int e = tid; e < 64 * 4; e += TH)
            a.trace[(size_t)g * 256 + e] = (e / 4 < min(j + 1, 64)) ? s_trace[e] : 0ull;
    if (have) {
        double *dst = a.B + pc * a.ldb;
        for (int t = 0; t < LT; ++t) dst[t] = __ldcg(&xt[t * TH]);
#pragma unroll
        for (int t = 0; t < LR; ++t) dst[R0 + t] = x[t];
        for (int t = 0; t < LS; ++t) dst[S0 + t] = xsm[t * TH + tid];
    }
    if (g == 0) {
        for (int e = tid; e < j * a.lpad; e += TH) {
            const int t = e % a.lpad, c = e / a.lpad;
            a.vhat[e] = (t < c || t >= L) ? 0.0 : (t == c ? 1.0 : comp[c * L + t]);
        }
        for (int e = tid; e < j * a.bbpad; e += TH) {
            const int t = e % a.bbpad, c = e / a.bbpad;
            a.rhat11[e] = (t <= c) ? comp[c * L + t] : 0.0;
        }
        for (int c = tid; c < j; c += TH) { a.piv[c] = s_piv[c]; a.tauhat[c] = s_tauh[c]; }
        if (tid == 0) s_np = 0;
        __syncthreads();
        const int nlow = a.bb;
        for (int e = tid; e < nlow + hi_n; e += TH) {
            int64_t xq, src;
            if (e < nlow) { xq = e; src = low[e]; }
            else { xq = hi_pos[e - nlow]; src = hi_phys[e - nlow]; }
            a.perm[xq] = src;
            if (src != xq) {
                const int slot = atomicAdd(&s_np, 1);
                a.swap_dst[slot] = xq;
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
