// sample_qrcp_reg.cuh -- S2 sample QRCP (Alg. 1, on the l x n'
// sample, Alg. 2 line P:147) over a cooperative GRID with ONE COLUMN PER
// THREAD: rows 0..LR-1 of the column in registers, rows LR..LR+LS-1 in
// shared memory ([row][thread], conflict-free); n' <= grid x 256.  Same
// arithmetic and outputs as sample_qrcp.cuh / sample_qrcp_cl.cuh (dlarfg
// reading R-G7, squared-norm downdates with the R-G6 recompute, lowest
// position on ties R-G5, stop rule R-G12); the per-step exchange is the grid
// kernel's, without fences: every CTA publishes its best candidate (header
// and column) in a global slot in which each 32-bit half of every word
// travels with the step's tag in one 64-bit store (two per 16-byte unit, the
// "low-latency" flag protocol), and warp 0 of every CTA polls the G headers
// with relaxed loads until the tags match, picks the winner, polls its
// column the same way and forms the reflector redundantly.  A 64-bit aligned
// store is single-copy atomic, so a matching tag proves its half is current;
// no release/acquire fence (each costs an L2 round trip per step) is needed.  CTA 0 holds no columns: it stages the
// reflectors and R-hat rows in shared memory and writes the outputs at the
// end (so its shared memory is free for them).  Used for samples larger than one
// cluster can hold in registers (C3: 16384 columns; C4: 32768 columns of
// 144 rows).
#pragma once
#include <climits>
#include "common.cuh"
#include "sample_qrcp.cuh"

namespace rq {

#ifndef SQR_TRACE_DETAIL
#define SQR_TRACE_DETAIL 0
#endif
constexpr int SQR_THREADS = 256;
constexpr int SQR_CH = 16;  // rows per skipped chunk of the register rows (as SQC_CH)
constexpr int SQR_UNITS = SQ_MAXL + 2;  // 16-byte units per slot: header (2) + column
constexpr int SQR_MAXG = 160;  // register-grid CTAs (headers polled by one warp: 5 per lane)

// SMT (shared-memory top): rows [0, LS) in shared memory, rows [LS, L) in
// registers.  Step j touches rows >= j only, so with the shared-memory rows on
// top they drop out of the per-step shared-memory traffic as the panel
// advances (l = 144, bb = 128: 2628 instead of 7676 row-steps per panel);
// the register rows cost no shared-memory bandwidth wherever they sit.
// The per-step exchange of the register grids, run by warp 0 of every CTA:
// poll the G candidate headers of step `want` (tagged units, no fences), pick
// the winner (largest norm, lowest position on ties, R-G5), and fetch its
// column.  With spec != 0 the column of the best candidate among the headers
// that have arrived is fetched while the others are still being polled (the
// same winner: sq_better is a total order).  Measured slower (C4 S2 51.0 vs
// 46.8 ms): the warp reduction in every poll round delays the detection of
// the last header by more than the column's L2 round trip it saves.  Five
// headers per lane (G <= 160) instead of eight: C4 S2 50.6 -> 46.8 ms.
struct SqWin {
    double v;
    int p, sl, wc;
    bool stop;
};
RQ_DEV SqWin sq_exchange(const uint4 *slots, int G, unsigned want, int l, double stop2, int spec, int lane,
                         double (&xv)[SQ_RPL]) {
    constexpr int HPL = SQR_MAXG / 32;
    bool ready[HPL];
    unsigned long long h0[HPL], h1[HPL];
#pragma unroll
    for (int u = 0; u < HPL; ++u) { ready[u] = (lane + 32 * u >= G); h0[u] = 0; h1[u] = 0; }
    bool ok[SQ_RPL];
#pragma unroll
    for (int qq = 0; qq < SQ_RPL; ++qq) { ok[qq] = true; xv[qq] = 0.0; }
    int csl = -1;  // slot whose column is being fetched
    SqWin w;
    while (true) {
        bool all = true;
#pragma unroll
        for (int u = 0; u < HPL; ++u) {
            if (!ready[u]) {
                const uint4 *hq = slots + (int64_t)(lane + 32 * u) * SQR_UNITS;
                const bool r0_ = ll_load(hq, want, h0[u]);
                const bool r1_ = ll_load(hq + 1, want, h1[u]);
                ready[u] = r0_ && r1_;
            }
            all = all && ready[u];
        }
        const bool allh = __all_sync(0xffffffffu, all);
        if (!allh && !spec) continue;
        // best among the headers that have arrived
        double v = -1.0;
        int p = INT_MAX, sl = -1, wc = -1;
#pragma unroll
        for (int u = 0; u < HPL; ++u) {
            const int q = lane + 32 * u;
            const double hv = __longlong_as_double((long long)h0[u]);
            const int hp = (int)(unsigned)(h1[u] & 0xffffffffull);
            if (ready[u] && q < G && hp != INT_MAX && sq_better(hv, hp, v, p)) {
                v = hv; p = hp; sl = q; wc = (int)(unsigned)(h1[u] >> 32);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            const int osl = __shfl_xor_sync(0xffffffffu, sl, o);
            const int owc = __shfl_xor_sync(0xffffffffu, wc, o);
            if (osl >= 0 && (sl < 0 || sq_better(ov, op, v, p))) { v = ov; p = op; sl = osl; wc = owc; }
        }
        const bool stop = allh && ((sl < 0) || !(v > stop2));
        if (allh && stop) {
            w = SqWin{v, p, sl, wc, true};
            break;
        }
        if (sl >= 0 && sl != csl) {  // (re)start the column fetch
            csl = sl;
#pragma unroll
            for (int qq = 0; qq < SQ_RPL; ++qq) ok[qq] = lane + 32 * qq >= l;
        }
        bool cdone = true;
        if (csl >= 0) {
            const uint4 *src = slots + (int64_t)csl * SQR_UNITS + 2;
#pragma unroll
            for (int qq = 0; qq < SQ_RPL; ++qq) {
                if (!ok[qq]) {
                    unsigned long long x;
                    ok[qq] = ll_load(src + lane + 32 * qq, want, x);
                    xv[qq] = __longlong_as_double((long long)x);
                }
                cdone = cdone && ok[qq];
            }
        }
        if (allh && __all_sync(0xffffffffu, cdone)) {  // csl == sl here
            w = SqWin{v, p, sl, wc, false};
            break;
        }
    }
    return w;
}

template <int LR, int LS, bool SMT = false>
__global__ void __launch_bounds__(SQR_THREADS, 1) sample_qrcp_reg_kernel(SqArgs a) {
    constexpr int L = LR + LS;
    constexpr int R0 = SMT ? LS : 0;   // first register row
    constexpr int S0 = SMT ? 0 : LR;   // first shared-memory row
    constexpr int SE = S0 + LS;        // end of the shared-memory rows
    extern __shared__ __align__(16) double sq_dyn[];  // max(LS x 256, bb x L) doubles
    __shared__ __align__(16) double xs[L + 1];
    __shared__ __align__(16) double xraw[L + (L & 1)];
    __shared__ double wv[SQ_WARPS];
    __shared__ int wpos[SQ_WARPS], wcol[SQ_WARPS];
    __shared__ double s_tau, s_beta, s_alpha;
    __shared__ int s_wpos, s_wcol, s_stop, s_np;
    __shared__ int64_t low[SQ_MAXB];
    __shared__ int hi_pos[SQ_MAXB];
    __shared__ int64_t hi_phys[SQ_MAXB];
    __shared__ int hi_n;
    __shared__ int s_piv[SQ_MAXB];
    __shared__ double s_tauh[SQ_MAXB];
    __shared__ unsigned long long s_trace[64 * 4];  // RQRCP_TRACE phase stamps

    const int G = gridDim.x, g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = a.l;
    const int64_t nn = a.nn;
    // CTA 0 records the outputs (no columns); CTAs 1.. hold cpb <= 256 columns each
    const int64_t cpb = (nn + G - 2) / (G - 1);
    const int64_t c_lo = (g == 0) ? 0 : min(nn, (int64_t)(g - 1) * cpb);
    const int64_t c_hi = (g == 0) ? 0 : min(nn, c_lo + cpb);
    const bool have = tid < (int)(c_hi - c_lo);
    const int64_t pc = c_lo + tid;
    double *xsm = sq_dyn;   // CTAs >= 1: [LS][256]
    double *comp = sq_dyn;  // CTA 0: [bb][L]
    if (*a.status != 0 || *a.done) {
        if (g == 0 && tid == 0) { *a.bb_eff = 0; *a.swap_np = 0; }
        return;
    }
    const double stop2 = *a.stop_tol2;

    double x[LR];
    // the column's entries are contiguous: 16-byte loads when aligned
    const bool vec = ((a.ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.B) & 15) == 0) && !(LR & 1) && !(LS & 1);
    if (have && vec) {
        const double2 *src = reinterpret_cast<const double2 *>(a.B + pc * a.ldb);
#pragma unroll
        for (int t = 0; t < LR; t += 2) {
            const double2 v = src[(R0 + t) / 2];
            x[t] = v.x;
            x[t + 1] = v.y;
        }
#pragma unroll 4
        for (int t = 0; t < LS; t += 2) {
            const double2 v = src[(S0 + t) / 2];
            xsm[t * SQR_THREADS + tid] = v.x;
            xsm[(t + 1) * SQR_THREADS + tid] = v.y;
        }
    } else {
#pragma unroll
        for (int t = 0; t < LR; ++t) x[t] = have ? a.B[(R0 + t) + pc * a.ldb] : 0.0;
#pragma unroll 4
        for (int t = 0; t < LS; ++t) xsm[t * SQR_THREADS + tid] = have ? a.B[(S0 + t) + pc * a.ldb] : 0.0;
    }
    double r = 0.0;
    if (SMT)  // ascending rows
        for (int t = 0; t < LS; ++t) r += xsm[t * SQR_THREADS + tid] * xsm[t * SQR_THREADS + tid];
#pragma unroll
    for (int t = 0; t < LR; ++t) r += x[t] * x[t];
    if (!SMT)
        for (int t = 0; t < LS; ++t) r += xsm[t * SQR_THREADS + tid] * xsm[t * SQR_THREADS + tid];
    double r0 = r;
    int lpos = (int)pc;
    bool act = have;
    if (have) a.perm[pc] = pc;
    if (g == 0) {
        for (int q = tid; q < a.bb; q += SQR_THREADS) low[q] = q;
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
        for (int w = 1; w < SQ_WARPS; ++w)
            if (sq_better(wv[w], wpos[w], bv, bp)) { bv = wv[w]; bp = wpos[w]; bc = wcol[w]; }
        // the owner stages its register rows in xraw (free until the next poll)
        if (act && (int)pc == bc) {
#pragma unroll
            for (int t = 0; t + 1 < LR; t += 2)  // 16-byte stores (xraw is 16-byte aligned; R0 even)
                *reinterpret_cast<double2 *>(&xraw[R0 + t]) = make_double2(x[t], x[t + 1]);
            if (LR & 1) xraw[R0 + LR - 1] = x[LR - 1];
        }
        __syncthreads();
        if (warp == 0) {
            uint4 *dst = a.ll + (int64_t)(par * G + g) * SQR_UNITS;
            const unsigned tg = a.tag0 + (unsigned)step;
            if (bc >= 0) {
                const int oc = bc - (int)c_lo;
                for (int t = lane; t < l; t += 32) {
                    const double xv = (t >= S0 && t < SE) ? xsm[(t - S0) * SQR_THREADS + oc] : xraw[t];
                    ll_store(dst + 2 + t, (unsigned long long)__double_as_longlong(xv), tg);
                }
            }
            if (lane == 0) ll_store(dst, (unsigned long long)__double_as_longlong(bv), tg);
            if (lane == 1) ll_store(dst + 1, (unsigned long long)(unsigned)bp | ((unsigned long long)(unsigned)bc << 32), tg);
        }
    };

    if (a.trace)
        for (int e = tid; e < 64 * 4; e += SQR_THREADS) s_trace[e] = 0ull;
    publish(0);

    int j = 0;
    // phase stamps (RQRCP_TRACE): kept in shared memory, written at the end so
    // the trace adds no global traffic to the steps it measures
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
#if SQR_TRACE_DETAIL
            stamp(2);
#endif
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
#if SQR_TRACE_DETAIL
        stamp(3);
#else
        stamp(1);
#endif
        if (s_stop) break;
        const int wp = s_wpos, wcl = s_wcol;
        const double tau = s_tau;
        if (g == 0) {
            for (int t = tid; t < L; t += SQR_THREADS) comp[j * L + t] = (t < j) ? xraw[t] : (t == j ? s_beta : xs[t]);
            if (tid == 0) { s_piv[j] = wp; s_tauh[j] = tau; }
        }
        if (g == 0 && warp == SQ_WARPS - 1) {
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
            // w = v^T x over rows >= j (xs is zero above row j); SQR_CH-row chunks
            // entirely above row j are skipped (uniform branches); four
            // independent accumulators
            double d[4] = {0.0, 0.0, 0.0, 0.0};
            // the shared-memory rows [max(j, S0), SE)
            auto smem_dot = [&]() {
                int t = (j > S0 ? j : S0);
                const double *xc = xsm + tid - S0 * SQR_THREADS;
                if ((t & 1) && t < SE) { d[1] += xs[t] * xc[t * SQR_THREADS]; ++t; }  // (S0 is even)
                // pairs of the reflector from one 16-byte broadcast load
                for (; t + 3 < SE; t += 4) {
                    const double2 v01 = *reinterpret_cast<const double2 *>(&xs[t]);
                    const double2 v23 = *reinterpret_cast<const double2 *>(&xs[t + 2]);
                    d[0] += v01.x * xc[t * SQR_THREADS];
                    d[1] += v01.y * xc[(t + 1) * SQR_THREADS];
                    d[2] += v23.x * xc[(t + 2) * SQR_THREADS];
                    d[3] += v23.y * xc[(t + 3) * SQR_THREADS];
                }
                for (; t < SE; ++t) d[0] += xs[t] * xc[t * SQR_THREADS];
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
            // x -= tw v; bj = x(j) picked in the chunk that holds row j
            double bj = 0.0;
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
                    double *q = &xsm[(t - S0) * SQR_THREADS + tid];
                    const double nv = *q - tw * xs[t];
                    *q = nv;
                    ++t;
                }
#pragma unroll 2
                for (; t + 1 < SE; t += 2) {
                    const double2 v01 = *reinterpret_cast<const double2 *>(&xs[t]);
                    double *q = &xsm[(t - S0) * SQR_THREADS + tid];
                    const double n0 = q[0] - tw * v01.x;
                    const double n1 = q[SQR_THREADS] - tw * v01.y;
                    q[0] = n0;
                    q[SQR_THREADS] = n1;
                }
                for (; t < SE; ++t) {
                    double *q = &xsm[(t - S0) * SQR_THREADS + tid];
                    const double nv = *q - tw * xs[t];
                    *q = nv;
                }
                // the updated x(j), read back once instead of selected in the loop
                if (j >= S0 && j < SE) bj = xsm[(j - S0) * SQR_THREADS + tid];
            }
            double rn = r - bj * bj;
            if (rn < 1e-6 * r0) {  // recompute from the updated rows (R-G6)
                double s0 = 0.0;
                auto smem_ss = [&]() {
                    for (int t = (j + 1 > S0 ? j + 1 : S0); t < SE; ++t)
                        s0 += xsm[(t - S0) * SQR_THREADS + tid] * xsm[(t - S0) * SQR_THREADS + tid];
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
#if !SQR_TRACE_DETAIL
        stamp(2);
#endif
        if (j + 1 < a.bb) publish(j + 1);
#if !SQR_TRACE_DETAIL
        stamp(3);
#endif
    }
    __syncthreads();

    // ---- results --------------------------------------------------------------
    if (a.trace)
        for (int e = tid; e < 64 * 4; e += SQR_THREADS)
            a.trace[(size_t)g * 256 + e] = (e / 4 < min(j + 1, 64)) ? s_trace[e] : 0ull;
    if (have && vec) {
        double2 *dst = reinterpret_cast<double2 *>(a.B + pc * a.ldb);
#pragma unroll
        for (int t = 0; t < LR; t += 2) dst[(R0 + t) / 2] = make_double2(x[t], x[t + 1]);
        for (int t = 0; t < LS; t += 2)
            dst[(S0 + t) / 2] = make_double2(xsm[t * SQR_THREADS + tid], xsm[(t + 1) * SQR_THREADS + tid]);
    } else if (have) {
#pragma unroll
        for (int t = 0; t < LR; ++t) a.B[(R0 + t) + pc * a.ldb] = x[t];
        for (int t = 0; t < LS; ++t) a.B[(S0 + t) + pc * a.ldb] = xsm[t * SQR_THREADS + tid];
    }
    if (g == 0) {
        for (int e = tid; e < j * a.lpad; e += SQR_THREADS) {
            const int t = e % a.lpad, c = e / a.lpad;
            a.vhat[e] = (t < c || t >= L) ? 0.0 : (t == c ? 1.0 : comp[c * L + t]);
        }
        for (int e = tid; e < j * a.bbpad; e += SQR_THREADS) {
            const int t = e % a.bbpad, c = e / a.bbpad;
            a.rhat11[e] = (t <= c) ? comp[c * L + t] : 0.0;
        }
        for (int c = tid; c < j; c += SQR_THREADS) { a.piv[c] = s_piv[c]; a.tauhat[c] = s_tauh[c]; }
        if (tid == 0) s_np = 0;
        __syncthreads();
        const int nlow = a.bb;
        for (int e = tid; e < nlow + hi_n; e += SQR_THREADS) {
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
