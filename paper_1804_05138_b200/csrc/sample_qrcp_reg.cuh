// sample_qrcp_reg.cuh -- S2 sample QRCP (Alg. 1, on the l x n'
// sample, Alg. 2 line P:147) over a cooperative GRID with ONE COLUMN PER
// THREAD: rows 0..LR-1 of the column in registers, rows LR..LR+LS-1 in
// shared memory ([row][thread], conflict-free); n' <= grid x 256.  Same
// arithmetic and outputs as sample_qrcp.cuh / sample_qrcp_cl.cuh (dlarfg
// reading R-G7, squared-norm downdates with the R-G6 recompute, lowest
// position on ties R-G5, stop rule R-G12); the per-step exchange is the grid
// kernel's: every CTA publishes its best candidate (column in a global slot,
// then a 16-byte header with a release store) and warp 0 of every CTA polls
// the G headers with acquire loads, picks the winner, loads its column and
// forms the reflector redundantly.  CTA 0 holds no columns: it stages the
// reflectors and R-hat rows in shared memory and writes the outputs at the
// end (so its shared memory is free for them).  Used for samples larger than one
// cluster can hold in registers (C3: 16384 columns; C4: 32768 columns of
// 144 rows).
#pragma once
#include <climits>
#include "common.cuh"
#include "sample_qrcp.cuh"

namespace rq {

constexpr int SQR_THREADS = 256;

template <int LR, int LS>
__global__ void __launch_bounds__(SQR_THREADS, 1) sample_qrcp_reg_kernel(SqArgs a) {
    constexpr int L = LR + LS;
    extern __shared__ __align__(16) double sq_dyn[];  // max(LS x 256, bb x L) doubles
    __shared__ __align__(16) double xs[L + 1];
    __shared__ __align__(16) double xe[2 * L];  // (v_t, [t == j]) pairs
    __shared__ double xraw[L];
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
#pragma unroll
    for (int t = 0; t < LR; ++t) x[t] = have ? a.B[t + pc * a.ldb] : 0.0;
#pragma unroll 4
    for (int t = 0; t < LS; ++t) xsm[t * SQR_THREADS + tid] = have ? a.B[(LR + t) + pc * a.ldb] : 0.0;
    double r = 0.0;
#pragma unroll
    for (int t = 0; t < LR; ++t) r += x[t] * x[t];
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
            for (int t = 0; t < LR; ++t) xraw[t] = x[t];
        }
        __syncthreads();
        if (warp == 0) {
            if (bc >= 0) {
                double *dst = a.slot_data + (int64_t)(par * G + g) * a.lpad;
                const int oc = bc - (int)c_lo;
                for (int t = lane; t < l; t += 32)
                    __stcg(dst + t, (t < LR) ? xraw[t] : xsm[(t - LR) * SQR_THREADS + oc]);
            }
            if (lane == 0) a.slot_col[par * G + g] = bc;
            __syncwarp();
            if (lane == 0) st_release_hdr(a.slot_hdr + (int64_t)(par * G + g) * a.hstride, bv, bp, a.tag0 + (unsigned)step);
        }
    };

    publish(0);

    int j = 0;
    for (; j < a.bb; ++j) {
        const int par = j & 1;
        // ---- 1. winner and its reflector (warp 0, redundantly per CTA) --------
        if (warp == 0) {
            const unsigned want = a.tag0 + (unsigned)j;
            constexpr int HPL = SQ_MAXG / 32;
            double v = -1.0;
            int p = INT_MAX, sl = -1;
            bool ready[HPL];
            double hv[HPL];
            int hp[HPL];
#pragma unroll
            for (int u = 0; u < HPL; ++u) { ready[u] = (lane + 32 * u >= G); hv[u] = -1.0; hp[u] = INT_MAX; }
            while (true) {
                bool all = true;
#pragma unroll
                for (int u = 0; u < HPL; ++u) {
                    if (!ready[u]) {
                        unsigned tg;
                        ld_acquire_hdr(a.slot_hdr + (int64_t)(par * G + lane + 32 * u) * a.hstride, hv[u], hp[u], tg);
                        ready[u] = (tg == want);
                    }
                    all = all && ready[u];
                }
                if (__all_sync(0xffffffffu, all)) break;
            }
#pragma unroll
            for (int u = 0; u < HPL; ++u) {
                const int q = lane + 32 * u;
                if (q < G && hp[u] != INT_MAX && sq_better(hv[u], hp[u], v, p)) { v = hv[u]; p = hp[u]; sl = q; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                const int osl = __shfl_xor_sync(0xffffffffu, sl, o);
                if (osl >= 0 && (sl < 0 || sq_better(ov, op, v, p))) { v = ov; p = op; sl = osl; }
            }
            const bool stop = (sl < 0) || !(v > stop2);
            double xv[SQ_RPL];
            const double *src = a.slot_data + (int64_t)(par * G + (sl >= 0 ? sl : 0)) * a.lpad;
#pragma unroll
            for (int qq = 0; qq < SQ_RPL; ++qq) {
                const int t = lane + 32 * qq;
                xv[qq] = (!stop && t < l) ? __ldcg(src + t) : 0.0;
            }
            const int wc = (sl >= 0) ? __ldcg(a.slot_col + par * G + sl) : -1;
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
                        xe[2 * t] = vt;
                        xe[2 * t + 1] = (t == j) ? 1.0 : 0.0;
                        xraw[t] = xv[qq];
                    }
                }
                if (lane == 0) { s_tau = tau; s_beta = beta; }
            }
        }
        __syncthreads();
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
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int c0 = 0; c0 < LR; c0 += 8) {
                if (j < c0 + 8) {
#pragma unroll
                    for (int t = c0; t < c0 + 8 && t + 1 < LR; t += 2) {
                        const double2 v2 = *reinterpret_cast<const double2 *>(&xs[t]);
                        d0 += v2.x * x[t];
                        d1 += v2.y * x[t + 1];
                    }
                    if ((LR & 1) && c0 + 8 >= LR) d0 += xs[LR - 1] * x[LR - 1];
                }
            }
            for (int t = (j > LR ? j : LR); t < L; ++t) d0 += xs[t] * xsm[(t - LR) * SQR_THREADS + tid];
            const double tw = tau * (d0 + d1);
            double bj = 0.0;
#pragma unroll
            for (int c0 = 0; c0 < LR; c0 += 8) {
                if (j < c0 + 8) {
#pragma unroll
                    for (int t = c0; t < c0 + 8 && t < LR; ++t) {
                        const double2 e2 = *reinterpret_cast<const double2 *>(&xe[2 * t]);
                        x[t] -= tw * e2.x;
                        bj += e2.y * x[t];
                    }
                }
            }
            for (int t = (j > LR ? j : LR); t < L; ++t) {
                double *p = &xsm[(t - LR) * SQR_THREADS + tid];
                const double nv = *p - tw * xs[t];
                *p = nv;
                if (t == j) bj = nv;
            }
            double rn = r - bj * bj;
            if (rn < 1e-6 * r0) {  // recompute from the updated rows (R-G6)
                double s0 = 0.0;
#pragma unroll
                for (int t = 0; t < LR; ++t)
                    if (t > j) s0 += x[t] * x[t];
                for (int t = (j + 1 > LR ? j + 1 : LR); t < L; ++t)
                    s0 += xsm[(t - LR) * SQR_THREADS + tid] * xsm[(t - LR) * SQR_THREADS + tid];
                rn = s0;
            }
            r = rn;
            if (lpos == j) lpos = wp;
        }
        if (j + 1 < a.bb) publish(j + 1);
    }
    __syncthreads();

    // ---- results --------------------------------------------------------------
    if (have) {
#pragma unroll
        for (int t = 0; t < LR; ++t) a.B[t + pc * a.ldb] = x[t];
        for (int t = 0; t < LS; ++t) a.B[(LR + t) + pc * a.ldb] = xsm[t * SQR_THREADS + tid];
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
