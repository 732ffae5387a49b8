// sample_qrcp_cl.cuh -- S2 sample QRCP (Alg. 1, on the l x n'
// sample, Alg. 2 line P:147) for samples that fit one thread-block cluster
// with ONE COLUMN PER THREAD held in registers: l <= SQC_L rows and
// n' <= 16 CTAs x 256 threads.  Same arithmetic and outputs as the grid
// kernel in sample_qrcp.cuh (dlarfg reading R-G7, squared-norm downdates with
// the R-G6 recompute, lowest-position ties R-G5, stop rule R-G12); the
// per-step exchange goes through distributed shared memory and one
// split-phase cluster barrier instead of L2:
//   publish(j): each CTA's best remaining column (value, position, physical
//     column, its l entries) into its own shared-memory slot (parity j & 1),
//     then barrier.cluster.arrive.release;
//   step j: barrier.cluster.wait.acquire; warp 0 reads the G candidate
//     headers and the winner's column with ld.shared::cluster, forms the
//     reflector redundantly in every CTA (same bits), then every thread
//     applies it to its register-resident column.
// Double-buffered slots + the barrier order every reuse (a slot of parity p
// is rewritten two steps later, after every CTA passed the barrier between).
#pragma once
#include <climits>
#include "common.cuh"
#include "sample_qrcp.cuh"

namespace rq {

constexpr int SQC_L = 80;         // max rows (l = b + p); kernels are instantiated for exact l
constexpr int SQC_THREADS = 256;  // columns per CTA
constexpr int SQC_MAXG = 16;      // CTAs (one cluster)
#ifndef SQC_CH
#define SQC_CH 16                 // rows per skipped chunk in the apply (uniform branches;
                                  // measured at C2: 8 / 16 / 24 / 32 rows -> S2 1.70 / 1.59 / 1.60 / 1.61 ms)
#endif

RQ_DEV unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
RQ_DEV void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
RQ_DEV void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
RQ_DEV unsigned cl_map(const void *p, unsigned rank) {
    unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
RQ_DEV double cl_ld_f64(unsigned addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
RQ_DEV int cl_ld_s32(unsigned addr) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

template <int L>
__global__ void __launch_bounds__(SQC_THREADS, 1) sample_qrcp_cluster_kernel(SqArgs a) {
    constexpr int RECW = (L + 2 + 1) / 2 * 2;  // pushed record: v, (pos, col) bits, the column, padded to pairs
    constexpr int NPAIR = RECW / 2;
    extern __shared__ __align__(16) double comp[];  // CTA 0: [bb][L] winner columns (LAPACK format)
    __shared__ int s_piv[SQ_MAXB];
    __shared__ double s_tauh[SQ_MAXB];
    __shared__ __align__(16) double rec[RECW];                   // this CTA's candidate record
    __shared__ __align__(16) double recv[2][SQC_MAXG][RECW];     // pushed records (slot = source CTA)
    __shared__ __align__(16) double vw[SQ_WARPS][SQC_L];         // per-warp copy of the reflector
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ double wv[SQ_WARPS];
    __shared__ int wpos[SQ_WARPS], wcol[SQ_WARPS];
    __shared__ int s_np;
    __shared__ int64_t low[SQ_MAXB];
    __shared__ int hi_pos[SQ_MAXB];
    __shared__ int64_t hi_phys[SQ_MAXB];
    __shared__ int hi_n;

    const int G = gridDim.x;
    const int g = (int)cl_rank();
    // the recorder CTA (stages the outputs, receives whole records): the last
    // one, which holds the ragged remainder of the columns (least apply work)
    const int rg0 = G - 1;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nn = a.nn;  // (a.l == L: the kernel is instantiated per sample height)
    const int64_t cpb = (nn + G - 1) / G;  // <= 256
    const int64_t c_lo = min(nn, (int64_t)g * cpb), c_hi = min(nn, c_lo + cpb);
    const bool have = tid < (int)(c_hi - c_lo);
    const int64_t pc = c_lo + tid;  // this thread's physical column
    // every CTA takes part in every exchange, so an early exit is uniform
    const bool noop = (*a.status != 0 || *a.done);
    if (noop) {
        if (g == 0 && tid == 0) { *a.bb_eff = 0; *a.swap_np = 0; }
        return;
    }
    const double stop2 = *a.stop_tol2;
    const unsigned mb0 = (unsigned)__cvta_generic_to_shared(&mbar[0]);
    // bytes a CTA receives for step st: the recorder rg0 gets every record whole
    // (it stages the R-hat rows); the others the header and rows >= (st & ~1) only
    auto step_bytes = [&](int st) -> unsigned {
        const int np = (g == rg0) ? NPAIR : NPAIR - (st & ~1) / 2;
        return (unsigned)(G * np * 16);
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb0 + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }

    double x[L];
#pragma unroll
    for (int t = 0; t < L; ++t) x[t] = 0.0;
    if (have) {  // the column's l entries are contiguous: 16-byte loads when aligned
        const double *src = a.B + pc * a.ldb;
        if (((a.ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.B) & 15) == 0)) {
#pragma unroll
            for (int t = 0; t + 1 < L; t += 2) {
                const double2 v = reinterpret_cast<const double2 *>(src)[t / 2];
                x[t] = v.x;
                x[t + 1] = v.y;
            }
            if (L & 1) x[L - 1] = src[L - 1];
        } else {
#pragma unroll
            for (int t = 0; t < L; ++t) x[t] = src[t];
        }
    }
    double r = 0.0;
#pragma unroll
    for (int t = 0; t < L; ++t) r += x[t] * x[t];
    double r0 = r;
    int lpos = (int)pc;
    bool act = have;
    if (have) a.perm[pc] = pc;
    if (g == rg0) {
        for (int q = tid; q < a.bb; q += SQC_THREADS) low[q] = q;
        if (tid == 0) hi_n = 0;
    }
    // every CTA's mbarriers are initialised before anyone pushes
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    cl_wait();
    if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb0), "r"(step_bytes(0)) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb0 + 8), "r"(step_bytes(1)) : "memory");
    }

    // CTA-best candidate (value, position, physical column, its l entries),
    // pushed into slot g of every CTA's receive buffer of parity (step & 1)
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
        // every thread reduces the SQ_WARPS candidates (same order: same result)
        double bv = wv[0];
        int bp = wpos[0], bc = wcol[0];
        for (int w = 1; w < SQ_WARPS; ++w)
            if (sq_better(wv[w], wpos[w], bv, bp)) { bv = wv[w]; bp = wpos[w]; bc = wcol[w]; }
        if (act && (int)pc == bc) {
            double2 *r2 = reinterpret_cast<double2 *>(&rec[2]);
#pragma unroll
            for (int t = 0; t + 1 < L; t += 2) r2[t / 2] = make_double2(x[t], x[t + 1]);
            if (L & 1) rec[2 + L - 1] = x[L - 1];
        }
        if (tid == 0) {
            rec[0] = bv;
            rec[1] = __longlong_as_double(((long long)bp << 32) | (unsigned)bc);
        }
        __syncthreads();
        const unsigned lm = mb0 + 8 * par;
        // pair 0 (header) and the column pairs: all of them to the recorder CTA
        // rg0, from the pair holding row (step & ~1) on to the others
        const int p0 = 1 + (step & ~1) / 2;      // first column pair sent to CTAs != 0
        const int np_o = NPAIR - p0 + 1;          // pairs per record for CTAs != 0
        const int ntot = NPAIR + (G - 1) * np_o;
        for (int e = tid; e < ntot; e += SQC_THREADS) {
            int d, w;
            if (e < NPAIR) { d = rg0; w = 2 * e; }
            else {
                const int f = e - NPAIR, q = f % np_o;
                d = f / np_o;  // 0 .. G-2: the CTAs other than rg0
                w = 2 * ((q == 0) ? 0 : p0 + q - 1);
            }
            const double2 val = *reinterpret_cast<const double2 *>(&rec[w]);
            const unsigned la = (unsigned)__cvta_generic_to_shared(&recv[par][g][w]);
            unsigned ra, rm;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(d));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rm) : "r"(lm), "r"(d));
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(ra),
                         "d"(val.x), "d"(val.y), "r"(rm)
                         : "memory");
        }
    };

    publish(0);

    int j = 0;
    auto stamp = [&](int ph) {
        if (a.trace && tid == 0 && j < 64) a.trace[((size_t)g * 64 + j) * 4 + ph] = clock64();
    };
    for (; j < a.bb; ++j) {
        const int par = j & 1;
        stamp(0);
        {
            unsigned ok = 0;
            const unsigned ph = (unsigned)((j >> 1) & 1);
            while (!ok)
                asm volatile(
                    "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                    " selp.u32 %0, 1, 0, p;\n}\n"
                    : "=r"(ok)
                    : "r"(mb0 + 8 * par), "r"(ph)
                    : "memory");
        }
        // step j+2 re-arms this mbarrier: its bytes can only come after every
        // CTA received this CTA's step j+1 record (sent after all reads below)
        if (tid == 0 && j + 2 < a.bb)
            asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb0 + 8 * par),
                         "r"(step_bytes(j + 2))
                         : "memory");
        // ---- 1. winner and its reflector, redundantly in EVERY warp (local
        //      shared memory only: same bits everywhere, no CTA barrier) ------
        double v = -1.0;
        int p = INT_MAX, sl = -1, wc = -1;
        if (lane < G) {
            v = recv[par][lane][0];
            const long long pcb = __double_as_longlong(recv[par][lane][1]);
            p = (int)(pcb >> 32);
            wc = (int)(unsigned)(pcb & 0xffffffffll);
            if (p != INT_MAX) sl = lane;
            else v = -1.0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            const int osl = __shfl_xor_sync(0xffffffffu, sl, o);
            const int owc = __shfl_xor_sync(0xffffffffu, wc, o);
            if (osl >= 0 && (sl < 0 || sq_better(ov, op, v, p))) { v = ov; p = op; sl = osl; wc = owc; }
        }
        const bool stop = (sl < 0) || !(v > stop2);
        stamp(1);
        if (stop) break;  // uniform: every warp of every CTA sees the same records
        const int wp = p, wcl = wc;
        const double *wx = &recv[par][sl][2];  // the winner column (rows < j: R-hat entries)
        double xv[SQ_RPL];
        double sx = 0.0, alpha = 0.0;
#pragma unroll
        for (int qq = 0; qq < SQ_RPL; ++qq) {
            const int t = lane + 32 * qq;
            xv[qq] = (t < L) ? wx[t] : 0.0;
            if (t > j && t < L) sx += xv[qq] * xv[qq];
        }
        alpha = wx[j];
        sx = warp_sum(sx);
        double tau = 0.0, beta = alpha, scal = 0.0;
        if (sx != 0.0) {
            const double nrm = sqrt(alpha * alpha + sx);
            beta = (alpha >= 0.0) ? -nrm : nrm;
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        // this warp's copy of the reflector (rows < j zero: the apply needs no predicates)
        double *xs = vw[warp];
#pragma unroll
        for (int qq = 0; qq < SQ_RPL; ++qq) {
            const int t = lane + 32 * qq;
            if (t < L) xs[t] = (t > j) ? xv[qq] * scal : (t == j ? 1.0 : 0.0);
        }
        __syncwarp();
        // ---- outputs (staged in CTA 0's shared memory, written at the end) -----
        if (g == rg0 && warp == 0) {
            // column j in LAPACK format: R-hat above the diagonal, beta, v below
#pragma unroll
            for (int qq = 0; qq < SQ_RPL; ++qq) {
                const int t = lane + 32 * qq;
                if (t < L) comp[j * L + t] = (t < j) ? xv[qq] : (t == j ? beta : xs[t]);
            }
            if (lane == 0) { s_piv[j] = wp; s_tauh[j] = tau; }
        }
        if (g == rg0 && warp == SQ_WARPS - 1) {
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
        if (act && (int)pc == wcl) act = false;  // retire the pivot
        if (act) {
            // w = v^T x over rows >= j (xs is zero above row j); SQC_CH-row chunks
            // entirely above row j are skipped (uniform branches)
            // four independent accumulators (row t goes to accumulator t mod 4)
            double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int c0 = 0; c0 < L; c0 += SQC_CH) {
                if (j < c0 + SQC_CH) {
#pragma unroll
                    for (int t = c0; t < c0 + SQC_CH && t + 1 < L; t += 2) {
                        const double2 v2 = *reinterpret_cast<const double2 *>(&xs[t]);
                        d[t & 3] += v2.x * x[t];
                        d[(t + 1) & 3] += v2.y * x[t + 1];
                    }
                    if ((L & 1) && c0 + SQC_CH >= L) d[(L - 1) & 3] += xs[L - 1] * x[L - 1];
                }
            }
            const double tw = tau * ((d[0] + d[1]) + (d[2] + d[3]));
            // x -= tw v (v is zero above row j); bj = the updated x(j), selected
            // inside the one 8-row chunk that holds row j (uniform branch)
            double bj = 0.0;
#pragma unroll
            for (int c0 = 0; c0 < L; c0 += SQC_CH) {
                if (j < c0 + SQC_CH) {
#pragma unroll
                    for (int t = c0; t < c0 + SQC_CH && t + 1 < L; t += 2) {
                        const double2 v2 = *reinterpret_cast<const double2 *>(&xs[t]);
                        x[t] -= tw * v2.x;
                        x[t + 1] -= tw * v2.y;
                    }
                    if ((L & 1) && c0 + SQC_CH >= L) x[L - 1] -= tw * xs[L - 1];
                    if (j >= c0) {
#pragma unroll
                        for (int t = c0; t < c0 + SQC_CH && t < L; ++t)
                            if (t == j) bj = x[t];
                    }
                }
            }
            double rn = r - bj * bj;
            if (rn < 1e-6 * r0) {  // recompute from the updated rows (R-G6)
                double s0 = 0.0;
#pragma unroll
                for (int t = 0; t < L; ++t)
                    if (t > j) s0 += x[t] * x[t];
                rn = s0;
            }
            r = rn;
            if (lpos == j) lpos = wp;  // position j moves to s*
        }
        stamp(2);
        if (j + 1 < a.bb) publish(j + 1);
        stamp(3);
    }
    // no CTA leaves while pushes into it may be in flight
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    cl_wait();

    // ---- results --------------------------------------------------------------
    if (have) {
        double *dst = a.B + pc * a.ldb;
        if (((a.ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.B) & 15) == 0)) {
#pragma unroll
            for (int t = 0; t + 1 < L; t += 2) reinterpret_cast<double2 *>(dst)[t / 2] = make_double2(x[t], x[t + 1]);
            if (L & 1) dst[L - 1] = x[L - 1];
        } else {
#pragma unroll
            for (int t = 0; t < L; ++t) dst[t] = x[t];
        }
    }
    if (g == rg0) {
        // Vhat (lpad x bbpad: unit diagonal, v below), Rhat11 (bbpad x bbpad), piv, tauhat
        for (int e = tid; e < j * a.lpad; e += SQC_THREADS) {
            const int t = e % a.lpad, c = e / a.lpad;
            a.vhat[e] = (t < c || t >= L) ? 0.0 : (t == c ? 1.0 : comp[c * L + t]);
        }
        for (int e = tid; e < j * a.bbpad; e += SQC_THREADS) {
            const int t = e % a.bbpad, c = e / a.bbpad;
            a.rhat11[e] = (t <= c) ? comp[c * L + t] : 0.0;
        }
        for (int c = tid; c < j; c += SQC_THREADS) { a.piv[c] = s_piv[c]; a.tauhat[c] = s_tauh[c]; }
        if (tid == 0) s_np = 0;
        __syncthreads();
        const int nlow = a.bb;
        for (int e = tid; e < nlow + hi_n; e += SQC_THREADS) {
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
