// sample_qrcp.cuh -- S2 (kernels K3+K4): bb steps of Businger-Golub QRCP
// (Alg. 1) on the l x n' sample B(:, i:n) (Alg. 2 line P:147).
//
// One persistent cooperative kernel; CTA g owns a contiguous range of the
// sample's PHYSICAL columns and keeps them in place for the whole panel (a
// transposition j <-> s* only relabels logical positions).
//
// Layout.  A CTA's columns are held TRANSPOSED (row-major, [row][column]) so
// that a group of TPC threads per column (TPC = 1..32, a power of two chosen
// by the host so that columns x TPC fills the 256 threads) reads rows
// t = h, h+TPC, ... of consecutive columns with conflict-free shared-memory
// accesses (row stride ncs = CPW mod 16, CPW = 32/TPC columns per warp).
// Columns that do not fit in shared memory live transposed in a global
// scratch (`spill`, L2-resident, coalesced across the column group).  Per-
// column state (squared norm, panel-start norm, logical position, active
// flag) lives in shared memory.
//
// Per step j (all sums in a fixed order: identical bits run to run):
//   1. warp 0 polls the G candidate headers of step j (16 bytes each: value,
//      logical position, step tag) until every tag is current -- no separate
//      grid barrier -- reduces them to the global argmax of the squared norms
//      (lowest logical position on exact ties, R-G5), loads the winner's
//      published column and forms dlarfg (R-G7) in registers; every CTA does
//      this redundantly on the same bits and gets the same reflector;
//   2. every thread group applies H_j to its active columns (dot over its rows
//      + butterfly over the group, then the AXPY) and downdates the squared
//      norm r_s -= B(j,s)^2, recomputing it from the updated rows when
//      r_s < 1e-6 r0_s (R-G6); the column at logical position j takes s*'s
//      position;
//   3. the CTA's best remaining column is published: warp 0 copies its l
//      values to the CTA's slot, then lane 0 stores the header with release
//      semantics (the readers' acquire loads of the header order the data).
// Stops early (bb_eff < bb) when the winning squared norm is <= stop_tol2
// = (1e3 eps)^2 ||Omega A||_F^2 (reading R-G12).
// CTA 0 tracks the logical -> physical map of the touched positions in
// shared memory; at the end it writes `perm` (consumed by S6) and the
// (dst, src) column moves that apply the same transpositions, in order, to A
// and Pi (S3).  Other outputs: piv[j] (s* of step j, relative to column i),
// tauhat, Vhat (l x bb reflectors), Rhat11 (bb x bb), bb_eff, rank, gaps.
#pragma once
#include <climits>
#include "common.cuh"

namespace rq {

constexpr int SQ_THREADS = 256;
constexpr int SQ_WARPS = SQ_THREADS / 32;
constexpr int SQ_MAXL = 160;  // l = b + p <= 160 rows
constexpr int SQ_RPL = 5;     // rows per lane of a warp-held column (SQ_MAXL / 32)
constexpr int SQ_MAXB = 128;  // panel width
constexpr int SQ_MAXG = 256;  // CTAs (headers scanned by one warp, 8 per lane)
constexpr int SQS_UNITS = SQ_MAXL + 3;  // tagged slot (poll_mode 3): v, pos | col << 32, v2, column
constexpr int SQ_SPB = 16;    // loads in flight per thread for L2-resident (spilled) columns

struct __align__(16) SqHdr {  // one candidate header (16 bytes, one vector store)
    double v;                 // squared norm of the best active column (-1: none)
    int pos;                  // its logical position (INT_MAX: none)
    unsigned tag;             // launch sequence * 256 + step: never repeats within a context
};

struct SqArgs {
    double *B;            // sample, physical columns, lpad x nn, ld ldb
    int64_t ldb;
    int l, lpad;
    int64_t nn;           // n' = trailing columns of this panel
    int bb;               // planned panel width
    int tpc;              // threads per column (power of two, <= 32)
    int nsm;              // columns per CTA held in shared memory
    int ncs;              // row stride of the shared-memory tile (>= nsm)
    double *spill;        // global scratch for the other columns (transposed, per CTA)
    uint4 *ll;            // [2][G][SQ_MAXL + 3] tagged 16-byte units (sample_qrcp_reg.cuh; poll_mode 3 here)
    const double *stop_tol2;
    SqHdr *slot_hdr;      // [2][G] x hstride
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
    unsigned tag0;        // launch sequence * 256 (distinct per launch)
    int hstride;          // header stride in headers (8: one header per 128-byte line)
    int poll_mode;        // 0: acquire polls; 1: relaxed polls + one acquire fence; 2: 1 + nanosleep backoff;
                          // 3: tagged 16-byte units (ll), no release / acquire fence on either side
    unsigned long long *trace;  // debug: [G][64 steps][4 phases] clock64 stamps, or nullptr
    int spec;             // register grids: fetch the column of the best candidate seen so far while
                          // the last headers are still arriving (0: only after every header)
};

RQ_DEV bool sq_better(double v, int pos, double bv, int bpos) { return (v > bv) || (v == bv && pos < bpos); }

// dynamic shared memory: l x ncs tile + state of cpb columns
__host__ __device__ inline size_t sq_smem_bytes(int ncs, int64_t cpb, int l) {
    return (size_t)l * ncs * sizeof(double) + (size_t)cpb * (2 * sizeof(double) + 2 * sizeof(int));
}

RQ_DEV void st_release_hdr(SqHdr *p, double v, int pos, unsigned tag) {
    const unsigned long long w0 = (unsigned long long)__double_as_longlong(v);
    const unsigned long long w1 = (unsigned long long)(unsigned)pos | ((unsigned long long)tag << 32);
    asm volatile("st.release.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
RQ_DEV void ld_relaxed_hdr(const SqHdr *p, double &v, int &pos, unsigned &tag) {
    unsigned long long a, b;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    v = __longlong_as_double((long long)a);
    pos = (int)(unsigned)(b & 0xffffffffull);
    tag = (unsigned)(b >> 32);
}
RQ_DEV void ld_acquire_hdr(const SqHdr *p, double &v, int &pos, unsigned &tag) {
    unsigned long long a, b;
    asm volatile("ld.acquire.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    v = __longlong_as_double((long long)a);
    pos = (int)(unsigned)(b & 0xffffffffull);
    tag = (unsigned)(b >> 32);
}

__global__ void __launch_bounds__(SQ_THREADS, 1) sample_qrcp_kernel(SqArgs a) {
    extern __shared__ __align__(16) double sq_dyn[];
    __shared__ double xs[SQ_MAXL];
    __shared__ double wv[SQ_WARPS], wv2[SQ_WARPS];
    __shared__ int wpos[SQ_WARPS], wcol[SQ_WARPS];
    __shared__ double s_tau, s_beta, s_alpha;
    __shared__ int s_wpos, s_wcol, s_stop, s_np;
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
    const int nov = ncol - nsm;  // spilled columns (row stride nov in the scratch)
    const int ncs = a.ncs;
    const bool want_v2 = a.gaps != nullptr;
    const int TPC = a.tpc, CPW = 32 / TPC;
    const int gh = lane / CPW;                   // row phase of this thread in its group
    const int gslot = warp * CPW + (lane % CPW);  // column slot within a round
    const int CPR = SQ_WARPS * CPW;              // columns per round
    const int nrounds = (ncol + CPR - 1) / CPR;

    if (*a.status != 0 || *a.done) {
        if (g == 0 && tid == 0) { *a.bb_eff = 0; *a.swap_np = 0; }
        return;
    }
    const double stop2 = *a.stop_tol2;

    double *tile = sq_dyn;  // [l][ncs]
    double *r = sq_dyn + (size_t)l * ncs;
    double *r0 = r + cpb;
    int *lpos = reinterpret_cast<int *>(r0 + cpb);
    int *act = lpos + cpb;
    double *spill = a.spill + c_lo * (int64_t)lpad;  // [l][nov]
    // element (t, cl) of this CTA's columns
    auto elem = [&](int t, int cl) -> double * {
        return (cl < nsm) ? tile + (size_t)t * ncs + cl : spill + (size_t)t * nov + (cl - nsm);
    };

    // ---- load (transpose) this CTA's columns --------------------------------
    for (int e = tid; e < ncol * l; e += SQ_THREADS) {
        const int t = e % l, cl = e / l;
        *elem(t, cl) = a.B[t + (c_lo + cl) * a.ldb];
    }
    for (int64_t x = c_lo + tid; x < c_hi; x += SQ_THREADS) a.perm[x] = x;
    if (g == 0) {
        for (int x = tid; x < a.bb; x += SQ_THREADS) low[x] = x;
        if (tid == 0) hi_n = 0;
    }
    __syncthreads();

    // group butterfly (lanes of one column differ in the bits CPW..16)
    auto gsum = [&](double v) {
        for (int o = CPW; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };

    // this thread's best active column (and second-best value)
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

    // ---- initial squared norms (K3) -----------------------------------------
    for (int rd = 0; rd < nrounds; ++rd) {
        const int cl = rd * CPR + gslot;
        const bool have = cl < ncol;
        double s0 = 0.0, s1 = 0.0;
        if (have) {
            int t = gh;
            for (; t + TPC < l; t += 2 * TPC) {
                const double x0 = *elem(t, cl), x1 = *elem(t + TPC, cl);
                s0 += x0 * x0;
                s1 += x1 * x1;
            }
            if (t < l) { const double x0 = *elem(t, cl); s0 += x0 * x0; }
        }
        const double s = gsum(s0 + s1);
        if (have) {
            if (gh == 0) { r[cl] = s; r0[cl] = s; lpos[cl] = (int)(c_lo + cl); act[cl] = 1; }
            consider(s, (int)(c_lo + cl), (int)(c_lo + cl));
        }
    }

    // CTA-best of this thread's candidates -> header + column of slot (step & 1).
    // Warp reduce, then warp 0 reduces the SQ_WARPS candidates, copies the
    // column and releases the header.
    auto publish = [&](int step) {
        const int parity = step & 1;
        double v = bv, v2 = bv2;
        int p = bpos, c = bcol;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const double ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            const int oc = __shfl_xor_sync(0xffffffffu, c, o);
            if (sq_better(ov, op, v, p)) {
                v2 = fmax(fmax(v2, ov2), (oc == c) ? ov2 : v);
                v = ov; p = op; c = oc;
            } else {
                v2 = fmax(fmax(v2, ov2), (oc == c) ? v2 : ov);
            }
        }
        if (lane == 0) { wv[warp] = v; wv2[warp] = v2; wpos[warp] = p; wcol[warp] = c; }
        __syncthreads();
        if (warp == 0) {
            v = -1.0; v2 = -1.0; p = INT_MAX; c = -1;
            if (lane < SQ_WARPS) { v = wv[lane]; v2 = wv2[lane]; p = wpos[lane]; c = wcol[lane]; }
#pragma unroll
            for (int o = SQ_WARPS / 2; o > 0; o >>= 1) {
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
            v = __shfl_sync(0xffffffffu, v, 0);  // lanes 0..7 hold the CTA best
            v2 = __shfl_sync(0xffffffffu, v2, 0);
            p = __shfl_sync(0xffffffffu, p, 0);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (a.poll_mode == 3) {  // tagged units: no fence waits for this CTA's outstanding stores
                uint4 *dst = a.ll + (int64_t)(parity * G + g) * SQS_UNITS;
                const unsigned tg = a.tag0 + (unsigned)step;
                if (c >= 0) {
                    const int cl = c - (int)c_lo;
                    for (int t = lane; t < l; t += 32)
                        ll_store(dst + 3 + t, (unsigned long long)__double_as_longlong(*elem(t, cl)), tg);
                }
                if (lane == 0) ll_store(dst, (unsigned long long)__double_as_longlong(v), tg);
                if (lane == 1) ll_store(dst + 1, (unsigned long long)(unsigned)p | ((unsigned long long)(unsigned)c << 32), tg);
                if (lane == 2 && want_v2) ll_store(dst + 2, (unsigned long long)__double_as_longlong(v2), tg);
            } else {
                if (c >= 0) {
                    double *dst = a.slot_data + (int64_t)(parity * G + g) * lpad;
                    const int cl = c - (int)c_lo;
                    for (int t = lane; t < l; t += 32) __stcg(dst + t, *elem(t, cl));
                }
                if (lane == 0) {
                    a.slot_col[parity * G + g] = c;
                    if (want_v2) a.slot_v2[parity * G + g] = v2;
                }
                __syncwarp();
                if (lane == 0) {
                    st_release_hdr(a.slot_hdr + (int64_t)(parity * G + g) * a.hstride, v, p, a.tag0 + (unsigned)step);
                }
            }
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
        // ---- 1. global winner and its Householder reflector (warp 0) ----------
        if (warp == 0) {
            const unsigned want = a.tag0 + (unsigned)j;
            constexpr int HPL = SQ_MAXG / 32;  // headers per lane
            double v = -1.0;
            int p = INT_MAX, sl = -1;
            bool stop;
            double xv[SQ_RPL];
            int wc = -1;
            if (a.poll_mode == 3) {
                // tagged units: poll the G headers, then the winner's column
                const uint4 *slots = a.ll + (int64_t)(par * G) * SQS_UNITS;
                bool ready[HPL];
                unsigned long long h0[HPL], h1[HPL];
#pragma unroll
                for (int u = 0; u < HPL; ++u) { ready[u] = (lane + 32 * u >= G); h0[u] = 0; h1[u] = 0; }
                while (true) {
                    bool all = true;
#pragma unroll
                    for (int u = 0; u < HPL; ++u) {
                        if (!ready[u]) {
                            const uint4 *hq = slots + (int64_t)(lane + 32 * u) * SQS_UNITS;
                            const bool r0_ = ll_load(hq, want, h0[u]);
                            const bool r1_ = ll_load(hq + 1, want, h1[u]);
                            ready[u] = r0_ && r1_;
                        }
                        all = all && ready[u];
                    }
                    if (__all_sync(0xffffffffu, all)) break;
                }
                double hvs[HPL];
#pragma unroll
                for (int u = 0; u < HPL; ++u) {
                    const int q = lane + 32 * u;
                    hvs[u] = __longlong_as_double((long long)h0[u]);
                    const int hp_ = (int)(unsigned)(h1[u] & 0xffffffffull);
                    if (q < G && hp_ != INT_MAX && sq_better(hvs[u], hp_, v, p)) {
                        v = hvs[u]; p = hp_; sl = q; wc = (int)(unsigned)(h1[u] >> 32);
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
                stop = (sl < 0) || !(v > stop2);
                {
                    const uint4 *src = slots + (int64_t)(sl >= 0 ? sl : 0) * SQS_UNITS + 3;
                    bool ok[SQ_RPL];
#pragma unroll
                    for (int qq = 0; qq < SQ_RPL; ++qq) { ok[qq] = stop || lane + 32 * qq >= l; xv[qq] = 0.0; }
                    while (true) {
                        bool all = true;
#pragma unroll
                        for (int qq = 0; qq < SQ_RPL; ++qq) {
                            if (!ok[qq]) {
                                unsigned long long w;
                                ok[qq] = ll_load(src + lane + 32 * qq, want, w);
                                xv[qq] = __longlong_as_double((long long)w);
                            }
                            all = all && ok[qq];
                        }
                        if (__all_sync(0xffffffffu, all)) break;
                    }
                }
                if (g == 0 && want_v2 && !stop) {  // gap of the step (diagnostic): runner-up over all slots
                    double m2 = -1.0;
#pragma unroll
                    for (int u = 0; u < HPL; ++u) {
                        const int q = lane + 32 * u;
                        if (q >= G) continue;
                        double val = hvs[u];
                        if (q == sl) {
                            unsigned long long w;
                            while (!ll_load(slots + (int64_t)q * SQS_UNITS + 2, want, w)) {}
                            val = __longlong_as_double((long long)w);
                        }
                        m2 = fmax(m2, val);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o));
                    if (lane == 0) a.gaps[j] = (m2 < 0.0 || v == 0.0) ? 1.0 : (v - m2) / v;
                }
                if (lane == 0) {
                    s_stop = stop;
                    s_wpos = p;
                    s_wcol = wc;
                }
            } else {
                bool ready[HPL];
                double hv[HPL];
                int hp[HPL];
#pragma unroll
                for (int u = 0; u < HPL; ++u) { ready[u] = (lane + 32 * u >= G); hv[u] = -1.0; hp[u] = INT_MAX; }
                // poll until every header of step j is visible (acquire loads)
                const int pm = a.poll_mode;
                while (true) {
                    bool all = true;
#pragma unroll
                    for (int u = 0; u < HPL; ++u) {
                        if (!ready[u]) {
                            unsigned tg;
                            const SqHdr *hp_ = a.slot_hdr + (int64_t)(par * G + lane + 32 * u) * a.hstride;
                            if (pm == 0) ld_acquire_hdr(hp_, hv[u], hp[u], tg);
                            else ld_relaxed_hdr(hp_, hv[u], hp[u], tg);
                            ready[u] = (tg == want);
                        }
                        all = all && ready[u];
                    }
                    if (__all_sync(0xffffffffu, all)) break;
                    if (pm == 2) __nanosleep(64);
                }
                if (pm != 0) asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
#pragma unroll
                for (int u = 0; u < HPL; ++u) {
                    const int q = lane + 32 * u;
                    if (q < G && hp[u] != INT_MAX && sq_better(hv[u], hp[u], v, p)) {
                        v = hv[u]; p = hp[u]; sl = q;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                    const int op = __shfl_xor_sync(0xffffffffu, p, o);
                    const int osl = __shfl_xor_sync(0xffffffffu, sl, o);
                    if (osl >= 0 && (sl < 0 || sq_better(ov, op, v, p))) { v = ov; p = op; sl = osl; }
                }
                stop = (sl < 0) || !(v > stop2);
                const double *src = a.slot_data + (int64_t)(par * G + (sl >= 0 ? sl : 0)) * lpad;
#pragma unroll
                for (int qq = 0; qq < SQ_RPL; ++qq) {
                    const int t = lane + 32 * qq;
                    xv[qq] = (!stop && t < l) ? __ldcg(src + t) : 0.0;
                }
                wc = (sl >= 0) ? __ldcg(a.slot_col + par * G + sl) : -1;
                if (lane == 0) {
                    s_stop = stop;
                    s_wpos = p;
                    s_wcol = wc;
                    if (g == 0 && want_v2 && !stop) {
                        double v2 = -1.0;
                        for (int q = 0; q < G; ++q) {
                            const double hv = __ldcg(&a.slot_hdr[(int64_t)(par * G + q) * a.hstride].v);
                            v2 = fmax(v2, (q == sl) ? __ldcg(a.slot_v2 + par * G + q) : hv);
                        }
                        a.gaps[j] = (v2 < 0.0 || v == 0.0) ? 1.0 : (v - v2) / v;
                    }
                }
            }
            if (!stop) {
                double sx = 0.0;
#pragma unroll
                for (int qq = 0; qq < SQ_RPL; ++qq) {
                    const int t = lane + 32 * qq;
                    if (t > j) sx += xv[qq] * xv[qq];
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
                    if (t < l) xs[t] = (t > j) ? xv[qq] * scal : (t == j ? 1.0 : xv[qq]);
                }
                if (lane == 0) { s_tau = tau; s_beta = beta; }
            }
        }
        __syncthreads();
        stamp(1);
        if (s_stop) break;
        const int wp = s_wpos, wcl = s_wcol;
        const double tau = s_tau;
        // ---- outputs + position map ------------------------------------------
        // step-j outputs written by CTA (j+1) mod G (spreads the extra work)
        if (g == (j + 1) % G) {
            for (int t = tid; t < lpad; t += SQ_THREADS)
                a.vhat[t + (int64_t)j * lpad] = (t < j) ? 0.0 : (t == j ? 1.0 : (t < l ? xs[t] : 0.0));
            for (int t = tid; t < a.bbpad; t += SQ_THREADS)
                a.rhat11[t + (int64_t)j * a.bbpad] = (t < j) ? xs[t] : (t == j ? s_beta : 0.0);
            if (tid == 0) { a.piv[j] = wp; a.tauhat[j] = tau; }
        }
        if (g == 0 && warp == SQ_WARPS - 1) {
            // transposition j <-> wp; q = phys column at position j (< bb)
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
        // ---- 2. apply H_j to own active columns, downdate norms -------------
        bv = -1.0; bv2 = -1.0; bpos = INT_MAX; bcol = -1;
        const int t0 = j + ((gh - j) % TPC + TPC) % TPC;  // first row >= j of this phase
        for (int rd = 0; rd < nrounds; ++rd) {
            const int cl = rd * CPR + gslot;
            const int64_t pc = c_lo + cl;
            bool live = cl < ncol;
            if (live && pc == wcl) { live = false; if (gh == 0) act[cl] = 0; }  // retire the pivot
            live = live && act[cl < ncol ? cl : 0];
            // dot over this thread's rows (two chains), then the group butterfly
            double d0 = 0.0, d1 = 0.0;
            double *base = nullptr;
            int rs = 0;
            if (live) {
                if (cl < nsm) { base = tile + cl; rs = ncs; }
                else { base = spill + (cl - nsm); rs = nov; }
                int t = t0;
                if (cl >= nsm) {
                    // L2-resident column: SQ_SPB loads in flight per thread (the
                    // loop below would expose one L2 latency per pair of rows)
                    for (; t + (SQ_SPB - 1) * TPC < l; t += SQ_SPB * TPC) {
                        double xv[SQ_SPB];
#pragma unroll
                        for (int u = 0; u < SQ_SPB; ++u) xv[u] = base[(size_t)(t + u * TPC) * rs];
#pragma unroll
                        for (int u = 0; u < SQ_SPB; u += 2) {
                            d0 += xs[t + u * TPC] * xv[u];
                            d1 += xs[t + (u + 1) * TPC] * xv[u + 1];
                        }
                    }
                }
                for (; t + TPC < l; t += 2 * TPC) {
                    d0 += xs[t] * base[(size_t)t * rs];
                    d1 += xs[t + TPC] * base[(size_t)(t + TPC) * rs];
                }
                if (t < l) d0 += xs[t] * base[(size_t)t * rs];
            }
            const double w = gsum(d0 + d1);
            double bj = 0.0, tail = 0.0;
            if (live) {
                const double tw = tau * w;
                int t = t0;
                if (cl >= nsm) {  // L2-resident column: batches of SQ_SPB loads
                    for (; t + (SQ_SPB - 1) * TPC < l; t += SQ_SPB * TPC) {
                        double xv[SQ_SPB];
#pragma unroll
                        for (int u = 0; u < SQ_SPB; ++u) xv[u] = base[(size_t)(t + u * TPC) * rs];
#pragma unroll
                        for (int u = 0; u < SQ_SPB; ++u) {
                            const int tt = t + u * TPC;
                            const double x = xv[u] - tw * xs[tt];
                            base[(size_t)tt * rs] = x;
                            if (tt == j) bj = x;
                            else tail += x * x;
                        }
                    }
                }
                for (; t < l; t += TPC) {
                    const double x = base[(size_t)t * rs] - tw * xs[t];
                    base[(size_t)t * rs] = x;
                    if (t == j) bj = x;
                    else tail += x * x;
                }
            }
            bj = gsum(bj);  // exactly one thread of the group holds row j
            const double rr = live ? r[cl] : 0.0, rr0 = live ? r0[cl] : 0.0;
            double rn = rr - bj * bj;
            const bool need = live && (rn < 1e-6 * rr0);
            if (__any_sync(0xffffffffu, need)) {
                const double ts = gsum(tail);
                if (need) rn = ts;
            }
            const int lp = live ? lpos[cl] : 0;
            __syncwarp();  // the group's reads of r/lpos precede the writes below
            if (live) {
                const int pos = (lp == j) ? wp : lp;  // position j moves to s*
                if (gh == 0) { r[cl] = rn; lpos[cl] = pos; }
                consider(rn, pos, (int)pc);
            }
        }
        stamp(2);
        // ---- 3. candidates for step j+1 -------------------------------------
        if (j + 1 < a.bb) publish(j + 1);
        stamp(3);
    }

    // ---- results --------------------------------------------------------------
    __syncthreads();
    // transformed columns back to global, column-major (S6 reads R-hat12/22)
    for (int e = tid; e < ncol * l; e += SQ_THREADS) {
        const int t = e % l, cl = e / l;
        a.B[t + (c_lo + cl) * a.ldb] = *elem(t, cl);
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
