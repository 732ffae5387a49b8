// panel_cl.cuh -- S4 (kernel K6) for panels that fit the registers of one
// thread-block cluster: unpivoted Householder QR of A(i:m, i:i+bb) (Alg. 2
// line P:149, PDGEQRF at P:760) plus the V^T v_j columns that build the
// compact-WY T (PDLARFT; T itself is formed by tri_kernel).  Same
// arithmetic contract and outputs as panel_qr_kernel (panel.cuh): dlarfg
// (reading R-G7), columns bb_eff..bb-1 still receive the reflectors (R-G12),
// outputs in place + tau + the explicit V / V^T + ybuf.
//
// Layout: the panel is held in REGISTERS, column-owner style.  CTA g of the
// cluster owns panel rows [g*RC, (g+1)*RC) with RC = RG*RPT; thread
// (rg, c) = (tid / BB, tid % BB) holds column c of the RPT rows
// [g*RC + rg*RPT, +RPT) in av[0..RPT-1] (static indices only).  A warp is 32
// consecutive columns of one row group, so row-dependent branches are
// warp-uniform.  Rows 0..bb-1 (the R rows) are row group 0 of CTA 0.
// Per column j:
//   1. the owners of column j have published x = A(r, j) masked to rows r > j
//      in shared memory (xs); every thread forms its partial Gram entry
//      g_c = sum_r A(r, c) x_r over its RPT rows (broadcast smem reads); CTA 0's
//      row group 0 also extracts a_jc (a select tree on the bits of j);
//   2. the RG row-group partials are summed (fixed order) and PUSHED into a
//      slot of every CTA's receive buffer with st.async (DSMEM), completing
//      bytes on the receiver's mbarrier; CTA 0 pushes row j the same way;
//   3. each CTA waits on its own mbarrier (no cluster barrier, no fence, no
//      remote loads), sums the G partials by a fixed tree (identical bits in
//      every CTA); thread j evaluates dlarfg: beta, tau, scal = 1/(alpha - beta);
//   4. column c > j: w_c = tau (a_jc + scal g_c); a_rc -= (w_c scal) x_r (x is
//      zero at rows <= j).  The row-j result a_jc - w_c is final, so CTA 0
//      keeps it in shared memory (Rrow) instead of patching the register;
//      column j itself is left unscaled (v = scal_j x is formed at the store,
//      beta_j is kept in shared memory); CTA 0 records
//      y_c = v_c^T v_j = scal_c (a_jc + scal_j g_c) for c < j (T's column j);
//   5. the owners of column j+1 publish its masked values (double buffer).
// The receive buffers are double buffered by step parity; a CTA can push step
// j+2 only after it received every CTA's step j+1 partial, which each CTA
// sends after it finished reading step j: the data flow orders buffer reuse.
// Global memory is touched only at the start (the panel, coalesced through a
// shared-memory transpose) and at the end (A in place, V, V^T).
#pragma once
#include "common.cuh"
#include "panel.cuh"
#include "sample_qrcp_cl.cuh"

namespace rq {

constexpr int PNC_THREADS = 256;
constexpr int PNC_MAXG = 16;

RQ_DEV void cl_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
RQ_DEV unsigned cl_map_u32(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
RQ_DEV void mbar_init(unsigned mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(count) : "memory");
}
RQ_DEV void mbar_expect_tx(unsigned mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
}
RQ_DEV void mbar_wait_cluster(unsigned mb, unsigned parity) {
    unsigned ok = 0;
    while (!ok)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(mb), "r"(parity)
            : "memory");
}
// 8-byte DSMEM push that completes its bytes on the destination's mbarrier
RQ_DEV void st_async_f64(unsigned raddr, double v, unsigned rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(raddr), "d"(v),
                 "r"(rmbar)
                 : "memory");
}

// pairwise tree sum of N (power of two) values in a fixed order
template <int N>
RQ_DEV double tree_sum(double (&v)[N]) {
    static_assert((N & (N - 1)) == 0, "power of two");
#pragma unroll
    for (int w = N / 2; w >= 1; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) v[i] = v[2 * i] + v[2 * i + 1];
    return v[0];
}

// av[j] for a runtime j < 2^LOG (binary select tree on the bits of j)
template <int N>
RQ_DEV double select_rt(const double (&av)[N], int j) {
    static_assert((N & (N - 1)) == 0, "power of two");
    double s[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) s[i] = (j & 1) ? av[2 * i + 1] : av[2 * i];
#pragma unroll
    for (int w = N / 4, bit = 2; w >= 1; w >>= 1, bit <<= 1) {
#pragma unroll
        for (int i = 0; i < w; ++i) s[i] = (j & bit) ? s[2 * i + 1] : s[2 * i];
    }
    return s[0];
}

template <int BB, int RPT, int CPT = 1>
__global__ void __launch_bounds__(PNC_THREADS, 1) panel_qr_cluster_kernel(PanelArgs a) {
    constexpr int CG = BB / CPT;          // column groups (CPT adjacent columns per thread)
    constexpr int RG = PNC_THREADS / CG;  // row groups
    constexpr int RC = RG * RPT;          // rows per CTA
    constexpr int LDS = RPT + 1;          // staging stride
    constexpr int PG = PNC_THREADS / BB;  // push groups (thread -> (push group, column))
    static_assert(CG % 32 == 0 && RG >= 1, "a warp is 32 column groups of one row group");
    static_assert(RC >= BB, "the R rows (0..bb-1) live in CTA 0");
    // dynamic: max(BB * LDS, BB * BB) doubles: [BB][LDS] staging, then Rrow [BB][BB] (CTA 0)
    extern __shared__ __align__(16) double stage[];
    __shared__ __align__(16) double xs[2][RC];       // masked column j (rows > j), double buffered
    __shared__ __align__(16) double part[RG][BB];
    __shared__ double rj_s[BB];
    __shared__ __align__(16) double recv[2][PNC_MAXG][BB];  // pushed CTA partials (slot = source CTA)
    __shared__ __align__(16) double recv_rj[2][BB];          // pushed row j (from CTA 0)
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ double gsum[BB], rjv[BB];
    __shared__ double scal_s[BB], beta_s[BB];
    __shared__ double s_hh[2];  // this step's tau, scal
    __shared__ int s_stop;

    if (a.skip && *a.skip == 0) return;  // uniform: the CholeskyQR2 path already factored the panel
    const int G = gridDim.x;
    const int g = (int)cl_rank();
    const int tid = threadIdx.x;
    const int cg = tid % CG, rg = tid / CG;
    const int bb = a.bb;
    const int bbe = min(bb, max(0, *a.bb_eff - a.col0));
    const int64_t ldvt = a.ldvt ? a.ldvt : a.bbpad, ldy = a.ldy ? a.ldy : a.bbpad;
    const int64_t mp = a.mp, lda = a.lda;
    const int64_t cta_r0 = (int64_t)g * RC;
    const int rowbase = (int)(cta_r0 + rg * RPT);  // panel row of av[.][0]
    double *Rrow = stage;                          // CTA 0: Rrow[j * BB + c] = R(j, c), c > j

    const unsigned mb0 = (unsigned)__cvta_generic_to_shared(&mbar[0]);
    const unsigned step_bytes = (unsigned)((G + 1) * BB * sizeof(double));
    if (tid == 0) {
        mbar_init(mb0, 1);
        mbar_init(mb0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    double av[CPT][RPT];
    // ---- load.  CPT = 2: straight into registers (each thread's 32 rows of a
    // column are 256 contiguous bytes; 16-byte loads, all in flight at once).
    // CPT = 1: coalesced column reads through the staging buffer, one row group
    // at a time.
    const bool vec_ok = ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.A) & 15) == 0);
    if (CPT == 2) {
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int c = cg * CPT + k;
            const double *src = a.A + rowbase + (int64_t)c * lda;
            if (c < bb && vec_ok && rowbase + RPT <= mp) {
#pragma unroll
                for (int t = 0; t < RPT; t += 2) {
                    const double2 v = reinterpret_cast<const double2 *>(src)[t / 2];
                    av[k][t] = v.x;
                    av[k][t + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int t = 0; t < RPT; ++t) av[k][t] = (c < bb && rowbase + t < mp) ? src[t] : 0.0;
            }
        }
    }
    for (int q = 0; q < (CPT == 2 ? 0 : RG); ++q) {
        const int64_t r0 = cta_r0 + (int64_t)q * RPT;
        for (int e = tid; e < BB * RPT; e += PNC_THREADS) {
            const int r = e % RPT, cc = e / RPT;
            stage[cc * LDS + r] = (cc < bb && r0 + r < mp) ? a.A[r0 + r + (int64_t)cc * lda] : 0.0;
        }
        __syncthreads();
        if (rg == q) {
#pragma unroll
            for (int k = 0; k < CPT; ++k)
#pragma unroll
                for (int t = 0; t < RPT; ++t) av[k][t] = stage[(cg * CPT + k) * LDS + t];
        }
        __syncthreads();
    }
    // every CTA's mbarriers are initialised before anyone pushes
    cl_arrive_relaxed();
    cl_wait();
    if (tid == 0) {
        mbar_expect_tx(mb0, step_bytes);      // step 0
        mbar_expect_tx(mb0 + 8, step_bytes);  // step 1
    }
    // owners of column `col`: x masked to rows > col.  Each of the CPT columns
    // is stored under its own predicate (no register-array selection).
    auto publish_x = [&](int col, int buf) {
        if (col / CPT != cg) return;
        const int kk = col % CPT;
        double2 *x2 = reinterpret_cast<double2 *>(&xs[buf][rg * RPT]);
        if (rowbase > col) {
#pragma unroll
            for (int k = 0; k < CPT; ++k)
                if (k == kk) {
#pragma unroll
                    for (int t = 0; t < RPT; t += 2) x2[t / 2] = make_double2(av[k][t], av[k][t + 1]);
                }
        } else {
#pragma unroll
            for (int k = 0; k < CPT; ++k)
                if (k == kk) {
#pragma unroll
                    for (int t = 0; t < RPT; t += 2)
                        x2[t / 2] = make_double2((rowbase + t > col) ? av[k][t] : 0.0,
                                                 (rowbase + t + 1 > col) ? av[k][t + 1] : 0.0);
                }
        }
    };
    if (bbe > 0) publish_x(0, 0);

    const int tsel = (g == 0) ? 0 : (g == G - 1 ? 1 : -1);
    const int pq = tid / BB, pc = tid % BB;  // push mapping
    const double tol2 = a.tol2 ? *a.tol2 : -1.0;
    int bbo = bbe;  // columns factored (bbe, or the R11-diagonal stop column)
    for (int j = 0; j < bbe; ++j) {
        auto stamp = [&](int ph) {
            if (a.trace && tsel >= 0 && tid == 0 && j < 64) a.trace[((size_t)tsel * 64 + j) * 8 + ph] = clock64();
        };
        stamp(0);
        const int par = j & 1;
        const bool rowj_here = (j >= rowbase && j < rowbase + RPT);  // warp-uniform
        __syncthreads();  // xs[par] published
        // ---- 1. partial Gram entries over this thread's rows ----------------
        {
            const double2 *x2 = reinterpret_cast<const double2 *>(&xs[par][rg * RPT]);
            double s[CPT][2];
#pragma unroll
            for (int k = 0; k < CPT; ++k) s[k][0] = s[k][1] = 0.0;
            double s2[CPT][2];
#pragma unroll
            for (int k = 0; k < CPT; ++k) s2[k][0] = s2[k][1] = 0.0;
#pragma unroll
            for (int t = 0; t < RPT; t += 4) {
                const double2 u = x2[t / 2], v = x2[t / 2 + 1];
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    s[k][0] = fma(av[k][t], u.x, s[k][0]);
                    s[k][1] = fma(av[k][t + 1], u.y, s[k][1]);
                    s2[k][0] = fma(av[k][t + 2], v.x, s2[k][0]);
                    s2[k][1] = fma(av[k][t + 3], v.y, s2[k][1]);
                }
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) part[rg][cg * CPT + k] = (s[k][0] + s[k][1]) + (s2[k][0] + s2[k][1]);
            if (rowj_here) {
#pragma unroll
                for (int k = 0; k < CPT; ++k) rj_s[cg * CPT + k] = select_rt(av[k], j - rowbase);
            }
        }
        stamp(1);
        __syncthreads();
        // ---- 2. CTA partial (and row j) pushed into every CTA's slot --------
        {
            double pv[RG];
#pragma unroll
            for (int q = 0; q < RG; ++q) pv[q] = part[q][pc];
            const double sum = tree_sum(pv);
            const unsigned la = (unsigned)__cvta_generic_to_shared(&recv[par][g][pc]);
            const unsigned lr = (unsigned)__cvta_generic_to_shared(&recv_rj[par][pc]);
            const unsigned lm = mb0 + 8 * par;
            const double r = rj_s[pc];
            for (int d = pq; d < G; d += PG) {
                const unsigned rm = cl_map_u32(lm, d);
                st_async_f64(cl_map_u32(la, d), sum, rm);
                if (g == 0) st_async_f64(cl_map_u32(lr, d), r, rm);
            }
        }
        stamp(2);
        mbar_wait_cluster(mb0 + 8 * par, (unsigned)((j >> 1) & 1));
        stamp(3);
        // ---- 3. cluster sum in CTA order ------------------------------------
        if (tid < BB) {
            // fixed pairwise tree over 16 slots (absent CTAs contribute +0.0):
            // the same order, hence the same bits, in every CTA
            double v[PNC_MAXG];
#pragma unroll
            for (int q = 0; q < PNC_MAXG; ++q) v[q] = (q < G) ? recv[par][q][tid] : 0.0;
            const double gs = tree_sum(v), rj = recv_rj[par][tid];
            gsum[tid] = gs;
            rjv[tid] = rj;
            if (tid == j) {  // dlarfg (reading R-G7) once per CTA, from the same bits everywhere
                const double alpha = rj, xn2 = gs;
                double tau = 0.0, beta = alpha, scal = 0.0;
                if (xn2 != 0.0) {
                    const double nrm = sqrt(alpha * alpha + xn2);
                    beta = (alpha >= 0.0) ? -nrm : nrm;
                    tau = (beta - alpha) / beta;
                    scal = 1.0 / (alpha - beta);
                }
                s_hh[0] = tau;
                s_hh[1] = scal;
                scal_s[j] = scal;
                beta_s[j] = beta;
                // R11-diagonal rank stop (reading R-G12b): the same bits in every CTA
                s_stop = (beta * beta < tol2) ? 1 : 0;
            }
        }
        __syncthreads();
        if (s_stop) {  // uniform across the cluster; column j and beyond untouched
            bbo = j;
            break;
        }
        // step j+2 reuses this mbarrier (every read of recv[par] is above)
        if (tid == 0 && j + 2 < bbe) mbar_expect_tx(mb0 + 8 * par, step_bytes);
        stamp(4);
        // ---- 4. the update with this step's reflector ------------------------
        const double tau = s_hh[0], scal = s_hh[1];
        double ws[CPT];
        bool any = false;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int c = cg * CPT + k;
            ws[k] = 0.0;
            if (g == 0 && rg == 0) {
                if (c == 0) a.tau[j] = tau;
                if (c < j) a.ybuf[c + (int64_t)j * ldy] = scal_s[c] * (rjv[c] + scal * gsum[c]);
            }
            if (c > j && c < bb) {
                const double w = tau * (rjv[c] + scal * gsum[c]);
                ws[k] = w * scal;
                any = true;
                if (g == 0 && rg == 0) Rrow[j * BB + c] = rjv[c] - w;  // R(j, c): final
            }
        }
        stamp(6);
        if (any) {  // columns <= j (or >= bb) have ws = 0: a - 0 x = a exactly
            const double2 *x2 = reinterpret_cast<const double2 *>(&xs[par][rg * RPT]);
#pragma unroll
            for (int t = 0; t < RPT; t += 2) {
                const double2 u = x2[t / 2];
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    av[k][t] = fma(-ws[k], u.x, av[k][t]);
                    av[k][t + 1] = fma(-ws[k], u.y, av[k][t + 1]);
                }
            }
        }
        stamp(7);
        if (j + 1 < bbe) publish_x(j + 1, par ^ 1);
        stamp(5);
    }
    // no CTA leaves while pushes into it may be in flight
    cl_arrive_relaxed();
    cl_wait();
    __syncthreads();  // the last step's Rrow / scal / beta writes are visible

    // ---- store: A in place (columns < bb), explicit V (m' x bbpad) and V^T.
    //      Element (r, c): r < bbe, c > r: R(r, c) (Rrow); r == c < bbe: beta;
    //      c < bbe, r > c: v = scal_c x; otherwise the updated value.
    // CTA 0: the final R rows live in Rrow (= the staging buffer); take them first
    if (g == 0 && rowbase < bbo) {
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int c = cg * CPT + k;
#pragma unroll
            for (int t = 0; t < RPT; ++t) {
                const int row = rowbase + t;
                if (row < bbo && c > row && c < bb) av[k][t] = Rrow[row * BB + c];
            }
        }
    }
    if (CPT == 2) {
        // straight from registers.  Element (gr, cc): A = scal_c x below the
        // diagonal, beta_c on it, x (or the R row) above; V = scal_c x below, 1
        // on, 0 above (and 0 for unfactored columns).  V^T: the two columns of
        // a row are adjacent (one 16-byte store; a warp writes 512 contiguous
        // bytes); A and V: 16-byte stores along this thread's rows.
        const bool vo = vec_ok && ((a.ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.vfull) & 15) == 0) &&
                        rowbase + RPT <= mp;
        const int c0 = cg * CPT;
        double sc[CPT], be[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            sc[k] = (c0 + k < bbo) ? scal_s[c0 + k] : 0.0;
            be[k] = (c0 + k < bbo) ? beta_s[c0 + k] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < RPT; t += 2) {  // rows gr, gr + 1
            const int64_t gr = rowbase + t;
            double o[CPT][2], v[CPT][2];
#pragma unroll
            for (int k = 0; k < CPT; ++k)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cc = c0 + k;
                    double x = av[k][t + h], w = 0.0;
                    if (cc < bbo) {
                        if (gr + h > cc) { w = sc[k] * x; x = w; }
                        else if (gr + h == cc) { w = 1.0; x = be[k]; }
                    }
                    o[k][h] = x;
                    v[k][h] = w;
                }
            if (c0 < a.bbpad) {  // bbpad is a multiple of 8: both columns present
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (gr + h < mp)
                        *reinterpret_cast<double2 *>(a.vt + c0 + (gr + h) * ldvt) = make_double2(v[0][h], v[CPT - 1][h]);
            }
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int cc = c0 + k;
                double *dst = a.A + gr + (int64_t)cc * lda;
                double *vd = a.vfull + gr + (int64_t)cc * a.ldv;
                if (vo) {
                    if (cc < bb) *reinterpret_cast<double2 *>(dst) = make_double2(o[k][0], o[k][1]);
                    if (cc < a.bbpad) *reinterpret_cast<double2 *>(vd) = make_double2(v[k][0], v[k][1]);
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if (gr + h < mp) {
                            if (cc < bb) dst[h] = o[k][h];
                            if (cc < a.bbpad) vd[h] = v[k][h];
                        }
                }
            }
        }
    }
    for (int q = 0; q < (CPT == 2 ? 0 : RG); ++q) {
        const int64_t r0 = cta_r0 + (int64_t)q * RPT;
        __syncthreads();
        if (rg == q) {
#pragma unroll
            for (int k = 0; k < CPT; ++k)
#pragma unroll
                for (int t = 0; t < RPT; ++t) stage[(cg * CPT + k) * LDS + t] = av[k][t];
        }
        __syncthreads();
        for (int e = tid; e < BB * RPT; e += PNC_THREADS) {
            const int r = e % RPT, cc = e / RPT;
            const int64_t gr = r0 + r;
            if (gr >= mp) continue;
            const double x = stage[cc * LDS + r];
            double v = 0.0, o = x;
            if (cc < bbo) {
                if (gr > cc) { v = scal_s[cc] * x; o = v; }
                else if (gr == cc) { v = 1.0; o = beta_s[cc]; }
            }
            if (cc < bb) a.A[gr + (int64_t)cc * lda] = o;
            if (cc < a.bbpad) a.vfull[gr + (int64_t)cc * a.ldv] = v;
        }
        for (int e = tid; e < a.bbpad * RPT; e += PNC_THREADS) {
            const int cc = e % a.bbpad, r = e / a.bbpad;
            const int64_t gr = r0 + r;
            if (gr >= mp) continue;
            const double x = stage[cc * LDS + r];
            a.vt[cc + gr * ldvt] = (cc < bbo) ? (gr > cc ? scal_s[cc] * x : (gr == cc ? 1.0 : 0.0)) : 0.0;
        }
    }
    if (g == 0) {
        for (int cc = bbo + tid; cc < bb; cc += PNC_THREADS) a.tau[cc] = 0.0;
        if (tid == 0 && a.count) atomicAdd(a.count, 1);
        if (tid == 0 && a.stop_col) *a.stop_col = (bbo < bbe) ? bbo : -1;
    }
}

}  // namespace rq
