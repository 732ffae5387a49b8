// panel.cuh -- S4 (kernel K6): unpivoted Householder QR of the panel
// A(i:m, i:i+bb) (Alg. 2 line P:149, PDGEQRF at P:760) with the compact-WY
// inputs of the compact-WY factor T (PDLARFT) gathered in the same
// pass: H_0 ... H_{bb-1} = I - V T V^T with T(j,j) = tau_j,
// T(0:j, j) = -tau_j T(0:j, 0:j) (V(:,0:j)^T v_j); the V^T v_j columns are
// recorded here and T itself is built by tri_kernel (tri.cuh).
//
// One persistent cooperative kernel; CTA g owns a contiguous block of panel
// rows, cached in shared memory when it fits (the panel is then read from
// and written to HBM exactly once); one grid barrier per column.  At step j
// each CTA writes the partial Gram row  g_c = sum_{r > j, r owned} A(r,c) A(r,j)
// for every panel column c (c > j: v_j^T a_c up to scaling; c = j: ||x||^2
// below the diagonal; c < j: V(:,c)^T x, which gives T's column j), and the
// owner of row j publishes that row.  After the barrier every CTA reduces
// the G partials (warp per column, fixed butterfly: identical bits in every
// CTA), forms beta, tau, v = x/(alpha - beta) (dlarfg, reading R-G7) and
// w_c = tau (a_jc + g_c/(alpha - beta)), and updates its own rows:
// a_rc -= w_c v_r.  Columns bb_eff..bb-1 of the panel (rank stop, R-G12)
// still receive the reflectors.
// Outputs: V below the diagonal and R11 on/above it, in place; tau; the
// explicit V (Vfull, m' x bbpad: unit diagonal, zeros above, K-contiguous for
// W = V^T A22) and its transpose Vt (bbpad x m', for A22 += V W2); ybuf.
#pragma once
#include "common.cuh"

namespace rq {

constexpr int PN_THREADS = 256;
constexpr int PN_WARPS = PN_THREADS / 32;
constexpr int PN_MAXB = 128;
constexpr int PN_MAXROWS = 1024;  // rows per CTA (x staging buffer)
constexpr int PN_MAXG = 152;      // CTAs of the cooperative grid (<= one per SM)
constexpr int PN_RMAX = (PN_MAXG + PN_WARPS - 1) / PN_WARPS;  // partial rows summed per warp

struct PanelArgs {
    double *A;          // &A[i + i*lda]
    int64_t lda;
    int64_t mp;         // m' rows
    int bb;             // planned panel width (columns present)
    int bbpad;
    const int *skip;    // non-null and *skip == 0: the CholeskyQR2 path (cqr.cuh) already factored the panel
    int *count;         // incremented (CTA 0) when this kernel factors the panel
    int nsm;            // rows per CTA cached in dynamic shared memory (grid kernel)
    const int *bb_eff;
    double *tau;        // tau + i
    double *vfull;      // mp x bbpad, ld ldv
    int64_t ldv;
    double *vt;         // bbpad x mp, ld bbpad
    double *ybuf;       // bbpad x bbpad: y(c, j) = v_c^T v_j for c < j (strict upper of V^T V)
    double *part;       // [2][G][bbpad] partial Gram rows (one contiguous row per CTA)
    double *rowj;       // [2][bbpad] published row j
    unsigned *bar;      // per-launch barrier counter (zeroed by the host)
    int col0;           // blocked panel: this launch factors panel columns col0.. (bb_eff is the panel's)
    int64_t ldvt;       // leading dimension of vt (0: bbpad)
    int64_t ldy;        // leading dimension of ybuf (0: bbpad)
    const double *tol2; // R11-diagonal rank stop (reading R-G12b): stop at the first column whose
                        // beta^2 < *tol2 (= (1e3 eps)^2 ||panel||_F^2); nullptr: no check
    int *stop_col;      // out: that column (-1 when none); written by CTA 0
    unsigned long long *trace;  // debug: [2 CTAs][64 steps][8 phases] clock64 stamps, or nullptr
};

// CB: panel columns per warp batch of the partial Gram row (8; 4 for the
// 32-column sub-panels of the blocked panel, so all 8 warps have columns)
template <int CB>
__global__ void __launch_bounds__(PN_THREADS) panel_qr_kernel(PanelArgs a) {
    constexpr int NU = (CB == 4) ? 1 : PN_MAXB / 32;  // 32-column groups of the reduce (bb <= 32 for CB 4)
    extern __shared__ __align__(16) double pn_dyn[];
    __shared__ double w[PN_MAXB], rjs[PN_MAXB];
    __shared__ double wred[PN_WARPS][PN_MAXB];
    __shared__ double s_scal, s_tau, s_beta;
    __shared__ int s_stop;
    if (a.skip && *a.skip == 0) return;
    const int G = gridDim.x, g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bb = a.bb;
    const int bbe = min(bb, max(0, *a.bb_eff - a.col0));
    const int64_t ldvt = a.ldvt ? a.ldvt : a.bbpad, ldy = a.ldy ? a.ldy : a.bbpad;
    const int64_t mp = a.mp;
    const int64_t rpb = (mp + G - 1) / G;
    const int64_t r_lo = min(mp, (int64_t)g * rpb), r_hi = min(mp, r_lo + rpb);
    const int nrows = (int)(r_hi - r_lo);
    const int64_t lda = a.lda;
    unsigned epoch = 0;

    // rows [0, nsm) of this CTA's block live in shared memory (Ps, ld nsm),
    // rows [nsm, nrows) stay in the panel itself (L2 / HBM)
    const int nsm = min(nrows, a.nsm);
    double *Ps = pn_dyn;
    const int64_t lds = nsm > 0 ? nsm : 1;
    double *Pg = a.A + r_lo;
    for (int c = warp; c < bb; c += PN_WARPS)
        for (int r = lane; r < nsm; r += 32) Ps[r + (int64_t)c * lds] = Pg[r + c * lda];
    __syncthreads();
    auto Pv = [&](int r, int c) -> double { return (r < nsm) ? Ps[r + (int64_t)c * lds] : Pg[r + (int64_t)c * lda]; };
    const int tsel = (g == 0) ? 0 : (g == G - 1 ? 1 : -1);
    const double tol2 = a.tol2 ? *a.tol2 : -1.0;
    int bbo = bbe;  // columns factored (bbe, or the R11-diagonal stop column)
    for (int j = 0; j < bbe; ++j) {
        auto stamp = [&](int ph) {
            if (a.trace && tsel >= 0 && tid == 0 && j < 64) a.trace[((size_t)tsel * 64 + j) * 8 + ph] = clock64();
        };
        stamp(0);
        const int par = j & 1;
        const int rj = (int)(j - r_lo);  // local index of row j (may be out of range)
        const int rs = max(0, rj + 1);
        // ---- partial Gram row over own rows r > j: thread per row, 32 columns
        //      per pass in registers, then a butterfly reduce-scatter inside the
        //      warp (lane l ends with column 32 q + l) and the 8 warp sums in
        //      warp order (one fixed order) ------------------------------------
        for (int q = 0; q * 32 < bb; ++q) {
            double acc[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) acc[u] = 0.0;
            const int cb = min(32, bb - 32 * q);
            for (int r = rs + tid; r < nrows; r += PN_THREADS) {
                const double xr = Pv(r, j);
                // one running pointer (no 32 precomputed 64-bit addresses: the
                // kernel sits at the register limit)
                const bool sm = r < nsm;
                const int64_t ld = sm ? lds : lda;
                const double *pr = sm ? Ps + r + (int64_t)(32 * q) * lds : Pg + r + (int64_t)(32 * q) * lda;
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    if (u < cb) acc[u] += *pr * xr;
                    pr += ld;
                }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int u = 0; u < o; ++u) {
                    const double send = up ? acc[u] : acc[u + o];
                    const double keep = up ? acc[u + o] : acc[u];
                    acc[u] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            wred[warp][32 * q + lane] = acc[0];
        }
        __syncthreads();
        for (int c = tid; c < bb; c += PN_THREADS) {
            double v = 0.0;
#pragma unroll
            for (int ww = 0; ww < PN_WARPS; ++ww) v += wred[ww][c];
            a.part[((int64_t)par * G + g) * a.bbpad + c] = v;
        }
        if (rj >= 0 && rj < nrows)
            for (int c = tid; c < bb; c += PN_THREADS) a.rowj[par * a.bbpad + c] = Pv(rj, c);
        stamp(1);
        grid_barrier(a.bar, G, epoch);
        stamp(2);
        // ---- reduce the G partial rows (each CTA's row contiguous, coalesced
        //      reads; warp w sums rows g = w, w+8, ... in order, then the 8 warp
        //      sums are added in warp order: one fixed order in every CTA) ------
        {
            // every load of this warp's rows (g = warp + 8 h) in flight at once:
            // one L2 round trip instead of one per batch of four rows
            const double *pp = a.part + (int64_t)par * G * a.bbpad;
            const int nu = (bb + 31) >> 5;
            double acc[NU];
#pragma unroll
            for (int u = 0; u < NU; ++u) acc[u] = 0.0;
            double v[PN_RMAX][NU];
#pragma unroll
            for (int h = 0; h < PN_RMAX; ++h) {
                const int gg = warp + h * PN_WARPS;
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    const int c = lane + 32 * u;
                    v[h][u] = (u < nu && gg < G && c < bb) ? ld_cg(pp + (int64_t)gg * a.bbpad + c) : 0.0;
                }
            }
#pragma unroll
            for (int h = 0; h < PN_RMAX; ++h)
#pragma unroll
                for (int u = 0; u < NU; ++u) acc[u] += v[h][u];
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                const int c = lane + 32 * u;
                if (c < bb) wred[warp][c] = acc[u];
            }
        }
        if (warp == PN_WARPS - 1)
            for (int c = lane; c < bb; c += 32) rjs[c] = ld_cg(a.rowj + par * a.bbpad + c);
        __syncthreads();
        for (int c = tid; c < bb; c += PN_THREADS) {
            double sacc = 0.0;
#pragma unroll
            for (int ww = 0; ww < PN_WARPS; ++ww) sacc += wred[ww][c];
            w[c] = sacc;
        }
        __syncthreads();
        stamp(3);
        if (tid == 0) {
            const double alpha = rjs[j];
            const double xn2 = w[j];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (xn2 != 0.0) {
                const double nrm = sqrt(alpha * alpha + xn2);
                beta = (alpha >= 0.0) ? -nrm : nrm;
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            // R11-diagonal rank stop: |R(j,j)| = |beta| below 1e3 eps ||panel||_F
            // (every CTA evaluates the same bits: a uniform decision)
            const int stop = (beta * beta < tol2) ? 1 : 0;
            s_stop = stop;
            s_tau = tau; s_beta = beta; s_scal = scal;
            if (g == 0) a.tau[j] = stop ? 0.0 : tau;
        }
        __syncthreads();
        if (s_stop) {  // column j and beyond stay as they are (tau = 0)
            bbo = j;
            break;
        }
        const double tau = s_tau, scal = s_scal;
        // CTA 0 records y_c = v_c^T v_j = A(j,c) + scal g_c (c < j): column j of
        // strict_upper(V^T V), from which tri_kernel builds T off the critical path
        if (g == 0)
            for (int c = tid; c < j; c += PN_THREADS) a.ybuf[c + (int64_t)j * ldy] = rjs[c] + scal * w[c];
        // w_c = tau * (a_jc + scal g_c) for c > j
        for (int c = j + 1 + tid; c < bb; c += PN_THREADS) w[c] = tau * (rjs[c] + scal * w[c]);
        __syncthreads();
        stamp(4);
        // ---- update own rows: thread per row (the row's x_r read first; no
        //      other thread touches the row) -----------------------------------
        if (tau != 0.0) {
            const double beta = s_beta;
            for (int r = max(rj, 0) + tid; r < nrows; r += PN_THREADS) {
                const double xr = Pv(r, j);
                const double vr = (r > rj) ? scal * xr : 1.0;
                if (r < nsm) {
                    double *pr = Ps + r;
#pragma unroll 8
                    for (int c = j + 1; c < bb; ++c) pr[(int64_t)c * lds] -= w[c] * vr;
                    pr[(int64_t)j * lds] = (r > rj) ? vr : beta;
                } else {
                    double *pr = Pg + r;
#pragma unroll 8
                    for (int c = j + 1; c < bb; ++c) pr[(int64_t)c * lda] -= w[c] * vr;
                    pr[(int64_t)j * lda] = (r > rj) ? vr : beta;
                }
            }
        }
        __syncthreads();
        stamp(5);
    }
    // ---- write back, explicit V / V^T, zero tails (rank stop) -----------
    for (int c = warp; c < bb; c += PN_WARPS)
        for (int r = lane; r < nsm; r += 32) Pg[r + c * lda] = Ps[r + (int64_t)c * lds];
    __syncthreads();
    for (int r = warp; r < nrows; r += PN_WARPS) {
        const int64_t gr = r_lo + r;
        for (int c = lane; c < a.bbpad; c += 32) {
            double v = 0.0;
            if (c < bbo) v = (gr > c) ? Pg[r + (int64_t)c * lda] : (gr == c ? 1.0 : 0.0);
            a.vt[c + gr * ldvt] = v;
        }
    }
    for (int c = warp; c < a.bbpad; c += PN_WARPS)
        for (int r = lane; r < nrows; r += 32) {
            const int64_t gr = r_lo + r;
            double v = 0.0;
            if (c < bbo) v = (gr > c) ? Pg[r + (int64_t)c * lda] : (gr == c ? 1.0 : 0.0);
            a.vfull[gr + c * a.ldv] = v;
        }
    if (g == 0)
        for (int c = bbo + tid; c < bb; c += PN_THREADS) a.tau[c] = 0.0;
    if (g == 0 && tid == 0 && a.count) atomicAdd(a.count, 1);
    if (g == 0 && tid == 0 && a.stop_col) *a.stop_col = (bbo < bbe) ? bbo : -1;
}

}  // namespace rq
