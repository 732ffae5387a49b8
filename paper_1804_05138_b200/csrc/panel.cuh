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

struct PanelArgs {
    double *A;          // &A[i + i*lda]
    int64_t lda;
    int64_t mp;         // m' rows
    int bb;             // planned panel width (columns present)
    int bbpad;
    int use_smem;       // cache own rows (rows x bb) in dynamic shared memory
    const int *bb_eff;
    double *tau;        // tau + i
    double *vfull;      // mp x bbpad, ld ldv
    int64_t ldv;
    double *vt;         // bbpad x mp, ld bbpad
    double *ybuf;       // bbpad x bbpad: y(c, j) = v_c^T v_j for c < j (strict upper of V^T V)
    double *part;       // [2][bbpad][G] partial Gram rows (column-major over CTAs)
    double *rowj;       // [2][bbpad] published row j
    unsigned *bar;      // per-launch barrier counter (zeroed by the host)
};

__global__ void __launch_bounds__(PN_THREADS) panel_qr_kernel(PanelArgs a) {
    extern __shared__ __align__(16) double pn_dyn[];
    __shared__ double w[PN_MAXB];
    __shared__ double xs[PN_MAXROWS];
    __shared__ double s_scal, s_tau, s_beta;
    const int G = gridDim.x, g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bb = a.bb;
    const int bbe = *a.bb_eff;
    const int64_t mp = a.mp;
    const int64_t rpb = (mp + G - 1) / G;
    const int64_t r_lo = min(mp, (int64_t)g * rpb), r_hi = min(mp, r_lo + rpb);
    const int nrows = (int)(r_hi - r_lo);
    const int64_t lda = a.lda;
    unsigned epoch = 0;

    // P(r, c) = A(r_lo + r, c): shared-memory copy or the panel itself
    double *P;
    int64_t ldp;
    if (a.use_smem) {
        P = pn_dyn;
        ldp = nrows;
        for (int c = warp; c < bb; c += PN_WARPS)
            for (int r = lane; r < nrows; r += 32) P[r + (int64_t)c * ldp] = a.A[r_lo + r + c * lda];
        __syncthreads();
    } else {
        P = a.A + r_lo;
        ldp = lda;
    }

    for (int j = 0; j < bbe; ++j) {
        const int par = j & 1;
        const int rj = (int)(j - r_lo);  // local index of row j (may be out of range)
        // ---- partial Gram row over own rows r > j -----------------------
        const int rs = max(0, rj + 1);
        for (int c = warp; c < bb; c += PN_WARPS) {
            double s = 0.0;
            for (int r = rs + lane; r < nrows; r += 32) s += P[r + (int64_t)c * ldp] * P[r + (int64_t)j * ldp];
            s = warp_sum(s);
            if (lane == 0) a.part[((int64_t)par * a.bbpad + c) * G + g] = s;
        }
        if (rj >= 0 && rj < nrows)
            for (int c = tid; c < bb; c += PN_THREADS) a.rowj[par * a.bbpad + c] = P[rj + (int64_t)c * ldp];
        grid_barrier(a.bar, G, epoch);
        // ---- reduce the G partials (warp per column, fixed order) ----------
        // (loads of up to 4 columns x 5 partials per lane issued before any add)
        for (int c0 = warp; c0 < bb; c0 += 4 * PN_WARPS) {
            double v[4][5];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int c = c0 + cc * PN_WARPS;
                const double *pc = a.part + ((int64_t)par * a.bbpad + c) * G;
#pragma unroll
                for (int u = 0; u < 5; ++u) {
                    const int q = lane + 32 * u;
                    v[cc][u] = (c < bb && q < G) ? ld_cg(pc + q) : 0.0;
                }
            }
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                double s = v[cc][0] + v[cc][1] + v[cc][2] + v[cc][3] + v[cc][4];
                s = warp_sum(s);
                const int c = c0 + cc * PN_WARPS;
                if (lane == 0 && c < bb) w[c] = s;
            }
        }
        __syncthreads();
        if (tid == 0) {
            const double alpha = ld_cg(a.rowj + par * a.bbpad + j);
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
        // CTA 0 records y_c = v_c^T v_j = A(j,c) + scal g_c (c < j): column j of
        // strict_upper(V^T V), from which tri_kernel builds T off the critical path
        if (g == 0)
            for (int c = tid; c < j; c += PN_THREADS)
                a.ybuf[c + (int64_t)j * a.bbpad] = ld_cg(a.rowj + par * a.bbpad + c) + scal * w[c];
        // w_c = tau * (a_jc + scal g_c) for c > j
        for (int c = j + 1 + tid; c < bb; c += PN_THREADS) w[c] = tau * (ld_cg(a.rowj + par * a.bbpad + c) + scal * w[c]);
        for (int r = tid; r < nrows; r += PN_THREADS) xs[r] = P[r + (int64_t)j * ldp];
        __syncthreads();
        // ---- update own rows ---------------------------------------------
        if (tau != 0.0) {
            for (int c = j + 1 + warp; c < bb; c += PN_WARPS) {
                const double wc = w[c];
                for (int r = lane; r < nrows; r += 32) {
                    if (r > rj) P[r + (int64_t)c * ldp] -= wc * (scal * xs[r]);
                    else if (r == rj) P[r + (int64_t)c * ldp] -= wc;
                }
            }
            for (int r = tid; r < nrows; r += PN_THREADS) {
                if (r > rj) P[r + (int64_t)j * ldp] = scal * xs[r];
                else if (r == rj) P[r + (int64_t)j * ldp] = s_beta;
            }
        }
        __syncthreads();
    }
    // ---- write back, explicit V / V^T, zero tails (rank stop) -----------
    if (a.use_smem) {
        for (int c = warp; c < bb; c += PN_WARPS)
            for (int r = lane; r < nrows; r += 32) a.A[r_lo + r + c * lda] = P[r + (int64_t)c * ldp];
    }
    for (int r = warp; r < nrows; r += PN_WARPS) {
        const int64_t gr = r_lo + r;
        for (int c = lane; c < a.bbpad; c += 32) {
            double v = 0.0;
            if (c < bbe) v = (gr > c) ? P[r + (int64_t)c * ldp] : (gr == c ? 1.0 : 0.0);
            a.vt[c + gr * a.bbpad] = v;
        }
    }
    for (int c = warp; c < a.bbpad; c += PN_WARPS)
        for (int r = lane; r < nrows; r += 32) {
            const int64_t gr = r_lo + r;
            double v = 0.0;
            if (c < bbe) v = (gr > c) ? P[r + (int64_t)c * ldp] : (gr == c ? 1.0 : 0.0);
            a.vfull[gr + c * a.ldv] = v;
        }
    if (g == 0)
        for (int c = bbe + tid; c < bb; c += PN_THREADS) a.tau[c] = 0.0;
}

}  // namespace rq
