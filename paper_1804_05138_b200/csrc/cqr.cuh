// cqr.cuh -- S4 panel factorization with a constant number of device-wide
// steps (the paper's future-work item "TSQR for the panel", realised
// as a communication-avoiding tall-skinny QR): CholeskyQR2 followed by
// Householder reconstruction, so the outputs keep the Householder contract of
// Alg. 2 line P:149 / PDGEQRF+PDLARFT: V unit lower trapezoidal
// below the diagonal, tau, R11 (and the compact-WY T) -- no per-column
// device-wide exchange.
//
//   G1 = P^T P                        (DMMA Gram GEMM, host-dispatched)
//   R1 = chol(G1), Q1 = P R1^{-1}     (cqr_chol_kernel, cqr_rowmul_kernel)
//   G2 = Q1^T Q1, R2 = chol(G2), Q = Q1 R2^{-1}, Rc = R2 R1    (CholeskyQR2)
//   modified LU without pivoting of the top block (Ballard et al.,
//   "Reconstructing Householder vectors from TSQR"):  S - Qtop = L U with
//   the sign S_jj = sign of the Schur pivot (|pivot| >= 1), then
//   V = [L; -Qbottom U^{-1}],  T = (U S) L^{-T},  tau_j = T_jj,  R = S Rc
//   (cqr_recon_kernel, cqr_rowmul_kernel).
// With this sign choice R_jj = -sign(alpha_j) |R_jj| as LAPACK dlarfg's
// beta (reading R-G7).
//
// The bb x bb factorizations run in one CTA with the matrix entries held in
// registers (a fixed set per thread) and one __syncthreads per column: the
// owners of row (and column) j+1 publish it to shared memory during step j.
// The triangular inverses are block-recursive doublings in shared memory, and
// the m' x bb products with them run on the FP64 tensor cores (DMMA).
//
// Guard: CholeskyQR2 is accurate when kappa(P) is well below u^{-1/2}.  The
// first Cholesky must succeed with a diagonal ratio <= CQR_MAX_DIAG_RATIO and
// the second Gram must satisfy max|G2 - I| <= CQR_MAX_ORTH_ERR; the panel must
// not be rank-stopped (bb_eff == bb).  Otherwise *status = 1 and nothing in A
// is written: the column-by-column Householder kernel (panel.cuh) runs
// instead (it reads *status and is a no-op when the CholeskyQR path succeeded).
#pragma once
#include "common.cuh"

namespace rq {

constexpr int CQR_THREADS = 256;
// debug: phase stamps (clock64) of cqr_chol_kernel / cqr_recon_kernel, set by tools only
__device__ unsigned long long *g_cqr_dbg = nullptr;
RQ_DEV void cqr_stamp(int ph) {
    if (g_cqr_dbg && threadIdx.x == 0) g_cqr_dbg[ph] = clock64();
}
constexpr double CQR_MAX_DIAG_RATIO = 1e5;
constexpr double CQR_MAX_ORTH_ERR = 1e-4;
constexpr int CQR_MAXB = 128;
constexpr int CQR_EPT_U = (CQR_MAXB * (CQR_MAXB + 1) / 2 + CQR_THREADS - 1) / CQR_THREADS;  // 33
constexpr int CQR_EPT_F = (CQR_MAXB * CQR_MAXB + CQR_THREADS - 1) / CQR_THREADS;            // 64

// ---------------------------------------------------------------------------
// In-place inverse of an upper-triangular nb x nb matrix in shared memory
// (nb = 8 * 2^k, ld nb; identity padding beyond the live size) by
// block-recursive doubling: invert the 8x8 diagonal blocks, then
// B <- -A^{-1} B D^{-1} for the off-diagonal block of every 2s x 2s block.
// tmp: nb^2/4 doubles (nb/(2s) blocks of s^2 per level).  All threads of the
// CTA must call it.
// ---------------------------------------------------------------------------
RQ_DEV void tri_inv_upper_smem(double *M, int nb, double *tmp) {
    const int ld = nb, tid = threadIdx.x;
    // base: 8x8 diagonal blocks, one warp each (lane = column of the block,
    // back substitution down the rows; 8 lanes active)
    {
        const int warp = tid >> 5, lane = tid & 31;
        for (int blk = warp; blk < nb / 8; blk += CQR_THREADS / 32) {
            const int k0 = blk * 8;
            if (lane < 8) {
                const int c = lane;
                double x[8];
#pragma unroll
                for (int r = 7; r >= 0; --r) {
                    double s = (r == c) ? 1.0 : 0.0;
#pragma unroll
                    for (int q = r + 1; q < 8; ++q) s -= M[(k0 + r) + (k0 + q) * ld] * x[q];
                    x[r] = (r <= c) ? s / M[(k0 + r) + (k0 + r) * ld] : 0.0;
                }
                __syncwarp(0xffu);
#pragma unroll
                for (int r = 0; r < 8; ++r) M[(k0 + r) + (k0 + c) * ld] = x[r];
            }
        }
    }
    __syncthreads();
    // levels: every thread owns up to TI_E elements (r, c, block k) of the
    // nblk s x s off-diagonal blocks; q-outer loops keep TI_E independent
    // accumulators in flight
    constexpr int TI_E = 8;
    for (int s = 8; s < nb; s *= 2) {
        const int ls = __ffs(s) - 1;
        const int nblk = nb / (2 * s);
        const int ne = nblk * s * s;  // <= nb^2 / 4 = 4096 for nb = 128 -> <= 16 per thread
        for (int e0 = 0; e0 < ne; e0 += TI_E * CQR_THREADS) {
            // tmp_k = A_k^{-1} B_k  (A^{-1} upper, already inverted)
            double acc[TI_E];
            int rr[TI_E], cc[TI_E], kk[TI_E];
#pragma unroll
            for (int u = 0; u < TI_E; ++u) {
                const int e = e0 + u * CQR_THREADS + tid;
                rr[u] = e & (s - 1);
                cc[u] = (e >> ls) & (s - 1);
                kk[u] = (e < ne) ? (e >> (2 * ls)) * 2 * s : -1;
                acc[u] = 0.0;
            }
            for (int q = 0; q < s; ++q) {
                double av[TI_E], bv[TI_E];
#pragma unroll
                for (int u = 0; u < TI_E; ++u) {
                    const int k = kk[u] < 0 ? 0 : kk[u];
                    av[u] = M[(k + rr[u]) + (k + q) * ld];
                    bv[u] = M[(k + q) + (k + s + cc[u]) * ld];
                }
#pragma unroll
                for (int u = 0; u < TI_E; ++u)
                    if (q >= rr[u]) acc[u] += av[u] * bv[u];
            }
#pragma unroll
            for (int u = 0; u < TI_E; ++u) {
                const int e = e0 + u * CQR_THREADS + tid;
                if (e < ne) tmp[e] = acc[u];
            }
        }
        __syncthreads();
        for (int e0 = 0; e0 < ne; e0 += TI_E * CQR_THREADS) {
            // B_k = -tmp_k D_k^{-1}  (D^{-1} upper, already inverted)
            double acc[TI_E];
            int rr[TI_E], cc[TI_E], kb[TI_E];
#pragma unroll
            for (int u = 0; u < TI_E; ++u) {
                const int e = e0 + u * CQR_THREADS + tid;
                rr[u] = e & (s - 1);
                cc[u] = (e >> ls) & (s - 1);
                kb[u] = (e < ne) ? (e >> (2 * ls)) : -1;
                acc[u] = 0.0;
            }
            for (int q = 0; q < s; ++q) {
                double tv[TI_E], dv[TI_E];
#pragma unroll
                for (int u = 0; u < TI_E; ++u) {
                    const int b = kb[u] < 0 ? 0 : kb[u], k = b * 2 * s;
                    tv[u] = tmp[b * s * s + rr[u] + (q << ls)];
                    dv[u] = M[(k + s + q) + (k + s + cc[u]) * ld];
                }
#pragma unroll
                for (int u = 0; u < TI_E; ++u)
                    if (q <= cc[u]) acc[u] += tv[u] * dv[u];
            }
#pragma unroll
            for (int u = 0; u < TI_E; ++u) {
                const int k = kb[u] * 2 * s;
                if (kb[u] >= 0) M[(k + rr[u]) + (k + s + cc[u]) * ld] = -acc[u];
            }
        }
        __syncthreads();
    }
}

// 1/d to ~1 ulp: hardware approximation + two Newton steps (no division
// subroutine on the critical path of the per-column steps)
RQ_DEV double fast_rcp(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}

// packed upper-triangle index e -> (a, c), a <= c, e = c (c + 1) / 2 + a
RQ_DEV void upper_index(int e, int &a, int &c) {
    int cc = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
    while (cc * (cc + 1) / 2 > e) --cc;
    while ((cc + 1) * (cc + 2) / 2 <= e) ++cc;
    c = cc;
    a = e - cc * (cc + 1) / 2;
}

// ---------------------------------------------------------------------------
// Cholesky of the bb x bb Gram matrix (pass 1: G1 = P^T P; pass 2: G2 =
// Q1^T Q1 with the orthogonality check), the accumulated R factor and the
// inverse of this pass's R.  One CTA.  The upper triangle is held in
// registers (element e = tid + 256 i of the packed triangle); step j applies
// M(a,c) -= M(j,a) M(j,c) / M(j,j) to the elements with a > j, using row j
// from shared memory, and the owners of row j+1 publish it for step j+1.
// Outputs (ld bbpad, zero padding): Rc = R (pass 1) or R Rc (pass 2); Rinv.
// smem: nb^2 + (nb/2)^2 doubles, nb = 8 * 2^k >= bb.
// ---------------------------------------------------------------------------
template <int EPT>
__global__ void __launch_bounds__(CQR_THREADS, 1) cqr_chol_kernel(const double *G /* bbpad x bbpad */, int bb, int bbpad,
                                                               int nb, int pass, const int *bb_eff, int *status,
                                                               double *Rc, double *Rinv, const double *tol2) {
    extern __shared__ __align__(16) double cq_sm[];
    double *M = cq_sm;              // nb x nb (R, then R^{-1})
    double *tmp = cq_sm + nb * nb;  // (nb/2)^2
    __shared__ double rowb[2][CQR_MAXB];
    __shared__ double s_d[CQR_MAXB];
    __shared__ double s_idl[2];
    __shared__ int s_fail;
    __shared__ double s_red[CQR_THREADS / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (pass == 1) {
        if (tid == 0) *status = (*bb_eff == bb) ? 0 : 1;
        __syncthreads();
    }
    if (*status != 0) return;
    cqr_stamp(0);
    const int ne = bb * (bb + 1) / 2;
    double v[EPT];
    int ea[EPT], ec[EPT];  // element (a, c), a <= c; a = -1: no element
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int e = tid + CQR_THREADS * i;
        int a = 0, c = 0;
        if (e < ne) upper_index(e, a, c);
        ea[i] = (e < ne) ? a : -1;
        ec[i] = c;
        v[i] = (e < ne) ? G[a + (int64_t)c * bbpad] : 0.0;
        if (e < ne) mx = fmax(mx, fabs(v[i] - (a == c ? 1.0 : 0.0)));
        if (e < ne && a == 0) rowb[0][c] = v[i];
    }
    for (int j = tid; j < CQR_MAXB; j += CQR_THREADS) s_d[j] = 0.0;
    if (pass == 2) {  // max |G2 - I| over the upper triangle
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) s_red[warp] = mx;
    }
    __syncthreads();
    if (pass == 2) {
        double m2 = 0.0;
        for (int w = 0; w < CQR_THREADS / 32; ++w) m2 = fmax(m2, s_red[w]);
        if (!(m2 <= CQR_MAX_ORTH_ERR)) {
            if (tid == 0) *status = 1;
            return;
        }
    }
    cqr_stamp(1);
    // step j: M(a,c) -= M(j,a) M(j,c) / M(j,j) for a > j; the owners of row
    // j+1 publish it, the owner of (j+1, j+1) also 1/M(j+1,j+1) (or a failure)
    if (tid == 0) {
        const double d0 = rowb[0][0];
        s_d[0] = d0;
        s_idl[0] = fast_rcp(d0);
        s_fail = !(d0 > 0.0);
    }
    __syncthreads();
    // (a failed pivot only poisons the remaining entries; checked after the loop)
    for (int j = 0; j < bb; ++j) {
        const double *rj = rowb[j & 1];
        double *rn = rowb[(j + 1) & 1];
        const double idl = s_idl[j & 1];
        // all loads first (the stores below may alias them for the compiler),
        // then the updates, then the publication of row j+1
        double ra[EPT], rc[EPT];
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            ra[i] = rj[ea[i] > 0 ? ea[i] : 0];
            rc[i] = rj[ec[i]];
        }
#pragma unroll
        for (int i = 0; i < EPT; ++i) v[i] -= (ea[i] > j) ? ra[i] * rc[i] * idl : 0.0;
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if (ea[i] == j + 1) rn[ec[i]] = v[i];
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if (ea[i] == j + 1 && ec[i] == j + 1) {  // next pivot (one thread)
                s_d[j + 1] = v[i];
                s_idl[(j + 1) & 1] = fast_rcp(v[i]);
                if (!(v[i] > 0.0)) s_fail = 1;
            }
        __syncthreads();
    }
    __syncthreads();
    cqr_stamp(2);
    // a failed (non-positive / NaN) pivot leaves s_fail set and s_d short
    {
        double dmax = 0.0, dmin = 1e308;
        bool ok = !s_fail;
        // a diagonal below the R11-diagonal stop threshold (reading R-G12b)
        // declines: the column-by-column kernel then stops at that column
        const double t2 = (pass == 1 && tol2) ? *tol2 : -1.0;
        for (int j = 0; j < bb; ++j) {
            const double dj = s_d[j];
            ok = ok && (dj > 0.0) && !(dj < t2);
            dmax = fmax(dmax, dj);
            dmin = fmin(dmin, dj);
        }
        // diag(R) = sqrt(d): ratio check on R (pass 1)
        if (!ok || (pass == 1 && !(dmax <= CQR_MAX_DIAG_RATIO * CQR_MAX_DIAG_RATIO * dmin))) {
            if (tid == 0) *status = 1;
            return;
        }
    }
    // R(a, c) = M(a, c) / sqrt(d_a) into smem (upper; identity padding)
    for (int e = tid; e < nb * nb; e += CQR_THREADS) {
        const int r = e % nb, c = e / nb;
        M[e] = (r >= bb || c >= bb) ? (r == c ? 1.0 : 0.0) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int a = ea[i], c = ec[i];
        if (a >= 0) M[a + c * nb] = (a == c) ? sqrt(s_d[a]) : v[i] / sqrt(s_d[a]);
    }
    __syncthreads();
    // Rc = R (pass 1) or R Rc_old (pass 2; staged in Rinv)
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int a = ea[i], c = ec[i];
        if (a < 0) continue;
        double acc;
        if (pass == 1) acc = M[a + c * nb];
        else {
            acc = 0.0;
            for (int q = a; q <= c; ++q) acc += M[a + q * nb] * Rc[q + (int64_t)c * bbpad];
        }
        Rinv[a + (int64_t)c * bbpad] = acc;
    }
    __syncthreads();
    for (int c = warp; c < bbpad; c += CQR_THREADS / 32)
        for (int r = lane; r < bbpad; r += 32)
            Rc[r + (int64_t)c * bbpad] = (r < bb && c < bb && r <= c) ? Rinv[r + (int64_t)c * bbpad] : 0.0;
    cqr_stamp(3);
    tri_inv_upper_smem(M, nb, tmp);
    __syncthreads();
    cqr_stamp(4);
    for (int c = warp; c < bbpad; c += CQR_THREADS / 32)
        for (int r = lane; r < bbpad; r += 32) Rinv[r + (int64_t)c * bbpad] = (r < bb && c < bb) ? M[r + c * nb] : 0.0;
}

// ---------------------------------------------------------------------------
// Y(r, :) = s X(r, :) R for rows r in [r0, rows), R bbpad x bbpad (entries
// with row or column >= bb are zero), on the FP64 tensor cores: each warp
// owns 16 rows and all bbpad columns (mma.sync m8n8k4, A fragments from X in
// global memory, B fragments from R in shared memory with a row stride = 4 mod
// 16 doubles: conflict-free).  In place allowed (a warp reads all its rows'
// entries before it writes).  Columns bb..bbpad-1 of Y are written as 0.
// mode 1 (V2 of the reconstruction): also A(r, c) = Y(r, c) (the panel below
// the top block) and Vt(c, r) = Y(r, c).  No-op when *status != 0.
// ---------------------------------------------------------------------------
constexpr int RM_ROWS = 16;  // rows per warp (2 m8 tiles)
__global__ void __launch_bounds__(CQR_THREADS, 1) cqr_rowmul_kernel(const double *X, int64_t ldx, int64_t r0, int64_t rows,
                                                                 int bb, int bbpad, const double *R, double s,
                                                                 double *Y, int64_t ldy, const int *status, int mode,
                                                                 double *A, int64_t lda, double *vt) {
    extern __shared__ __align__(16) double rm_sm[];  // bbpad x (bbpad + pad)
    if (*status != 0) return;
    const int ldr = bbpad + 4;  // bbpad is a multiple of 8: ldr = 4 or 12 mod 16
    for (int e = threadIdx.x; e < bbpad * bbpad; e += blockDim.x) {
        const int k = e % bbpad, c = e / bbpad;
        rm_sm[k + c * ldr] = R[k + (int64_t)c * bbpad];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t rbase = r0 + ((int64_t)blockIdx.x * (CQR_THREADS / 32) + warp) * RM_ROWS;
    if (rbase >= rows) return;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[2][16][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const int NT = bbpad / 8;
    // all A fragments of this warp's rows first (one round trip), then the MMAs
    double af[2][CQR_MAXB / 4];
#pragma unroll
    for (int kk = 0; kk < CQR_MAXB / 4; ++kk) {
        const int k = kk * 4 + fk;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const int64_t r = rbase + mt * 8 + fr;
            af[mt][kk] = (kk * 4 < bbpad && r < rows && k < bb) ? X[r + (int64_t)k * ldx] : 0.0;
        }
    }
#pragma unroll
    for (int kk = 0; kk < CQR_MAXB / 4; ++kk) {
        if (kk * 4 >= bbpad) break;
        const int k = kk * 4 + fk;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            if (nt < NT) {
                const double b = rm_sm[k + (nt * 8 + fr) * ldr];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt][kk], b);
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
        const int64_t r = rbase + mt * 8 + fr;
        if (r >= rows) continue;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            if (nt >= NT) continue;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int c = nt * 8 + 2 * fk + hh;
                const double y = (c < bb) ? s * acc[mt][nt][hh] : 0.0;
                Y[r + (int64_t)c * ldy] = y;
                if (mode == 1) {
                    if (c < bb) A[r + (int64_t)c * lda] = y;
                    vt[c + r * bbpad] = y;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Householder reconstruction of the top bb x bb block (one CTA):
//   X = -Q(0:bb, 0:bb); for j: S_j = sign(X_jj) (1 if 0); pivot X_jj + S_j;
//   L(:, j) = X(j+1:, j) / pivot; Schur update  ->  S - Qtop = L U.
// The entries live in registers (element e = tid + 256 i, row-major index
// (e / bb, e mod bb)); row and column j+1 are published during step j.
//   T = (U S) L^{-T}, tau_j = T_jj, R = S Rc, U^{-1} (for V2 = -Qbottom U^{-1}).
// Writes: the top block of the panel in A (L strictly below, R on/above), the
// top bb rows of Vfull (after reading Q's) and Vt, tau, tneg = -T, Uinv; sets
// *status = 1 (and writes none of the outputs) on a non-finite pivot.
// smem: nb^2 + (nb/2)^2 doubles.
// ---------------------------------------------------------------------------
template <int EPT>
__global__ void __launch_bounds__(CQR_THREADS, 1) cqr_recon_kernel(double *vfull /* holds Q; ld ldq */, int64_t ldq, int bb,
                                                                int bbpad, int nb, const double *Rc, int *status,
                                                                double *A, int64_t lda, double *tau, double *tneg,
                                                                double *Uinv, double *vt) {
    extern __shared__ __align__(16) double rc_sm[];
    double *M = rc_sm;             // nb x nb
    double *tmp = rc_sm + nb * nb; // (nb/2)^2
    __shared__ double rowb[2][CQR_MAXB], colb[2][CQR_MAXB];
    __shared__ double sgn[CQR_MAXB], s_piv[CQR_MAXB];
    __shared__ double s_ip[2];
    __shared__ int s_fail;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (*status != 0) return;
    const int ne = bb * bb;
    double v[EPT];
    int erc[EPT];  // r | c << 16 (r = 0xffff: no element)
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int e = tid + CQR_THREADS * i;
        const int r = (e < ne) ? e / bb : -1, c = (e < ne) ? e % bb : 0;
        erc[i] = (r & 0xffff) | (c << 16);
        v[i] = (e < ne) ? -vfull[r + (int64_t)c * ldq] : 0.0;
        if (r == 0) rowb[0][c] = v[i];
        if (e < ne && c == 0) colb[0][r] = v[i];
    }
    __syncthreads();
    // step j: X(r,c) -= X(r,j) X(j,c) / piv_j for r, c > j; the owners of row
    // and column j+1 publish them, the owner of (j+1, j+1) the next pivot
    // (with its sign S_{j+1}) and its reciprocal
    if (tid == 0) {
        const double a0 = rowb[0][0];
        const double sj = (a0 < 0.0) ? -1.0 : 1.0;
        sgn[0] = sj;
        s_piv[0] = a0 + sj;
        s_ip[0] = fast_rcp(a0 + sj);
        s_fail = !isfinite(a0);
    }
    __syncthreads();
    for (int j = 0; j < bb; ++j) {
        const double *rj = rowb[j & 1], *cj = colb[j & 1];
        double *rn = rowb[(j + 1) & 1], *cn = colb[(j + 1) & 1];
        const double ip = s_ip[j & 1];
        // all loads first, then the updates, then the publication
        double xr[EPT], xc[EPT];
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            xr[i] = cj[(erc[i] & 0xffff) & 127];
            xc[i] = rj[erc[i] >> 16];
        }
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int r = erc[i] & 0xffff, c = erc[i] >> 16;  // r = 0xffff: no element
            const bool act = (r > j) && (c > j) && (r != 0xffff);
            v[i] -= act ? xr[i] * ip * xc[i] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int r = erc[i] & 0xffff, c = erc[i] >> 16;
            const bool act = (r > j) && (c > j) && (r != 0xffff);
            if (act && r == j + 1) rn[c] = v[i];
            if (act && c == j + 1) cn[r] = v[i];
        }
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if ((erc[i] & 0xffff) == j + 1 && (erc[i] >> 16) == j + 1) {  // next pivot (one thread)
                const double sn = (v[i] < 0.0) ? -1.0 : 1.0;
                sgn[j + 1] = sn;
                s_piv[j + 1] = v[i] + sn;
                s_ip[(j + 1) & 1] = fast_rcp(v[i] + sn);
                if (!isfinite(v[i])) s_fail = 1;
            }
        __syncthreads();
    }
    const bool bad = s_fail;
    __syncthreads();
    if (bad) {
        if (tid == 0) *status = 1;
        return;
    }
    // final entries: L(r, c) = X(r, c) / piv_c (r > c); U(r, c) = X(r, c) (r < c), U(c, c) = piv_c
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int r = erc[i] & 0xffff, c = erc[i] >> 16;
        if (r == 0xffff) continue;
        if (r > c) v[i] /= s_piv[c];
        else if (r == c) v[i] = s_piv[c];
    }
    // U -> smem -> U^{-1} -> Uinv (global)
    for (int e = tid; e < nb * nb; e += CQR_THREADS) {
        const int r = e % nb, c = e / nb;
        M[e] = (r >= bb || c >= bb) ? (r == c ? 1.0 : 0.0) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int r = erc[i] & 0xffff, c = erc[i] >> 16;
        if (r != 0xffff && r <= c) M[r + c * nb] = v[i];
    }
    __syncthreads();
    tri_inv_upper_smem(M, nb, tmp);
    __syncthreads();
    for (int c = warp; c < bbpad; c += CQR_THREADS / 32)
        for (int r = lane; r < bbpad; r += 32) Uinv[r + (int64_t)c * bbpad] = (r < bb && c < bb) ? M[r + c * nb] : 0.0;
    __syncthreads();
    // L^T (unit upper) -> smem -> L^{-T}
    for (int e = tid; e < nb * nb; e += CQR_THREADS) {
        const int r = e % nb, c = e / nb;
        M[e] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int r = erc[i] & 0xffff, c = erc[i] >> 16;
        if (r != 0xffff && r > c) M[c + r * nb] = v[i];
    }
    __syncthreads();
    tri_inv_upper_smem(M, nb, tmp);
    __syncthreads();
    // T(r, c) = sum_{r <= q <= c} U(r, q) S_q Linv^T(q, c): U from registers via tmp? -> use vt scratch:
    // stage U (upper) row-major in Vt's top block rows (they are rewritten below)
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int r = erc[i] & 0xffff, c = erc[i] >> 16;
        if (r != 0xffff && r <= c) vt[c + (int64_t)r * bbpad] = v[i] * sgn[c];
    }
    __syncthreads();
    for (int e = tid; e < bbpad * bbpad; e += CQR_THREADS) {
        const int r = e / bbpad, c = e % bbpad;
        double acc = 0.0;
        if (r < bb && c < bb && r <= c)
            for (int q = r; q <= c; ++q) acc += vt[q + (int64_t)r * bbpad] * M[q + c * nb];
        tneg[r + (int64_t)c * bbpad] = -acc;
        if (r == c && r < bb) tau[r] = acc;
    }
    __syncthreads();
    // panel top block: L strictly below, R = S Rc on/above; Vt / Vfull top rows
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int r = erc[i] & 0xffff, c = erc[i] >> 16;
        if (r == 0xffff) continue;
        A[r + (int64_t)c * lda] = (r > c) ? v[i] : sgn[r] * Rc[r + (int64_t)c * bbpad];
        const double vv = (r > c) ? v[i] : (r == c ? 1.0 : 0.0);
        vt[c + (int64_t)r * bbpad] = vv;
        vfull[r + (int64_t)c * ldq] = vv;
    }
    for (int e = tid; e < bb * (bbpad - bb); e += CQR_THREADS) {
        const int r = e % bb, c = bb + e / bb;
        vt[c + (int64_t)r * bbpad] = 0.0;
        vfull[r + (int64_t)c * ldq] = 0.0;
    }
}

}  // namespace rq
