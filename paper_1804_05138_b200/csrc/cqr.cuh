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
// The bb x bb factorizations run in one CTA on a shared-memory copy of the
// matrix (leading dimension nb + 1: row and column walks both free of bank
// conflicts), right-looking, one __syncthreads per column, two threads per
// row of the trailing block.  The triangular inverses are block-recursive
// doublings in shared memory, and every m' x bb or bb x bb product with them
// (Q1 = P R1^{-1}, V2 = -Qbottom U^{-1}, T = (U S) L^{-T}) runs on the FP64
// tensor cores (DMMA, cqr_rowmul_kernel).
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
// shared memory of the one-CTA kernels: nb x (nb + 1) matrix + (nb/2)^2 scratch
inline size_t cqr_smem_bytes(int nb) { return ((size_t)nb * (nb + 1) + (size_t)(nb / 2) * (nb / 2)) * sizeof(double); }

// ---------------------------------------------------------------------------
// In-place inverse of an upper-triangular nb x nb matrix in shared memory
// (nb = 8 * 2^k, leading dimension ld; identity padding beyond the live size)
// by block-recursive doubling: invert the 8x8 diagonal blocks, then
// B <- -A^{-1} B D^{-1} for the off-diagonal block of every 2s x 2s block.
// Only the upper triangle is written (a strictly lower part stays as it is).
// tmp: nb^2/4 doubles (nb/(2s) blocks of s^2 per level).  All threads of the
// CTA must call it.
// ---------------------------------------------------------------------------
RQ_DEV void tri_inv_upper_smem(double *M, int nb, double *tmp, int ld) {
    const int tid = threadIdx.x;
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
                for (int r = 0; r < 8; ++r)
                    if (r <= c) M[(k0 + r) + (k0 + c) * ld] = x[r];
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
// inverse of this pass's R.  One CTA, the upper triangle in shared memory:
// step j applies M(a,c) -= M(j,a) M(j,c) / M(j,j) to j < a <= c (two threads
// per row a, alternate columns), so M ends as D U with R = D^{1/2} U.
// Outputs (ld bbpad, zero padding): Rc = R (pass 1) or R Rc (pass 2; the old
// Rc staged nb/4 columns at a time); Rinv = R^{-1}.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CQR_THREADS, 1) cqr_chol_kernel(const double *G /* bbpad x bbpad */, int bb, int bbpad,
                                                               int nb, int pass, const int *bb_eff, int *status,
                                                               double *Rc, double *Rinv, const double *tol2) {
    extern __shared__ __align__(16) double cq_sm[];
    const int ld = nb + 1;
    double *M = cq_sm;                   // nb x nb, ld nb + 1
    double *tmp = cq_sm + (size_t)nb * ld;  // (nb/2)^2
    __shared__ double s_sq[CQR_MAXB];
    __shared__ double s_red[CQR_THREADS / 32];
    __shared__ int s_bad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (pass == 1) {
        if (tid == 0) *status = (*bb_eff == bb) ? 0 : 1;
        __syncthreads();
    }
    if (*status != 0) return;
    cqr_stamp(0);
    double mx = 0.0;
    for (int e = tid; e < nb * nb; e += CQR_THREADS) {
        const int r = e % nb, c = e / nb;
        double v = (r == c) ? 1.0 : 0.0;
        if (r < bb && c < bb) {
            v = (r <= c) ? G[r + (int64_t)c * bbpad] : 0.0;
            if (r <= c) mx = fmax(mx, fabs(v - (r == c ? 1.0 : 0.0)));
        }
        M[r + c * ld] = v;
    }
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
    // trailing block as a 16 x 16 thread grid: thread (ta, tc) owns rows
    // j+1+ta+16p and columns j+1+tc+16q (p, q < 8): all loads of a step in flight
    const int ta = tid & 15, tc = tid >> 4;
    for (int j = 0; j < bb; ++j) {
        const double idl = fast_rcp(M[j + j * ld]);
        const int n0 = j + 1;
        double ma[8], rq[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int a = n0 + ta + 16 * u, c = n0 + tc + 16 * u;
            ma[u] = (a < bb) ? M[j + a * ld] * idl : 0.0;
            rq[u] = (c < bb) ? M[j + c * ld] : 0.0;
        }
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
            const int a = n0 + ta + 16 * pp;
            if (a >= bb) break;
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) {
                const int c = n0 + tc + 16 * qq;
                if (c >= bb) break;
                if (c >= a) M[a + c * ld] -= ma[pp] * rq[qq];
            }
        }
        __syncthreads();
    }
    cqr_stamp(2);
    // checks: every pivot positive, none below the R11-diagonal stop threshold
    // (reading R-G12b: the column-by-column kernel then stops at it), and the
    // diagonal ratio of R (pass 1)
    if (warp == 0) {
        const double t2 = (pass == 1 && tol2) ? *tol2 : -1.0;
        bool ok = true;
        double dmax = 0.0, dmin = 1e308;
        for (int q = lane; q < bb; q += 32) {
            const double d = M[q + q * ld];
            ok = ok && (d > 0.0) && !(d < t2);
            dmax = fmax(dmax, d);
            dmin = fmin(dmin, d);
        }
        for (int o = 16; o > 0; o >>= 1) {
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
            dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        }
        ok = __all_sync(0xffffffffu, ok);
        if (lane == 0)
            s_bad = !ok || (pass == 1 && !(dmax <= CQR_MAX_DIAG_RATIO * CQR_MAX_DIAG_RATIO * dmin));
    }
    for (int q = tid; q < bb; q += CQR_THREADS) s_sq[q] = sqrt(M[q + q * ld]);
    __syncthreads();
    if (s_bad) {
        if (tid == 0) *status = 1;
        return;
    }
    // R(a, c) = M(a, c) / sqrt(d_a), R(a, a) = sqrt(d_a)
    for (int e = tid; e < bb * bb; e += CQR_THREADS) {
        const int r = e % bb, c = e / bb;
        if (r < c) M[r + c * ld] /= s_sq[r];
        else if (r == c) M[r + c * ld] = s_sq[r];
    }
    __syncthreads();
    if (pass == 1) {
        for (int e = tid; e < bbpad * bbpad; e += CQR_THREADS) {
            const int r = e % bbpad, c = e / bbpad;
            Rc[e] = (r <= c && c < bb) ? M[r + c * ld] : 0.0;
        }
    } else {
        // Rc <- R Rc: nb/4 columns of the old Rc at a time in tmp (written back
        // only after their own chunk has been staged)
        const int cw = nb / 4;
        for (int c0 = 0; c0 < bb; c0 += cw) {
            const int w = min(cw, bb - c0);
            for (int e = tid; e < nb * w; e += CQR_THREADS) {
                const int q = e % nb, cc = e / nb;
                tmp[e] = (q < bb) ? Rc[q + (int64_t)(c0 + cc) * bbpad] : 0.0;
            }
            __syncthreads();
            // a thread takes row r = tid mod nb of four chunk columns at once
            // (e = e0 + tid + 256 u: nb divides 256, so r is the same for all four):
            // four independent chains
            for (int e0 = 0; e0 < nb * w; e0 += 4 * CQR_THREADS) {
                int cc[4];
                double acc[4];
                const int r = (e0 + tid) % nb;
                int cmax = -1;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + tid + u * CQR_THREADS;
                    cc[u] = (e < nb * w) ? e / nb : -1;
                    acc[u] = 0.0;
                    if (cc[u] >= 0) cmax = max(cmax, c0 + cc[u]);
                }
                for (int q = r; q <= cmax; ++q) {
                    const double mv = M[r + q * ld];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (cc[u] >= 0 && q <= c0 + cc[u]) acc[u] += mv * tmp[q + cc[u] * nb];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = c0 + cc[u];
                    if (cc[u] >= 0 && r <= c && r < bb) Rc[r + (int64_t)c * bbpad] = acc[u];
                }
            }
            __syncthreads();
        }
    }
    cqr_stamp(3);
    tri_inv_upper_smem(M, nb, tmp, ld);
    __syncthreads();
    cqr_stamp(4);
    for (int e = tid; e < bbpad * bbpad; e += CQR_THREADS) {
        const int r = e % bbpad, c = e / bbpad;
        Rinv[e] = (r <= c && c < bb) ? M[r + c * ld] : 0.0;
    }
}

// ---------------------------------------------------------------------------
// Y(r, :) = s X(r, :) R for rows r in [r0, rows), R bbpad x bbpad (entries
// with row or column >= bb are zero), on the FP64 tensor cores: each warp
// takes 8-row tiles (grid-strided) with all bbpad columns (mma.sync m8n8k4, A fragments from X in
// global memory, B fragments from R in shared memory with a row stride = 4 mod
// 16 doubles: conflict-free).  In place allowed (a warp reads all its rows'
// entries before it writes).  Columns bb..bbpad-1 of Y are written as 0.
// mode 1 (V2 of the reconstruction): also A(r, c) = Y(r, c) (the panel below
// the top block) and Vt(c, r) = Y(r, c).  No-op when *status != 0.
// ---------------------------------------------------------------------------
constexpr int RM_ROWS = 8;   // rows per warp (one m8 tile: no register spills)
constexpr int RM_MT = RM_ROWS / 8;
__global__ void __launch_bounds__(CQR_THREADS, 1) cqr_rowmul_kernel(const double *X, int64_t ldx, int64_t r0, int64_t rows,
                                                                 int bb, int bbpad, const double *R, double s,
                                                                 double *Y, int64_t ldy, const int *status, int mode,
                                                                 double *A, int64_t lda, double *vt) {
    extern __shared__ __align__(16) double rm_sm[];  // bbpad x (bbpad + pad)
    if (*status != 0) return;
    const int ldr = bbpad + 4;  // bbpad is a multiple of 8: ldr = 4 or 12 mod 16
    // R staged by 16-byte cp.async copies, all in flight at once (a plain copy
    // loop waits one L2 round trip per iteration: tens of microseconds per
    // launch); R and its padded image are 16-byte aligned (bbpad, ldr even)
    for (int e = threadIdx.x; e < bbpad * bbpad / 2; e += blockDim.x) {
        const int k = (2 * e) % bbpad, c = (2 * e) / bbpad;
        cp_async16(&rm_sm[k + c * ldr], &R[k + (int64_t)c * bbpad], 16);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fr = lane >> 2, fk = lane & 3;
    const int64_t tstride = (int64_t)gridDim.x * (CQR_THREADS / 32) * RM_ROWS;
    const int NT = bbpad / 8;
    // column slices (gridDim.y > 1, small products): this CTA's 8-column tiles
    const int nts = (NT + (int)gridDim.y - 1) / (int)gridDim.y;
    const int nt0 = (int)blockIdx.y * nts, nt1 = min(NT, nt0 + nts);
    // the A fragments of a warp's rows (one round trip), prefetched one tile
    // ahead so the loads of tile t + 1 are in flight during tile t's MMAs
    double af[RM_MT][CQR_MAXB / 4], an[RM_MT][CQR_MAXB / 4];
    auto load_frag = [&](double (&f)[RM_MT][CQR_MAXB / 4], int64_t rb) {
#pragma unroll
        for (int kk = 0; kk < CQR_MAXB / 4; ++kk) {
            const int k = kk * 4 + fk;
#pragma unroll
            for (int mt = 0; mt < RM_MT; ++mt) {
                const int64_t r = rb + mt * 8 + fr;
                f[mt][kk] = (kk * 4 < bbpad && r < rows && k < bb) ? X[r + (int64_t)k * ldx] : 0.0;
            }
        }
    };
    int64_t rbase = r0 + ((int64_t)blockIdx.x * (CQR_THREADS / 32) + warp) * RM_ROWS;
    if (rbase < rows) load_frag(af, rbase);
    for (; rbase < rows; rbase += tstride) {
        if (rbase + tstride < rows) load_frag(an, rbase + tstride);
        double acc[RM_MT][16][2];
#pragma unroll
        for (int mt = 0; mt < RM_MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < CQR_MAXB / 4; ++kk) {
            if (kk * 4 >= bbpad) break;
            const int k = kk * 4 + fk;
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) {
                if (nt >= nt0 && nt < nt1) {
                    const double b = rm_sm[k + (nt * 8 + fr) * ldr];
#pragma unroll
                    for (int mt = 0; mt < RM_MT; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt][kk], b);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int mt = 0; mt < RM_MT; ++mt) {
            const int64_t r = rbase + mt * 8 + fr;
            if (r >= rows) continue;
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) {
                if (nt < nt0 || nt >= nt1) continue;
                double yv[2];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int c = nt * 8 + 2 * fk + hh;
                    const double y = (c < bb) ? s * acc[mt][nt][hh] : 0.0;
                    yv[hh] = y;
                    Y[r + (int64_t)c * ldy] = y;
                    if (mode == 1 && c < bb) A[r + (int64_t)c * lda] = y;
                }
                // Vt(c, r), Vt(c + 1, r): one 16-byte store (c even, bbpad even)
                if (mode == 1)
                    *reinterpret_cast<double2 *>(&vt[nt * 8 + 2 * fk + r * bbpad]) = make_double2(yv[0], yv[1]);
            }
        }
#pragma unroll
        for (int mt = 0; mt < RM_MT; ++mt)
#pragma unroll
            for (int kk = 0; kk < CQR_MAXB / 4; ++kk) af[mt][kk] = an[mt][kk];
    }
}

// ---------------------------------------------------------------------------
// The m'-row products of the panel (Q1 = P R1^{-1}, V2 = -Q1bottom C): same
// arithmetic and epilogue as cqr_rowmul_kernel (for every output element the
// same ascending-k DMMA chain, so the same bits), with 512 threads: 16 warps,
// two per 8-row tile, each owning half of the 8-column tiles -- four warps per
// SM sub-partition instead of two, so one warp's fragment loads and epilogue
// stores overlap the others' DMMAs.  No prefetch (128 registers per thread).
// In place (V2) is safe: a CTA barrier separates each round's loads from its
// stores (the warp pair of a row tile reads all columns, writes half each).
// ---------------------------------------------------------------------------
constexpr int RM2_THREADS = 512;
__global__ void __launch_bounds__(RM2_THREADS, 1) cqr_rowmul2_kernel(const double *X, int64_t ldx, int64_t r0, int64_t rows,
                                                                   int bb, int bbpad, const double *R, double s,
                                                                   double *Y, int64_t ldy, const int *status, int mode,
                                                                   double *A, int64_t lda, double *vt) {
    constexpr int NH = 2, NTW = 16 / NH;
    extern __shared__ __align__(16) double rm_sm[];  // bbpad x (bbpad + pad)
    if (*status != 0) return;
    const int ldr = bbpad + 4;
    for (int e = threadIdx.x; e < bbpad * bbpad / 2; e += blockDim.x) {
        const int k = (2 * e) % bbpad, c = (2 * e) / bbpad;
        cp_async16(&rm_sm[k + c * ldr], &R[k + (int64_t)c * bbpad], 16);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fr = lane >> 2, fk = lane & 3;
    const int rt = warp / NH, h = warp % NH;
    constexpr int RPC = (RM2_THREADS / 32 / NH) * 8;  // rows per CTA round
    const int NT = bbpad / 8;
    const int ntb = h * NTW;  // this warp's first 8-column tile
    // rounds are uniform over the CTA: the two warps of a row tile read ALL
    // columns of their rows, so (in place: V2 overwrites its input) every
    // fragment load of a round precedes the round's stores (CTA barrier)
    for (int64_t base = r0 + (int64_t)blockIdx.x * RPC; base < rows; base += (int64_t)gridDim.x * RPC) {
        const int64_t rbase = base + rt * 8;
        const int64_t r = rbase + fr;
        double af[CQR_MAXB / 4];
#pragma unroll
        for (int kk = 0; kk < CQR_MAXB / 4; ++kk) {
            const int k = kk * 4 + fk;
            af[kk] = (kk * 4 < bbpad && r < rows && k < bb) ? X[r + (int64_t)k * ldx] : 0.0;
        }
        __syncthreads();
        double acc[NTW][2];
#pragma unroll
        for (int j = 0; j < NTW; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < CQR_MAXB / 4; ++kk) {
            if (kk * 4 >= bbpad) break;
            const int k = kk * 4 + fk;
#pragma unroll
            for (int j = 0; j < NTW; ++j) {
                if (ntb + j < NT) {
                    const double b = rm_sm[k + ((ntb + j) * 8 + fr) * ldr];
                    dmma(acc[j][0], acc[j][1], af[kk], b);
                }
            }
        }
        __syncwarp();
        if (r < rows) {
#pragma unroll
            for (int j = 0; j < NTW; ++j) {
                const int nt = ntb + j;
                if (nt >= NT) continue;
                double yv[2];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int c = nt * 8 + 2 * fk + hh;
                    const double y = (c < bb) ? s * acc[j][hh] : 0.0;
                    yv[hh] = y;
                    Y[r + (int64_t)c * ldy] = y;
                    if (mode == 1 && c < bb) A[r + (int64_t)c * lda] = y;
                }
                if (mode == 1)
                    *reinterpret_cast<double2 *>(&vt[nt * 8 + 2 * fk + r * bbpad]) = make_double2(yv[0], yv[1]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Householder reconstruction of the top bb x bb block (one CTA):
//   X = -Q(0:bb, 0:bb); for j: S_j = sign(X_jj) (1 if 0); pivot X_jj + S_j;
//   L(:, j) = X(j+1:, j) / pivot; Schur update  ->  S - Qtop = L U
// (right-looking in shared memory, two threads per row of the trailing block,
// one __syncthreads per column).  Then tau_j = T_jj = U_jj S_j, R = S Rc, and
// for the host's DMMA products: U S (us), U^{-1} (Uinv; V2 = -Qbottom U^{-1})
// and L^{-T} (linvt; T = (U S) L^{-T}).
// Writes: the top block of the panel in A (L strictly below, R on/above), the
// top bb rows of Vfull (after reading Q's) and Vt, tau, us, Uinv, linvt; sets
// *status = 1 (and writes none of the outputs) on a non-finite pivot.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CQR_THREADS, 1) cqr_recon_kernel(double *vfull /* holds Q; ld ldq */, int64_t ldq, int bb,
                                                                int bbpad, int nb, const double *Rc, int *status,
                                                                double *A, int64_t lda, double *tau, double *us,
                                                                double *Uinv, double *linvt, double *vt) {
    extern __shared__ __align__(16) double rc_sm[];
    const int ld = nb + 1;
    double *M = rc_sm;                       // nb x nb, ld nb + 1
    double *tmp = rc_sm + (size_t)nb * ld;   // (nb/2)^2
    __shared__ double sgn[CQR_MAXB], s_piv[CQR_MAXB];
    __shared__ int s_fail;
    const int tid = threadIdx.x;
    const int ta = tid & 15, tc = tid >> 4;  // 16 x 16 thread grid over the trailing block
    if (*status != 0) return;
    cqr_stamp(0);
    for (int e = tid; e < nb * nb; e += CQR_THREADS) {
        const int r = e % nb, c = e / nb;
        M[r + c * ld] = (r < bb && c < bb) ? -vfull[r + (int64_t)c * ldq] : (r == c ? 1.0 : 0.0);
    }
    if (tid == 0) s_fail = 0;
    __syncthreads();
    for (int j = 0; j < bb; ++j) {
        const double xjj = M[j + j * ld];
        const double sj = (xjj < 0.0) ? -1.0 : 1.0;
        const double piv = xjj + sj;
        const double ip = fast_rcp(piv);
        if (tid == 0) {
            sgn[j] = sj;
            s_piv[j] = piv;
            if (!isfinite(xjj)) s_fail = 1;
        }
        const int n0 = j + 1;
        double xr[8], xc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int r = n0 + ta + 16 * u, c = n0 + tc + 16 * u;
            xr[u] = (r < bb) ? M[r + j * ld] * ip : 0.0;
            xc[u] = (c < bb) ? M[j + c * ld] : 0.0;
        }
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
            const int r = n0 + ta + 16 * pp;
            if (r >= bb) break;
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) {
                const int c = n0 + tc + 16 * qq;
                if (c >= bb) break;
                M[r + c * ld] -= xr[pp] * xc[qq];
            }
        }
        __syncthreads();
    }
    cqr_stamp(1);
    if (s_fail) {
        if (tid == 0) *status = 1;
        return;
    }
    // L(r, c) = X(r, c) / piv_c (r > c); U(c, c) = piv_c; U(r, c) = X(r, c) (r < c)
    for (int e = tid; e < bb * bb; e += CQR_THREADS) {
        const int r = e % bb, c = e / bb;
        if (r > c) M[r + c * ld] /= s_piv[c];
        else if (r == c) M[r + c * ld] = s_piv[c];
    }
    __syncthreads();
    // panel top block: L strictly below, R = S Rc on/above; Vt / Vfull top rows
    for (int e = tid; e < bb * bb; e += CQR_THREADS) {
        const int r = e % bb, c = e / bb;
        const double x = M[r + c * ld];
        A[r + (int64_t)c * lda] = (r > c) ? x : sgn[r] * Rc[r + (int64_t)c * bbpad];
        const double vv = (r > c) ? x : (r == c ? 1.0 : 0.0);
        vt[c + (int64_t)r * bbpad] = vv;
        vfull[r + (int64_t)c * ldq] = vv;
    }
    for (int e = tid; e < bb * (bbpad - bb); e += CQR_THREADS) {
        const int r = e % bb, c = bb + e / bb;
        vt[c + (int64_t)r * bbpad] = 0.0;
        vfull[r + (int64_t)c * ldq] = 0.0;
    }
    for (int c = tid; c < bb; c += CQR_THREADS) tau[c] = s_piv[c] * sgn[c];
    for (int e = tid; e < bbpad * bbpad; e += CQR_THREADS) {
        const int r = e % bbpad, c = e / bbpad;
        us[e] = (r <= c && c < bb) ? M[r + c * ld] * sgn[c] : 0.0;
    }
    __syncthreads();
    // U^{-1} (upper, in place; L below untouched)
    tri_inv_upper_smem(M, nb, tmp, ld);
    __syncthreads();
    for (int e = tid; e < bbpad * bbpad; e += CQR_THREADS) {
        const int r = e % bbpad, c = e / bbpad;
        Uinv[e] = (r <= c && c < bb) ? M[r + c * ld] : 0.0;
    }
    __syncthreads();
    // upper := L^T (unit upper) from the strict lower part, then L^{-T}
    for (int e = tid; e < nb * nb; e += CQR_THREADS) {
        const int r = e % nb, c = e / nb;
        if (r < c) M[r + c * ld] = (c < bb) ? M[c + r * ld] : 0.0;
        else if (r == c) M[r + c * ld] = 1.0;
    }
    __syncthreads();
    tri_inv_upper_smem(M, nb, tmp, ld);
    __syncthreads();
    for (int e = tid; e < bbpad * bbpad; e += CQR_THREADS) {
        const int r = e % bbpad, c = e / bbpad;
        linvt[e] = (r <= c && c < bb) ? M[r + c * ld] : 0.0;
    }
    cqr_stamp(2);
}

}  // namespace rq
