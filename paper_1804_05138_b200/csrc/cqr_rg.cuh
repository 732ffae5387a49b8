// cqr_rg.cuh -- the one-CTA bb x bb factorizations of the CholeskyQR2 panel
// (cqr.cuh: CholeskyQR2 + Householder reconstruction, reading R-G24 of the
// paper's "TSQR for the panel") with the matrix held in REGISTERS.
//
// The shared-memory kernels of cqr.cuh read-modify-write the whole trailing
// block in shared memory at every step (~2100 SM cycles per step at bb = 128:
// bound by shared-memory wavefronts) and then invert the triangular factors in
// separate block-recursive passes.  Here a 16 x 16 thread grid owns the
// NB x NB matrix as E x E register tiles (thread (ta, tc) holds rows
// ta + 16p and columns tc + 16q, E = NB / 16); a step only broadcasts row j
// (and column j) through shared memory -- one __syncthreads per step, the
// next row published by its owners right after their update -- and the
// inverses are carried along instead of computed afterwards:
//
//   Cholesky (pass 1: G1 = P^T P, pass 2: G2 = Q1^T Q1):  symmetric
//   elimination M(a,c) -= M(j,a) M(j,c) / M(j,j) (j < a <= c), the same
//   update as cqr_chol_kernel, applied as a row operation to [G | I]: the
//   upper triangle ends as D U and the strict lower triangle as Y = U^{-T}
//   (the elimination matrix), so R = D^{1/2} U and R^{-1} = Y^T D^{-1/2}.
//
//   Reconstruction (Ballard et al.): LU without pivoting of S - Qtop with
//   S_j = sign of the Schur pivot, then L^{-1} (forward, in place in the
//   strict lower triangle) and U^{-1} (column-oriented, in place in the upper
//   triangle) in ONE sweep: step j reads row j and column j of the square.
//
// Block pruning: step j (in 16-row block jb) only touches the register tiles
// that can change (compile-time p / q ranges), so the work per step shrinks
// with the trailing block.  Outputs and their layouts are those of
// cqr_chol_kernel / cqr_recon_kernel (the host calls either).
#pragma once
#include "cqr.cuh"

namespace rq {

constexpr int RG_THREADS = 256;
// dynamic shared memory of cqr_chol_rg_kernel (pass 2: R2 and the old Rc,
// both packed upper triangles)
inline size_t cqr_rg_smem_bytes(int nb) { return (size_t)nb * (nb + 1) * sizeof(double); }

RQ_DEV int upk(int r, int c) { return c * (c + 1) / 2 + r; }  // packed upper, column-major, r <= c

template <int NB>
__global__ void __launch_bounds__(RG_THREADS, 1) cqr_chol_rg_kernel(const double *G, int bb, int bbpad, int pass,
                                                                  const int *bb_eff, int *status, double *Rc,
                                                                  double *Rinv, double *tol2, int tol_from_gram) {
    constexpr int E = NB / 16;
    static_assert(NB % 16 == 0 && E >= 1 && E <= 8, "NB in 16..128");
    extern __shared__ __align__(16) double rg_sm[];  // pass 2: R2 packed | old Rc packed
    __shared__ double rowb[2][NB];
    __shared__ double dsq[NB], rsq[NB];
    __shared__ double s_red[RG_THREADS / 32];
    __shared__ int s_bad;
    const int tid = threadIdx.x, ta = tid & 15, tc = tid >> 4, warp = tid >> 5, lane = tid & 31;
    if (pass == 1) {
        if (tid == 0) {
            *status = (*bb_eff == bb) ? 0 : 1;
            if (tol_from_gram) {
                // the R11-diagonal stop scale (reading R-G12b) from the Gram diagonal:
                // ||panel||_F^2 = trace(P^T P), ascending columns (replaces colsumsq +
                // panel_tol_kernel; also read by the column-by-column fallback)
                double sg = 0.0;
                for (int c = 0; c < bb; ++c) sg += G[c + (int64_t)c * bbpad];
                const double eps = 0x1p-52;
                *tol2 = (*bb_eff == 0) ? 0.0 : (1e3 * eps) * (1e3 * eps) * sg;
            }
        }
        __syncthreads();
    }
    if (*status != 0) return;
    cqr_stamp(0);
    double x[E][E];
    double mx = 0.0;
#pragma unroll
    for (int p = 0; p < E; ++p)
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const int a = ta + 16 * p, c = tc + 16 * q;
            double v = (a == c) ? 1.0 : 0.0;
            if (a < bb && c < bb && a <= c) {
                v = G[a + (int64_t)c * bbpad];
                mx = fmax(mx, fabs(v - (a == c ? 1.0 : 0.0)));
            }
            x[p][q] = v;
        }
    if (pass == 2) {  // max |G2 - I| over the upper triangle
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) s_red[warp] = mx;
    }
    if (ta == 0) {
#pragma unroll
        for (int q = 0; q < E; ++q) rowb[0][tc + 16 * q] = x[0][q];
    }
    __syncthreads();
    if (pass == 2) {
        double m2 = 0.0;
        for (int w = 0; w < RG_THREADS / 32; ++w) m2 = fmax(m2, s_red[w]);
        if (!(m2 <= CQR_MAX_ORTH_ERR)) {
            if (tid == 0) *status = 1;
            return;
        }
    }
    cqr_stamp(1);
    // ---- symmetric elimination on [G | I] ---------------------------------
#pragma unroll
    for (int jb = 0; jb < E; ++jb) {
        if (16 * jb >= bb) break;
        for (int s = 0; s < 16; ++s) {
            const int j = 16 * jb + s;
            if (j >= bb) break;
            const double *rb = rowb[j & 1];
            const double idl = fast_rcp(rb[j]);
            double lv[E], rv[E];
#pragma unroll
            for (int p = jb; p < E; ++p) lv[p] = rb[ta + 16 * p] * idl;  // M(j, a) / d_j (upper part)
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int c = tc + 16 * q;
                rv[q] = (c == j) ? 1.0 : rb[c];  // M(j, c) for c > j, Y(j, c) for c < j, Y(j, j) = 1
            }
            // tiles classified at compile time: only tiles in block row / column
            // jb or on the block diagonal need an element predicate
#pragma unroll
            for (int p = jb; p < E; ++p) {
                const int a = ta + 16 * p;
#pragma unroll
                for (int q = 0; q < E; ++q) {
                    if (!(q >= p || q <= jb)) continue;
                    const int c = tc + 16 * q;
                    bool on = true;
                    if (p == jb) on = on && (a > j);
                    if (q == p) on = on && (c >= a || (q == jb && c <= j));
                    else if (q < p && q == jb) on = on && (c <= j);
                    if (on) x[p][q] = fma(-lv[p], rv[q], x[p][q]);
                }
            }
            // publish row j + 1 (its owners' values after this step)
            const int jn = j + 1;
            if (ta == (jn & 15) && jn < bb) {
                if (s < 15) {
#pragma unroll
                    for (int q = 0; q < E; ++q) rowb[jn & 1][tc + 16 * q] = x[jb][q];
                } else if (jb + 1 < E) {
#pragma unroll
                    for (int q = 0; q < E; ++q) rowb[jn & 1][tc + 16 * q] = x[jb + 1 < E ? jb + 1 : jb][q];
                }
            }
            __syncthreads();
        }
    }
    cqr_stamp(2);
    // ---- checks: pivots positive, not below the R11-diagonal stop (R-G12b),
    //      diagonal ratio (pass 1) -------------------------------------------
    if (ta == tc) {
#pragma unroll
        for (int p = 0; p < E; ++p) dsq[ta + 16 * p] = x[p][p];
    }
    __syncthreads();
    if (warp == 0) {
        const double t2 = (pass == 1 && tol2) ? *tol2 : -1.0;
        bool ok = true;
        double dmax = 0.0, dmin = 1e308;
        for (int q = lane; q < bb; q += 32) {
            const double d = dsq[q];
            ok = ok && (d > 0.0) && !(d < t2);
            dmax = fmax(dmax, d);
            dmin = fmin(dmin, d);
        }
        for (int o = 16; o > 0; o >>= 1) {
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
            dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        }
        ok = __all_sync(0xffffffffu, ok);
        if (lane == 0) s_bad = !ok || (pass == 1 && !(dmax <= CQR_MAX_DIAG_RATIO * CQR_MAX_DIAG_RATIO * dmin));
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) *status = 1;
        return;
    }
    for (int q = tid; q < bb; q += RG_THREADS) dsq[q] = sqrt(dsq[q]);
    __syncthreads();
    cqr_stamp(3);
    // ---- R = D^{-1/2} (D U) (registers), R^{-1} = Y^T D^{-1/2}: every thread
    //      writes the transposed position of each of its elements into a
    //      shared-memory image (ld NB + 1), copied out coalesced -------------
    {
        double *S = rg_sm;
        constexpr int LS = NB + 1;
        for (int q = tid; q < bb; q += RG_THREADS) rsq[q] = 1.0 / dsq[q];
        __syncthreads();
#pragma unroll
        for (int p = 0; p < E; ++p) {
            const int a = ta + 16 * p;
            const double ra = (a < bb) ? rsq[a] : 0.0;
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int c = tc + 16 * q;
                // Rinv(c, a) = Y(a, c) / sqrt(d_a) from the strict lower element (a, c)
                S[c + a * LS] = (c < a) ? x[p][q] * ra : ((c == a) ? ra : 0.0);
                if (c > a) x[p][q] = (c < bb) ? x[p][q] * ra : 0.0;
                else if (c == a) x[p][q] = (a < bb) ? dsq[a] : 0.0;
                else x[p][q] = 0.0;
            }
        }
        __syncthreads();
        for (int e = tid; e < bbpad * bbpad; e += RG_THREADS) {
            const int r = e % bbpad, c = e / bbpad;
            Rinv[e] = S[r + c * LS];
        }
        __syncthreads();
    }
    if (pass == 1) {
#pragma unroll
        for (int p = 0; p < E; ++p)
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int a = ta + 16 * p, c = tc + 16 * q;
                if (a < bbpad && c < bbpad) Rc[a + (int64_t)c * bbpad] = x[p][q];
            }
    } else {
        // Rc <- R2 Rc: both upper triangular, packed in shared memory; thread
        // tile (p, q) only receives the 16-row t blocks with p <= tb <= q
        double *S2 = rg_sm, *S1 = rg_sm + NB * (NB + 1) / 2;
#pragma unroll
        for (int p = 0; p < E; ++p)
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int a = ta + 16 * p, c = tc + 16 * q;
                if (a <= c) {
                    S2[upk(a, c)] = x[p][q];
                    S1[upk(a, c)] = (c < bb) ? Rc[a + (int64_t)c * bbpad] : 0.0;
                }
            }
        __syncthreads();
        double acc[E][E];
#pragma unroll
        for (int p = 0; p < E; ++p)
#pragma unroll
            for (int q = 0; q < E; ++q) acc[p][q] = 0.0;
#pragma unroll
        for (int tb = 0; tb < E; ++tb) {
            for (int s = 0; s < 16; ++s) {
                const int t = 16 * tb + s;
                double r2[E], r1[E];
#pragma unroll
                for (int p = 0; p <= tb; ++p) {
                    const int a = ta + 16 * p;
                    r2[p] = (a <= t) ? S2[upk(a, t)] : 0.0;
                }
#pragma unroll
                for (int q = tb; q < E; ++q) {
                    const int c = tc + 16 * q;
                    r1[q] = (t <= c) ? S1[upk(t, c)] : 0.0;
                }
#pragma unroll
                for (int p = 0; p <= tb; ++p)
#pragma unroll
                    for (int q = tb; q < E; ++q) acc[p][q] = fma(r2[p], r1[q], acc[p][q]);
            }
        }
#pragma unroll
        for (int p = 0; p < E; ++p)
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int a = ta + 16 * p, c = tc + 16 * q;
                if (a < bbpad && c < bbpad) Rc[a + (int64_t)c * bbpad] = (a <= c && c < bb) ? acc[p][q] : 0.0;
            }
    }
    cqr_stamp(4);
}

// ---------------------------------------------------------------------------
// Householder reconstruction of the top bb x bb block (one CTA, registers):
// same outputs as cqr_recon_kernel (cqr.cuh).
// ---------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(RG_THREADS, 1) cqr_recon_rg_kernel(const double *qtop /* Q(0:bb, 0:bb), ld ldqt */,
                                                                   int64_t ldqt, double *vfull /* ld ldq */, int64_t ldq,
                                                                   int bb, int bbpad, const double *Rc, int *status,
                                                                   double *A, int64_t lda, double *tau, double *us,
                                                                   double *Uinv, double *linvt, double *vt,
                                                                   const double *r2inv, double *cmat) {
    constexpr int E = NB / 16;
    static_assert(NB % 16 == 0 && E >= 1 && E <= 8, "NB in 16..128");
    extern __shared__ __align__(16) double rc_img[];  // NB x (NB + 1): transposed outputs, copied out coalesced
    constexpr int LS = NB + 1;
    __shared__ double rowb[2][NB], colb[2][NB];
    __shared__ double sgn[NB], piv[NB];
    __shared__ int s_fail;
    const int tid = threadIdx.x, ta = tid & 15, tc = tid >> 4;
    if (*status != 0) return;
    cqr_stamp(0);
    double x[E][E];
#pragma unroll
    for (int p = 0; p < E; ++p)
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const int a = ta + 16 * p, c = tc + 16 * q;
            x[p][q] = (a < bb && c < bb) ? -qtop[a + (int64_t)c * ldqt] : (a == c ? 1.0 : 0.0);
        }
    if (tid == 0) s_fail = 0;
    cqr_stamp(1);
    // row 0 and column 0
    if (ta == 0) {
#pragma unroll
        for (int q = 0; q < E; ++q) rowb[0][tc + 16 * q] = x[0][q];
    }
    if (tc == 0) {
#pragma unroll
        for (int p = 0; p < E; ++p) colb[0][ta + 16 * p] = x[p][0];
    }
    __syncthreads();
    // publish row / column jn (values after the step that precedes it)
    // (jb is a compile-time constant at every call: the register tile of row /
    // column jn is x[jb] or x[jb + 1])
    auto publish = [&](int jn, int jb, int s) {
        if (jn >= bb) return;
        const int pb = (s < 15) ? jb : (jb + 1 < E ? jb + 1 : jb);
        if (ta == (jn & 15)) {
            if (pb == jb) {
#pragma unroll
                for (int q = 0; q < E; ++q) rowb[jn & 1][tc + 16 * q] = x[jb][q];
            } else {
#pragma unroll
                for (int q = 0; q < E; ++q) rowb[jn & 1][tc + 16 * q] = x[jb + 1 < E ? jb + 1 : jb][q];
            }
        }
        if (tc == (jn & 15)) {
            if (pb == jb) {
#pragma unroll
                for (int p = 0; p < E; ++p) colb[jn & 1][ta + 16 * p] = x[p][jb];
            } else {
#pragma unroll
                for (int p = 0; p < E; ++p) colb[jn & 1][ta + 16 * p] = x[p][jb + 1 < E ? jb + 1 : jb];
            }
        }
    };
    // ---- LU without pivoting of S - Qtop (S added to each pivot) -----------
#pragma unroll
    for (int jb = 0; jb < E; ++jb) {
        if (16 * jb >= bb) break;
        for (int s = 0; s < 16; ++s) {
            const int j = 16 * jb + s;
            if (j >= bb) break;
            const double *rb = rowb[j & 1], *cb = colb[j & 1];
            const double xjj = rb[j];
            const double sj = (xjj < 0.0) ? -1.0 : 1.0;
            const double pv = xjj + sj;
            const double ip = fast_rcp(pv);
            if (tid == 0) {
                sgn[j] = sj;
                piv[j] = pv;
                if (!isfinite(xjj)) s_fail = 1;
            }
            double lv[E], rv[E];
#pragma unroll
            for (int p = jb; p < E; ++p) lv[p] = cb[ta + 16 * p] * ip;  // L(a, j)
#pragma unroll
            for (int q = jb; q < E; ++q) rv[q] = rb[tc + 16 * q];      // U(j, c)
#pragma unroll
            for (int p = jb; p < E; ++p) {
                const int a = ta + 16 * p;
#pragma unroll
                for (int q = jb; q < E; ++q) {
                    const int c = tc + 16 * q;
                    const bool arow = (p > jb) || (a > j);
                    if (q > jb) {
                        if (arow) x[p][q] = fma(-lv[p], rv[q], x[p][q]);
                    } else if (arow) {
                        if (c > j) x[p][q] = fma(-lv[p], rv[q], x[p][q]);
                        else if (c == j) x[p][q] = lv[p];
                    }
                }
            }
            publish(j + 1, jb, s);
            __syncthreads();
        }
    }
    cqr_stamp(2);
    if (s_fail) {
        if (tid == 0) *status = 1;
        return;
    }
    // Two CTAs (gridDim.x == 2) run the same LU; CTA 0 then writes the
    // factorization outputs and inverts L, CTA 1 inverts U (half the sweep's
    // work each).  One CTA does all of it.
    const bool do_low = (blockIdx.x == 0), do_up = (blockIdx.x == gridDim.x - 1);
    // ---- outputs of the factorization (before the in-place inversions) ------
#pragma unroll
    for (int p = 0; p < E; ++p)
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const int a = ta + 16 * p, c = tc + 16 * q;
            if (do_low && a < bb && c < bbpad) {
                const double xv = x[p][q];
                const double lvv = (a > c && c < bb) ? xv : (a == c ? 1.0 : 0.0);
                if (c < bb) A[a + (int64_t)c * lda] = (a > c) ? xv : sgn[a] * Rc[a + (int64_t)c * bbpad];
                rc_img[c + a * LS] = lvv;  // vt(c, a)
                vfull[a + (int64_t)c * ldq] = lvv;
            }
            if (do_low && a < bbpad && c < bbpad) {
                const double u = (a < c) ? x[p][q] : piv[c < bb ? c : 0];
                us[a + (int64_t)c * bbpad] = (a <= c && c < bb) ? u * sgn[c] : 0.0;
            }
            if (a == c && a < bb) x[p][q] = piv[a];  // U(j, j) = the Schur pivot
        }
    if (do_low)
        for (int c = tid; c < bb; c += RG_THREADS) tau[c] = piv[c] * sgn[c];
    __syncthreads();
    if (do_low)
    for (int e = tid; e < bb * bbpad; e += RG_THREADS) {  // vt: bbpad x bb (rows of Vt = columns of V)
        const int r = e % bbpad, c = e / bbpad;
        vt[r + (int64_t)c * bbpad] = rc_img[r + c * LS];
    }
    // row 0 / column 0 of the factored square for the inversion sweep
    __syncthreads();
    cqr_stamp(3);
    if (ta == 0) {
#pragma unroll
        for (int q = 0; q < E; ++q) rowb[0][tc + 16 * q] = x[0][q];
    }
    if (tc == 0) {
#pragma unroll
        for (int p = 0; p < E; ++p) colb[0][ta + 16 * p] = x[p][0];
    }
    __syncthreads();
    // ---- L^{-1} (strict lower, unit) and U^{-1} (upper), one sweep ----------
    // step j:  lower  Y(a, c) = [c < j] Y(a, c) - L(a, j) [c == j ? 1 : Y(j, c)]   (a > j, c <= j)
    //          upper  column j of Z = U^{-1} completes: Z(r, j) = -acc(r, j) / U(j, j) (r < j),
    //                 Z(j, j) = 1 / U(j, j);  acc(r, a) = [r < j] acc(r, a) + Z(r, j) U(j, a)
    //                 (r <= j, a > j)
#pragma unroll
    for (int jb = 0; jb < E; ++jb) {
        if (16 * jb >= bb) break;
        for (int s = 0; s < 16; ++s) {
            const int j = 16 * jb + s;
            if (j >= bb) break;
            const double *rb = rowb[j & 1], *cb = colb[j & 1];
            const double iu = fast_rcp(rb[j]);  // 1 / U(j, j)
            // one column array (rows a > j: -L(a, j); a < j: Z(a, j) = -acc(a, j) / U(j, j);
            // a = j: Z(j, j)) and one row array (c <= j: Y(j, c) with Y(j, j) = 1;
            // c > j: U(j, c)): the lower and upper updates use disjoint halves
            double cv[E], rv[E];
#pragma unroll
            for (int p = 0; p < E; ++p) {
                const int a = ta + 16 * p;
                const double v = cb[a];
                cv[p] = (a > j) ? -v : ((a < j) ? -v * iu : iu);
            }
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int c = tc + 16 * q;
                rv[q] = (c == j) ? 1.0 : rb[c];
            }
#pragma unroll
            for (int p = 0; p < E; ++p) {
                const int a = ta + 16 * p;
#pragma unroll
                for (int q = 0; q < E; ++q) {
                    const int c = tc + 16 * q;
                    if (do_low && p >= jb && q <= jb) {  // lower part: a > j, c <= j
                        const bool arow = (p > jb) || (a > j);
                        const bool ccol = (q < jb) || (c <= j);
                        if (arow && ccol) x[p][q] = fma(cv[p], rv[q], (q == jb && c == j) ? 0.0 : x[p][q]);
                    }
                    if (do_up && p <= jb && q >= jb) {  // upper part: a <= j, c > j; column j finalised
                        const bool arow = (p < jb) || (a <= j);
                        if (arow) {
                            if (q > jb) x[p][q] = fma(cv[p], rv[q], (p == jb && a == j) ? 0.0 : x[p][q]);
                            else if (c > j) x[p][q] = fma(cv[p], rv[q], (p == jb && a == j) ? 0.0 : x[p][q]);
                            else if (c == j) x[p][q] = cv[p];
                        }
                    }
                }
            }
            publish(j + 1, jb, s);
            __syncthreads();
        }
    }
    cqr_stamp(4);
    // ---- U^{-1} and L^{-T} (transposed through the shared-memory image) -------
#pragma unroll
    for (int p = 0; p < E; ++p)
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const int a = ta + 16 * p, c = tc + 16 * q;
            if (do_up && a < bbpad && c < bbpad) Uinv[a + (int64_t)c * bbpad] = (a <= c && c < bb) ? x[p][q] : 0.0;
            // L^{-T}(c, a) = Y(a, c) from the strict lower element (a, c)
            rc_img[c + a * LS] = (a > c) ? ((a < bb) ? x[p][q] : 0.0) : ((a == c && a < bb) ? 1.0 : 0.0);
        }
    __syncthreads();
    if (do_low)
    for (int e = tid; e < bbpad * bbpad; e += RG_THREADS) {
        const int r = e % bbpad, c = e / bbpad;
        linvt[e] = rc_img[r + c * LS];
    }
    // CTA 1 (the U^{-1} one) also forms C = R2^{-1} U^{-1} for V2 = -Q1bottom C:
    // both upper triangular, packed in shared memory, register-grid product with
    // the 16-row t blocks pruned to p <= tb <= q (as the Cholesky's Rc product)
    if (do_up && cmat) {
        __syncthreads();  // (one CTA: the L^{-T} copy above still reads the image)
        double *S2 = rc_img, *S1 = rc_img + NB * (NB + 1) / 2;
#pragma unroll
        for (int p = 0; p < E; ++p)
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int a = ta + 16 * p, c = tc + 16 * q;
                if (a <= c) {
                    S2[upk(a, c)] = (c < bb) ? r2inv[a + (int64_t)c * bbpad] : 0.0;
                    S1[upk(a, c)] = (c < bb) ? x[p][q] : 0.0;
                }
            }
        __syncthreads();
        double acc[E][E];
#pragma unroll
        for (int p = 0; p < E; ++p)
#pragma unroll
            for (int q = 0; q < E; ++q) acc[p][q] = 0.0;
#pragma unroll
        for (int tb = 0; tb < E; ++tb) {
            for (int s = 0; s < 16; ++s) {
                const int t = 16 * tb + s;
                double r2[E], r1[E];
#pragma unroll
                for (int p = 0; p <= tb; ++p) {
                    const int a = ta + 16 * p;
                    r2[p] = (a <= t) ? S2[upk(a, t)] : 0.0;
                }
#pragma unroll
                for (int q = tb; q < E; ++q) {
                    const int c = tc + 16 * q;
                    r1[q] = (t <= c) ? S1[upk(t, c)] : 0.0;
                }
#pragma unroll
                for (int p = 0; p <= tb; ++p)
#pragma unroll
                    for (int q = tb; q < E; ++q) acc[p][q] = fma(r2[p], r1[q], acc[p][q]);
            }
        }
#pragma unroll
        for (int p = 0; p < E; ++p)
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int a = ta + 16 * p, c = tc + 16 * q;
                if (a < bbpad && c < bbpad) cmat[a + (int64_t)c * bbpad] = (a <= c && c < bb) ? acc[p][q] : 0.0;
            }
    }
    cqr_stamp(5);
}

}  // namespace rq
