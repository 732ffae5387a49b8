// moves.cuh -- S3 (kernel K5) as pack / exchange / unpack of whole columns,
// the same code for one GPU and for the 1D column-block-cyclic layout of
// SURVEY.md §8(e), and the per-panel helpers around the panel buffer.
//
// The sample QRCP (S2) leaves, on the device, its bb_eff transpositions
// (applied in order, reading R-G5) as
//   perm[q]            the ORIGINAL trailing position whose column ends at
//                      position q (q < bb: the panel slots),
//   (dst <- src) moves over the <= 2 bb touched positions.
// Two facts of the transposition sequence j <-> s_j (s_j >= j, j = 0..bb-1)
// make the exchange a fixed-size one:
//   (a) every column that ends in a slot q < bb comes from position perm[q];
//   (b) every touched position dst >= bb receives an ORIGINAL slot column
//       (src < bb): a column from >= bb only ever moves into a slot, and a
//       slot is final after its own step.
// So panel t ("swap ... in A, Pi" then the panel QR) is
//   pack:      Pbuf(:, q) = A(:, perm[q])          (full height m; on P > 1
//              each rank packs the slots it owns, zeros elsewhere, and an
//              integer-sum reduce delivers the exact bits to the owner)
//   [narrow:   Pbuf(i:m, :) += V_prev W2_prev(:, perm) -- look-ahead only]
//   panel QR on Pbuf(i:m, :)                       (owner)
//   displaced: A(:, dst) = A_slot(:, src) for dst >= bb (owner broadcasts its
//              bb slot columns on P > 1)
//   copy back: A(:, slot q) = Pbuf(:, q)           (owner)
//   jpvt:      the same moves on the replicated jpvt.
// Full-height columns move (earlier R12 rows move with them, LAPACK
// semantics, as swap_fused_kernel did).
#pragma once
#include "common.cuh"
#include "dist.cuh"

namespace rq {

// dst[r] = src[r] (or 0 when !own) for r < m over the grid's x dimension;
// 16-byte accesses when both columns are 16-byte aligned (the leading
// dimensions are even on every path the bench takes).
RQ_DEV void copy_col(double *dst, const double *src, int64_t m, bool own = true) {
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, ts = (int64_t)gridDim.x * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const int64_t m2 = m >> 1;
        double2 *d2 = reinterpret_cast<double2 *>(dst);
        const double2 *s2 = reinterpret_cast<const double2 *>(src);
        int64_t r = t0;
        for (; r + 3 * ts < m2; r += 4 * ts) {  // four 16-byte loads in flight per thread
            double2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = own ? s2[r + u * ts] : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < 4; ++u) d2[r + u * ts] = v[u];
        }
        for (; r < m2; r += ts) d2[r] = own ? s2[r] : make_double2(0.0, 0.0);
        if ((m & 1) && t0 == 0) dst[m - 1] = own ? src[m - 1] : 0.0;
    } else {
        for (int64_t r = t0; r < m; r += ts) dst[r] = own ? src[r] : 0.0;
    }
}

// Pbuf(:, q) = A(:, local(i + perm[q])) for the slots this rank owns (zeros
// otherwise); W2g(:, q) = W2(:, local - lj0w) likewise when w2 != nullptr (the
// look-ahead's narrow update; lj0w = first local trailing column of the
// previous panel).  No-op when *bb_eff == 0 (the factorization has stopped).
__global__ void pack_pivots_kernel(const double *A, int64_t lda, int64_t m, int64_t i, const int64_t *perm, int bb,
                                   const int *bb_eff, int b, int P, int me, double *pbuf, int64_t ldp,
                                   const double *w2, int64_t ldw2, int w2rows, int64_t lj0w, double *w2g) {
    if (*bb_eff == 0) return;
    const int q = blockIdx.y;
    if (q >= bb) return;
    const int64_t jg = i + perm[q];
    const bool own = dist_owner(jg, b, P) == me;
    const int64_t lj = own ? dist_local(jg, b, P) : 0;
    copy_col(pbuf + (int64_t)q * ldp, A + lj * lda, m, own);
    if (w2 && blockIdx.x == 0)
        for (int r = threadIdx.x; r < w2rows; r += blockDim.x)
            w2g[r + (int64_t)q * w2rows] = own ? w2[r + (lj - lj0w) * ldw2] : 0.0;
}

// dispbuf(:, q) = A(:, ljs + q), q < bb: the owner's original slot columns
// (after the trailing update of the previous panel).
__global__ void pack_slots_kernel(const double *A, int64_t lda, int64_t m, int64_t ljs, int bb, const int *bb_eff,
                                  double *dispbuf, int64_t ldd) {
    if (*bb_eff == 0) return;
    const int q = blockIdx.y;
    if (q >= bb) return;
    copy_col(dispbuf + (int64_t)q * ldd, A + (ljs + q) * lda, m);
}

// A(:, local(i + dst)) = S(:, src) for the moves with dst >= bb whose
// destination this rank owns; S = dispbuf (ld lds), or on one GPU the slot
// columns of A itself (S = A + i lda, lds = lda: by fact (b) the sources
// are slots and the destinations are not, so reads and writes never meet).
__global__ void place_displaced_kernel(double *A, int64_t lda, int64_t m, int64_t i, const int64_t *mdst,
                                       const int64_t *msrc, const int *np, int bb, const int *bb_eff, int b, int P,
                                       int me, const double *S, int64_t lds) {
    if (*bb_eff == 0) return;
    const int e = blockIdx.y;
    if (e >= *np) return;
    const int64_t d = mdst[e], s = msrc[e];
    if (d < bb) return;
    const int64_t jg = i + d;
    if (dist_owner(jg, b, P) != me) return;
    copy_col(A + dist_local(jg, b, P) * lda, S + s * lds, m);
}

// A(:, ljs + q) = Pbuf(:, q) (owner; all m rows)
__global__ void copy_back_kernel(double *A, int64_t lda, int64_t m, int64_t ljs, int bb, const int *bb_eff,
                                 const double *pbuf, int64_t ldp) {
    if (*bb_eff == 0) return;
    const int q = blockIdx.y;
    if (q >= bb) return;
    copy_col(A + (ljs + q) * lda, pbuf + (int64_t)q * ldp, m);
}

// replicated jpvt (+ i): the same moves; also the trace's per-panel pivots
__global__ void jpvt_moves_kernel(int64_t *jpvt, const int64_t *mdst, const int64_t *msrc, const int *np,
                                  const int *bb_eff, int bb, int64_t *piv_out) {
    __shared__ int64_t v[2 * 128 + 2];
    if (*bb_eff == 0) return;
    const int n = *np;
    for (int q = threadIdx.x; q < n; q += blockDim.x) v[q] = jpvt[msrc[q]];
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) jpvt[mdst[q]] = v[q];
    if (piv_out) {
        __syncthreads();
        for (int q = threadIdx.x; q < bb; q += blockDim.x) piv_out[q] = jpvt[q];
    }
}

// ||panel||_F^2 per column, fixed order (thread-strided rows, then a fixed
// tree): the R11-diagonal rank stop's scale (reading R-G12b).
__global__ void colsumsq_kernel(const double *P, int64_t ldp, int64_t rows, int bb, const int *bb_eff, double *out) {
    __shared__ double red[32];
    if (*bb_eff == 0) return;
    const int c = blockIdx.x;
    const double *x = P + (int64_t)c * ldp;
    // eight independent partial sums (eight loads in flight per thread), then a fixed tree
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int64_t step = (int64_t)blockDim.x;
    int64_t r = threadIdx.x;
    for (; r + 7 * step < rows; r += 8 * step) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = x[r + u * step];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += v[u] * v[u];
    }
    for (; r < rows; r += step) a[0] += x[r] * x[r];  // (constant index: a[] stays in registers)
    double s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) out[c] = t;
    }
    (void)bb;
}

// tol2 = (1e3 eps)^2 sum_c colss[c] (ascending c), then the caller compares
// beta_j^2 < tol2.  Written to *tol2 by one thread.
__global__ void panel_tol_kernel(const double *colss, int bb, const int *bb_eff, double *tol2) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (*bb_eff == 0) { *tol2 = 0.0; return; }
    double s = 0.0;
    for (int c = 0; c < bb; ++c) s += colss[c];
    const double eps = 0x1p-52;
    *tol2 = (1e3 * eps) * (1e3 * eps) * s;
}

// The R11-diagonal stop found in the panel at column jstop (< bb_eff): the
// panel kernel wrote *stop_col; fold it into the panel state (one thread,
// after the panel kernel): bb_eff = jstop, rank -= (old bb_eff - jstop), done.
__global__ void panel_stop_apply_kernel(const int *stop_col, int off, int *bb_eff, int *rank, int *done) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (*stop_col < 0) return;
    const int js = *stop_col + off;  // the column within the panel (blocked panels: + sub-panel offset)
    if (js >= *bb_eff) return;
    *rank -= (*bb_eff - js);
    *bb_eff = js;
    *done = 1;
}

// Blocked panel helpers: the columns a sub-panel factors, and zeros above the
// diagonal blocks of the explicit V / V^T (each sub-panel writes its rows only)
__global__ void sub_eff_kernel(const int *bb_eff, int c0, int w, int *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = min(w, max(0, *bb_eff - c0));
}
__global__ void zero_top_kernel(double *vfull, int64_t ldv, double *vt, int64_t ldvt, int bbpad) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bbpad * bbpad; e += gridDim.x * blockDim.x) {
        const int r = e % bbpad, c = e / bbpad;
        vfull[r + (int64_t)c * ldv] = 0.0;
        vt[c + (int64_t)r * ldvt] = 0.0;
    }
}

// ---------------------------------------------------------------------------
// Trace hook (rqrcp_factor_ex): snapshots of the sample in pivoted order.
// ---------------------------------------------------------------------------
// R-hat after S2: out(r, c) for c < nn (positions relative to i), r < l:
//   c < bbe: the R-hat11 column (upper, zeros below the diagonal);
//   c >= bbe: the transformed physical column perm[c] of the sample.
__global__ void trace_rhat_kernel(const double *B, int64_t ldb, const int64_t *perm, const double *rhat11, int bbpad,
                                  int l, int64_t nn, const int *bb_eff, double *out) {
    const int bbe = *bb_eff;
    const int64_t total = (int64_t)l * nn;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % l);
        const int64_t c = e / l;
        double v;
        if (c < bbe) v = (r <= c) ? rhat11[r + c * bbpad] : 0.0;
        else v = B[r + perm[c] * ldb];
        out[e] = v;
    }
}
// plain l x nn copy (ld ldb -> l)
__global__ void trace_copy_kernel(const double *B, int64_t ldb, int l, int64_t nn, double *out) {
    const int64_t total = (int64_t)l * nn;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = B[(e % l) + (e / l) * ldb];
}

}  // namespace rq
