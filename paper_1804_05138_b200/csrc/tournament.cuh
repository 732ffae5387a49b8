// tournament.cuh -- tournament pivoting on the sample (the paper's future
// work; reading R-TP of DESIGN.md), on top of the S2 kernels:
//   groups: position c of the panel's trailing sample belongs to group
//     ((i + c) / b) mod G (the columns one rank owns in a G-rank block-cyclic
//     layout); each group's columns are gathered and reduced to <= bb
//     candidates by the sample QRCP kernels (Alg. 1);
//   merges: pairs (g, g + span), span = 1, 2, 4, ...: the union (left list,
//     then right list) of ORIGINAL sample columns, zero-padded to 2 bb, is
//     reduced to bb candidates by the sample QRCP again; the root's pivot
//     order is the panel's pivot order, and its reflectors V-hat, tau-hat and
//     R-hat11 are the Householder QR of the sample's chosen columns;
//   the sample becomes R-hat = Q-hat^T B by three DMMA contractions (driver),
//   and tp_finish_kernel writes perm, the (dst <- src) moves and the panel
//   state exactly as the S2 kernels do, so S3-S6 run unchanged.
#pragma once
#include "common.cuh"
#include "dist.cuh"

namespace rq {

// S(:, q) = B(:, pos_q), idx[q] = pos_q for the n_g columns of group g
// (positions relative to the panel start i, ascending)
__global__ void tp_gather_group_kernel(const double *B, int64_t ldb, int lpad, int64_t i, int b, int G, int g,
                                       int64_t lq0, int64_t ng, double *S, int64_t *idx) {
    const int64_t total = ng * lpad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % lpad);
        const int64_t q = e / lpad;
        const int64_t pos = dist_global(lq0 + q, b, G, g) - i;
        S[r + q * lpad] = B[r + pos * ldb];
        if (r == 0) idx[q] = pos;
    }
}

// cand[q] = idx[perm[q]] for q < *cnt_in (the selection of one QRCP), *cnt_out
__global__ void tp_collect_kernel(const int64_t *perm, const int *cnt_in, const int64_t *idx, int64_t *cand,
                                  int *cnt_out) {
    const int c = *cnt_in;
    for (int q = threadIdx.x; q < c; q += blockDim.x) cand[q] = idx[perm[q]];
    if (threadIdx.x == 0) *cnt_out = c;
}

// U(:, q) = B(:, u_q) for the union u = [candL(0:cntL), candR(0:cntR)],
// zero columns up to ncols (the padded width the QRCP runs on); uidx likewise
__global__ void tp_union_kernel(const double *B, int64_t ldb, int lpad, const int64_t *candL, const int *cntL,
                                const int64_t *candR, const int *cntR, int ncols, double *U, int64_t *uidx) {
    const int nl = *cntL, nr = *cntR;
    const int total = ncols * lpad;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int r = e % lpad, q = e / lpad;
        int64_t pos = -1;
        if (q < nl) pos = candL[q];
        else if (q - nl < nr) pos = candR[q - nl];
        U[r + (int64_t)q * lpad] = (pos >= 0) ? B[r + pos * ldb] : 0.0;
        if (r == 0) uidx[q] = pos;
    }
}

// vt (bbpad x lpad) = vhat^T (vhat: lpad x bbpad)
__global__ void tp_transpose_kernel(const double *vhat, int lpad, int bbpad, double *vt) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < lpad * bbpad; e += gridDim.x * blockDim.x) {
        const int r = e % lpad, c = e / lpad;
        vt[c + r * bbpad] = vhat[e];
    }
}

__global__ void tp_iota_kernel(int64_t *perm, int64_t n) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        perm[e] = e;
}

// The chosen positions F[0..cnt) (root pivot order) as transpositions
// j <-> current position of F[j], in order (reading R-G5): perm of the touched
// positions (the rest stays the identity written by tp_iota_kernel), the
// (dst <- src) moves, and the panel state (bb_eff, rank, done) -- what the S2
// kernels leave.  One warp; the <= 2 bb touched positions are kept in shared
// memory (position -> its current original column).  No-op (bb_eff = 0) when
// the factorization has stopped.
__global__ void tp_finish_kernel(const int64_t *F, const int *cnt, int bb, const int *status, int *done, int *bb_eff,
                                 int *rank, int64_t *perm, int64_t *mdst, int64_t *msrc, int *np) {
    __shared__ int64_t tpos[2 * 128 + 2], torig[2 * 128 + 2];
    __shared__ int s_nt;
    const int lane = threadIdx.x;
    if (*status != 0 || *done) {
        if (lane == 0) { *bb_eff = 0; *np = 0; }
        return;
    }
    const int c = *cnt;
    if (lane == 0) s_nt = 0;
    __syncwarp();
    // content(p): the original column now at position p
    auto find = [&](int64_t p) -> int {
        int found = -1;
        for (int e0 = 0; e0 < s_nt; e0 += 32) {
            const int e = e0 + lane;
            const unsigned msk = __ballot_sync(0xffffffffu, e < s_nt && tpos[e] == p);
            if (msk) { found = e0 + __ffs(msk) - 1; break; }
        }
        return found;
    };
    for (int j = 0; j < c; ++j) {
        // where is original column F[j] now?  (it is untouched, or recorded)
        const int64_t want = F[j];
        int64_t s = want;
        {
            int found = -1;
            for (int e0 = 0; e0 < s_nt; e0 += 32) {
                const int e = e0 + lane;
                const unsigned msk = __ballot_sync(0xffffffffu, e < s_nt && torig[e] == want);
                if (msk) { found = e0 + __ffs(msk) - 1; break; }
            }
            if (found >= 0) s = tpos[found];
        }
        if (s != j) {
            const int ej = find(j), es = find(s);
            const int64_t cj = (ej >= 0) ? torig[ej] : j;
            const int64_t cs = (es >= 0) ? torig[es] : s;
            __syncwarp();
            if (lane == 0) {
                int n_ = s_nt;
                if (ej >= 0) torig[ej] = cs; else { tpos[n_] = j; torig[n_] = cs; ++n_; }
                if (es >= 0) torig[es] = cj; else { tpos[n_] = s; torig[n_] = cj; ++n_; }
                s_nt = n_;
            }
            __syncwarp();
        }
    }
    __syncwarp();
    int nm = 0;
    for (int e = 0; e < s_nt; ++e) {
        const int64_t p = tpos[e], o = torig[e];
        if (lane == 0) {
            perm[p] = o;
            if (o != p) { mdst[nm] = p; msrc[nm] = o; }
        }
        if (o != p) ++nm;
    }
    if (lane == 0) {
        *np = nm;
        *bb_eff = c;
        *rank += c;
        if (c < bb) *done = 1;
    }
}

}  // namespace rq
