// gemm_dmma.cuh -- the FP64 tensor-core (DMMA) contraction used by every
// dense step of the hot path:
//   S1 sketch           B  = Omega A        X = Omega^T, Y = A
//   S5 W                W  = V^T A22          (PDLARFB P:761)  X = V, Y = A22
//   S5 W2               W2 = -T^T W                          X = -T,  Y = W
//   S5 update           A22 += V W2  (i.e. A22 - V T^T V^T A22)       X = W2, Y = V^T
// All four are "C = X^T Y" with both operands K-contiguous (column-major
// K x M and K x N), which is the layout the m8n8k4 fragments want:
// A[m][k] = X[k + m ldx], B[k][n] = Y[k + n ldy].
//
// Tiling: CTA tile BM x BN = (8 MT WM) x (8 NT WN), warps WM x WN, each warp
// MT x NT tiles of 8x8.  K is staged through shared memory by cp.async in
// BK-deep stages (STAGES-deep pipeline).  Shared layout per stage and
// operand: [BK/8][rows][8] doubles, so a quarter-warp's double2 fragment
// loads (rows r, r+1 x 4 chunks) cover 128 contiguous bytes: conflict-free.
// Each double2 feeds two DMMAs (even k, odd k): the 8 k-values of a k8 block
// are consumed as two k4 MMAs with the same permutation on both operands.
//
// Epilogues: STORE (C = acc), PARTIAL (split-K slice to workspace, summed
// later in fixed order -> deterministic), ACCUM_T (C^T += acc: element (m, n)
// of the product is added to C[n + m ldc]; used by the trailing update where
// the product is A22^T's tile).
#pragma once
#include "common.cuh"

namespace rq {

enum GemmEpi { EPI_STORE = 0, EPI_PARTIAL = 1, EPI_ACCUM_T = 2, EPI_ACCUM_T_PRE = 3 };

struct GemmArgs {
    int64_t M, N, K;
    const double *X;
    int64_t ldx;
    const double *Y;
    int64_t ldy;
    double *C;
    int64_t ldc;
    int64_t k_per_split;  // multiple of BK
    int64_t split_stride; // elements between split-K partial slices (EPI_PARTIAL)
};

template <int MT, int NT, int WM, int WN, int BK, int STAGES, int EPI>
__global__ void __launch_bounds__(WM *WN * 32) gemm_tn_kernel(GemmArgs g) {
    constexpr int BM = 8 * MT * WM;
    constexpr int BN = 8 * NT * WN;
    constexpr int NTHR = WM * WN * 32;
    constexpr int KB = BK / 8;
    constexpr int XS = KB * BM * 8;  // doubles per stage, X operand
    constexpr int YS = KB * BN * 8;
    extern __shared__ __align__(16) double smem[];
    double *xs = smem;
    double *ys = smem + STAGES * XS;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp / WN, wn = warp % WN;
    const int64_t m0 = (int64_t)blockIdx.y * BM;
    const int64_t n0 = (int64_t)blockIdx.x * BN;
    const int64_t kbeg = (int64_t)blockIdx.z * g.k_per_split;
    const int64_t kend = min(g.K, kbeg + g.k_per_split);
    const int64_t nk = (kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;

    auto load_stage = [&](int stage, int64_t kt) {
        const int64_t k0 = kbeg + kt * BK;
        double *xd = xs + stage * XS;
        double *yd = ys + stage * YS;
        // element e -> (row, k): consecutive threads walk k (contiguous in global)
#pragma unroll 4
        for (int e = tid; e < BM * BK; e += NTHR) {
            const int r = e / BK, k = e % BK;
            const int64_t gm = m0 + r, gk = k0 + k;
            const bool ok = (gm < g.M) && (gk < kend);
            const double *src = ok ? (g.X + gk + gm * g.ldx) : g.X;
            cp_async8(xd + ((k >> 3) * BM + r) * 8 + (k & 7), src, ok);
        }
#pragma unroll 4
        for (int e = tid; e < BN * BK; e += NTHR) {
            const int r = e / BK, k = e % BK;
            const int64_t gn = n0 + r, gk = k0 + k;
            const bool ok = (gn < g.N) && (gk < kend);
            const double *src = ok ? (g.Y + gk + gn * g.ldy) : g.Y;
            cp_async8(yd + ((k >> 3) * BN + r) * 8 + (k & 7), src, ok);
        }
    };

    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int fr = lane >> 2;        // fragment row within an 8x8 tile
    const int fk = (lane & 3) * 2;   // fragment k pair within a k8 block
    // EPI_ACCUM_T_PRE: the C tile (A22^T) is loaded into registers before the
    // K loop, so its HBM latency overlaps the DMMAs instead of the epilogue.
    double cpre[EPI == EPI_ACCUM_T_PRE ? MT : 1][EPI == EPI_ACCUM_T_PRE ? NT : 1][2];
    if (EPI == EPI_ACCUM_T_PRE) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int64_t gm = m0 + wm * 8 * MT + i * 8 + fr;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t gn = n0 + wn * 8 * NT + j * 8 + fk + h;
                    cpre[i][j][h] = (gm < g.M && gn < g.N) ? g.C[gn + gm * g.ldc] : 0.0;
                }
        }
    }

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }

    for (int64_t kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        // refill the slot consumed in iteration kt-1 (everyone is past it)
        {
            const int64_t nxt = kt + STAGES - 1;
            if (nxt < nk) load_stage((int)(nxt % STAGES), nxt);
            cp_async_commit();
        }
        const int stage = (int)(kt % STAGES);
        const double *xd = xs + stage * XS;
        const double *yd = ys + stage * YS;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            double2 a[MT], b[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i)
                a[i] = *reinterpret_cast<const double2 *>(xd + (kb * BM + wm * 8 * MT + i * 8 + fr) * 8 + fk);
#pragma unroll
            for (int j = 0; j < NT; ++j)
                b[j] = *reinterpret_cast<const double2 *>(yd + (kb * BN + wn * 8 * NT + j * 8 + fr) * 8 + fk);
            // all even-k MMAs, then all odd-k ones: MT*NT independent
            // accumulators between two dependent DMMAs (hides DMMA latency)
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
        }
    }
    cp_async_wait<0>();

    // epilogue: thread holds C[fr][2(lane&3) + {0,1}] of each 8x8 tile
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int64_t gm = m0 + wm * 8 * MT + i * 8 + fr;
        if (gm >= g.M) continue;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gn = n0 + wn * 8 * NT + j * 8 + fk + h;
                if (gn >= g.N) continue;
                if (EPI == EPI_STORE) {
                    g.C[gm + gn * g.ldc] = acc[i][j][h];
                } else if (EPI == EPI_PARTIAL) {
                    g.C[(int64_t)blockIdx.z * g.split_stride + gm + gn * g.M] = acc[i][j][h];
                } else if (EPI == EPI_ACCUM_T) {
                    double *c = g.C + gn + gm * g.ldc;
                    *c = *c + acc[i][j][h];
                } else {  // EPI_ACCUM_T_PRE
                    g.C[gn + gm * g.ldc] = cpre[i][j][h] + acc[i][j][h];
                }
            }
        }
    }
}

// Fixed-order sum of split-K slices: C[m + n ldc] = sum_s P[s][m + n M].
__global__ void splitk_reduce_kernel(const double *P, int64_t M, int64_t N, int splits, int64_t stride, double *C,
                                     int64_t ldc) {
    const int64_t total = M * N;
    // pairs of consecutive elements (same column: M even) by 16-byte loads / stores
    const bool vec = ((M | ldc | stride) & 1) == 0 && ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(C)) & 15) == 0;
    if (vec) {
        for (int64_t e = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); e < total;
             e += 2 * (int64_t)gridDim.x * blockDim.x) {
            // slices added in order q = 0, 1, ... (fixed: deterministic)
            double s0 = 0.0, s1 = 0.0;
            int q = 0;
            for (; q + 4 <= splits; q += 4) {
                double2 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const double2 *>(P + (int64_t)(q + u) * stride + e);
#pragma unroll
                for (int u = 0; u < 4; ++u) { s0 += v[u].x; s1 += v[u].y; }
            }
            for (; q < splits; ++q) {
                const double2 v = *reinterpret_cast<const double2 *>(P + (int64_t)q * stride + e);
                s0 += v.x;
                s1 += v.y;
            }
            const int64_t m = e % M, n = e / M;
            *reinterpret_cast<double2 *>(C + m + n * ldc) = make_double2(s0, s1);
        }
        return;
    }
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        // slices added in order q = 0, 1, ... (fixed: deterministic); loads in
        // batches of 8 so a many-slice reduce is not one L2 latency per slice
        double s = 0.0;
        int q = 0;
        for (; q + 8 <= splits; q += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = P[(int64_t)(q + u) * stride + e];
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; q < splits; ++q) s += P[(int64_t)q * stride + e];
        const int64_t m = e % M, n = e / M;
        C[m + n * ldc] = s;
    }
}

}  // namespace rq
