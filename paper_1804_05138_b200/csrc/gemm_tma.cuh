// gemm_tma.cuh -- persistent FP64 DMMA contraction fed by TMA.
//
// Same product as gemm_dmma.cuh (C = X^T Y, both operands K-contiguous) but:
//  * operands are staged by the Tensor Memory Accelerator: per k8 block one
//    cp.async.bulk.tensor.2d of box {8 doubles, rows} lands a dense [rows][8]
//    slab -- exactly the conflict-free fragment layout -- and signals an
//    mbarrier with its byte count; out-of-range rows/columns are zero-filled
//    by the TMA unit (ragged M, N, K tails need no predication);
//  * the kernel is persistent (grid = #SMs): each CTA walks its tiles and
//    their K chunks as ONE stage stream, so the loads of the next tile are in
//    flight while the current tile finishes and stores its epilogue;
//  * EPI_ACCUM_T_PRE issues the C-tile loads (A22) into registers when a tile
//    starts, hiding HBM latency behind the tile's DMMAs.
// One elected thread issues the TMA copies; a __syncthreads per stage guards
// slot reuse (plus fence.proxy.async before the async-proxy overwrite).
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "gemm_dmma.cuh"

namespace rq {

struct TmaGemmArgs {
    int64_t M, N, K;       // product sizes
    int64_t xk0, xm0;      // operand X element (k, m) -> tensor coords (xk0 + k, xm0 + m)
    int64_t yk0, yn0;      // operand Y element (k, n) -> tensor coords (yk0 + k, yn0 + n)
    double *C;
    int64_t ldc;
    int64_t k_per_split;   // multiple of BK
    int splits;
    int64_t split_stride;
    int vec2;              // EPI_ACCUM_T_PRE: C 16-byte aligned with even ldc -> double2 accesses
    int *tile_ctr;         // DYN kernels: tiles are claimed from this zeroed counter (atomicAdd)
};

RQ_DEV unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

RQ_DEV void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
RQ_DEV void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
RQ_DEV void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
RQ_DEV void tma_load_2d(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <int MT, int NT, int WM, int WN, int BK, int ST>
constexpr size_t tma_gemm_smem() {
    return 128 + (size_t)ST * BK * (8 * MT * WM + 8 * NT * WN) * sizeof(double) + ST * sizeof(uint64_t);
}

// DYN: tiles are claimed dynamically (atomicAdd on g.tile_ctr) instead of the
// static stride-gridDim walk, so CTAs that become resident late (the GPU is
// shared with a concurrent kernel) simply take fewer tiles.  The producer
// thread records each stage's tile in shared memory and ends the stream with
// a data-less stage (tile -1).  Same per-tile arithmetic: same bits.
template <int MT, int NT, int WM, int WN, int BK, int ST, int EPI, bool DYN = false>
__global__ void __launch_bounds__(WM *WN * 32, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY, TmaGemmArgs g) {
    constexpr int BM = 8 * MT * WM;
    constexpr int BN = 8 * NT * WN;
    constexpr int KB = BK / 8;
    constexpr int XS = KB * BM * 8;  // doubles per stage
    constexpr int YS = KB * BN * 8;
    constexpr unsigned STAGE_BYTES = (unsigned)((XS + YS) * sizeof(double));
    // dynamic smem: [pad to 128 B][X stages][Y stages][ST mbarriers]
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // align through the shared-window offset so the pointer stays a shared
    // pointer (LDS, not generic LD) for the compiler
    const unsigned pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
    double *xs = reinterpret_cast<double *>(smem_raw + pad);
    double *ys = xs + ST * XS;
    uint64_t *full = reinterpret_cast<uint64_t *>(ys + ST * YS);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp / WN, wn = warp % WN;
    const int fr = lane >> 2, fk = (lane & 3) * 2;
    const int64_t tilesN = (g.N + BN - 1) / BN, tilesM = (g.M + BM - 1) / BM;
    const int64_t ntiles = tilesN * tilesM * g.splits;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // tile t -> (split, m-tile, n-tile); n fastest so concurrent CTAs share X
    struct It {
        int64_t t;
        int64_t kc, nk, m0, n0, kbeg;
        int split;
    };
    auto set_tile = [&](It &it, int64_t t) {
        it.t = t;
        it.kc = 0;
        if (t >= ntiles) return;
        const int64_t per = tilesN * tilesM;
        it.split = (int)(t / per);
        const int64_t r = t % per;
        it.m0 = (r / tilesN) * BM;
        it.n0 = (r % tilesN) * BN;
        it.kbeg = (int64_t)it.split * g.k_per_split;
        const int64_t kend = min(g.K, it.kbeg + g.k_per_split);
        it.nk = (kend > it.kbeg) ? (kend - it.kbeg + BK - 1) / BK : 0;
    };
    __shared__ int64_t stage_t[ST];  // DYN: the tile of each stage slot (-1: end of stream)
    auto next_tile = [&](int64_t cur) -> int64_t {
        if (DYN) return (int64_t)atomicAdd(g.tile_ctr, 1);
        return cur + gridDim.x;
    };
    auto advance = [&](It &it) {
        if (++it.kc >= it.nk) set_tile(it, next_tile(it.t));
    };
    auto issue = [&](const It &it, int slot) {
        const int64_t k0 = it.kbeg + it.kc * BK;
        if (DYN) stage_t[slot] = it.t;
        mbar_expect_tx(&full[slot], STAGE_BYTES);
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            tma_load_2d(xs + slot * XS + kb * BM * 8, &tmX, (int)(g.xk0 + k0 + kb * 8), (int)(g.xm0 + it.m0), &full[slot]);
            tma_load_2d(ys + slot * YS + kb * BN * 8, &tmY, (int)(g.yk0 + k0 + kb * 8), (int)(g.yn0 + it.n0), &full[slot]);
        }
    };

    It P, Cn;
    if (tid == 0) set_tile(P, DYN ? next_tile(0) : (int64_t)blockIdx.x);
    set_tile(Cn, blockIdx.x);
    // skip tiles with no K work (cannot happen for K >= 1, kept for safety)
    int64_t sp = 0, sc = 0;
    bool pend_end = DYN;  // DYN: the end-of-stream stage is still to be issued
    auto issue_end = [&](int slot) {  // DYN: a data-less stage carrying tile -1
        stage_t[slot] = -1;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&full[slot])) : "memory");
        pend_end = false;
    };
    if (tid == 0) {
        for (int s = 0; s < ST - 1; ++s) {
            if (P.t < ntiles) {
                issue(P, (int)(sp % ST));
                ++sp;
                advance(P);
            } else {
                if (DYN && pend_end) { issue_end((int)(sp % ST)); ++sp; }
                break;
            }
        }
    }

    double acc[MT][NT][2];
    double cpre[EPI == EPI_ACCUM_T_PRE ? MT : 1][EPI == EPI_ACCUM_T_PRE ? NT : 1][2];
    while (DYN || Cn.t < ntiles) {
        const int slot = (int)(sc % ST);
        mbar_wait(&full[slot], (unsigned)((sc / ST) & 1));
        __syncthreads();  // everyone is past stage sc-1: its slot may be refilled
        if (DYN) {
            const int64_t tt = stage_t[slot];
            if (tt < 0) break;  // uniform: every thread read the same slot
            if (Cn.kc == 0) set_tile(Cn, tt);
        }
        if (tid == 0) {
            if (P.t < ntiles) {
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                issue(P, (int)(sp % ST));
                ++sp;
                advance(P);
            } else if (DYN && pend_end) {
                issue_end((int)(sp % ST));
                ++sp;
            }
        }
        if (Cn.kc == 0) {
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            if (EPI == EPI_ACCUM_T_PRE) {
                const bool interior = g.vec2 && Cn.m0 + BM <= g.M && Cn.n0 + BN <= g.N;
                if (interior) {  // no predicates, 16-byte loads of (row, row+1) pairs
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const int64_t gm = Cn.m0 + wm * 8 * MT + i * 8 + fr;
#pragma unroll
                        for (int j = 0; j < NT; ++j) {
                            const int64_t gn = Cn.n0 + wn * 8 * NT + j * 8 + fk;
                            const double2 c2 = *reinterpret_cast<const double2 *>(g.C + gn + gm * g.ldc);
                            cpre[i][j][0] = c2.x;
                            cpre[i][j][1] = c2.y;
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const int64_t gm = Cn.m0 + wm * 8 * MT + i * 8 + fr;
#pragma unroll
                        for (int j = 0; j < NT; ++j)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int64_t gn = Cn.n0 + wn * 8 * NT + j * 8 + fk + h;
                                cpre[i][j][h] = (gm < g.M && gn < g.N) ? g.C[gn + gm * g.ldc] : 0.0;
                            }
                    }
                }
            }
        }
        const double *xd = xs + slot * XS;
        const double *yd = ys + slot * YS;
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
        if (Cn.kc == Cn.nk - 1) {
            // epilogue of this tile (stores overlap the next tile's loads)
            if (EPI == EPI_ACCUM_T_PRE && g.vec2 && Cn.m0 + BM <= g.M && Cn.n0 + BN <= g.N) {
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const int64_t gm = Cn.m0 + wm * 8 * MT + i * 8 + fr;
#pragma unroll
                    for (int j = 0; j < NT; ++j) {
                        const int64_t gn = Cn.n0 + wn * 8 * NT + j * 8 + fk;
                        *reinterpret_cast<double2 *>(g.C + gn + gm * g.ldc) =
                            make_double2(cpre[i][j][0] + acc[i][j][0], cpre[i][j][1] + acc[i][j][1]);
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < MT; ++i) {
                    const int64_t gm = Cn.m0 + wm * 8 * MT + i * 8 + fr;
                    if (gm >= g.M) continue;
#pragma unroll
                    for (int j = 0; j < NT; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int64_t gn = Cn.n0 + wn * 8 * NT + j * 8 + fk + h;
                            if (gn >= g.N) continue;
                            if (EPI == EPI_STORE) {
                                g.C[gm + gn * g.ldc] = acc[i][j][h];
                            } else if (EPI == EPI_PARTIAL) {
                                g.C[(int64_t)Cn.split * g.split_stride + gm + gn * g.M] = acc[i][j][h];
                            } else if (EPI == EPI_ACCUM_T_PRE) {
                                g.C[gn + gm * g.ldc] = cpre[i][j][h] + acc[i][j][h];
                            }
                        }
                }
            }
        }
        ++sc;
        if (DYN) {  // the next stage's tile comes from stage_t
            if (++Cn.kc >= Cn.nk) Cn.kc = 0;
        } else {
            advance(Cn);
        }
    }
}

}  // namespace rq

namespace rq {

// ---------------------------------------------------------------------------
// The S5 rank-bb update A22 += V W2 (as A22^T += W2^T Vt) with the C tile
// moved by TMA in both directions, so the compute warps issue no global
// loads or stores: per tile (BM = 64 columns x BN = 128 rows of A22) the
// elected thread loads the next tile's C into the other of two shared-memory
// buffers (16 boxes of {8 rows, 64 columns}: the fragment reads of a warp
// cover 512 contiguous bytes), the warps add their accumulators into the
// current buffer, and the elected thread stores it back with bulk tensor
// stores (out-of-range rows / columns are skipped by the TMA unit).
// Operands as in gemm_tma_kernel (persistent, one stage stream over tiles).
// ---------------------------------------------------------------------------
RQ_DEV void tma_store_2d(const CUtensorMap *tm, int c0, int c1, const void *src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(tm), "r"(c0),
                 "r"(c1), "r"(smem_u32(src))
                 : "memory");
}

template <int MT, int NT, int WM, int WN, int BK, int ST, int CB = 2>
constexpr size_t tma_upd_smem() {
    return 128 + (size_t)ST * BK * (8 * MT * WM + 8 * NT * WN) * sizeof(double) +
           CB * (size_t)(8 * MT * WM) * (8 * NT * WN) * sizeof(double) + (ST + 2) * sizeof(uint64_t);
}

// CB = 2: the next tile's C loads into the other buffer during this tile;
// CB = 1: one buffer, the next tile's load is issued once this tile's stores
// have read it (frees shared memory for a deeper operand ring)
template <int MT, int NT, int WM, int WN, int BK, int ST, int CB = 2>
__global__ void __launch_bounds__(WM *WN * 32, 1)
    gemm_upd_tma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                        const __grid_constant__ CUtensorMap tmC, TmaGemmArgs g) {
    constexpr int BM = 8 * MT * WM;  // columns of A22 per tile
    constexpr int BN = 8 * NT * WN;  // rows of A22 per tile
    constexpr int KB = BK / 8;
    constexpr int XS = KB * BM * 8;
    constexpr int YS = KB * BN * 8;
    constexpr int CS = BM * BN;      // doubles per C buffer: BN/8 slabs of [BM][8]
    constexpr unsigned STAGE_BYTES = (unsigned)((XS + YS) * sizeof(double));
    constexpr unsigned C_BYTES = (unsigned)(CS * sizeof(double));
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
    double *xs = reinterpret_cast<double *>(smem_raw + pad);
    double *ys = xs + ST * XS;
    double *cb = ys + ST * YS;  // [CB][CS]
    uint64_t *full = reinterpret_cast<uint64_t *>(cb + CB * CS);
    uint64_t *cfull = full + ST;  // [2]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp / WN, wn = warp % WN;
    const int fr = lane >> 2, fk = (lane & 3) * 2;
    const int64_t tilesN = (g.N + BN - 1) / BN, tilesM = (g.M + BM - 1) / BM;
    const int64_t ntiles = tilesN * tilesM;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
        mbar_init(&cfull[0], 1);
        mbar_init(&cfull[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    struct It {
        int64_t t, kc, nk, m0, n0;
    };
    auto set_tile = [&](It &it, int64_t t) {
        it.t = t;
        it.kc = 0;
        if (t >= ntiles) return;
        it.m0 = (t / tilesN) * BM;
        it.n0 = (t % tilesN) * BN;
        it.nk = (g.K + BK - 1) / BK;
    };
    auto advance = [&](It &it) {
        if (++it.kc >= it.nk) set_tile(it, it.t + gridDim.x);
    };
    auto issue = [&](const It &it, int slot) {
        const int64_t k0 = it.kc * BK;
        mbar_expect_tx(&full[slot], STAGE_BYTES);
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            tma_load_2d(xs + slot * XS + kb * BM * 8, &tmX, (int)(g.xk0 + k0 + kb * 8), (int)(g.xm0 + it.m0), &full[slot]);
            tma_load_2d(ys + slot * YS + kb * BN * 8, &tmY, (int)(g.yk0 + k0 + kb * 8), (int)(g.yn0 + it.n0), &full[slot]);
        }
    };
    // C tile of tile t into buffer b: BN/8 boxes {8 rows, BM columns} of A22
    auto issue_c = [&](int64_t t, int b) {
        const int64_t m0 = (t / tilesN) * BM, n0 = (t % tilesN) * BN;
        mbar_expect_tx(&cfull[b], C_BYTES);
#pragma unroll
        for (int s = 0; s < BN / 8; ++s)
            tma_load_2d(cb + b * CS + s * BM * 8, &tmC, (int)(n0 + 8 * s), (int)m0, &cfull[b]);
    };

    It P, Cn;
    set_tile(P, blockIdx.x);
    set_tile(Cn, blockIdx.x);
    int64_t sp = 0, sc = 0;
    if (tid == 0) {
        if (Cn.t < ntiles) issue_c(Cn.t, 0);
        for (int s = 0; s < ST - 1 && P.t < ntiles; ++s) {
            issue(P, (int)(sp % ST));
            ++sp;
            advance(P);
        }
    }
    int64_t ntile_local = 0;  // tiles this CTA has finished (buffer = ntile_local & 1)
    double acc[MT][NT][2];
    while (Cn.t < ntiles) {
        const int slot = (int)(sc % ST);
        mbar_wait(&full[slot], (unsigned)((sc / ST) & 1));
        __syncthreads();
        if (tid == 0 && P.t < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(P, (int)(sp % ST));
            ++sp;
            advance(P);
        }
        if (Cn.kc == 0) {
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            // CB = 2: the next tile's C into the other buffer (its previous
            // stores must have finished reading it)
            if (CB == 2 && tid == 0) {
                const int64_t tn = Cn.t + gridDim.x;
                if (tn < ntiles) {
                    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    issue_c(tn, (int)((ntile_local + 1) & 1));
                }
            }
        }
        const double *xd = xs + slot * XS;
        const double *yd = ys + slot * YS;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            double2 a[MT], b[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i)
                a[i] = *reinterpret_cast<const double2 *>(xd + (kb * BM + wm * 8 * MT + i * 8 + fr) * 8 + fk);
#pragma unroll
            for (int j = 0; j < NT; ++j)
                b[j] = *reinterpret_cast<const double2 *>(yd + (kb * BN + wn * 8 * NT + j * 8 + fr) * 8 + fk);
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
        }
        if (Cn.kc == Cn.nk - 1) {
            // epilogue: C (shared) += acc, then bulk tensor stores
            const int bsel = (CB == 2) ? (int)(ntile_local & 1) : 0;
            mbar_wait(&cfull[bsel], (unsigned)(((CB == 2) ? (ntile_local >> 1) : ntile_local) & 1));
            double *cbuf = cb + bsel * CS;
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const int cm = wm * 8 * MT + i * 8 + fr;  // column within the tile
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const int s = wn * NT + j;  // 8-row slab
                    double2 *p = reinterpret_cast<double2 *>(cbuf + s * BM * 8 + cm * 8 + fk);
                    double2 c2 = *p;
                    c2.x += acc[i][j][0];
                    c2.y += acc[i][j][1];
                    *p = c2;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
            if (tid == 0) {
#pragma unroll
                for (int s = 0; s < BN / 8; ++s)
                    tma_store_2d(&tmC, (int)(Cn.n0 + 8 * s), (int)Cn.m0, cbuf + s * BM * 8);
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                if (CB == 1) {  // the next tile's C into the same buffer once the stores have read it
                    const int64_t tn = Cn.t + gridDim.x;
                    if (tn < ntiles) {
                        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                        issue_c(tn, 0);
                    }
                }
            }
            ++ntile_local;
        }
        ++sc;
        advance(Cn);
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

}  // namespace rq

namespace rq {

// ---------------------------------------------------------------------------
// The S5 rank-bb update A22 += V W2 (as A22^T += W2^T Vt), warp-specialised:
//  * one producer warp streams the operand stages by TMA into a ring guarded
//    by full (transaction bytes) and empty (one arrive per consumer warp)
//    mbarriers -- no CTA-wide barrier anywhere in the main loop;
//  * each of the WM x WN consumer warps owns a 32 x 32 sub-tile of the C tile
//    and moves it ITSELF by TMA: its next tile's C is prefetched into the
//    other of two private shared-memory buffers while it computes, and its
//    finished sub-tile is added in shared memory and stored by bulk tensor
//    stores -- so one warp's epilogue overlaps the other warps' DMMAs (the
//    CTA-wide epilogue + per-stage __syncthreads of gemm_upd_tma_kernel cost
//    ~20% of the tensor pipe at C4, ncu).
// Same per-element arithmetic as every other update kernel: acc = sum over k
// (ascending, DMMA k4 steps) from zero, then C + acc.
// ---------------------------------------------------------------------------
template <int WM, int WN, int BK, int ST>
constexpr size_t upd_ws_smem() {
    return 128 + (size_t)ST * BK * (32 * WM + 32 * WN) * sizeof(double) + (size_t)WM * WN * 2 * 32 * 32 * sizeof(double) +
           (2 * ST + 2 * WM * WN) * sizeof(uint64_t);
}

RQ_DEV void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int WM, int WN, int BK, int ST>
__global__ void __launch_bounds__((WM * WN + 1) * 32, 1)
    gemm_upd_ws_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                       const __grid_constant__ CUtensorMap tmC /* box {8, 32} */, TmaGemmArgs g) {
    constexpr int MT = 4, NT = 4;
    constexpr int BM = 8 * MT * WM;  // columns of A22 per tile
    constexpr int BN = 8 * NT * WN;  // rows of A22 per tile
    constexpr int KB = BK / 8;
    constexpr int XS = KB * BM * 8;
    constexpr int YS = KB * BN * 8;
    constexpr int CW = 32 * 32;      // doubles per warp C buffer: 4 slabs of [32 cols][8 rows]
    constexpr int NCW = WM * WN;     // consumer warps
    constexpr unsigned STAGE_BYTES = (unsigned)((XS + YS) * sizeof(double));
    constexpr unsigned CW_BYTES = (unsigned)(CW * sizeof(double));
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
    double *xs = reinterpret_cast<double *>(smem_raw + pad);
    double *ys = xs + ST * XS;
    double *cb = ys + ST * YS;  // [NCW][2][CW]
    uint64_t *full = reinterpret_cast<uint64_t *>(cb + NCW * 2 * CW);
    uint64_t *empty = full + ST;
    uint64_t *cfull = empty + ST;  // [NCW][2]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t tilesN = (g.N + BN - 1) / BN, tilesM = (g.M + BM - 1) / BM;
    const int64_t ntiles = tilesN * tilesM;
    const int nk = (int)((g.K + BK - 1) / BK);

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        for (int w = 0; w < 2 * NCW; ++w) mbar_init(&cfull[w], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {  // ---------------- producer ----------------
        if (lane != 0) return;
        int64_t sp = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t m0 = (t / tilesN) * BM, n0 = (t % tilesN) * BN;
            for (int kc = 0; kc < nk; ++kc, ++sp) {
                const int slot = (int)(sp % ST);
                if (sp >= ST) mbar_wait(&empty[slot], (unsigned)(((sp / ST) - 1) & 1));
                mbar_expect_tx(&full[slot], STAGE_BYTES);
                const int k0 = kc * BK;
#pragma unroll
                for (int kb = 0; kb < KB; ++kb) {
                    tma_load_2d(xs + slot * XS + kb * BM * 8, &tmX, (int)(g.xk0 + k0 + kb * 8), (int)(g.xm0 + m0), &full[slot]);
                    tma_load_2d(ys + slot * YS + kb * BN * 8, &tmY, (int)(g.yk0 + k0 + kb * 8), (int)(g.yn0 + n0), &full[slot]);
                }
            }
        }
        return;
    }
    // ---------------- consumers ----------------
    const int wm = warp / WN, wn = warp % WN;
    const int fr = lane >> 2, fk = (lane & 3) * 2;
    double *mycb = cb + (int64_t)warp * 2 * CW;
    uint64_t *mycf = cfull + 2 * warp;
    auto issue_c = [&](int64_t t, int buf) {  // lane 0: this warp's sub-tile of tile t
        const int64_t m0 = (t / tilesN) * BM + wm * 32, n0 = (t % tilesN) * BN + wn * 32;
        mbar_expect_tx(&mycf[buf], CW_BYTES);
#pragma unroll
        for (int s = 0; s < 4; ++s) tma_load_2d(mycb + buf * CW + s * 256, &tmC, (int)(n0 + 8 * s), (int)m0, &mycf[buf]);
    };
    if (lane == 0 && (int64_t)blockIdx.x < ntiles) issue_c(blockIdx.x, 0);
    int64_t sc = 0, nt = 0;
    double acc[MT][NT][2];
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
        const int buf = (int)(nt & 1);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kc = 0; kc < nk; ++kc, ++sc) {
            const int slot = (int)(sc % ST);
            mbar_wait(&full[slot], (unsigned)((sc / ST) & 1));
            const double *xd = xs + slot * XS;
            const double *yd = ys + slot * YS;
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                double2 a[MT], b[NT];
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    a[i] = *reinterpret_cast<const double2 *>(xd + (kb * BM + wm * 8 * MT + i * 8 + fr) * 8 + fk);
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    b[j] = *reinterpret_cast<const double2 *>(yd + (kb * BN + wn * 8 * NT + j * 8 + fr) * 8 + fk);
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            // after the first stage, prefetch this warp's next C sub-tile into the
            // other buffer (its previous stores have had a stage to drain)
            if (kc == 0 && lane == 0 && t + gridDim.x < ntiles) {
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                issue_c(t + gridDim.x, buf ^ 1);
            }
        }
        // epilogue of this warp's sub-tile
        mbar_wait(&mycf[buf], (unsigned)((nt >> 1) & 1));
        double *cbuf = mycb + buf * CW;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                double2 *p = reinterpret_cast<double2 *>(cbuf + j * 256 + (i * 8 + fr) * 8 + fk);
                double2 c2 = *p;
                c2.x += acc[i][j][0];
                c2.y += acc[i][j][1];
                *p = c2;
            }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            const int64_t m0 = (t / tilesN) * BM + wm * 32, n0 = (t % tilesN) * BN + wn * 32;
#pragma unroll
            for (int s = 0; s < 4; ++s) tma_store_2d(&tmC, (int)(n0 + 8 * s), (int)m0, cbuf + s * 256);
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

}  // namespace rq

namespace rq {

// ---------------------------------------------------------------------------
// C = X^T Y (skinny M: S1 sketch, S5 W = V^T A22), warp-specialised like
// gemm_upd_ws_kernel: a producer warp streams the (tile, K-slice) stages by
// TMA into a full / empty mbarrier ring, the consumer warps never meet at a
// CTA-wide barrier, and each writes its own fragments at a tile's end
// (EPI_STORE: C; EPI_PARTIAL: the split-K slice).  Same tiles, same K slices
// and the same per-element DMMA order as gemm_tma_kernel: the same bits.
// ---------------------------------------------------------------------------
template <int MT, int NT, int WM, int WN, int BK, int ST>
constexpr size_t ws_gemm_smem() {
    return 128 + (size_t)ST * BK * (8 * MT * WM + 8 * NT * WN) * sizeof(double) + 2 * ST * sizeof(uint64_t);
}

template <int MT, int NT, int WM, int WN, int BK, int ST, int EPI>
__global__ void __launch_bounds__((WM * WN + 1) * 32, 1)
    gemm_ws_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY, TmaGemmArgs g) {
    constexpr int BM = 8 * MT * WM;
    constexpr int BN = 8 * NT * WN;
    constexpr int KB = BK / 8;
    constexpr int XS = KB * BM * 8;
    constexpr int YS = KB * BN * 8;
    constexpr int NCW = WM * WN;
    constexpr unsigned STAGE_BYTES = (unsigned)((XS + YS) * sizeof(double));
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
    double *xs = reinterpret_cast<double *>(smem_raw + pad);
    double *ys = xs + ST * XS;
    uint64_t *full = reinterpret_cast<uint64_t *>(ys + ST * YS);
    uint64_t *empty = full + ST;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t tilesN = (g.N + BN - 1) / BN, tilesM = (g.M + BM - 1) / BM;
    const int64_t per = tilesN * tilesM;
    const int64_t ntiles = per * g.splits;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // tile t -> (split, m-tile, n-tile), n fastest (as gemm_tma_kernel)
    auto tile_geom = [&](int64_t t, int &split, int64_t &m0, int64_t &n0, int64_t &kbeg, int &nk) {
        split = (int)(t / per);
        const int64_t r = t % per;
        m0 = (r / tilesN) * BM;
        n0 = (r % tilesN) * BN;
        kbeg = (int64_t)split * g.k_per_split;
        const int64_t kend = min(g.K, kbeg + g.k_per_split);
        nk = (kend > kbeg) ? (int)((kend - kbeg + BK - 1) / BK) : 0;
    };
    if (warp == NCW) {  // producer
        if (lane != 0) return;
        int64_t sp = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int split, nk;
            int64_t m0, n0, kbeg;
            tile_geom(t, split, m0, n0, kbeg, nk);
            for (int kc = 0; kc < nk; ++kc, ++sp) {
                const int slot = (int)(sp % ST);
                if (sp >= ST) mbar_wait(&empty[slot], (unsigned)(((sp / ST) - 1) & 1));
                mbar_expect_tx(&full[slot], STAGE_BYTES);
                const int64_t k0 = kbeg + (int64_t)kc * BK;
#pragma unroll
                for (int kb = 0; kb < KB; ++kb) {
                    tma_load_2d(xs + slot * XS + kb * BM * 8, &tmX, (int)(g.xk0 + k0 + kb * 8), (int)(g.xm0 + m0), &full[slot]);
                    tma_load_2d(ys + slot * YS + kb * BN * 8, &tmY, (int)(g.yk0 + k0 + kb * 8), (int)(g.yn0 + n0), &full[slot]);
                }
            }
        }
        return;
    }
    const int wm = warp / WN, wn = warp % WN;
    const int fr = lane >> 2, fk = (lane & 3) * 2;
    int64_t sc = 0;
    double acc[MT][NT][2];
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int split, nk;
        int64_t m0, n0, kbeg;
        tile_geom(t, split, m0, n0, kbeg, nk);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kc = 0; kc < nk; ++kc, ++sc) {
            const int slot = (int)(sc % ST);
            mbar_wait(&full[slot], (unsigned)((sc / ST) & 1));
            const double *xd = xs + slot * XS;
            const double *yd = ys + slot * YS;
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                double2 a[MT], b[NT];
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    a[i] = *reinterpret_cast<const double2 *>(xd + (kb * BM + wm * 8 * MT + i * 8 + fr) * 8 + fk);
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    b[j] = *reinterpret_cast<const double2 *>(yd + (kb * BN + wn * 8 * NT + j * 8 + fr) * 8 + fk);
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int64_t gm = m0 + wm * 8 * MT + i * 8 + fr;
            if (gm >= g.M) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t gn = n0 + wn * 8 * NT + j * 8 + fk + h;
                    if (gn >= g.N) continue;
                    if (EPI == EPI_STORE) g.C[gm + gn * g.ldc] = acc[i][j][h];
                    else g.C[(int64_t)split * g.split_stride + gm + gn * g.M] = acc[i][j][h];
                }
        }
    }
}

}  // namespace rq
