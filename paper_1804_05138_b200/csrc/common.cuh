// common.cuh -- device helpers shared by the RQRCP kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define RQ_DEV __device__ __forceinline__

namespace rq {

// ---------------------------------------------------------------------------
// FP64 tensor core: mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4 on sm_100a (the
// only FP64 MMA shape Blackwell has; tcgen05 has no f64 kind).
// A fragment: thread t holds A[t/4][t%4]; B: B[t%4][t/4]; C/D: C[t/4][2(t%4)+{0,1}].
// ---------------------------------------------------------------------------
RQ_DEV void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// cp.async (LDGSTS): 8-byte element copies with zero fill when !pred.
RQ_DEV void cp_async8(void *smem, const void *gmem, bool pred) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
RQ_DEV void cp_async16(void *smem, const void *gmem, int src_bytes) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
RQ_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RQ_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Deterministic warp sum (fixed butterfly: identical bits on every run/CTA).
RQ_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// Grid barrier for cooperative (co-resident) launches: arrival counter +
// generation word, release/acquire through gpu-scope fences.
// bar[0] = arrival count, bar[1] = generation.
// ---------------------------------------------------------------------------
RQ_DEV void grid_barrier(unsigned *bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        unsigned g = *gen;
        __threadfence();
        unsigned arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

RQ_DEV double ld_cg(const double *p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
    return v;
}

}  // namespace rq
