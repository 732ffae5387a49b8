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
// Grid barrier for cooperative (co-resident) launches.  `count` is a
// per-launch counter zeroed by the host before the launch; barrier number e
// (1, 2, ...) completes when count reaches e * nblocks.  Arrival is a
// release reduction (orders this CTA's prior writes, made CTA-visible by the
// preceding __syncthreads), the wait an acquire load: no full fences.
// ---------------------------------------------------------------------------
RQ_DEV void grid_barrier(unsigned *count, unsigned nblocks, unsigned &epoch) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        const unsigned target = epoch * nblocks;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(count) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(count) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

RQ_DEV double2 ld_volatile_v2(const double2 *p) {
    double2 v;
    asm volatile("ld.volatile.global.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}
RQ_DEV void st_cg_v2(double2 *p, double2 v) {
    asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// Tagged 16-byte units for fence-free exchanges between CTAs: a 64-bit
// value travels as two 32-bit halves, each beside the step tag, in one
// single-copy-atomic 16-byte store; a reader polls until both tags match.
// unit = {lo32 | tag << 32, hi32 | tag << 32}
RQ_DEV void ll_store(uint4 *p, unsigned long long w, unsigned tag) {
    const unsigned long long t = (unsigned long long)tag << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"((w & 0xffffffffull) | t),
                 "l"((w >> 32) | t)
                 : "memory");
}
RQ_DEV bool ll_load(const uint4 *p, unsigned tag, unsigned long long &w) {
    unsigned long long a, b;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    w = (a & 0xffffffffull) | (b << 32);
    return (unsigned)(a >> 32) == tag && (unsigned)(b >> 32) == tag;
}

// L2 load for data written by other CTAs (after a grid barrier); not
// volatile, so the compiler may batch several in flight.
RQ_DEV double ld_cg(const double *p) { return __ldcg(p); }

}  // namespace rq
