// tools/lat_bench.cu -- latencies of the building blocks of the latency-bound
// kernels (diagnostic): dependent FP64 chains (DFMA, sqrt, division), shared
// memory load-use, __syncthreads, barrier.cluster (release/acquire vs relaxed)
// and an all-to-all DSMEM exchange by st.async + mbarrier complete_tx, per
// step, for clusters of 2..16 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void chain_kernel(long long *out, double *sink, int n) {
    double x = 1.0 + threadIdx.x * 1e-9, y = 0.5;
    __shared__ double s[64];
    __shared__ int idx[64];
    if (threadIdx.x < 64) { s[threadIdx.x] = 1.0; idx[threadIdx.x] = (threadIdx.x + 1) & 63; }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 0.9999999, 1e-7);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
    long long t3 = clock64();
    int p = 0;
    for (int i = 0; i < n; ++i) p = idx[p];
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) { y = s[p & 63] * y + 1e-9; p = (int)y; }
    long long t6 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = t6 - t5;
    }
    sink[threadIdx.x] = x + p + y;
}

__device__ __forceinline__ unsigned cl_rank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned cl_map(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

// variant 0: barrier.cluster arrive.release / wait.acquire; 1: relaxed arrive / wait
__global__ void clbar_kernel(long long *out, int n, int variant) {
    long long t0 = clock64();
    if (variant == 0) {
        for (int i = 0; i < n; ++i)
            asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        for (int i = 0; i < n; ++i)
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;\n" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && cl_rank() == 0) out[0] = t1 - t0;
}

// all-to-all: every CTA pushes `words` doubles (its step value) into a slot of
// every CTA's receive buffer with st.async; receivers wait on their mbarrier
// (phase per step, two parities), then sum the G slots.
__global__ void a2a_kernel(long long *out, double *sink, int n, int words) {
    __shared__ __align__(16) double recv[2][16][128];
    __shared__ __align__(8) unsigned long long mb[2];
    const int G = gridDim.x, g = (int)cl_rank(), tid = threadIdx.x;
    const unsigned mba0 = (unsigned)__cvta_generic_to_shared(&mb[0]);
    const unsigned bytes = (unsigned)(G * words * 8);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mba0));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mba0 + 8));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;\n" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mba0), "r"(bytes) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mba0 + 8), "r"(bytes) : "memory");
    }
    __syncthreads();
    double acc = 0.0;
    long long t0 = clock64();
    for (int s = 0; s < n; ++s) {
        const int par = s & 1;
        // push: thread e -> (destination, word pair)
        const int pairs = words / 2;
        for (int e = tid; e < G * pairs; e += blockDim.x) {
            const int dst = e / pairs, w = 2 * (e % pairs);
            const unsigned la = (unsigned)__cvta_generic_to_shared(&recv[par][g][w]);
            const unsigned ra = cl_map(la, dst), rm = cl_map(mba0 + 8 * par, dst);
            const double v = acc + s + w;
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(ra),
                         "d"(v), "d"(v), "r"(rm) : "memory");
        }
        unsigned ok = 0;
        const unsigned ph = (unsigned)((s >> 1) & 1);
        while (!ok)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"(mba0 + 8 * par), "r"(ph) : "memory");
        double t = 0.0;
        for (int q = 0; q < G; ++q) t += recv[par][q][tid % words];
        acc = t * 1e-3;
        __syncthreads();
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(mba0 + 8 * par), "r"(bytes) : "memory");
    }
    long long t1 = clock64();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;\n" ::: "memory");
    if (tid == 0 && g == 0) out[0] = t1 - t0;
    sink[tid] = acc;
}

// pull: every CTA writes its `words` doubles into its own slot (parity s & 1),
// fence.release.sync_restrict::shared::cta.cluster, relaxed arrive, wait;
// then every thread reads its word from all G CTAs (ld.shared::cluster).
__global__ void pull_kernel(long long *out, double *sink, int n, int words) {
    __shared__ __align__(16) double slot[2][128];
    const int G = gridDim.x, tid = threadIdx.x;
    double acc = 0.0;
    long long t0 = clock64();
    for (int s = 0; s < n; ++s) {
        const int par = s & 1;
        if (tid < words) slot[par][tid] = acc + s + tid;
        asm volatile("fence.release.sync_restrict::shared::cta.cluster;\n" ::: "memory");
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;\n" ::: "memory");
        const unsigned la = (unsigned)__cvta_generic_to_shared(&slot[par][tid % words]);
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (q < G) {
                const unsigned ra = cl_map(la, q);
                asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v[q]) : "r"(ra) : "memory");
            }
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (q < G) t += v[q];
        acc = t * 1e-3;
    }
    long long t1 = clock64();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;\n" ::: "memory");
    if (tid == 0 && cl_rank() == 0) out[0] = t1 - t0;
    sink[tid] = acc;
}

// shared-memory load throughput with 256 threads (8 warps): LDS.128 broadcast
// (every lane the same address) vs distinct conflict-free addresses, and the
// DFMA issue rate, in SM cycles per warp-instruction (whole SM).
__global__ void lds_tput_kernel(long long *out, unsigned *sink, int n, int mode) {
    __shared__ __align__(16) uint4 buf[1024];
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) buf[e] = make_uint4(e, e + 1, e + 2, e + 3);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint4 acc = make_uint4(0, 0, 0, 0);
    double d[16];
    for (int k = 0; k < 16; ++k) d[k] = threadIdx.x + k;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {
        for (int i = 0; i < n; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint4 v = buf[(i * 8 + k) & 1023];  // broadcast
                acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
            }
        }
    } else if (mode == 1) {
        for (int i = 0; i < n; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint4 v = buf[((i * 8 + k) * 32 + lane) & 1023];  // 32 distinct 16-byte words
                acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
            }
        }
    } else {
        for (int i = 0; i < n; ++i) {
#pragma unroll
            for (int k = 0; k < 16; ++k) d[k] = fma(d[k], 0.999999, 1e-9);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    double s = 0;
    for (int k = 0; k < 16; ++k) s += d[k];
    sink[threadIdx.x] = acc.x ^ acc.y ^ acc.z ^ acc.w ^ (unsigned)s;
}

int main() {
    long long *d_out, h[8];
    double *sink;
    CK(cudaMalloc(&d_out, 64));
    CK(cudaMalloc(&sink, 8192));
    const int n = 1000;
    chain_kernel<<<1, 256>>>(d_out, sink, n);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d_out, 48, cudaMemcpyDeviceToHost));
    printf("{\"cycles_per_op\": {\"dfma_dep\": %.1f, \"sqrt_dep\": %.1f, \"div_dep\": %.1f, \"lds_chase\": %.1f, "
           "\"syncthreads_256\": %.1f, \"lds_dfma_dep\": %.1f}",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
    CK(cudaFuncSetAttribute(clbar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(a2a_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int variant = 0; variant < 2; ++variant) {
        printf(", \"cluster_barrier_%s\": {", variant ? "relaxed" : "release_acquire");
        int first = 1;
        for (int cs : {2, 4, 8, 16}) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(cs);
            lc.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            lc.attrs = at; lc.numAttrs = 1;
            CK(cudaLaunchKernelEx(&lc, clbar_kernel, d_out, n, variant));
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
            printf("%s\"%d\": %.1f", first ? "" : ", ", cs, h[0] / (double)n);
            first = 0;
        }
        printf("}");
    }
    for (int words : {64, 128}) {
        printf(", \"a2a_stasync_%dw\": {", words);
        int first = 1;
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(cs);
            lc.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            lc.attrs = at; lc.numAttrs = 1;
            CK(cudaLaunchKernelEx(&lc, a2a_kernel, d_out, sink, n, words));
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
            printf("%s\"%d\": %.1f", first ? "" : ", ", cs, h[0] / (double)n);
            first = 0;
        }
        printf("}");
    }
    CK(cudaFuncSetAttribute(pull_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int words : {64, 128}) {
        printf(", \"a2a_pull_restrictfence_%dw\": {", words);
        int first = 1;
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(cs);
            lc.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            lc.attrs = at; lc.numAttrs = 1;
            CK(cudaLaunchKernelEx(&lc, pull_kernel, d_out, sink, n, words));
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
            printf("%s\"%d\": %.1f", first ? "" : ", ", cs, h[0] / (double)n);
            first = 0;
        }
        printf("}");
    }
    {
        unsigned *usink;
        CK(cudaMalloc(&usink, 4096));
        const char *names[3] = {"lds128_broadcast", "lds128_distinct", "dfma"};
        const double per[3] = {8.0 * 8, 8.0 * 8, 16.0 * 8};  // warp-instructions per iteration (8 warps)
        printf(", \"sm_cycles_per_warp_instr_256thr\": {");
        for (int mode = 0; mode < 3; ++mode) {
            lds_tput_kernel<<<1, 256>>>(d_out, usink, n, mode);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost));
            printf("%s\"%s\": %.2f", mode ? ", " : "", names[mode], h[0] / (n * per[mode]));
        }
        printf("}");
    }
    printf(", \"unit\": \"SM cycles per op / per step\"}\n");
    return 0;
}
