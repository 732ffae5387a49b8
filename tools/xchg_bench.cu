// tools/xchg_bench.cu -- per-step cost of the all-to-all "argmax + winner
// column" exchange the sample-QRCP and panel kernels do once per pivot step,
// on one B200, for several protocols and grid sizes (diagnostic; not product).
//
// Each step: every CTA publishes a 16-byte candidate header and a column of L
// doubles; every CTA then waits for all G headers of this step, picks the
// winner (max value) and reads its column.  Protocols:
//   0 "rel/acq"     : st.release header after the column; ld.acquire polls
//   1 "rel/rlx+fence": st.release header; ld.relaxed polls + one fence.acq_rel
//   2 "LL"          : every 8-byte word carries the step tag (32-bit payload
//                     halves); plain relaxed stores and loads, no fences
//   3 "barrier"     : red.release counter barrier + ld.acquire spin, then
//                     plain ld.cg of headers and column (the original design)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xchg_bench tools/xchg_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int L = 80;
constexpr int MAXG = 256;

__device__ __forceinline__ void st_rel_v2(void *p, unsigned long long a, unsigned long long b) {
    asm volatile("st.release.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_rlx_v2(void *p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_acq_v2(const void *p, unsigned long long &a, unsigned long long &b) {
    asm volatile("ld.acquire.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_rlx_v2(const void *p, unsigned long long &a, unsigned long long &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

struct Buf {
    unsigned long long *hdr;   // [2][G][16] (stride 128 B)
    unsigned long long *col;   // [2][G][2L] (protocol 2: (hi|tag, lo|tag) per double)
    unsigned *bar;
    double *out;
};

__global__ void __launch_bounds__(256, 1) xchg_kernel(Buf b, int steps, int proto, int work) {
    const int G = gridDim.x, g = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double s_w;
    __shared__ double col_s[L];
    double acc = 0.0;
    unsigned epoch = 0;
    for (int j = 0; j < steps; ++j) {
        const unsigned tag = 1000u + (unsigned)j;  // distinct per launch via host memset
        const int par = j & 1;
        // fake apply work (DFMA chain per thread)
        double x = (double)threadIdx.x;
        for (int i = 0; i < work; ++i) x = fma(x, 0.999999, 1e-3);
        acc += x;
        __syncthreads();
        const double myv = (double)((g * 7919 + j * 104729) % 1000003);
        if (warp == 0) {
            unsigned long long *hp = b.hdr + ((size_t)(par * G + g)) * 16;
            unsigned long long *cp = b.col + ((size_t)(par * G + g)) * 2 * L;
            if (proto == 2) {
                for (int t = lane; t < L; t += 32) {
                    const unsigned long long bits = __double_as_longlong(myv + t);
                    const unsigned long long w0 = (bits >> 32) | ((unsigned long long)tag << 32);
                    const unsigned long long w1 = (bits & 0xffffffffull) | ((unsigned long long)tag << 32);
                    st_rlx_v2(cp + 2 * t, w0, w1);
                }
                if (lane == 0) {
                    const unsigned long long bits = __double_as_longlong(myv);
                    st_rlx_v2(hp, (bits >> 32) | ((unsigned long long)tag << 32),
                              (bits & 0xffffffffull) | ((unsigned long long)tag << 32));
                }
            } else {
                for (int t = lane; t < L; t += 32) __stcg(reinterpret_cast<double *>(cp) + t, myv + t);
                __syncwarp();
                if (lane == 0) {
                    if (proto == 3) {
                        __stcg(reinterpret_cast<double *>(hp), myv);
                    } else {
                        st_rel_v2(hp, __double_as_longlong(myv), (unsigned long long)tag);
                    }
                }
            }
        }
        if (proto == 3) {
            __syncthreads();
            ++epoch;
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(b.bar) : "memory");
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(b.bar) : "memory");
                } while (v < epoch * G);
            }
            __syncthreads();
        }
        if (warp == 0) {
            double best = -1.0;
            int bs = -1;
            constexpr int HPL = MAXG / 32;
            bool ready[HPL];
            double hv[HPL];
#pragma unroll
            for (int u = 0; u < HPL; ++u) { ready[u] = lane + 32 * u >= G; hv[u] = -1.0; }
            while (true) {
                bool all = true;
#pragma unroll
                for (int u = 0; u < HPL; ++u) {
                    if (!ready[u]) {
                        const unsigned long long *hp = b.hdr + ((size_t)(par * G + lane + 32 * u)) * 16;
                        unsigned long long a0, a1;
                        if (proto == 3) {
                            hv[u] = __ldcg(reinterpret_cast<const double *>(hp));
                            ready[u] = true;
                        } else {
                            if (proto == 0) ld_acq_v2(hp, a0, a1);
                            else ld_rlx_v2(hp, a0, a1);
                            if (proto == 2) {
                                if ((a0 >> 32) == tag && (a1 >> 32) == tag) {
                                    hv[u] = __longlong_as_double((long long)((a0 << 32) | (a1 & 0xffffffffull)));
                                    ready[u] = true;
                                }
                            } else if ((unsigned)a1 == tag) {
                                hv[u] = __longlong_as_double((long long)a0);
                                ready[u] = true;
                            }
                        }
                    }
                    all = all && ready[u];
                }
                if (__all_sync(0xffffffffu, all)) break;
            }
#pragma unroll
            for (int u = 0; u < HPL; ++u)
                if (lane + 32 * u < G && hv[u] > best) { best = hv[u]; bs = lane + 32 * u; }
            if (proto == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int os = __shfl_xor_sync(0xffffffffu, bs, o);
                if (ob > best || (ob == best && os < bs)) { best = ob; bs = os; }
            }
            const unsigned long long *cp = b.col + ((size_t)(par * G + bs)) * 2 * L;
            for (int t = lane; t < L; t += 32) {
                double v;
                if (proto == 2) {
                    while (true) {
                        unsigned long long a0, a1;
                        ld_rlx_v2(cp + 2 * t, a0, a1);
                        if ((a0 >> 32) == tag && (a1 >> 32) == tag) {
                            v = __longlong_as_double((long long)((a0 << 32) | (a1 & 0xffffffffull)));
                            break;
                        }
                    }
                } else {
                    v = __ldcg(reinterpret_cast<const double *>(cp) + t);
                }
                col_s[t] = v;
            }
            if (lane == 0) s_w = best;
        }
        __syncthreads();
        acc += s_w + col_s[threadIdx.x % L];
    }
    if (acc == 1234.5) b.out[0] = acc;
}

// protocol 4: one thread-block cluster (G <= 16); headers + columns in each
// CTA's own shared memory (double-buffered), one barrier.cluster per step,
// readers use DSMEM loads (ld.shared::cluster).
__global__ void __launch_bounds__(256, 1) xchg_cluster_kernel(double *out, int steps, int work) {
    __shared__ double hdr[2];
    __shared__ double col[2][L];
    __shared__ double s_w;
    __shared__ double col_s[L];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned rank, G;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(G));
    double acc = 0.0;
    for (int j = 0; j < steps; ++j) {
        const int par = j & 1;
        double x = (double)threadIdx.x;
        for (int i = 0; i < work; ++i) x = fma(x, 0.999999, 1e-3);
        acc += x;
        __syncthreads();
        const double myv = (double)((rank * 7919 + j * 104729) % 1000003);
        if (warp == 0) {
            for (int t = lane; t < L; t += 32) col[par][t] = myv + t;
            if (lane == 0) hdr[par] = myv;
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (warp == 0) {
            double best = -1.0;
            int bs = -1;
            if (lane < (int)G) {
                unsigned a = (unsigned)__cvta_generic_to_shared(&hdr[par]), ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"((unsigned)lane));
                asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(best) : "r"(ra));
                bs = lane;
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int os = __shfl_xor_sync(0xffffffffu, bs, o);
                if (ob > best || (ob == best && os < bs)) { best = ob; bs = os; }
            }
            for (int t = lane; t < L; t += 32) {
                unsigned a = (unsigned)__cvta_generic_to_shared(&col[par][t]), ra;
                double v;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"((unsigned)bs));
                asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
                col_s[t] = v;
            }
            if (lane == 0) s_w = best;
        }
        __syncthreads();
        acc += s_w + col_s[threadIdx.x % L];
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (acc == 1234.5) out[0] = acc;
}

int main() {
    Buf b;
    CK(cudaMalloc(&b.hdr, sizeof(unsigned long long) * 2 * MAXG * 16));
    CK(cudaMalloc(&b.col, sizeof(unsigned long long) * 2 * MAXG * 2 * L));
    CK(cudaMalloc(&b.bar, sizeof(unsigned)));
    CK(cudaMalloc(&b.out, sizeof(double)));
    const char *names[4] = {"rel/acq", "rel/rlx+fence", "LL", "barrier"};
    const int steps = 2000;
    printf("{\"L\": %d, \"steps\": %d, \"us_per_step\": {", L, steps);
    bool first = true;
    for (int work : {0, 200}) {
        for (int proto = 0; proto < 4; ++proto) {
            for (int G : {16, 32, 64, 148}) {
                float best = 1e9;
                for (int rep = 0; rep < 3; ++rep) {
                    CK(cudaMemset(b.hdr, 0, sizeof(unsigned long long) * 2 * MAXG * 16));
                    CK(cudaMemset(b.col, 0, sizeof(unsigned long long) * 2 * MAXG * 2 * L));
                    CK(cudaMemset(b.bar, 0, sizeof(unsigned)));
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    int st = steps, pr = proto, wk = work;
                    void *args[] = {&b, &st, &pr, &wk};
                    cudaEventRecord(e0);
                    CK(cudaLaunchCooperativeKernel((void *)xchg_kernel, dim3(G), dim3(256), args, 0, 0));
                    cudaEventRecord(e1);
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                printf("%s\"%s/G%d/work%d\": %.3f", first ? "" : ", ", names[proto], G, work, best * 1e3 / steps);
                first = false;
                fflush(stdout);
            }
        }
    }
    cudaFuncSetAttribute(xchg_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int work : {0, 200}) {
        for (int G : {2, 4, 8, 16}) {
            float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                cudaLaunchConfig_t lc = {};
                lc.gridDim = dim3(G);
                lc.blockDim = dim3(256);
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = G;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                CK(cudaLaunchKernelEx(&lc, xchg_cluster_kernel, b.out, steps, work));
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf(", \"cluster/G%d/work%d\": %.3f", G, work, best * 1e3 / steps);
            fflush(stdout);
        }
    }
    printf("}}\n");
    return 0;
}
