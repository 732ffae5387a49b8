// tools/microbench.cu -- B200 measurements that MEASURED_PEAKS.json lacks:
//   1. FP64 DMMA.8x8x4 throughput (mma.sync m8n8k4 f64), all SMs, register
//      operands, independent accumulator chains -> the FP64 tensor peak;
//   2. DFMA throughput, same protocol -> the FP64 vector peak;
//   3. grid-barrier round trip (the barrier the cooperative sample-QRCP and
//      panel kernels use once per pivot step) for several grid sizes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
// Prints one JSON object.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dmma_kernel(double *out, int iters) {
    double d[8][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_kernel(double *out, int iters) {
    double x[8];
    const double a = 1.0000001, b = 1e-9 * threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ void grid_barrier_old(unsigned *bar, unsigned nblocks) {
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

__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned nblocks, unsigned &epoch) {
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

__global__ void barrier_kernel(unsigned *bar, int iters, int variant) {
    unsigned epoch = 0;
    if (variant == 0)
        for (int i = 0; i < iters; ++i) grid_barrier_old(bar, gridDim.x);
    else
        for (int i = 0; i < iters; ++i) grid_barrier(bar, gridDim.x, epoch);
}

// exchange pattern of the sample QRCP step: publish 16-byte header, grid
// barrier, warp 0 reads all G headers + argmax reduce, CTA barrier.
__global__ void exchange_kernel(double2 *hdr, unsigned *bar, int iters, double *out) {
    unsigned epoch = 0;
    const int G = gridDim.x, g = blockIdx.x;
    double best = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        if (threadIdx.x == 0) hdr[par * G + g] = make_double2((double)((g * 7 + it) % G), (double)g);
        grid_barrier(bar, G, epoch);
        if (threadIdx.x < 32) {
            double v = -1, p = 1e9;
            for (int q = threadIdx.x; q < G; q += 32) {
                const double2 h = __ldcg(hdr + par * G + q);
                if (h.x > v || (h.x == v && h.y < p)) { v = h.x; p = h.y; }
            }
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(~0u, v, o), op = __shfl_xor_sync(~0u, p, o);
                if (ov > v || (ov == v && op < p)) { v = ov; p = op; }
            }
            best += v + p;
        }
        __syncthreads();
    }
    if (best == 12345.0) out[0] = best;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    double *out;
    unsigned *bar;
    CK(cudaMalloc(&out, 64));
    CK(cudaMalloc(&bar, 64));
    CK(cudaMemset(bar, 0, 64));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
    // DMMA: blocks x warps sweep, report best
    {
        double best = 0;
        int bw = 0;
        const int iters = 20000;
        for (int warps : {4, 8, 16}) {
            for (int bps : {1, 2}) {
                dim3 grid(sms * bps), block(32 * warps);
                dmma_kernel<<<grid, block>>>(out, 100);
                CK(cudaDeviceSynchronize());
                float best_ms = 1e30f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(e0);
                    dmma_kernel<<<grid, block>>>(out, iters);
                    cudaEventRecord(e1);
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best_ms) best_ms = ms;
                }
                const double flops = 2.0 * 256 * 8 * (double)iters * grid.x * warps;
                const double tf = flops / (best_ms * 1e-3) / 1e12;
                if (tf > best) { best = tf; bw = warps * 100 + bps; }
            }
        }
        printf(", \"dmma_tflops\": %.3f, \"dmma_best_cfg\": %d", best, bw);
    }
    {
        double best = 0;
        const int iters = 20000;
        for (int warps : {8, 16, 32}) {
            dim3 grid(sms * 2), block(32 * warps);
            dfma_kernel<<<grid, block>>>(out, 100);
            CK(cudaDeviceSynchronize());
            float best_ms = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                dfma_kernel<<<grid, block>>>(out, iters);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best_ms) best_ms = ms;
            }
            const double flops = 2.0 * 8 * (double)iters * grid.x * block.x;
            const double tf = flops / (best_ms * 1e-3) / 1e12;
            if (tf > best) best = tf;
        }
        printf(", \"dfma_tflops\": %.3f", best);
    }
    for (int variant = 0; variant < 2; ++variant) {
        printf(", \"grid_barrier_%s_us\": {", variant == 0 ? "fence_atomic" : "release_acquire");
        bool first = true;
        for (int g : {16, 32, 64, 128, sms}) {
            int iters = 2000;
            void *args[] = {&bar, (void *)&iters, (void *)&variant};
            CK(cudaMemset(bar, 0, 64));
            cudaEventRecord(e0);
            CK(cudaLaunchCooperativeKernel((void *)barrier_kernel, dim3(g), dim3(256), args, 0, 0));
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s\"%d\": %.3f", first ? "" : ", ", g, ms * 1e3 / iters);
            first = false;
        }
        printf("}");
    }
    printf(", \"exchange_us\": {");
    {
        double2 *hdr;
        CK(cudaMalloc(&hdr, 2 * 160 * sizeof(double2)));
        bool first = true;
        for (int g : {8, 16, 32, 64, 96, 128, sms}) {
            int iters = 2000;
            void *args[] = {&hdr, &bar, (void *)&iters, &out};
            CK(cudaMemset(bar, 0, 64));
            cudaEventRecord(e0);
            CK(cudaLaunchCooperativeKernel((void *)exchange_kernel, dim3(g), dim3(256), args, 0, 0));
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s\"%d\": %.3f", first ? "" : ", ", g, ms * 1e3 / iters);
            first = false;
        }
        printf("}");
    }
    printf("}\n");
    return 0;
}
