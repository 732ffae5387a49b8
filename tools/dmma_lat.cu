// tools/dmma_lat.cu -- DMMA.8x8x4 issue model on B200: cycles per DMMA per SM
// for C independent accumulator chains per warp and W warps per CTA (one CTA
// per SM, 148 CTAs): how many independent chains a warp / an SM sub-partition
// needs to keep the FP64 tensor pipe full (the GEMM inner loops' design).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat tools/dmma_lat.cu
#include <cuda_runtime.h>
#include <cstdio>

template <int C>
__global__ void chains(double *out, int iters, unsigned long long *cyc) {
    double d[C][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < C; ++i) d[i][0] = d[i][1] = 0.0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.0) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps, double *out, unsigned long long *cyc) {
    const int iters = 4096 / C * 8;
    chains<C><<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    chains<C><<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i];
    mean /= 148;
    const double n = (double)iters * C * warps;  // DMMAs per SM
    printf("{\"chains_per_warp\": %d, \"warps\": %d, \"cycles_per_dmma_per_sm\": %.3f}\n", C, warps, mean / n);
}

int main() {
    double *out;
    unsigned long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 8);
    for (int w : {1, 2, 4, 8, 16}) {
        run<1>(w, out, cyc);
        run<2>(w, out, cyc);
        run<4>(w, out, cyc);
        run<8>(w, out, cyc);
        run<16>(w, out, cyc);
    }
    return 0;
}
