// clock64 rate vs CUDA events (diagnostic): spins N clock64 cycles in one
// thread (optionally with all SMs busy) and prints cycles / elapsed ns.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long n, unsigned long long *out) {
    const long long t0 = clock64();
    unsigned long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    while (clock64() - t0 < n) {}
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = g1 - g0;
}
int main() {
    unsigned long long *d, h;
    cudaMalloc(&d, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int grid : {1, 148, 296}) {
        for (int rep = 0; rep < 2; ++rep) {
            const long long n = 400000000LL;
            cudaEventRecord(a);
            spin<<<grid, 256>>>(n, d);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("grid %d: %lld cycles in %.3f ms (events) / %.3f ms (globaltimer): %.3f GHz (events), %.3f GHz (globaltimer)\n",
                   grid, n, ms, h * 1e-6, n / (ms * 1e6), n / (h * 1.0));
        }
    }
    return 0;
}
