// globaltimer vs clock64 vs CUDA events: a 148-CTA kernel that spins ~N SM clocks; each CTA records
// globaltimer / clock64 at its start and end.  Checks that in-kernel globaltimer spans agree with
// event timing (used by the per-CTA timelines of scripts/trace_*.py).
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_t[148][4];
__global__ void spin(long long n) {
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const long long c0 = clock64();
    while (clock64() - c0 < n) {}
    const long long c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) { g_t[blockIdx.x][0] = g0; g_t[blockIdx.x][1] = g1; g_t[blockIdx.x][2] = c0; g_t[blockIdx.x][3] = c1; }
}
// the same spin with 226 KB of dynamic shared memory and 512 threads (the persistent kernels' shape),
// optionally allocating 256 TMEM columns
template <bool TMEM>
__global__ void __launch_bounds__(512, 1) spin_big(long long n) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    __shared__ unsigned int tbase;
    if (TMEM && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((unsigned)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    const long long c0 = clock64();
    while (clock64() - c0 < n) {}
    if (threadIdx.x == 0) sm[0] = 1;
    __syncthreads();
    if (TMEM && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) { g_t[blockIdx.x][0] = g0; g_t[blockIdx.x][1] = g1; g_t[blockIdx.x][2] = 0; g_t[blockIdx.x][3] = sm[0]; }
}
template <bool TMEM>
void run_big(long long n) {
    const int smem = 226 * 1024;
    cudaFuncSetAttribute(spin_big<TMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    spin_big<TMEM><<<148, 512, smem>>>(n);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    spin_big<TMEM><<<148, 512, smem>>>(n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[148][4];
    cudaMemcpyFromSymbol(t, g_t, sizeof(t));
    unsigned long long gmin = ~0ull, gmax = 0;
    for (int i = 0; i < 148; ++i) { if (t[i][0] < gmin) gmin = t[i][0]; if (t[i][1] > gmax) gmax = t[i][1]; }
    printf("big%s n=%lld: events %.2f us, globaltimer span %.2f us (%s)\n", TMEM ? "+tmem" : "", n, 1e3 * ms,
           (gmax - gmin) / 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (long long n : {20000LL, 200000LL, 2000000LL}) {
        spin<<<148, 128>>>(n);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        spin<<<148, 128>>>(n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long t[148][4];
        cudaMemcpyFromSymbol(t, g_t, sizeof(t));
        unsigned long long gmin = ~0ull, gmax = 0;
        for (int i = 0; i < 148; ++i) { if (t[i][0] < gmin) gmin = t[i][0]; if (t[i][1] > gmax) gmax = t[i][1]; }
        double clk = (double)(t[0][3] - t[0][2]), gt = (double)(t[0][1] - t[0][0]);
        printf("n=%lld: events %.2f us, globaltimer span %.2f us, CTA0 clock %.0f over %.0f ns -> %.3f GHz\n", n,
               1e3 * ms, (gmax - gmin) / 1e3, clk, gt, clk / gt);
    }
    run_big<false>(20000);
    run_big<true>(20000);
    return 0;
}
