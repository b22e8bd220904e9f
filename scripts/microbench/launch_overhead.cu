// Launch cost of a persistent big-shared-memory kernel (148 CTAs x 512 threads, ~226 KB dynamic smem)
// on its own and after a small kernel that uses no shared memory (the shared-memory carveout then
// differs between consecutive kernels).  nvcc -gencode arch=compute_100a,code=sm_100a -o lo launch_overhead.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void small_k(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }
__global__ void __launch_bounds__(512, 1) big_k(int* p) {
    extern __shared__ int s[];
    if (threadIdx.x == 0) s[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main() {
    const int smem = 226 * 1024;
    cudaFuncSetAttribute(big_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int* d;
    cudaMalloc(&d, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int N = 200;
    float ms;
    auto run = [&](const char* name, auto body) {
        for (int i = 0; i < 10; ++i) body();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int i = 0; i < N; ++i) body();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("%-44s %8.2f us per iteration\n", name, 1e3 * ms / N);
    };
    run("small (1 CTA, no smem)", [&] { small_k<<<1, 1024>>>(d); });
    run("small (148 CTAs, no smem)", [&] { small_k<<<148, 256>>>(d); });
    run("big (148 CTAs, 226 KB smem)", [&] { big_k<<<148, 512, smem>>>(d); });
    run("small + big", [&] { small_k<<<1, 1024>>>(d); big_k<<<148, 512, smem>>>(d); });
    cudaFuncSetAttribute(small_k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    run("small (carveout max shared) + big", [&] { small_k<<<1, 1024>>>(d); big_k<<<148, 512, smem>>>(d); });
    run("small (carveout max shared, 148 CTAs) + big", [&] { small_k<<<148, 256>>>(d); big_k<<<148, 512, smem>>>(d); });
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
