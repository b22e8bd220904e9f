// Exp body of the softmax kernel (64 keys per thread: FFMA2, MUFU.EX2, FADD2, F2FP, tcgen05.st
// 16x32bx2) timed in isolation: 4 warps (1 per SMSP) or 8 warps (2 per SMSP), with and without the
// TMEM store.  nvcc -gencode arch=compute_100a,code=sm_100a -I ../../paper_2510_22049_b200/csrc -o expbody2 expbody2.cu
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace vista;
template <int STORE>
__device__ __forceinline__ float body(const uint32_t (&r)[2][32], float sl2, float neg, uint32_t tP) {
    const uint64_t sl2x2 = ptx::f2_pack(sl2, sl2);
    const uint64_t negx2 = ptx::f2_pack(neg, neg);
    uint64_t acc[2] = {ptx::f2_pack(0.f, 0.f), ptx::f2_pack(0.f, 0.f)};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint64_t x2 = ptx::f2_fma(ptx::f2_pack(__uint_as_float(r[c][2 * j]), __uint_as_float(r[c][2 * j + 1])), sl2x2, negx2);
            float x0, x1;
            ptx::f2_unpack(x2, x0, x1);
            const uint64_t p2 = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
            acc[j & 1] = ptx::f2_add(acc[j & 1], p2);
            float p0, p1;
            ptx::f2_unpack(p2, p0, p1);
            pk[j] = ptx::pack_bf16x2(p0, p1);
        }
        if (STORE) ptx::tmem_st16x32bx2_x16<32>(tP + c * 16, pk);
        else {
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[0] = ptx::f2_add(acc[0], ptx::f2_pack(__uint_as_float(pk[j]), 0.f));
        }
    }
    float la, lb, lc, ld;
    ptx::f2_unpack(acc[0], la, lb);
    ptx::f2_unpack(acc[1], lc, ld);
    return (la + lb) + (lc + ld);
}
template <int STORE>
__global__ void k(float* out, long long* cyc, int iters) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = base + ((uint32_t)((warp % 4) * 32 + (warp / 4) * 16) << 16) + 384;
    uint32_t r[2][32];
    for (int c = 0; c < 2; ++c)
        for (int j = 0; j < 32; ++j) r[c][j] = __float_as_uint(-1.0f * (j + c + lane) * 0.01f);
    float s = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        s += body<STORE>(r, 1.4427f, -0.5f - it * 1e-6f, tm);
        if (STORE) ptx::tmem_wait_st();
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}
template <int STORE>
void run(int warps) {
    float* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
    const int iters = 2000;
    k<STORE><<<1, warps * 32>>>(o, c, iters);
    k<STORE><<<1, warps * 32>>>(o, c, iters);
    long long h; cudaError_t e = cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("store=%d warps=%d: %.1f clk per 64-key body per warp (%s)\n", STORE, warps, (double)h / iters, cudaGetErrorString(e));
}
int main() { run<1>(4); run<1>(8); run<0>(4); run<0>(8); }
