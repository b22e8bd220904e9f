// The softmax kernel's exp_tile (sm100_softmax.cu) in isolation, one warp per SMSP, with and without
// its TMEM stores of P (tcgen05.st 32x32b.x16 per 32 scores) and with the S load from TMEM, to see
// which part of the in-kernel exp phase (~1600 clk) exceeds the MUFU floor (1024 clk).
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace vista;
template <int MODE>  // all modes load S from TMEM every iteration. 2: ld+max+exp+st+wait  3: ld+max  4: ld+max+exp (no st)  5: ld+exp+st+wait (no max)  6: ld only
__global__ void __launch_bounds__(128, 1) k(float* out, long long* cyc, float sl2, int iters) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc(&tbase, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tS = tbase + ((uint32_t)(warp * 32) << 16);
    uint32_t r[4][32];
    for (int c = 0; c < 4; ++c)
        for (int i = 0; i < 32; ++i) r[c][i] = __float_as_uint((threadIdx.x + c * 32 + i) * 1e-3f);
    {
        for (int c = 0; c < 4; ++c) ptx::tmem_st32(tS + c * 32, r[c]);
        ptx::tmem_wait_st();
    }
    uint32_t sink = 0;
    float lsum = 0.f, neg = -2.f;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        {
#pragma unroll
            for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tS + c * 32, r[c]);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 4; ++c) ptx::reg_fence(r[c]);
        }
        if (MODE == 6) { sink ^= r[0][it & 31]; continue; }
        if (MODE != 5) {
            float m = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int j = 0; j < 32; j += 2) m = ptx::max3(m, __uint_as_float(r[c][j]), __uint_as_float(r[c][j + 1]));
            neg = -m * sl2;
            if (MODE == 3) { sink ^= __float_as_uint(neg); continue; }
        }
        const uint64_t sl2x2 = ptx::f2_pack(sl2, sl2);
        const uint64_t negx2 = ptx::f2_pack(neg, neg);
        uint64_t acc[2] = {ptx::f2_pack(0.f, 0.f), ptx::f2_pack(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint64_t x2 = ptx::f2_fma(ptx::f2_pack(__uint_as_float(r[c][2 * j]), __uint_as_float(r[c][2 * j + 1])),
                                                sl2x2, negx2);
                float x0, x1;
                ptx::f2_unpack(x2, x0, x1);
                const uint64_t p2 = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
                acc[j & 1] = ptx::f2_add(acc[j & 1], p2);
                float p0, p1;
                ptx::f2_unpack(p2, p0, p1);
                pk[j] = ptx::pack_bf16x2(p0, p1);
            }
            if (MODE != 4) ptx::tmem_st16(tS + 128 + c * 16, pk);
            else {
#pragma unroll
                for (int j = 0; j < 16; ++j) sink ^= pk[j];
            }
        }
        if (MODE != 4) ptx::tmem_wait_st();
        float la, lb, lc, ld;
        ptx::f2_unpack(acc[0], la, lb);
        ptx::f2_unpack(acc[1], lc, ld);
        lsum += (la + lb) + (lc + ld);
        asm volatile("" : "+r"(sink));
    }
    long long t1 = clock64();
    out[threadIdx.x] = lsum + sink;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tbase, 256);
}
template <int MODE> void run(const char* name) {
    float* o; long long* c; cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 8);
    k<MODE><<<1, 128>>>(o, c, 1.4427f, 200);
    k<MODE><<<1, 128>>>(o, c, 1.4427f, 200);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-44s %s cycles per 128-score row = %.1f\n", name, cudaGetErrorString(e), h / 200.0);
}
int main() {
    run<6>("tcgen05.ld S (4 x 32x32b.x32) + wait");
    run<3>("ld + row max");
    run<4>("ld + max + exp (P to a sink)");
    run<5>("ld + exp + st P + wait (no max)");
    run<2>("ld + max + exp + st P + wait (kernel order)");
}
