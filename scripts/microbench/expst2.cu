// Softmax per-tile body (tcgen05.ld S -> row max -> exp2 -> bf16 P -> tcgen05.st P -> wait::st), one
// warp per SMSP, with different ways of storing P to TMEM:
//   ST 0: no store (P to a sink)   1: 4 x st.32x32b.x16 right after each 32-score chunk (kernel)
//   ST 2: 2 x st.x32 (after chunks 1, 3)   3: all P kept, 2 x st.x32 at the end
//   ST 4: 4 x st.x16, each deferred until the next chunk's exponentials are issued
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace vista;
template <int ST>
__global__ void __launch_bounds__(128, 1) k(float* out, long long* cyc, float sl2, int iters) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc(&tbase, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tS = tbase + ((uint32_t)(warp * 32) << 16);
    {
        uint32_t r[32];
        for (int c = 0; c < 4; ++c) {
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint((threadIdx.x + c * 32 + i) * 1e-3f);
            ptx::tmem_st32(tS + c * 32, r);
        }
        ptx::tmem_wait_st();
    }
    uint32_t sink = 0;
    float lsum = 0.f;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        uint32_t r[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tS + c * 32, r[c]);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::reg_fence(r[c]);
        float m = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int j = 0; j < 32; j += 2) m = ptx::max3(m, __uint_as_float(r[c][j]), __uint_as_float(r[c][j + 1]));
        const float neg = -m * sl2;
        const uint64_t sl2x2 = ptx::f2_pack(sl2, sl2);
        const uint64_t negx2 = ptx::f2_pack(neg, neg);
        uint64_t acc[2] = {ptx::f2_pack(0.f, 0.f), ptx::f2_pack(0.f, 0.f)};
        uint32_t pk[4][16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
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
                pk[c][j] = ptx::pack_bf16x2(p0, p1);
            }
            if (ST == 1) ptx::tmem_st16(tS + 128 + c * 16, pk[c]);
            if (ST == 4 && c > 0) ptx::tmem_st16(tS + 128 + (c - 1) * 16, pk[c - 1]);
            if (ST == 2 && (c & 1)) {
                uint32_t w[32];
#pragma unroll
                for (int j = 0; j < 16; ++j) { w[j] = pk[c - 1][j]; w[16 + j] = pk[c][j]; }
                ptx::tmem_st32(tS + 128 + (c - 1) * 16, w);
            }
        }
        if (ST == 4) ptx::tmem_st16(tS + 128 + 48, pk[3]);
        if (ST == 3) {
            uint32_t w[32];
#pragma unroll
            for (int j = 0; j < 16; ++j) { w[j] = pk[0][j]; w[16 + j] = pk[1][j]; }
            ptx::tmem_st32(tS + 128, w);
#pragma unroll
            for (int j = 0; j < 16; ++j) { w[j] = pk[2][j]; w[16 + j] = pk[3][j]; }
            ptx::tmem_st32(tS + 160, w);
        }
        if (ST == 5) {  // stores without the per-tile wait::st
            uint32_t w[32];
#pragma unroll
            for (int j = 0; j < 16; ++j) { w[j] = pk[0][j]; w[16 + j] = pk[1][j]; }
            ptx::tmem_st32(tS + 128, w);
#pragma unroll
            for (int j = 0; j < 16; ++j) { w[j] = pk[2][j]; w[16 + j] = pk[3][j]; }
            ptx::tmem_st32(tS + 160, w);
        } else if (ST == 0) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int j = 0; j < 16; ++j) sink ^= pk[c][j];
        } else if (ST != 5) {
            ptx::tmem_wait_st();
        }
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
template <int ST> void run(const char* name, int threads = 128) {
    float* o; long long* c; cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 8);
    k<ST><<<1, threads>>>(o, c, 1.4427f, 200);
    k<ST><<<1, threads>>>(o, c, 1.4427f, 200);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-44s warps=%d %s cycles per 128-score row = %.1f\n", name, threads / 32, cudaGetErrorString(e), h / 200.0);
}
int main() {
    run<0>("no P store (sink)");
    run<1>("4 x st.x16 inline (kernel)");
    run<2>("2 x st.x32");
    run<3>("2 x st.x32 at the end");
    run<4>("4 x st.x16 deferred one chunk");
    run<5>("2 x st.x32 at the end, no wait::st", 128);
    run<6>("ld + max + exp, wait::st only (no st)", 128);
    run<0>("no P store (sink)", 32);
    run<1>("4 x st.x16 inline (kernel)", 32);
    run<3>("2 x st.x32 at the end", 32);
}
