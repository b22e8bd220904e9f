// Exp body of the softmax (128 scores per thread -> bf16 P + row sum), one warp per SMSP (4 warps),
// with EMU of every 8 pairs computed by the FMA-pipe polynomial (ptx::exp2_emu2) instead of
// MUFU.EX2.  Prints cycles per 128-element row.  Same code as sm100_softmax.cu exp_tile minus the
// TMEM store (results XORed into a sink).
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace vista;
template <int EMU>
__global__ void k(float* out, long long* cyc, float sl2, float neg, int iters) {
    uint32_t r[4][32];
    for (int c = 0; c < 4; ++c)
        for (int i = 0; i < 32; ++i) r[c][i] = __float_as_uint((threadIdx.x + c * 32 + i) * 1e-3f);
    uint32_t sink = 0;
    float lsum = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
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
                uint64_t p2;
                if (EMU > 0 && (j & 7) >= 8 - EMU) {
                    p2 = ptx::exp2_emu2(x2);
                } else {
                    float x0, x1;
                    ptx::f2_unpack(x2, x0, x1);
                    p2 = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
                }
                acc[j & 1] = ptx::f2_add(acc[j & 1], p2);
                float p0, p1;
                ptx::f2_unpack(p2, p0, p1);
                pk[j] = ptx::pack_bf16x2(p0, p1);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) sink ^= pk[j];
        }
        float la, lb, lc, ld;
        ptx::f2_unpack(acc[0], la, lb);
        ptx::f2_unpack(acc[1], lc, ld);
        lsum += (la + lb) + (lc + ld);
        neg -= 1e-7f;
        asm volatile("" : "+r"(sink));
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = lsum + sink;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int EMU> void run(int warps) {
    float* o; long long* c; cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 8);
    k<EMU><<<1, warps * 32>>>(o, c, 1.4427f, -2.f, 200);
    k<EMU><<<1, warps * 32>>>(o, c, 1.4427f, -2.f, 200);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("EMU %d/8 warps=%d  cycles per 128-element row = %.1f\n", EMU, warps, h / 200.0);
}
int main() {
    for (int w : {4, 8}) { run<0>(w); run<1>(w); run<2>(w); run<3>(w); run<4>(w); }
}
