// Cycles for the softmax exp body on 128 fp32 scores per thread (one warp per SMSP, W warps per SM).
// Variants: 0 packed (FFMA2, 2x MUFU.EX2, FADD2, F2FP) as in the kernel; 1 scalar FFMA/FADD;
// 2 packed without the F2FP pack; 3 MUFU only.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t pk2(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void up2(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int V>
__global__ void k(float* out, long long* cyc, float sl2, float neg, int iters) {
    float r[128];
    for (int i = 0; i < 128; ++i) r[i] = (threadIdx.x + i) * 1e-3f;
    uint32_t sink = 0; float lsum = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint64_t acc0 = pk2(0.f, 0.f), acc1 = pk2(0.f, 0.f);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            float p0, p1;
            if (V == 1) {
                p0 = ex2(fmaf(r[2 * j], sl2, neg)); p1 = ex2(fmaf(r[2 * j + 1], sl2, neg));
                a0 += p0; a1 += p1;
            } else if (V == 3) {
                p0 = ex2(r[2 * j]); p1 = ex2(r[2 * j + 1]);
            } else {
                uint64_t x2; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x2) : "l"(pk2(r[2*j], r[2*j+1])), "l"(pk2(sl2, sl2)), "l"(pk2(neg, neg)));
                float x0, x1; up2(x2, x0, x1);
                p0 = ex2(x0); p1 = ex2(x1);
                uint64_t& acc = (j & 1) ? acc1 : acc0;
                asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(pk2(p0, p1)));
            }
            if (V != 2 && V != 3) { uint32_t pk; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk) : "f"(p1), "f"(p0)); sink ^= pk; }
            else sink ^= __float_as_uint(p0) ^ __float_as_uint(p1);
        }
        float b0, b1, c0, c1; up2(acc0, b0, b1); up2(acc1, c0, c1);
        lsum += a0 + a1 + b0 + b1 + c0 + c1;
        neg -= 1e-7f;
    }
    long long t1 = clock64();
    out[threadIdx.x] = lsum + sink;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int V> void run(const char* name, int warps) {
    float* o; long long* c; cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 8);
    k<V><<<1, warps * 32>>>(o, c, 1.4427f, -2.f, 200);
    k<V><<<1, warps * 32>>>(o, c, 1.4427f, -2.f, 200);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s warps=%d  cycles per 128-element row = %.1f\n", name, warps, h / 200.0);
}
int main() {
    for (int w : {4, 8}) {
        run<0>("packed ffma2+ex2+fadd2+f2fp", w); run<1>("scalar ffma+ex2+fadd+f2fp", w);
        run<2>("packed, no f2fp", w); run<3>("ex2 only", w);
    }
}
