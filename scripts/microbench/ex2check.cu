// Does ex2.approx.f16x2 / bf16x2 compute both halves? (one MUFU.EX2.F16 per 32-bit register)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
__global__ void k(uint32_t* out, uint32_t a, uint32_t b) {
    uint32_t x = a, y = b;
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(y));
    out[0] = x; out[1] = y;
}
int main() {
    __half2 h = __floats2half2_rn(-1.0f, -3.0f);
    __nv_bfloat162 b = __floats2bfloat162_rn(-1.0f, -3.0f);
    uint32_t a, bb; memcpy(&a, &h, 4); memcpy(&bb, &b, 4);
    uint32_t* d; cudaMalloc(&d, 8);
    k<<<1, 1>>>(d, a, bb);
    uint32_t r[2]; cudaMemcpy(r, d, 8, cudaMemcpyDeviceToHost);
    __half2 rh; __nv_bfloat162 rb; memcpy(&rh, &r[0], 4); memcpy(&rb, &r[1], 4);
    printf("f16x2: %f %f   bf16x2: %f %f  (expect 0.5 0.125)\n", __low2float(rh), __high2float(rh), __low2float(rb), __high2float(rb));
}
