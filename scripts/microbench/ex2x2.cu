// MUFU.EX2 throughput per SMSP: f32 vs f16x2 vs bf16x2 (cycles per warp-instruction, 1 and 2 warps/SMSP)
#include <cstdio>
#include <cstdint>
#define N 4096
template <int OP>
__global__ void k(float* out, long long* cyc, float a) {
    float x[8];
    uint32_t h[8];
    for (int i = 0; i < 8; ++i) { x[i] = -a * (threadIdx.x + i) * 1e-3f; h[i] = 0xBC00BC00u ^ (i << 3); }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            if (OP == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
            if (OP == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i] + h[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int OP> void run(const char* name, int warps) {
    float* o; long long* c; cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 8);
    k<OP><<<1, warps * 32>>>(o, c, 0.5f);
    k<OP><<<1, warps * 32>>>(o, c, 0.5f);
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    const double per_smsp = (double)(warps / 4) * N * 8;
    printf("%-10s warps=%d  cycles per warp-instr per SMSP = %.2f  (exps per clk per SMSP = %.1f)\n", name, warps,
           hc / per_smsp, per_smsp * 32 * (OP ? 2 : 1) / hc);
}
int main() {
    for (int w : {4, 8}) { run<0>("f32", w); run<1>("f16x2", w); run<2>("bf16x2", w); }
}
