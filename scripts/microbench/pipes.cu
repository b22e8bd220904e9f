// Pipe throughput microbenchmark on one SM: cycles per warp-instruction for MUFU.EX2, FFMA, FFMA2,
// FADD2, F2FP(bf16x2) with W warps (W/4 per SMSP).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#define N 4096
template <int OP>
__global__ void k(float* out, long long* cyc, float a) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = a + threadIdx.x * 1e-3f + i;
    uint64_t y[8];
    for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1, %2};" : "=l"(y[i]) : "f"(x[i]), "f"(x[i] + 1.f));
    uint32_t z[8] = {0};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0fBF000000;" : "+f"(x[i]));
            if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(y[i]));
            if (OP == 3) asm volatile("add.rn.f32x2 %0, %0, %0;" : "+l"(y[i]));
            if (OP == 4) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(z[i]) : "f"(x[i]), "f"(x[(i + 1) & 7]));
            if (OP == 4) asm volatile("" : "+f"(x[i]) : "r"(z[i]));
            if (OP == 5) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(x[(i + 1) & 7]), "f"(x[(i + 2) & 7]));
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) { s += x[i]; float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(y[i])); s += p + q + z[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
void run(const char* name, int warps) {
    float* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8 * 148);
    k<OP><<<1, warps * 32>>>(o, c, 0.5f);
    k<OP><<<1, warps * 32>>>(o, c, 0.5f);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    // instructions per SMSP = (warps/4) * N * 8
    double per_smsp = (double)((warps + 3) / 4) * N * 8;
    printf("%-8s warps=%2d  cycles/warp-instr per SMSP = %.2f\n", name, warps, h / per_smsp);
    cudaFree(o); cudaFree(c);
}
int main() {
    for (int w : {4, 8, 16}) {
        run<0>("ex2", w); run<1>("ffma", w); run<2>("ffma2", w); run<3>("fadd2", w); run<4>("f2fp", w); run<5>("fmnmx3", w);
    }
}
