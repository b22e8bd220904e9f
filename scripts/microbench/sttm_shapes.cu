// tcgen05.st throughput/latency by shape: one warp per SMSP (4 warps), each stores 64 columns x 32
// lanes x 4 B = 8 KB per iteration, then tcgen05.wait::st.  Cycles per iteration on warp 0.
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace vista;
template <int SH>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int iters, int do_wait) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc(&tbase, 128);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t t = tbase + ((uint32_t)(warp * 32) << 16);
    uint32_t r[64];
    for (int i = 0; i < 64; ++i) r[i] = threadIdx.x * 64 + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        r[0] += it;
        if (SH == 0) {  // 4 x 32x32b.x16
            for (int c = 0; c < 4; ++c) {
                uint32_t w[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) w[j] = r[c * 16 + j];
                ptx::tmem_st16(t + c * 16, w);
            }
        } else if (SH == 1) {  // 2 x 32x32b.x32
            for (int c = 0; c < 2; ++c) {
                uint32_t w[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) w[j] = r[c * 32 + j];
                ptx::tmem_st32(t + c * 32, w);
            }
        } else if (SH == 2) {  // 16x256b.x8 twice (lanes 0-15 and 16-31 of the quarter): 32 regs each
            for (int hh = 0; hh < 2; ++hh) {
                asm volatile(
                    "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                    "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t + ((uint32_t)(16 * hh) << 16)),
                    "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                    "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                    "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                    "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
                    : "memory");
            }
        }
        if (do_wait) ptx::tmem_wait_st();
    }
    ptx::tmem_wait_st();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tbase, 128);
}
template <int SH> void run(const char* name, int w) {
    long long* c; cudaMalloc(&c, 8);
    k<SH><<<1, 128>>>(c, 1000, w);
    k<SH><<<1, 128>>>(c, 1000, w);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s wait=%d %s cycles per 8 KB per warp = %.1f\n", name, w, cudaGetErrorString(e), h / 1000.0);
}
int main() {
    for (int w = 0; w < 2; ++w) {
        run<0>("4 x 32x32b.x16", w);
        run<1>("2 x 32x32b.x32", w);
        run<2>("2 x 16x256b.x8", w);
    }
}
