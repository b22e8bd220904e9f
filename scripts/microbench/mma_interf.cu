// Tensor-core rate under interference (B200): warp 1 issues the PV+S pattern (8 TS + 8 SS MMAs,
// M128 N128 K16) back to back; warps 4..7 optionally generate
//   mode 1: TMEM reads  (tcgen05.ld 32x32b.x32 x4 + wait, like the softmax S load), continuous
//   mode 2: TMEM writes (tcgen05.st 32x32b.x16 x4 + wait, like the P store), continuous
//   mode 3: bulk global->smem copies (cp.async.bulk, 32 KB per round, like the K/V TMA loads)
//   mode 4: modes 1+2 with a softmax-like duty cycle (one S load + one P store per 1000 clk)
// Prints cycles per MMA on CTA 0 (all 148 SMs run the same).
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace vista;
constexpr int R = 1000;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(long long* out, const uint8_t* gsrc) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bar, bbar;
    __shared__ uint32_t tbase;
    __shared__ volatile int done;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::mbar_init(&bbar, 1); ptx::fence_mbar_init(); done = 0; }
    if (warp == 0) ptx::tmem_alloc(&tbase, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tbase;
    long long t0 = 0, t1 = 0;
    if (warp == 1) {
        constexpr uint32_t idS = ptx::idesc_bf16_f32(128, 128, 0, 0);
        constexpr uint32_t idP = ptx::idesc_bf16_f32(128, 128, 0, 1);
        const uint32_t sA = base, sB = base + 65536;
        for (int r = -10; r < R; ++r) {
            if (r == 0) t0 = clock64();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                ptx::mma_ts_w(tmem + 128, tmem + 256 + kk * 8, ptx::sdesc_sw128(sB + kk * 2048, 16384, 1024), idP, kk > 0);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                ptx::mma_ss_w(tmem, ptx::sdesc_sw128(sA + off, 16, 1024), ptx::sdesc_sw128(sB + off, 16, 1024), idS, kk > 0);
            }
        }
        ptx::mma_commit_w(&bar);
        ptx::mbar_wait(&bar, 0);
        t1 = clock64();
        if (lane == 0) done = 1;
    } else if (warp >= 4) {
        const uint32_t lanes = (uint32_t)((warp % 4) * 32) << 16;
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) r[j] = j;
        uint32_t ph = 0;
        while (!done) {
            if (MODE == 1 || MODE == 4) {
                uint32_t a[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tmem + lanes + 384 + c * 32 - 384 + 384, a[c]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::reg_fence(a[c]);
                r[0] += a[0][0] + a[3][31];
            }
            if (MODE == 2 || MODE == 4) {
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) pk[j] = r[j] + j;
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_st16(tmem + lanes + 448 + c * 16, pk);
                ptx::tmem_wait_st();
            }
            if (MODE == 3 && warp == 4) {
                if (lane == 0) {
                    ptx::mbar_arrive_expect_tx(&bbar, 32768);
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(base + 131072), "l"(gsrc + (blockIdx.x % 64) * 32768), "r"(32768),
                                 "r"(ptx::smem_u32(&bbar)) : "memory");
                }
                ptx::mbar_wait(&bbar, ph);
                ph ^= 1;
            }
            if (MODE == 4) __nanosleep(400);
        }
        if (r[0] == 12345) out[1000] = 1;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name) {
    long long* d; cudaMalloc(&d, 8 * 2048);
    uint8_t* g; cudaMalloc(&g, 64 * 32768 + 4096); cudaMemset(g, 0, 64 * 32768 + 4096);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<MODE><<<148, 256, smem>>>(d, g);
    k<MODE><<<148, 256, smem>>>(d, g);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("%-44s %s  cyc/MMA %.1f\n", name, cudaGetErrorString(e), (double)h[0] / R / 16);
    cudaFree(d); cudaFree(g);
}
int main() {
    run<0>("PV+S alone");
    run<1>("+ continuous TMEM reads (4 warps)");
    run<2>("+ continuous TMEM writes (4 warps)");
    run<3>("+ continuous 32 KB bulk copies");
    run<4>("+ softmax-like TMEM ld/st duty cycle");
    return 0;
}
