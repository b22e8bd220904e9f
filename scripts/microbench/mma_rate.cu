// tcgen05.mma issue/execute rate on B200 (cta_group::1, bf16 -> f32), all SMs busy, one CTA/SM.
// Modes: 0 SS M128 N128 (the S GEMM), 1 TS M128 N128 (the PV GEMM, A = P in TMEM), 2 SS M128 N256,
// 3 PV+S pattern (8 TS then 8 SS), 4 SS M128 N128 K-major A, MN-major B (like PV's V operand, SS).
// Prints cycles per MMA instruction (K = 16) measured on CTA 0 over R rounds of 8 MMAs + commit/wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2510_22049_b200/csrc
#include <cstdio>
#include <cstdint>
#include "sm100_ptx.cuh"
using namespace vista;
constexpr int R = 2000;
__device__ int g_fill;

template <int MODE, bool WAIT>
__global__ void __launch_bounds__(128, 1) k(long long* out) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc(&tbase, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tbase;
    if (g_fill) {  // random bf16 in [-2, 2) in all operand smem and in the TMEM P columns
        uint32_t x = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
        for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            const uint32_t lo = 0x3f80u | ((x & 0x7f) ) | ((x >> 7 & 1) << 15), hi = 0x3f80u | ((x >> 8) & 0x7f) | ((x >> 15 & 1) << 15);
            reinterpret_cast<uint32_t*>(smem_raw + (base - ptx::smem_u32(smem_raw)))[i] = lo | (hi << 16);
        }
        const uint32_t lanes = (uint32_t)((warp % 4) * 32) << 16;
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; r[j] = (0x3f80u | (x & 0x7f)) | ((0x3f80u | ((x >> 8) & 0x7f)) << 16); }
        ptx::tmem_st32(tmem + lanes + 256, r);
        ptx::tmem_st32(tmem + lanes + 288, r);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
    }
    long long t0 = 0, t1 = 0;
    if (warp == 1) {
        constexpr uint32_t idS = ptx::idesc_bf16_f32(128, 128, 0, 0);
        constexpr uint32_t idS256 = ptx::idesc_bf16_f32(128, 256, 0, 0);
        constexpr uint32_t idP = ptx::idesc_bf16_f32(128, 128, 0, 1);
        const uint32_t sA = base, sB = base + 65536;
        uint32_t ph = 0;
        for (int r = -10; r < R; ++r) {
            if (r == 0) t0 = clock64();
            if (MODE == 0 || MODE == 3) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    ptx::mma_ss_w(tmem, ptx::sdesc_sw128(sA + off, 16, 1024), ptx::sdesc_sw128(sB + off, 16, 1024), idS, kk > 0);
                }
            }
            if (MODE == 1 || MODE == 3) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    ptx::mma_ts_w(tmem + 128, tmem + 256 + kk * 8, ptx::sdesc_sw128(sB + kk * 2048, 16384, 1024), idP, kk > 0);
            }
            if (MODE == 5) {  // SS M128 N64
                constexpr uint32_t idS64 = ptx::idesc_bf16_f32(128, 64, 0, 0);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    ptx::mma_ss_w(tmem, ptx::sdesc_sw128(sA + off, 16, 1024), ptx::sdesc_sw128(sB + off, 16, 1024), idS64, kk > 0);
                }
            }
            if (MODE == 6) {  // TS M128 N128 with K=64 keys (4 MMAs) -- half-tile PV
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    ptx::mma_ts_w(tmem + 128, tmem + 256 + kk * 8, ptx::sdesc_sw128(sB + kk * 2048, 16384, 1024), idP, kk > 0);
            }
            if (MODE == 2) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                    ptx::mma_ss_w(tmem, ptx::sdesc_sw128(sA + off, 16, 1024), ptx::sdesc_sw128(sB + 2 * off, 16, 1024), idS256, kk > 0);
                }
            }
            if (WAIT || r == R - 1) {
                ptx::mma_commit_w(&bar);
                ptx::mbar_wait(&bar, ph);
                ph ^= 1;
            }
        }
        t1 = clock64();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
}

template <int MODE, bool WAIT>
void run(const char* name, int mmas_per_round) {
    long long* d; cudaMalloc(&d, 8 * 148);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k<MODE, WAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<MODE, WAIT><<<148, 128, smem>>>(d);
    k<MODE, WAIT><<<148, 128, smem>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-34s %s  cyc/MMA (CTA0) %.1f  (max CTA) %.1f\n", name, cudaGetErrorString(e), (double)h[0] / R / mmas_per_round,
           mx / R / mmas_per_round);
    cudaFree(d);
}
int main() {
    for (int fill = 1; fill < 2; ++fill) {
    cudaMemcpyToSymbol(g_fill, &fill, 4);
    printf("fill=%d\n", fill);
    run<0, false>("SS M128 N128 K16 (S GEMM)", 8);
    run<1, false>("TS M128 N128 K16 (PV GEMM)", 8);
    run<2, false>("SS M128 N256 K16", 8);
    run<3, false>("PV+S pattern (8 TS + 8 SS)", 16);
    run<5, false>("SS M128 N64 K16", 8);
    run<6, false>("TS M128 N128 K16 (4 per round)", 4);
    run<0, true>("SS M128 N128, wait per 8", 8);
    run<1, true>("TS M128 N128, wait per 8", 8);
    run<3, true>("PV+S, wait per 16", 16);
    }
    return 0;
}
