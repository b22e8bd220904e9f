// Is tcgen05.mma kind::f16 with A = f16 and B = bf16 (mixed formats in the instruction descriptor)
// computed correctly?  SS and TS (A from TMEM) variants, M128 N128 K16, integer-valued operands.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include "sm100_ptx.cuh"
using namespace vista;

__device__ __forceinline__ uint32_t sw_off(int r, int c) {  // bf16/f16 element (row r, col c < 64), SW128 K-major
    return r * 128 + (((c / 8) ^ (r % 8)) * 16) + (c % 8) * 2;
}
template <bool TS>
__global__ void k(float* out, uint32_t afmt, uint32_t bfmt) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sm = smem_raw + (base - ptx::smem_u32(smem_raw));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // A: rows r, k: value (r + k) % 5 - 2 ; B: rows n, k: (3n + k) % 7 - 3
    for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) {
        const int r = i / 16, c = i % 16;
        const float a = (float)((r + c) % 5 - 2), b = (float)((3 * r + c) % 7 - 3);
        uint16_t ab, bb;
        if (afmt == 0) { __half h = __float2half(a); memcpy(&ab, &h, 2); } else { __nv_bfloat16 h = __float2bfloat16(a); memcpy(&ab, &h, 2); }
        if (bfmt == 0) { __half h = __float2half(b); memcpy(&bb, &h, 2); } else { __nv_bfloat16 h = __float2bfloat16(b); memcpy(&bb, &h, 2); }
        *reinterpret_cast<uint16_t*>(sm + sw_off(r, c)) = ab;
        *reinterpret_cast<uint16_t*>(sm + 16384 + sw_off(r, c)) = bb;
    }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc(&tbase, 256);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tbase;
    if (TS) {  // A into TMEM cols [128, 136): lane r, col j holds k = 2j, 2j+1
        const int r = warp * 32 + lane;
        uint32_t v[16];
        for (int j = 0; j < 8; ++j) {
            uint16_t lo = *reinterpret_cast<uint16_t*>(sm + sw_off(r, 2 * j));
            uint16_t hi = *reinterpret_cast<uint16_t*>(sm + sw_off(r, 2 * j + 1));
            v[j] = lo | ((uint32_t)hi << 16);
        }
        for (int j = 8; j < 16; ++j) v[j] = 0;
        ptx::tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 128, v);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
    }
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 1) {
        const uint32_t id = (1u << 4) | (afmt << 7) | (bfmt << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        if (TS) ptx::mma_ts_w(tmem, tmem + 128, ptx::sdesc_sw128(base + 16384, 16, 1024), id, 0);
        else ptx::mma_ss_w(tmem, ptx::sdesc_sw128(base, 16, 1024), ptx::sdesc_sw128(base + 16384, 16, 1024), id, 0);
        ptx::mma_commit_w(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    const int r = warp * 32 + lane;
    for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32_sync(tmem + ((uint32_t)(warp * 32) << 16) + c * 32, v);
        for (int j = 0; j < 32; ++j) out[r * 128 + c * 32 + j] = __uint_as_float(v[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 256);
}
template <bool TS> void run(uint32_t af, uint32_t bf) {
    float* d; cudaMalloc(&d, 128 * 128 * 4);
    cudaFuncSetAttribute(k<TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<TS><<<1, 128, 64 * 1024>>>(d, af, bf);
    cudaError_t e = cudaDeviceSynchronize();
    static float h[128 * 128];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0; double maxe = 0;
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < 128; ++n) {
            double ref = 0;
            for (int c = 0; c < 16; ++c) ref += (double)((r + c) % 5 - 2) * (double)((3 * n + c) % 7 - 3);
            const double err = fabs(h[r * 128 + n] - ref);
            maxe = err > maxe ? err : maxe;
            bad += err > 1e-3;
        }
    printf("%s A=%s B=%s: %s  mismatches %d / 16384  max err %.3g\n", TS ? "TS" : "SS", af ? "bf16" : "f16",
           bf ? "bf16" : "f16", cudaGetErrorString(e), bad, maxe);
    cudaFree(d);
}
int main() {
    run<false>(1, 1); run<false>(0, 0); run<false>(0, 1); run<false>(1, 0);
    run<true>(1, 1); run<true>(0, 0); run<true>(0, 1);
}
