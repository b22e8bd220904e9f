// sm100_gemm.cu -- the dense projections of the multi-layer summarizer (NEXT-3) on tcgen05.
//
// C[M, N] = A[M, K] B[N, K]^T (+ R) in bf16 with fp32 accumulation in TMEM, A and B both K-major
// (row-major activations, weights stored [out][in]):
//   projections  [Q | K | V | G] = X [Wq | Wk | Wv | Wg]^T: the N tiles are routed to NSPLIT separate
//                output tensors of width N / NSPLIT (so K and V come out as plain [R, H, d] tensors the
//                QLA state kernel streams with TMA)
//   output       X <- X + O Wo^T with the residual added in the epilogue (O already SGLU-gated by the
//                rows kernel, reading R23)
// Persistent, one CTA per SM; 128 x 128 output tiles (n fastest, so consecutive tiles of a CTA reuse
// the A rows from L2), K in blocks of 64 (one 128-B swizzle atom), a 6-stage TMA ring of A / B blocks.
//   warp 0       TMA producer          warp 1   MMA issuer (accumulator double-buffered in TMEM)
//   warps 8-15   epilogue: TMEM -> (+ residual) -> bf16, coalesced through a TMEM round trip
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdlib.h>

#include <algorithm>

#include "internal.h"
#include "sm100_ptx.cuh"

namespace vista {

bool make_map_bf16(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                   const cuuint32_t* box);

namespace {

constexpr int kBlk = 128 * 128;  // a 128-row x 64-column bf16 block (16 KB)
constexpr int kThreads = 512;
constexpr int kEpi = 256;
constexpr int kStages = 6;
constexpr int kStageBytes = 2 * kBlk;  // A, B
constexpr int kBarOff = kStages * kStageBytes;
constexpr int kSmem = kBarOff + 256 + 1024;
static_assert(kSmem <= 232448, "shared memory");

struct GemmBars {
    uint64_t full[kStages], empty[kStages];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};

struct GemmParams {
    int M, N, K;
    int nsplit;                      // outputs: N / nsplit columns each
    __nv_bfloat16* out[4];           // [M, N / nsplit] row-major each
    const __nv_bfloat16* resid;      // [M, N] or NULL (may alias out[0])
};

// P.out[which] without a dynamically indexed copy of the parameter array in local memory
__device__ __forceinline__ __nv_bfloat16* out_sel(const GemmParams& P, int which) {
    return which == 0 ? P.out[0] : which == 1 ? P.out[1] : which == 2 ? P.out[2] : P.out[3];
}

__device__ __forceinline__ void st_v8(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// Epilogue of one 64-column block of a 128-row accumulator (this warp: 32 rows, TMEM address tc):
// fp32 -> bf16 (+ residual) -> global, coalesced through a permuted TMEM round trip (after a
// 16x256b load a quad of threads holds 128 contiguous bytes of one row).  row0 = the warp's first
// global row; col0 = the block's first global column (residual), c_out its column in `outp`.
template <bool RESID>  // RESID: P.resid is set (a separate instantiation: no prefetch registers otherwise)
__device__ __forceinline__ void store_block64(const GemmParams& P, uint32_t tc, int row0, int lane,
                                              __nv_bfloat16* outp, int nw, int col0, int c_out) {
    // the residual rows this thread adds, loaded first: their latency overlaps the TMEM round trip
    // (loaded after it, every half waited for its own loads -- the output GEMM was latency-bound)
    uint4 xr[2][2][2];
    if constexpr (RESID) {
#pragma unroll
        for (int half = 0; half < 2; ++half)
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int row = row0 + 16 * half + (lane >> 2) + 8 * rr;
                if (row < P.M) {
                    const uint4* rs = reinterpret_cast<const uint4*>(P.resid + (size_t)row * P.N + col0 + 16 * (lane & 3));
                    xr[half][rr][0] = rs[0];
                    xr[half][rr][1] = rs[1];
                }
            }
    }
    uint32_t a[32];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32_sync(tc + c * 32, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int w = 16 * c + j;  // packed word w = columns 2w, 2w + 1
            const int g = (w >> 1) & 3, p = w >> 3, e = w & 1;
            a[8 * g + 2 * p + e] = ptx::pack_bf16x2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        }
    }
    ptx::tmem_st32(tc, a);
    ptx::tmem_wait_st();
    const int p = lane & 3;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        uint32_t r[16];
        ptx::tmem_ld16x256b_x4(tc + ((uint32_t)(16 * half) << 16), r);
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
        const int ra = row0 + 16 * half + (lane >> 2);
        uint32_t v0[8] = {r[0], r[1], r[4], r[5], r[8], r[9], r[12], r[13]};
        uint32_t v1[8] = {r[2], r[3], r[6], r[7], r[10], r[11], r[14], r[15]};
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int row = ra + 8 * rr;
            uint32_t* v = rr ? v1 : v0;
            if (row >= P.M) continue;
            if constexpr (RESID) {  // + residual (16 contiguous bf16 of the row), added in f32
                const uint4 x0 = xr[half][rr][0], x1 = xr[half][rr][1];
                const uint32_t xw[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    v[e] = ptx::pack_bf16x2(__uint_as_float(v[e] << 16) + __uint_as_float(xw[e] << 16),
                                            __uint_as_float(v[e] & 0xFFFF0000u) + __uint_as_float(xw[e] & 0xFFFF0000u));
            }
            st_v8(outp + (size_t)row * nw + c_out + 16 * p, *reinterpret_cast<const uint32_t(*)[8]>(v));
        }
    }
}

template <int SB, int ST>
__device__ __forceinline__ void issue_kblock(uint32_t tacc, uint32_t base, bool acc) {
    const uint32_t a = base + ST * SB, b = a + kBlk;
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 0);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
        ptx::mma_ss_w(tacc, ptx::sdesc_sw128(a + kk * 32, 16, 1024), ptx::sdesc_sw128(b + kk * 32, 16, 1024), id,
                      (acc || kk > 0) ? 1u : 0u);
}
__device__ __forceinline__ void issue_kblock_d(int st, uint32_t tacc, uint32_t base, bool acc) {
    switch (st) {
        case 0: issue_kblock<kStageBytes, 0>(tacc, base, acc); break;
        case 1: issue_kblock<kStageBytes, 1>(tacc, base, acc); break;
        case 2: issue_kblock<kStageBytes, 2>(tacc, base, acc); break;
        case 3: issue_kblock<kStageBytes, 3>(tacc, base, acc); break;
        case 4: issue_kblock<kStageBytes, 4>(tacc, base, acc); break;
        default: issue_kblock<kStageBytes, 5>(tacc, base, acc); break;
    }
}

template <bool RESID>
__global__ void __launch_bounds__(kThreads, 1)
    sm100_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      const GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = ptx::smem_u32(smem);
    GemmBars* bars = reinterpret_cast<GemmBars*>(smem + kBarOff);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bars->full[s], 1);
            ptx::mbar_init(&bars->empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->acc_full[b], 1);
            ptx::mbar_init(&bars->acc_empty[b], kEpi);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);
    const int num_m = (P.M + 127) / 128, num_n = P.N / 128, nk = P.K / 64;
    const int num_tiles = num_m * num_n;

    if (warp == 0) {
        // ---------------- TMA producer
        ptx::tma_prefetch(&mapA);
        ptx::tma_prefetch(&mapB);
        // A rows are shared by the CTAs on the N tiles of an M block: kept in L2 (as in the pair kernel)
        const uint64_t pol_a = ptx::policy_evict_last(), pol_b = ptx::policy_evict_last();
        int st = 0;
        uint32_t ph = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const int m = t / num_n, n = t % num_n;
            for (int kb = 0; kb < nk; ++kb) {
                ptx::mbar_wait(&bars->empty[st], ph ^ 1);
                ptx::mbar_arrive_expect_tx_w(&bars->full[st], kStageBytes);
                uint8_t* s = smem + st * kStageBytes;
                ptx::tma_load_3d_w(s, &mapA, &bars->full[st], kb * 64, m * 128, 0, pol_a);
                ptx::tma_load_3d_w(s + kBlk, &mapB, &bars->full[st], kb * 64, n * 128, 0, pol_b);
                if (++st == kStages) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        int st = 0, ab = 0;
        uint32_t ph = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            ptx::mbar_wait(&bars->acc_empty[ab], ((aphm >> ab) & 1u) ^ 1);
            aphm ^= 1u << ab;
            const uint32_t tacc = tmem + ab * 128;
            for (int kb = 0; kb < nk; ++kb) {
                ptx::mbar_wait(&bars->full[st], ph);
                ptx::tc_fence_after();
                issue_kblock_d(st, tacc, base, kb > 0);
                ptx::mma_commit_w(&bars->empty[st]);
                if (++st == kStages) { st = 0; ph ^= 1; }
            }
            ptx::mma_commit_w(&bars->acc_full[ab]);
            ab ^= 1;
        }
    } else if (warp >= 8) {
        // ---------------- epilogue
        const int wq = warp % 4;
        const int chalf = (warp - 8) / 4;  // columns [64 chalf, 64 chalf + 64) of the tile
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const int nw = P.N / P.nsplit;  // columns of one output tensor
        int ab = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const int m = t / num_n, n = t % num_n;
            const int col0 = n * 128 + chalf * 64;       // global column of this warp's first column
            const int which = col0 / nw, c_out = col0 % nw;
            __nv_bfloat16* outp = out_sel(P, which);
            ptx::mbar_wait(&bars->acc_full[ab], ((aphm >> ab) & 1u));
            aphm ^= 1u << ab;
            ptx::tc_fence_after();
            store_block64<RESID>(P, tmem + lane_bits + ab * 128 + chalf * 64, m * 128 + wq * 32, lane, outp, nw, col0,
                                 c_out);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bars->acc_empty[ab]);
            ab ^= 1;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 256);
}


// ---- CTA pair (cta_group::2): 256 x 256 output tiles.  CTA r of the pair loads the A rows
// [256 m + 128 r, + 128) and the B rows [256 n + 128 r, + 128) of every 64-wide K block; the leader
// issues M = 256, N = 256 MMAs over both CTAs' shared memory, each CTA accumulating its 128 rows x 256
// columns in TMEM (double-buffered: 2 x 256 columns).  Per K block each SM reads 16 KB of A and 16 KB
// of B from shared memory per 512 MMA clocks (64 B/clk) instead of 32 KB per 256 clocks in the
// 128 x 128 kernel, which is shared-memory bound at half the tensor rate.
template <int ST>
__device__ __forceinline__ void issue_kblock2(uint32_t tacc, uint32_t base, bool acc) {
    const uint32_t a = base + ST * kStageBytes, b = a + kBlk;
    constexpr uint32_t id = ptx::idesc_bf16_f32(256, 256, 0, 0);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
        ptx::mma2_ss_w(tacc, ptx::sdesc_sw128(a + kk * 32, 16, 1024), ptx::sdesc_sw128(b + kk * 32, 16, 1024), id,
                       (acc || kk > 0) ? 1u : 0u);
}
__device__ __forceinline__ void issue_kblock2_d(int st, uint32_t tacc, uint32_t base, bool acc) {
    switch (st) {
        case 0: issue_kblock2<0>(tacc, base, acc); break;
        case 1: issue_kblock2<1>(tacc, base, acc); break;
        case 2: issue_kblock2<2>(tacc, base, acc); break;
        case 3: issue_kblock2<3>(tacc, base, acc); break;
        case 4: issue_kblock2<4>(tacc, base, acc); break;
        default: issue_kblock2<5>(tacc, base, acc); break;
    }
}

template <bool RESID>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    sm100_gemm2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                       const GemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = ptx::smem_u32(smem);
    GemmBars* bars = reinterpret_cast<GemmBars*>(smem + kBarOff);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rank = (int)ptx::cluster_ctarank();
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bars->full[s], 1);   // the leader's expect_tx + both CTAs' TMA bytes
            ptx::mbar_init(&bars->empty[s], 1);  // the leader's MMA commit, multicast to both CTAs
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->acc_full[b], 1);
            ptx::mbar_init(&bars->acc_empty[b], 16);  // 8 epilogue warps of each CTA, one arrive per warp
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc2(&bars->tmem_base, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // both CTAs' barriers exist before any remote signal
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);
    const int num_m = (P.M + 255) / 256, num_n = P.N / 256, nk = P.K / 64;
    const int num_tiles = num_m * num_n;

    if (warp == 0) {
        // ---------------- TMA producer (both CTAs): this CTA's A rows and B rows of each K block
        ptx::tma_prefetch(&mapA);
        ptx::tma_prefetch(&mapB);
        // A rows are read by the pairs working on the num_n output tiles of an M block at about the
        // same time: kept in L2 for the others (A/B: evict_first read A ~3x from DRAM, QKVG GEMM
        // 1.18 ms; evict_normal 1.04; evict_last 1.03)
#ifndef VISTA_GEMM_APOL
#define VISTA_GEMM_APOL 2
#endif
        const uint64_t pol_a = VISTA_GEMM_APOL == 0 ? ptx::policy_evict_first()
                             : VISTA_GEMM_APOL == 1 ? ptx::policy_evict_normal() : ptx::policy_evict_last();
        const uint64_t pol_b = ptx::policy_evict_last();
        int st = 0;
        uint32_t ph = 0;
        for (int t = pair; t < num_tiles; t += npairs) {
            const int m = t / num_n, n = t % num_n;
            for (int kb = 0; kb < nk; ++kb) {
                ptx::mbar_wait(&bars->empty[st], ph ^ 1);
                const uint32_t fl = ptx::mapa(ptx::smem_u32(&bars->full[st]), 0);
                if (rank == 0) ptx::mbar_arrive_expect_tx_w(&bars->full[st], 2 * kStageBytes);
                const uint32_t s = base + st * kStageBytes;
                ptx::tma_load_3d_2sm_w(s, &mapA, fl, kb * 64, m * 256 + rank * 128, 0, pol_a);
                ptx::tma_load_3d_2sm_w(s + kBlk, &mapB, fl, kb * 64, n * 256 + rank * 128, 0, pol_b);
                if (++st == kStages) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ---------------- MMA issuer (leader CTA)
        int st = 0, ab = 0;
        uint32_t ph = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        for (int t = pair; t < num_tiles; t += npairs) {
            ptx::mbar_wait(&bars->acc_empty[ab], ((aphm >> ab) & 1u) ^ 1);
            aphm ^= 1u << ab;
            const uint32_t tacc = tmem + ab * 256;
            for (int kb = 0; kb < nk; ++kb) {
                ptx::mbar_wait(&bars->full[st], ph);
                ptx::tc_fence_after();
                issue_kblock2_d(st, tacc, base, kb > 0);
                ptx::mma2_commit_mc_w(&bars->empty[st]);
                if (++st == kStages) { st = 0; ph ^= 1; }
            }
            ptx::mma2_commit_mc_w(&bars->acc_full[ab]);
            ab ^= 1;
        }
    } else if (warp >= 8) {
        // ---------------- epilogue (both CTAs): this CTA's 128 rows x 256 columns of the tile
        const int wq = warp % 4;
        const int cq = (warp - 8) / 4;  // columns [128 cq, 128 cq + 128) of the tile
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const int nw = P.N / P.nsplit;
        const uint32_t acc_empty_l = ptx::mapa(ptx::smem_u32(&bars->acc_empty[0]), 0);
        int ab = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        for (int t = pair; t < num_tiles; t += npairs) {
            const int m = t / num_n, n = t % num_n;
            ptx::mbar_wait(&bars->acc_full[ab], ((aphm >> ab) & 1u));
            aphm ^= 1u << ab;
            ptx::tc_fence_after();
#pragma unroll 1
            for (int sb = 0; sb < 2; ++sb) {
                const int col0 = n * 256 + cq * 128 + sb * 64;
                const int which = col0 / nw, c_out = col0 % nw;
                store_block64<RESID>(P, tmem + lane_bits + ab * 256 + cq * 128 + sb * 64, m * 256 + rank * 128 + wq * 32,
                              lane, out_sel(P, which), nw, col0, c_out);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) ptx::mbar_arrive(&bars->acc_empty[ab]);
                else ptx::mbar_arrive_cluster(acc_empty_l + ab * 8, 1);
            }
            ab ^= 1;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // no CTA leaves (deallocates) while the pair's MMAs may still target it
    if (warp == 1) ptx::tmem_dealloc2(tmem, 512);
}

// bf16 row-major [rows, cols] as a TMA map with 64 x 128 boxes and the 128-B swizzle
bool make_mat_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld) {
    const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1), 1};
    const cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)ld * 2 * (rows > 0 ? rows : 1)};
    const cuuint32_t box[3] = {64, 128, 1};
    return make_map_bf16(map, base, 3, dims, strides, box);
}

}  // namespace

// C = A B^T (+ resid); A [M, K] (lda), B [N, K], outputs: nsplit tensors [M, N / nsplit].
// K % 64 == 0, N % 128 == 0, (N / nsplit) % 64 == 0.
cudaError_t launch_sm100_gemm(int M, int N, int K, const void* A, int64_t lda, const void* Bw, int nsplit,
                              void* const* outs, const void* resid, int num_sms, cudaStream_t stream) {
    if (M == 0) return cudaSuccess;
    if (K % 64 || N % 128 || nsplit < 1 || nsplit > 4 || (N / nsplit) % 64) return cudaErrorInvalidValue;
    CUtensorMap ma, mb;
    if (!make_mat_map(&ma, A, M, K, lda) || !make_mat_map(&mb, Bw, N, K, K)) return cudaErrorInvalidValue;
    GemmParams P;
    P.M = M;
    P.N = N;
    P.K = K;
    P.nsplit = nsplit;
    for (int i = 0; i < 4; ++i) P.out[i] = reinterpret_cast<__nv_bfloat16*>(outs[i < nsplit ? i : 0]);
    P.resid = reinterpret_cast<const __nv_bfloat16*>(resid);
    static const bool pair_off = [] {
        const char* e = getenv("VISTA_GEMM_PAIR");
        return e && e[0] == '0';
    }();
    if (N % 256 == 0 && !pair_off) {  // CTA-pair 256 x 256 tiles
        const int tiles = ((M + 255) / 256) * (N / 256);
        const int pairs = std::min(tiles, num_sms / 2);
        const void* fn2 = P.resid ? reinterpret_cast<const void*>(sm100_gemm2_kernel<true>)
                                  : reinterpret_cast<const void*>(sm100_gemm2_kernel<false>);
        const cudaError_t a = set_smem_attr(fn2, kSmem);
        if (a != cudaSuccess) return a;
        if (P.resid) sm100_gemm2_kernel<true><<<2 * pairs, kThreads, kSmem, stream>>>(ma, mb, P);
        else sm100_gemm2_kernel<false><<<2 * pairs, kThreads, kSmem, stream>>>(ma, mb, P);
        return cudaGetLastError();
    }
    const int tiles = ((M + 127) / 128) * (N / 128);
    const int grid = tiles < num_sms ? tiles : num_sms;
    const void* fn = P.resid ? reinterpret_cast<const void*>(sm100_gemm_kernel<true>)
                             : reinterpret_cast<const void*>(sm100_gemm_kernel<false>);
    const cudaError_t a = set_smem_attr(fn, kSmem);
    if (a != cudaSuccess) return a;
    if (P.resid) sm100_gemm_kernel<true><<<grid, kThreads, kSmem, stream>>>(ma, mb, P);
    else sm100_gemm_kernel<false><<<grid, kThreads, kSmem, stream>>>(ma, mb, P);
    return cudaGetLastError();
}

}  // namespace vista
