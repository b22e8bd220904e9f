// sm100_qla_bwd.cu -- QLA backward dK / dV on B200 (NEXT-2; gradients in qla_bwd.cu's header):
//     dV_j = phi1(k_j) dZ          dK_j = (v_j dZ^T) . phi1'(k_j)        (per user u, head h)
// Two 128x128x128 tcgen05 GEMMs per 128-item tile, both with dZ (bf16, pre-swizzled by
// qla_bwd_unit_kernel) as the B operand: MN-major ([K = c1][N = c2]) for dV, K-major
// ([N = c1][K = c2]) for dK'.  HBM-bound: per item-head 512 B of K+V read, 512 B of dK+dV written
// (bf16), 4 d^2 = 65,536 flop.
//
//   warp 0        TMA producer: K, V tiles (3 stages, freed by the MMA commit); dZ of the unit
//                 (bulk copy) on unit change
//   warp 1        MMA issuer (warp-wide, one elected lane); dV / dK' double-buffered in TMEM
//   warps 4..7    transform: phi1(K) in place (bf16)
//   warps 8..15   epilogue: TMEM -> bf16 rows of dV and of dK' . phi1'(K) (phi1' recomputed from
//                 the raw K rows re-read through L2), coalesced through a TMEM round trip
// Tiles are independent (no split partials): a CTA walks its stream-K range (work.cuh).
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "qla_common.cuh"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

bool make_kv_map(CUtensorMap* map, const void* base, int64_t total_len, int H);

namespace {

constexpr int kHalf = 128 * 128;       // one 64-column half of a 128 x 128 bf16 tile
constexpr int kTile = 2 * kHalf;       // 32 KB
#ifndef VISTA_QLA_BWD_KP
#define VISTA_QLA_BWD_KP 1
#endif
// kKp: the transform also writes phi1'(K) (bf16) into a third tile of the stage, which the epilogue
// reads from shared memory (2 stages); else 3 stages and the epilogue re-reads raw K through L2
constexpr bool kKp = VISTA_QLA_BWD_KP;
constexpr int kStages = kKp ? 2 : 3;
constexpr int kStageBytes = (kKp ? 3 : 2) * kTile;  // K (-> phi1(K) in place), V [, phi1'(K)]
constexpr int kDzOff = kStages * kStageBytes;
constexpr int kBarOff = kDzOff + kTile;
constexpr int kSmem = kBarOff + 256 + 1024;
constexpr int kThreads = 512;
constexpr int kXform = 128;  // transform threads (warps 4..7)
constexpr int kEpi = 256;    // epilogue threads (warps 8..15)

struct Bars {
    uint64_t kv_full[kStages], k_ready[kStages], kv_empty[kStages];
    uint64_t acc_full[2], acc_empty[2];
    uint64_t dz_full, dz_empty;
    uint32_t tmem_base;
};

struct Params {
    const int64_t* offsets;
    const int64_t* uts;
    const __nv_bfloat16* k;  // raw K (the epilogue re-reads it for phi1'(K))
    const uint8_t* dz_op;  // [B*H][32 KB]
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    int B, H;
};

// phi1 and phi1' of one value with shared work: SiLU through sigma(x) = (1 + tanh(x/2)) / 2 (one
// MUFU op), shifted ELU through one exp.
template <int PHI>
__device__ __forceinline__ void phi_and_prime(float x, float& f, float& fp) {
    if constexpr (PHI == VISTA_ACT_SILU) {
        float t;
        asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
        const float sg = fmaf(0.5f, t, 0.5f);
        f = x * sg;
        fp = sg * fmaf(x, 1.f - sg, 1.f);
    } else if constexpr (PHI == VISTA_ACT_SHIFTED_ELU) {
        const float e = ptx::ex2((x - 1.f) * 1.4426950408889634f);
        f = x >= 1.f ? x : e;
        fp = x >= 1.f ? 1.f : e;
    } else {
        f = x;
        fp = 1.f;
    }
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// phi1(K) in place, 16-B chunk by chunk (the 128-B swizzle only permutes chunks within a row, so
// the transform is layout-agnostic).  phi1'(K) is recomputed in the epilogue from the raw K rows
// (re-read through L2), so a stage is free as soon as its GEMMs complete.
template <int PHI>
__device__ __forceinline__ void xform_tile(uint32_t kbuf, int xt) {
#pragma unroll 4
    for (int i = 0; i < (2 * kTile / 16) / kXform / 2; ++i) {
        const uint32_t off = (uint32_t)(xt + i * kXform) * 16;
        const uint4 raw = lds128(kbuf + off);
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
        uint32_t ph[4], pp[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float lo = __uint_as_float(w[e] << 16), hi = __uint_as_float(w[e] & 0xFFFF0000u);
            float f0, p0, f1, p1;
            phi_and_prime<PHI>(lo, f0, p0);
            phi_and_prime<PHI>(hi, f1, p1);
            ph[e] = ptx::pack_bf16x2(f0, f1);
            pp[e] = ptx::pack_bf16x2(p0, p1);
        }
        sts128(kbuf + off, make_uint4(ph[0], ph[1], ph[2], ph[3]));
        if constexpr (kKp) sts128(kbuf + 2 * kTile + off, make_uint4(pp[0], pp[1], pp[2], pp[3]));
    }
}

template <int ST, int AB>
__device__ __forceinline__ void issue_tile(uint32_t tmem, uint32_t base) {
    const uint32_t kb = base + ST * kStageBytes, vb = kb + kTile, pb = kb, dz = base + kDzOff;
    constexpr uint32_t idV = ptx::idesc_bf16_f32(128, 128, 0, 1);  // A K-major, B MN-major
    constexpr uint32_t idK = ptx::idesc_bf16_f32(128, 128, 0, 0);  // both K-major
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t ak = (kk >> 2) * kHalf + (kk & 3) * 32;
        // dV = phi1(K) dZ : A [item][c1] K-major, B = dZ [K = c1][N = c2] MN-major
        ptx::mma_ss_w(tmem + AB * 256, ptx::sdesc_sw128(pb + ak, 16, 1024), ptx::sdesc_sw128(dz + kk * 2048, kHalf, 1024),
                      idV, kk > 0);
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t ak = (kk >> 2) * kHalf + (kk & 3) * 32;
        // dK' = V dZ^T : A = V [item][c2] K-major, B = dZ [N = c1][K = c2] K-major
        ptx::mma_ss_w(tmem + AB * 256 + 128, ptx::sdesc_sw128(vb + ak, 16, 1024), ptx::sdesc_sw128(dz + ak, 16, 1024),
                      idK, kk > 0);
    }
}
__device__ __forceinline__ void issue_tile_d(int st, int ab, uint32_t tmem, uint32_t base) {
    if (st == 0) { if (ab == 0) issue_tile<0, 0>(tmem, base); else issue_tile<0, 1>(tmem, base); }
    else if (kStages == 2 || st == 1) { if (ab == 0) issue_tile<1, 0>(tmem, base); else issue_tile<1, 1>(tmem, base); }
    else { if (ab == 0) issue_tile<2, 0>(tmem, base); else issue_tile<2, 1>(tmem, base); }
}

__device__ __forceinline__ void st_v8(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

template <int PHI1>
__global__ void __launch_bounds__(kThreads, 1)
    sm100_qla_bwd_kv_kernel(const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                            const Params P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = ptx::smem_u32(smem);
    Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cta = blockIdx.x, num_ctas = gridDim.x;
    const int HG = P.H;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bars->kv_full[s], 1);
            ptx::mbar_init(&bars->k_ready[s], kXform);
            ptx::mbar_init(&bars->kv_empty[s], kKp ? 1 + kEpi : 1);  // MMA commit [+ epilogue read phi1'(K)]
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->acc_full[b], 1);
            ptx::mbar_init(&bars->acc_empty[b], kEpi);
        }
        ptx::mbar_init(&bars->dz_full, 1);
        ptx::mbar_init(&bars->dz_empty, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);

    ItemIter iter;
    iter.init(P.uts, P.B, HG, cta, num_ctas);
    Item it;
    if (warp == 0) {
        // ============================ TMA producer ============================
        ptx::tma_prefetch(&mapK);
        ptx::tma_prefetch(&mapV);
        const uint64_t pol = ptx::policy_evict_first();
        const uint64_t pol_k = kKp ? pol : ptx::policy_evict_last();  // !kKp: re-read by the epilogue for phi1'(K)
        int stage = 0;
        uint32_t phase = 0;
        int k = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int h = it.hg;
            // dZ of this unit (the MMAs of the previous unit must be done with the buffer)
            if (k > 0) ptx::mbar_wait(&bars->dz_empty, (k - 1) & 1);
            ptx::mbar_arrive_expect_tx_w(&bars->dz_full, kTile);
            ptx::bulk_g2s_w(base + kDzOff, P.dz_op + (size_t)(it.u * HG + it.hg) * kTile, kTile, &bars->dz_full);
            const int64_t row0 = P.offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->kv_empty[stage], phase ^ 1);
                ptx::mbar_arrive_expect_tx_w(&bars->kv_full[stage], 2 * kTile);
                uint8_t* sk = smem + stage * kStageBytes;
                const int32_t row = (int32_t)(row0 + (int64_t)t * 128);
                for (int half = 0; half < 2; ++half) {
                    ptx::tma_load_3d_w(sk + half * kHalf, &mapK, &bars->kv_full[stage], half * 64, h, row, pol_k);
                    ptx::tma_load_3d_w(sk + kTile + half * kHalf, &mapV, &bars->kv_full[stage], half * 64, h, row, pol);
                }
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            ++k;
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ============================
        int stage = 0;
        uint32_t phase = 0;
        int ab = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        int k = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            ptx::mbar_wait(&bars->dz_full, k & 1);
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->k_ready[stage], phase);
                ptx::mbar_wait(&bars->acc_empty[ab], ((aphm >> ab) & 1u) ^ 1);
                aphm ^= 1u << ab;
                ptx::tc_fence_after();
                issue_tile_d(stage, ab, tmem, base);
                ptx::mma_commit_w(&bars->acc_full[ab]);
                ptx::mma_commit_w(&bars->kv_empty[stage]);  // K, V stage free once the GEMMs complete
                ab ^= 1;
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            ptx::mma_commit_w(&bars->dz_empty);  // dZ free once this unit's GEMMs complete
            ++k;
        }
    } else if (warp >= 4 && warp < 8) {
        // ============================ transform ============================
        const int xt = threadIdx.x - 128;
        int stage = 0;
        uint32_t phase = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->kv_full[stage], phase);
                xform_tile<PHI1>(base + stage * kStageBytes, xt);
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&bars->k_ready[stage]);
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp >= 8) {
        // ============================ epilogue ============================
        const int wq = warp % 4;
        const int chalf = (warp - 8) / 4;  // columns [64 chalf, 64 chalf + 64)
        const int row = wq * 32 + lane;    // item row within the tile = TMEM lane
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        int ab = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        // Coalesced row stores (see sm100_softmax.cu store_rows_coalesced): the 32 packed words of a
        // thread's 64-column row segment go back into the (already read) accumulator columns at
        // tcol in a permuted order and come out with the 16x256b shape, a quad of threads then
        // holding 128 contiguous bytes of one row: each warp store writes 8 full lines.
        auto store32 = [&](uint32_t tcol, const uint32_t (&w)[32], __nv_bfloat16* gbase, int valid) {
            uint32_t a[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const int g = c >> 3, p = (c & 7) >> 1, e = c & 1;
                a[c] = w[8 * p + 2 * g + e];
            }
            ptx::tmem_st32(tcol, a);
            ptx::tmem_wait_st();
            const int p = lane & 3;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t r[16];
                ptx::tmem_ld16x256b_x4(tcol + ((uint32_t)(16 * half) << 16), r);
                ptx::tmem_wait_ld();
                ptx::reg_fence(r);
                const int ra = wq * 32 + 16 * half + (lane >> 2);
                const uint32_t v0[8] = {r[0], r[1], r[4], r[5], r[8], r[9], r[12], r[13]};
                const uint32_t v1[8] = {r[2], r[3], r[6], r[7], r[10], r[11], r[14], r[15]};
                if (ra < valid) st_v8(gbase + (size_t)ra * P.H * 128 + 16 * p, v0);
                if (ra + 8 < valid) st_v8(gbase + (size_t)(ra + 8) * P.H * 128 + 16 * p, v1);
            }
        };
        auto epilogue = [&](int est, int eab, int64_t grow0, int valid, int h) {
            // raw k of this thread's row, columns [64 chalf, +64): 8 x 16 B through L2 (issued before the wait for the GEMMs)
            uint4 kraw[8];
            if constexpr (!kKp) {
                const int rr = row < valid ? row : 0;
                const uint4* src = reinterpret_cast<const uint4*>(P.k + ((size_t)(grow0 + rr) * P.H + h) * 128 +
                                                                  chalf * 64);
#pragma unroll
                for (int q = 0; q < 8; ++q) kraw[q] = __ldg(src + q);
            }
            ptx::mbar_wait(&bars->acc_full[eab], ((aphm >> eab) & 1u));
            aphm ^= 1u << eab;
            ptx::tc_fence_after();
            if constexpr (kKp) {  // phi1'(K) of this row's 64 columns from the stage (swizzled 16-B chunks)
                const uint32_t kp = base + est * kStageBytes + 2 * kTile + chalf * kHalf + row * 128;
#pragma unroll
                for (int q = 0; q < 8; ++q) kraw[q] = lds128(kp + ((q ^ (row & 7)) << 4));
                ptx::mbar_arrive(&bars->kv_empty[est]);
            }
            const size_t gcol = ((size_t)grow0 * P.H + h) * 128 + chalf * 64;  // row 0 of the tile
            const uint32_t tv = tmem + lane_bits + eab * 256 + chalf * 64;
            const uint32_t tk = tv + 128;
            {  // dV
                uint32_t w[32];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t rv[32];
                    ptx::tmem_ld32_sync(tv + c * 32, rv);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        w[16 * c + j] = ptx::pack_bf16x2(__uint_as_float(rv[2 * j]), __uint_as_float(rv[2 * j + 1]));
                }
                store32(tv, w, P.dv + gcol, valid);
            }
            {  // dK = (V dZ^T) . phi1'(K)
                uint32_t w[32];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t rk[32];
                    ptx::tmem_ld32_sync(tk + c * 32, rk);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 kr = kraw[4 * c + q];
                        const uint32_t kw[4] = {kr.x, kr.y, kr.z, kr.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int j = 4 * q + e;
                            float d0, d1;
                            if constexpr (kKp) {  // phi1'(k) (bf16) from the transform
                                d0 = __uint_as_float(kw[e] << 16);
                                d1 = __uint_as_float(kw[e] & 0xFFFF0000u);
                            } else {
                                float f;  // phi1(k): not needed here
                                phi_and_prime<PHI1>(__uint_as_float(kw[e] << 16), f, d0);
                                phi_and_prime<PHI1>(__uint_as_float(kw[e] & 0xFFFF0000u), f, d1);
                            }
                            w[16 * c + j] = ptx::pack_bf16x2(__uint_as_float(rk[2 * j]) * d0,
                                                             __uint_as_float(rk[2 * j + 1]) * d1);
                        }
                    }
                }
                store32(tk, w, P.dk + gcol, valid);
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bars->acc_empty[eab]);
            (void)est;
        };
        int est = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int64_t L = P.offsets[it.u + 1] - P.offsets[it.u];
            const int64_t row0 = P.offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                const int64_t rem = L - (int64_t)t * 128;
                epilogue(est, ab, row0 + (int64_t)t * 128, rem < 128 ? (int)rem : 128, it.hg);
                ab ^= 1;
                if (++est == kStages) est = 0;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

template <int PHI1>
cudaError_t launch_phi(const Problem& p, int num_ctas, const CUtensorMap& mk, const CUtensorMap& mv, const Params& P) {
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(sm100_qla_bwd_kv_kernel<PHI1>), kSmem);
    if (attr != cudaSuccess) return attr;
    sm100_qla_bwd_kv_kernel<PHI1><<<num_ctas, kThreads, kSmem, p.stream>>>(mk, mv, P);
    return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Per-unit backward on the tensor cores (one CTA of 128 threads per (u, h); S % 128 == 0):
//   W = phi2(Zbar) (bf16, K-major [N = c1][K = c2]) built from Z by the threads,
//   per 128-row block b:  dW += phi1(Q)_b^T dO_b  (both MN-major, K = the block's rows)
//                         dA_b = dO_b W^T       (dO_b K-major [M = i][K = c2], W K-major)
//                         dQ_u rows = dA_b . phi1'(Q)            -> f32 dqu
//   then dZ = dW . phi2'(Zbar) / N_u -> the bf16 operand of the dK / dV kernel.
namespace {
namespace ub {
constexpr int kW = 0, kA = kTile, kG = 2 * kTile;
constexpr int kSmemU = 3 * kTile + 1024;
}

// 8 consecutive dO values as 4 packed bf16x2 words (16-B / 2 x 16-B vector loads)
template <typename TO>
__device__ __forceinline__ uint4 ld8_bf16(const TO* p);
template <>
__device__ __forceinline__ uint4 ld8_bf16<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
}
template <>
__device__ __forceinline__ uint4 ld8_bf16<float>(const float* p) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    return make_uint4(ptx::pack_bf16x2(a.x, a.y), ptx::pack_bf16x2(a.z, a.w), ptx::pack_bf16x2(b.x, b.y),
                      ptx::pack_bf16x2(b.z, b.w));
}

__device__ __forceinline__ float act_any(int kind, float x) {
    if (kind == VISTA_ACT_SILU) return x * __frcp_rn(1.f + __expf(-x));
    if (kind == VISTA_ACT_SHIFTED_ELU) return x >= 1.f ? x : __expf(x - 1.f);
    return x;
}
__device__ __forceinline__ float act_prime_any(int kind, float x) {
    if (kind == VISTA_ACT_SILU) {
        const float s = __frcp_rn(1.f + __expf(-x));
        return s * (1.f + x * (1.f - s));
    }
    if (kind == VISTA_ACT_SHIFTED_ELU) return x >= 1.f ? 1.f : __expf(x - 1.f);
    return 1.f;
}

template <typename TO>
__global__ void __launch_bounds__(128) sm100_qla_bwd_unit_kernel(const __nv_bfloat16* __restrict__ q,
                                                                 int64_t q_user_stride, const TO* __restrict__ dout,
                                                                 const float* __restrict__ z,
                                                                 const uint8_t* __restrict__ abuf,
                                                                 const int64_t* __restrict__ offsets, int S, int H,
                                                                 int phi1, int phi2, int normalize,
                                                                 uint8_t* __restrict__ dz_op, float* __restrict__ dqu) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sm = smem_raw + (base - ptx::smem_u32(smem_raw));
    __shared__ uint64_t bar_a, bar_mma;
    __shared__ uint32_t tmem_slot;
    const int r = threadIdx.x, warp = r / 32;
    const int unit = blockIdx.x, u = unit / H, h = unit % H;
    const int nblk = S / 128;
    const int64_t N = offsets[u + 1] - offsets[u];
    const float inv = (normalize && N > 0) ? 1.f / (float)N : 1.f;
    if (warp == 0) ptx::tmem_alloc(&tmem_slot, 256);
    if (r == 0) {
        ptx::mbar_init(&bar_a, 1);
        ptx::mbar_init(&bar_mma, 1);
        ptx::fence_mbar_init();
    }
    // W = phi2(Zbar): thread r builds row c1 = r (K-major [N = c1][K = c2])
    const float* zrow = z + ((size_t)unit * 128 + r) * 128;
#pragma unroll 4
    for (int c = 0; c < 128; c += 8) {
        const float4 a = *reinterpret_cast<const float4*>(zrow + c), b = *reinterpret_cast<const float4*>(zrow + c + 4);
        uint4 pk;
        pk.x = ptx::pack_bf16x2(act_any(phi2, a.x * inv), act_any(phi2, a.y * inv));
        pk.y = ptx::pack_bf16x2(act_any(phi2, a.z * inv), act_any(phi2, a.w * inv));
        pk.z = ptx::pack_bf16x2(act_any(phi2, b.x * inv), act_any(phi2, b.y * inv));
        pk.w = ptx::pack_bf16x2(act_any(phi2, b.z * inv), act_any(phi2, b.w * inv));
        *reinterpret_cast<uint4*>(sm + ub::kW + qla_w_swz(r, c)) = pk;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_slot, 0);
    const uint32_t tdW = tmem, tdA = tmem + 128;
    const uint32_t lane_bits = (uint32_t)(warp * 32) << 16;
    const __nv_bfloat16* qu = q + (size_t)(q_user_stride ? u : 0) * q_user_stride;
    const uint8_t* au = abuf + (size_t)((q_user_stride ? u : 0) * H + h) * nblk * kTile;
    for (int b = 0; b < nblk; ++b) {
        // phi1(Q) block by bulk copy; dO block (row i = 128 b + r) by the threads, swizzled
        if (warp == 0) {
            ptx::mbar_arrive_expect_tx_w(&bar_a, kTile);
            ptx::bulk_g2s_w(base + ub::kA, au + (size_t)b * kTile, kTile, &bar_a);
        }
        const int i = b * 128 + r;
        const TO* go = dout + (((size_t)u * S + i) * H + h) * 128;
        uint4 gv[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) gv[c] = ld8_bf16<TO>(go + 8 * c);
#pragma unroll
        for (int c = 0; c < 16; ++c) *reinterpret_cast<uint4*>(sm + ub::kG + qla_w_swz(r, 8 * c)) = gv[c];
        ptx::fence_proxy_async_smem();
        __syncthreads();
        if (warp == 0) {
            ptx::mbar_wait(&bar_a, b & 1);
            ptx::tc_fence_after();
            constexpr uint32_t idW = ptx::idesc_bf16_f32(128, 128, 1, 1);  // both MN-major
            constexpr uint32_t idA = ptx::idesc_bf16_f32(128, 128, 0, 0);  // both K-major
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                ptx::mma_ss_w(tdW, ptx::sdesc_sw128(base + ub::kA + kk * 2048, kHalf, 1024),
                              ptx::sdesc_sw128(base + ub::kG + kk * 2048, kHalf, 1024), idW, (b > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t ak = (kk >> 2) * kHalf + (kk & 3) * 32;
                ptx::mma_ss_w(tdA, ptx::sdesc_sw128(base + ub::kG + ak, 16, 1024),
                              ptx::sdesc_sw128(base + ub::kW + ak, 16, 1024), idA, kk > 0);
            }
            ptx::mma_commit_w(&bar_mma);
        }
        ptx::mbar_wait(&bar_mma, b & 1);
        ptx::tc_fence_after();
        // dQ rows of this block: dA . phi1'(q)
        const __nv_bfloat16* qi = qu + ((size_t)i * H + h) * 128;
        float* dst = dqu + (((size_t)u * S + i) * H + h) * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint4 qv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) qv[e] = __ldg(reinterpret_cast<const uint4*>(qi + c * 32) + e);
            uint32_t o[32];
            ptx::tmem_ld32_sync(tdA + lane_bits + c * 32, o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t w[4] = {qv[e].x, qv[e].y, qv[e].z, qv[e].w};
#pragma unroll
                for (int f = 0; f < 4; f += 2) {
                    const int j = 8 * e + 2 * f;
                    float4 v;
                    v.x = __uint_as_float(o[j]) * act_prime_any(phi1, __uint_as_float(w[f] << 16));
                    v.y = __uint_as_float(o[j + 1]) * act_prime_any(phi1, __uint_as_float(w[f] & 0xFFFF0000u));
                    v.z = __uint_as_float(o[j + 2]) * act_prime_any(phi1, __uint_as_float(w[f + 1] << 16));
                    v.w = __uint_as_float(o[j + 3]) * act_prime_any(phi1, __uint_as_float(w[f + 1] & 0xFFFF0000u));
                    *reinterpret_cast<float4*>(dst + c * 32 + j) = v;
                }
            }
        }
        ptx::tc_fence_before();
        __syncthreads();  // smem blocks and the dA columns are reused by the next block
        ptx::tc_fence_after();
    }
    // dZ = dW . phi2'(Zbar) / N -> bf16 operand row c1 = r
    uint8_t* dzu = dz_op + (size_t)unit * kTile;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        ptx::tmem_ld32_sync(tdW + lane_bits + c * 32, o);
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            const float4 za = __ldg(reinterpret_cast<const float4*>(zrow + c * 32 + j));
            const float4 zb = __ldg(reinterpret_cast<const float4*>(zrow + c * 32 + j + 4));
            const float zz[8] = {za.x, za.y, za.z, za.w, zb.x, zb.y, zb.z, zb.w};
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float g0 = __uint_as_float(o[j + 2 * e]) * act_prime_any(phi2, zz[2 * e] * inv) * inv;
                const float g1 = __uint_as_float(o[j + 2 * e + 1]) * act_prime_any(phi2, zz[2 * e + 1] * inv) * inv;
                w[e] = ptx::pack_bf16x2(g0, g1);
            }
            *reinterpret_cast<uint4*>(dzu + qla_w_swz(r, c * 32 + j)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 256);
}
}  // namespace

cudaError_t launch_sm100_qla_bwd_unit(const Problem& p, bool dout_bf16, const void* dout, const float* z,
                                      const uint8_t* abuf, uint8_t* dz_op, float* dqu) {
    if (p.B == 0) return cudaSuccess;
    const int smem = ub::kSmemU;
    if (dout_bf16) {
        const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(sm100_qla_bwd_unit_kernel<__nv_bfloat16>), smem);
        if (attr != cudaSuccess) return attr;
        sm100_qla_bwd_unit_kernel<__nv_bfloat16><<<p.B * p.H, 128, smem, p.stream>>>(
            reinterpret_cast<const __nv_bfloat16*>(p.q), p.q_user_stride, reinterpret_cast<const __nv_bfloat16*>(dout),
            z, abuf, p.offsets, p.S, p.H, p.phi1, p.phi2, p.normalize, dz_op, dqu);
    } else {
        const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(sm100_qla_bwd_unit_kernel<float>), smem);
        if (attr != cudaSuccess) return attr;
        sm100_qla_bwd_unit_kernel<float><<<p.B * p.H, 128, smem, p.stream>>>(
            reinterpret_cast<const __nv_bfloat16*>(p.q), p.q_user_stride, reinterpret_cast<const float*>(dout), z, abuf,
            p.offsets, p.S, p.H, p.phi1, p.phi2, p.normalize, dz_op, dqu);
    }
    return cudaGetLastError();
}

bool qla_bwd_uses_tc(const Problem& p) {
    return p.in_bf16 && p.d == 128 && p.total_len < (int64_t(1) << 31);
}

cudaError_t launch_sm100_qla_bwd_kv(const Problem& p, const Workspace& w, char* ws, const uint8_t* dz_op, void* dk,
                                    void* dv) {
    CUtensorMap mk, mv;
    if (!make_kv_map(&mk, p.k, p.total_len, p.H) || !make_kv_map(&mv, p.v, p.total_len, p.H))
        return cudaErrorInvalidValue;
    Params P;
    P.offsets = p.offsets;
    P.uts = reinterpret_cast<const int64_t*>(ws + w.uts_off);
    P.dz_op = dz_op;
    P.k = reinterpret_cast<const __nv_bfloat16*>(p.k);
    P.dk = reinterpret_cast<__nv_bfloat16*>(dk);
    P.dv = reinterpret_cast<__nv_bfloat16*>(dv);
    P.B = p.B;
    P.H = p.H;
    return p.phi1 == VISTA_ACT_SILU ? launch_phi<VISTA_ACT_SILU>(p, w.num_ctas, mk, mv, P)
         : p.phi1 == VISTA_ACT_SHIFTED_ELU ? launch_phi<VISTA_ACT_SHIFTED_ELU>(p, w.num_ctas, mk, mv, P)
                                           : launch_phi<VISTA_ACT_IDENTITY>(p, w.num_ctas, mk, mv, P);
}

}  // namespace vista
