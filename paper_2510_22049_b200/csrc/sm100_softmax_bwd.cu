// sm100_softmax_bwd.cu -- softmax backward on B200 (NEXT-2, stage-1 training): the gradients of
// o_i = sum_j p_ij v_j, p_ij = softmax_j(scale q_i . k_j) over each user's
// history, flash-attention style (P recomputed from the forward's lse, never stored):
//   P = exp(scale Q K^T - lse);  dP = dO V^T;  D_i = sum_c dO_ic O_ic;  dS = P . (dP - D)
//   dV = P^T dO;   dK = scale dS^T Q;   dQ = scale dS K
// Two passes, each a persistent TMA + tcgen05 kernel over the flat key tiles (work.cuh):
//
//   sm100_softmax_bwd_kv_kernel  (dK, dV; one work unit = (user, head), all S <= 256 seed rows
//     resident in shared memory).  The key-major products are computed transposed so that the
//     tensor core's M dimension is the 128 keys of a tile and every operand fits the TMEM / SMEM
//     forms:  S^T = K Q_g^T,  dP^T = V dO_g^T  (SS);  P^T, dS^T go to TMEM as bf16 over S^T, dP^T
//     and feed  dV += P^T dO_g,  dK += dS^T Q_g  as TS MMAs (A from TMEM), g over the 128-row
//     query blocks.  The softmax is column-wise here (lse_i, D_i per query column; no reduction).
//   sm100_softmax_bwd_dq_kernel  (dQ; one unit = (user, head, 128-row query block), like the
//     forward with one Q tile):  S = Q_g K^T, dP = dO_g V^T (SS) -> dS (bf16 over S in TMEM) ->
//     dQ += dS K (TS, K tile as the MN-major B operand).  Split units (stream-K) write partial
//     slots, summed by the QLA slot merge into the [B, H, S, d] dQ buffer.
//
// TMEM, pass 1: two buffers of 128 columns, each a 64-query half block (S^T in its first 64
// columns with bf16 P^T over the first 32; dP^T in the last 64 with bf16 dS^T over its first 32),
// then dV [256,384), dK [384,512).  Pass 2: [0,128) S (bf16 dS over its first 64), [128,256) dP,
// [256,384) dQ.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>

#include "internal.h"
#include "qla_common.cuh"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

bool make_kv_map(CUtensorMap* map, const void* base, int64_t total_len, int H);
bool make_q_map(CUtensorMap* map, const void* base, int S, int H, int B, int64_t q_user_stride);

namespace {

constexpr int kHalf = 128 * 128;
constexpr int kTileB = 2 * kHalf;  // 32 KB: 128 rows x 128 bf16
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void st_v8(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// Coalesced bf16 row store of 32 packed words (64 columns of this thread's TMEM lane row), through
// a TMEM round trip at tcol (already read; see sm100_softmax.cu store_rows_coalesced).  Rows >= valid
// are not stored.  gbase: element (row 0, first column); row stride in elements.
__device__ __forceinline__ void store32_rows(uint32_t tcol, const uint32_t (&w)[32], __nv_bfloat16* gbase,
                                             size_t row_stride, int valid, int wq, int lane) {
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
        if (ra < valid) st_v8(gbase + (size_t)ra * row_stride + 16 * p, v0);
        if (ra + 8 < valid) st_v8(gbase + (size_t)(ra + 8) * row_stride + 16 * p, v1);
    }
}

__device__ __forceinline__ void named_sync_sm() { asm volatile("bar.sync 1, 256;" ::: "memory"); }  // the softmax warps

// ============================================================================ pass 1: dK, dV
namespace kv {
#ifdef VISTA_BWD_PROF  // cycles each role waits per barrier, averaged per CTA, printed by the last CTA
__device__ unsigned long long g_bwd_prof[16];
__device__ unsigned int g_bwd_done;
#define PWAIT(i, x)                            \
    do {                                       \
        const long long _t0 = clock64();       \
        x;                                     \
        prof[i] += clock64() - _t0;            \
    } while (0)
#else
#define PWAIT(i, x) x
#endif
// S <= 256 (RESIDENT): Q and dO of the unit stay in shared memory, [0, 64 KB) and [64, 128 KB).
// S > 256 (STREAM): the (Q_g, dO_g) pairs of each 128-row block stream through a 2-stage ring of
// 64 KB in the same 128 KB (L2-resident reloads per key tile).
constexpr int kResidentMaxS = 256;
constexpr int kMaxS = 1024;
constexpr int kQOff = 0;                            // Q blocks (RESIDENT) / ring stages (STREAM)
constexpr int kGOff = kQOff + 2 * kTileB;            // dO blocks (RESIDENT)
constexpr int kKOff = 4 * kTileB;                    // K ring, 2 stages
constexpr int kVOff = kKOff + 2 * kTileB;            // V, 1 stage
constexpr int kTiles = kVOff + kTileB;               // 224 KB of 1024-B aligned operand tiles
// Barriers and the unit's lse*log2e / D rows (RESIDENT, 2 x 256 floats) sit in front of the tiles:
// with the dynamic shared memory base 1024-B aligned this is exactly the 227 KB maximum.
constexpr int kHead = 3072;
constexpr int kSmem = kHead + kTiles;
constexpr int kThreads = 512;  // 0 TMA, 1 MMA, 4-11 softmax (two column halves), 12-15 epilogue

struct Bars {
    uint64_t q_full, q_empty, k_full[2], k_empty[2], v_full, v_empty;
    uint64_t s_full, dp_full, p_ready, ds_ready;
    uint64_t dv_full, dv_empty, dk_full, dk_empty;
    uint64_t qg_full[2], qg_empty[2];  // STREAM: Q_g of a ring stage
    uint64_t go_full[2], go_empty[2];  // STREAM: dO_g of a ring stage
    uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barriers overlap the lse / D rows");

struct Params {
    const int64_t* offsets;
    const int64_t* uts;
    const float* lse;  // [B, H, S] natural log
    const float* dd;   // D [B, H, S]
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    int B, S, H;
    float scale_log2, scale;
    int q_per_user;
};

// One 128-query block g of a 128-key tile: S^T = K Q_g^T -> cols [0,128), dP^T = V dO_g^T ->
// [128,256) (SS, all operands K-major).  The softmax warpgroup of query half sg writes bf16 P^T of
// its 64 queries over [64 sg, 64 sg + 32) (the start of the S^T columns it read itself), dS^T
// likewise over [128 + 64 sg, ...); dV += P^T dO_g -> [256,384), dK += dS^T Q_g -> [384,512) (A from
// TMEM: K steps 0-3 at columns 0-31, 4-7 at 64-95; B MN-major).
template <int KS>
__device__ __forceinline__ void issue_s(uint32_t tmem, uint32_t base, uint32_t qa) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t ka = base + kKOff + KS * kTileB;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
        ptx::mma_ss_w(tmem, ptx::sdesc_sw128(ka + off, 16, 1024), ptx::sdesc_sw128(qa + off, 16, 1024), id, kk > 0);
    }
}
__device__ __forceinline__ void issue_dp(uint32_t tmem, uint32_t base, uint32_t ga) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t va = base + kVOff;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
        ptx::mma_ss_w(tmem + 128, ptx::sdesc_sw128(va + off, 16, 1024), ptx::sdesc_sw128(ga + off, 16, 1024), id,
                      kk > 0);
    }
}
// acc: accumulate onto the tile's earlier blocks
__device__ __forceinline__ void issue_dv(uint32_t tmem, uint32_t ga, bool acc) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 1);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma_ts_w(tmem + 256, tmem + kk * 8 + (kk >> 2) * 32, ptx::sdesc_sw128(ga + kk * 2048, kHalf, 1024), id,
                      (acc || kk > 0) ? 1u : 0u);
}
__device__ __forceinline__ void issue_dk(uint32_t tmem, uint32_t qa, bool acc) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 1);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma_ts_w(tmem + 384, tmem + 128 + kk * 8 + (kk >> 2) * 32, ptx::sdesc_sw128(qa + kk * 2048, kHalf, 1024),
                      id, (acc || kk > 0) ? 1u : 0u);
}

template <bool STREAM>
__global__ void __launch_bounds__(kThreads, 1)
    sm100_softmax_bwd_kv_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapG,
                                const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                                const Params P) {
    extern __shared__ uint8_t smem_raw[];
    Bars* bars = reinterpret_cast<Bars*>(smem_raw);
    float* lsd = reinterpret_cast<float*>(smem_raw + 256);  // [2][256]: lse * log2e, D
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + kHead + 1023) & ~uintptr_t(1023));
    if (smem + kTiles > smem_raw + kSmem) __trap();  // dynamic smem base not 1024-B aligned
    const uint32_t base = ptx::smem_u32(smem);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cta = blockIdx.x, num_ctas = gridDim.x;
    const int HG = P.H, G = P.S / 128;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars->q_full, 1);
        ptx::mbar_init(&bars->q_empty, 1);
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&bars->k_full[s], 1);
            ptx::mbar_init(&bars->k_empty[s], 1);
            ptx::mbar_init(&bars->qg_full[s], 1);
            ptx::mbar_init(&bars->qg_empty[s], 1);
            ptx::mbar_init(&bars->go_full[s], 1);
            ptx::mbar_init(&bars->go_empty[s], 1);
        }
        ptx::mbar_init(&bars->v_full, 1);
        ptx::mbar_init(&bars->v_empty, 1);
        ptx::mbar_init(&bars->s_full, 1);
        ptx::mbar_init(&bars->dp_full, 1);
        ptx::mbar_init(&bars->p_ready, 256);
        ptx::mbar_init(&bars->ds_ready, 256);
        ptx::mbar_init(&bars->dv_full, 1);
        ptx::mbar_init(&bars->dv_empty, 128);
        ptx::mbar_init(&bars->dk_full, 1);
        ptx::mbar_init(&bars->dk_empty, 128);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);
#ifdef VISTA_BWD_PROF
    long long prof[16] = {};
    const long long tstart = clock64();
#endif
    ItemIter iter;
    iter.init(P.uts, P.B, HG, cta, num_ctas);
    Item it;
    if (warp == 0) {
        // ---------------- TMA producer: Q, dO (resident per unit, or streamed per block);
        //                  K (2 stages), V (1 stage) per tile
        ptx::tma_prefetch(&mapQ);
        ptx::tma_prefetch(&mapG);
        ptx::tma_prefetch(&mapK);
        ptx::tma_prefetch(&mapV);
        const uint64_t pol = ptx::policy_evict_first(), pol_q = ptx::policy_evict_last();
        int ks = 0;
        uint32_t kph = 0, vph = 0;
        int k = 0;
        int qs = 0;
        uint32_t qph = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int h = it.hg;
            if constexpr (!STREAM) {
                if (k > 0) PWAIT(3, ptx::mbar_wait(&bars->q_empty, (k - 1) & 1));
                ptx::mbar_arrive_expect_tx_w(&bars->q_full, 2 * G * kTileB);
                for (int g = 0; g < G; ++g)
                    for (int half = 0; half < 2; ++half) {
                        ptx::tma_load_4d_w(smem + kQOff + g * kTileB + half * kHalf, &mapQ, &bars->q_full, half * 64,
                                           h, g * 128, P.q_per_user ? it.u : 0, pol_q);
                        ptx::tma_load_4d_w(smem + kGOff + g * kTileB + half * kHalf, &mapG, &bars->q_full, half * 64,
                                           h, g * 128, it.u, pol_q);
                    }
            }
            const int64_t row0 = P.offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                const int32_t row = (int32_t)(row0 + (int64_t)t * 128);
                PWAIT(0, ptx::mbar_wait(&bars->k_empty[ks], kph ^ 1));
                ptx::mbar_arrive_expect_tx_w(&bars->k_full[ks], kTileB);
                for (int half = 0; half < 2; ++half)
                    ptx::tma_load_3d_w(smem + kKOff + ks * kTileB + half * kHalf, &mapK, &bars->k_full[ks], half * 64,
                                       h, row, pol);
                if (++ks == 2) { ks = 0; kph ^= 1; }
                PWAIT(1, ptx::mbar_wait(&bars->v_empty, vph ^ 1));
                vph ^= 1;
                ptx::mbar_arrive_expect_tx_w(&bars->v_full, kTileB);
                for (int half = 0; half < 2; ++half)
                    ptx::tma_load_3d_w(smem + kVOff + half * kHalf, &mapV, &bars->v_full, half * 64, h, row, pol);
                // V has one stage: pull the next tile's V into L2 now so its load after this tile's
                // last dP^T MMA is an L2 hit
                if (t + 1 < it.t1)
                    for (int half = 0; half < 2; ++half) ptx::tma_prefetch_l2_3d_w(&mapV, half * 64, h, row + 128);
                if constexpr (STREAM) {  // (Q_g, dO_g) for every 128-row block of this tile, each half
                    for (int g = 0; g < G; ++g) {  // freed separately (Q_g after dK, dO_g after dV)
                        PWAIT(2, ptx::mbar_wait(&bars->qg_empty[qs], qph ^ 1));
                        ptx::mbar_arrive_expect_tx_w(&bars->qg_full[qs], kTileB);
                        for (int half = 0; half < 2; ++half)
                            ptx::tma_load_4d_w(smem + kQOff + qs * 2 * kTileB + half * kHalf, &mapQ, &bars->qg_full[qs],
                                               half * 64, h, g * 128, P.q_per_user ? it.u : 0, pol_q);
                        PWAIT(2, ptx::mbar_wait(&bars->go_empty[qs], qph ^ 1));
                        ptx::mbar_arrive_expect_tx_w(&bars->go_full[qs], kTileB);
                        for (int half = 0; half < 2; ++half)
                            ptx::tma_load_4d_w(smem + kQOff + qs * 2 * kTileB + kTileB + half * kHalf, &mapG,
                                               &bars->go_full[qs], half * 64, h, g * 128, it.u, pol_q);
                        if (++qs == 2) { qs = 0; qph ^= 1; }
                    }
                }
            }
            ++k;
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer, software-pipelined over the (tile, block) sequence:
        //   S(n) dP(n) | P(n) ready: dV(n) S(n+1) | dS(n) ready: dK(n) dP(n+1) | ...
        // so the tensor core computes the next block's S^T / dP^T while the softmax warps turn this
        // block's into P^T / dS^T.  S(n+1) overwrites P^T(n) only after dV(n) (MMAs execute in order);
        // dP(n+1) overwrites dS^T(n) only after dK(n).
        int ks = 0;
        uint32_t kph = 0, vph = 0, pph = 0, dsph = 0, dvph = 0, dkph = 0;
        int qs = 0;
        uint32_t qph = 0;
        int k = 0;
        bool pend = false, p_first = false, p_last = false;
        uint32_t p_qa = 0, p_ga = 0;
        int p_qs = 0;
        // TS MMAs of the pending block: dV, then (optionally) the next block's S^T, then dK
        auto pend_dv = [&]() {
            PWAIT(4, ptx::mbar_wait(&bars->p_ready, pph));
            pph ^= 1;
            if (p_first) {  // the epilogue has drained dV of the previous tile
                PWAIT(6, ptx::mbar_wait(&bars->dv_empty, dvph ^ 1));
                dvph ^= 1;
            }
            ptx::tc_fence_after();
            issue_dv(tmem, p_ga, !p_first);
            if (p_last) ptx::mma_commit_w(&bars->dv_full);
            if constexpr (STREAM) ptx::mma_commit_w(&bars->go_empty[p_qs]);  // dO_g consumed (dP, dV)
        };
        auto pend_dk = [&]() {
            PWAIT(5, ptx::mbar_wait(&bars->ds_ready, dsph));
            dsph ^= 1;
            if (p_first) {
                PWAIT(6, ptx::mbar_wait(&bars->dk_empty, dkph ^ 1));
                dkph ^= 1;
            }
            ptx::tc_fence_after();
            issue_dk(tmem, p_qa, !p_first);
            if (p_last) ptx::mma_commit_w(&bars->dk_full);
            if constexpr (STREAM) ptx::mma_commit_w(&bars->qg_empty[p_qs]);  // Q_g consumed (S, dK)
            pend = false;
        };
        while (iter.next(it, P.uts, P.B, HG)) {
            if constexpr (!STREAM) {
                if (k > 0) {  // Q, dO of the previous unit are free once its last TS MMAs complete
                    if (pend) { pend_dv(); pend_dk(); }
                    ptx::mma_commit_w(&bars->q_empty);
                }
                PWAIT(7, ptx::mbar_wait(&bars->q_full, k & 1));
            }
            for (int t = it.t0; t < it.t1; ++t) {
                // K (2 stages) is loaded well ahead; V (1 stage) only after the previous tile's last
                // dP^T, so it is waited for just before this tile's first dP^T
                PWAIT(7, ptx::mbar_wait(&bars->k_full[ks], kph));
#pragma unroll 1
                for (int g = 0; g < G; ++g) {
                    uint32_t qa, ga;
                    if constexpr (STREAM) {
                        PWAIT(8, ptx::mbar_wait(&bars->qg_full[qs], qph));
                        ptx::tc_fence_after();
                        qa = base + kQOff + qs * 2 * kTileB;
                        ga = qa + kTileB;
                    } else {
                        qa = base + kQOff + g * kTileB;
                        ga = base + kGOff + g * kTileB;
                    }
                    if (pend) pend_dv();
                    ptx::tc_fence_after();
                    if (ks == 0) issue_s<0>(tmem, base, qa); else issue_s<1>(tmem, base, qa);
                    ptx::mma_commit_w(&bars->s_full);
                    if (g == G - 1) ptx::mma_commit_w(&bars->k_empty[ks]);  // K only feeds S^T
                    if (pend) pend_dk();
                    if (g == 0) {
                        PWAIT(12, ptx::mbar_wait(&bars->v_full, vph));
                        vph ^= 1;
                        ptx::tc_fence_after();
                    }
                    if constexpr (STREAM) {
                        PWAIT(8, ptx::mbar_wait(&bars->go_full[qs], qph));
                        ptx::tc_fence_after();
                    }
                    issue_dp(tmem, base, ga);
                    ptx::mma_commit_w(&bars->dp_full);
                    if (g == G - 1) ptx::mma_commit_w(&bars->v_empty);  // V only feeds dP^T
                    pend = true;
                    p_qa = qa;
                    p_ga = ga;
                    p_first = g == 0;
                    p_last = g == G - 1;
                    p_qs = qs;
                    if constexpr (STREAM)
                        if (++qs == 2) { qs = 0; qph ^= 1; }
                }
                if (++ks == 2) { ks = 0; kph ^= 1; }
            }
            ++k;
        }
        if (pend) { pend_dv(); pend_dk(); }
    } else if (warp >= 4 && warp < 12) {
        // ---------------- column softmax, in two phases per block:
        //   P^T = exp2(S^T scale log2e - lse_i log2e)  (-> bf16 in TMEM, kept in registers)
        //   dS^T = P^T (dP^T - D_i)
        // warpgroup sg = 0, 1 handles query columns [64 sg, 64 sg + 64) of each block
        const int wq = warp % 4, sg = (warp - 4) / 4, st = threadIdx.x - 128;  // st: 0..255
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const uint32_t ts = tmem + lane_bits;
        uint32_t sph = 0, dph = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const size_t lrow = ((size_t)it.u * P.H + it.hg) * P.S;
            if constexpr (!STREAM) {  // the unit's lse * log2e and D rows into shared memory
                named_sync_sm();      // the previous unit's chunks are done with them
                for (int e = st; e < P.S; e += 256) {  // negated: the FFMA2 / FADD2 addends below
                    lsd[e] = -__ldg(P.lse + lrow + e) * kLog2e;
                    lsd[256 + e] = -__ldg(P.dd + lrow + e);
                }
                named_sync_sm();
            }
            for (int t = it.t0; t < it.t1; ++t) {
#pragma unroll 1
                for (int g = 0; g < G; ++g) {
                    if constexpr (STREAM) {  // this block's 128 lse * log2e and D values into shared memory
                        const int e = st & 127;
                        const float lv = -__ldg(P.lse + lrow + g * 128 + e) * kLog2e;
                        const float dv = -__ldg(P.dd + lrow + g * 128 + e);
                        named_sync_sm();
                        if (st < 128) lsd[e] = lv; else lsd[256 + e] = dv;
                        named_sync_sm();
                    }
                    const uint64_t sl2x2 = ptx::f2_pack(P.scale_log2, P.scale_log2), zero2 = ptx::f2_pack(0.f, 0.f);
                    const float* ls = lsd + (STREAM ? 0 : g * 128) + sg * 64;
                    const float* dl = lsd + 256 + (STREAM ? 0 : g * 128) + sg * 64;
                    const uint32_t tsp = ts + sg * 64, tsd = ts + 128 + sg * 64;  // this half's S^T / dP^T columns
                    uint32_t pk[32];  // bf16x2 P^T of this warpgroup's 64 query columns
                    PWAIT(9, ptx::mbar_wait(&bars->s_full, sph));
                    sph ^= 1;
                    ptx::tc_fence_after();
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t sr[32];
                        ptx::tmem_ld32(tsp + c * 32, sr);
                        ptx::tmem_wait_ld();
                        ptx::reg_fence(sr);
#pragma unroll
                        for (int j = 0; j < 16; ++j) {  // x = s scale log2e - lse log2e (FFMA2), p = 2^x
                            const uint64_t nl2 = *reinterpret_cast<const uint64_t*>(ls + c * 32 + 2 * j);
                            float x0, x1;
                            ptx::f2_unpack(ptx::f2_fma(ptx::f2_pack(__uint_as_float(sr[2 * j]), __uint_as_float(sr[2 * j + 1])),
                                                       sl2x2, nl2),
                                           x0, x1);
                            pk[16 * c + j] = ptx::pack_bf16x2(ptx::ex2(x0), ptx::ex2(x1));
                        }
                        ptx::tmem_st16(tsp + c * 16, *reinterpret_cast<uint32_t(*)[16]>(pk + 16 * c));
                    }
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&bars->p_ready);
                    PWAIT(10, ptx::mbar_wait(&bars->dp_full, dph));
                    dph ^= 1;
                    ptx::tc_fence_after();
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t dr[32];
                        ptx::tmem_ld32(tsd + c * 32, dr);
                        ptx::tmem_wait_ld();
                        ptx::reg_fence(dr);
                        uint32_t sw[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {  // dS = P (dP - D): FADD2 then FFMA2 (+0)
                            const uint64_t nd2 = *reinterpret_cast<const uint64_t*>(dl + c * 32 + 2 * j);
                            const uint32_t pw = pk[16 * c + j];
                            const uint64_t t2 =
                                ptx::f2_add(ptx::f2_pack(__uint_as_float(dr[2 * j]), __uint_as_float(dr[2 * j + 1])), nd2);
                            float d0, d1;
                            ptx::f2_unpack(ptx::f2_fma(ptx::f2_pack(__uint_as_float(pw << 16), __uint_as_float(pw & 0xffff0000u)),
                                                       t2, zero2),
                                           d0, d1);
                            sw[j] = ptx::pack_bf16x2(d0, d1);
                        }
                        ptx::tmem_st16(tsd + c * 16, sw);
                    }
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&bars->ds_ready);
                }
            }
        }
    } else if (warp >= 12) {
        // ---------------- epilogue: dV, then dK (x scale) rows -> bf16; each accumulator is released
        // as soon as it is drained, so the next tile's dV MMAs need not wait for the dK drain
        const int wq = warp % 4;
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        uint32_t vph = 0, kph = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int64_t L = P.offsets[it.u + 1] - P.offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                const int64_t rem = L - (int64_t)t * 128;
                const int valid = rem < 128 ? (int)rem : 128;
                const size_t g0 = ((size_t)(P.offsets[it.u] + (int64_t)t * 128) * P.H + it.hg) * 128;
                for (int m = 0; m < 2; ++m) {  // 0: dV, 1: dK
                    if (m == 0) {
                        PWAIT(11, ptx::mbar_wait(&bars->dv_full, vph));
                        vph ^= 1;
                    } else {
                        PWAIT(11, ptx::mbar_wait(&bars->dk_full, kph));
                        kph ^= 1;
                    }
                    ptx::tc_fence_after();
                    const float sc = m ? P.scale : 1.f;
                    __nv_bfloat16* dst = (m ? P.dk : P.dv) + g0;
                    for (int hh = 0; hh < 2; ++hh) {  // 64-column halves
                        const uint32_t tc = tmem + lane_bits + 256 + m * 128 + hh * 64;
                        uint32_t w[32];
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            uint32_t r[32];
                            ptx::tmem_ld32_sync(tc + c * 32, r);
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                w[16 * c + j] = ptx::pack_bf16x2(__uint_as_float(r[2 * j]) * sc,
                                                                 __uint_as_float(r[2 * j + 1]) * sc);
                        }
                        store32_rows(tc, w, dst + hh * 64, (size_t)P.H * 128, valid, wq, lane);
                    }
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(m ? &bars->dk_empty : &bars->dv_empty);
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
#ifdef VISTA_BWD_PROF
    if (lane == 0 && (warp == 0 || warp == 1 || warp == 4 || warp == 12))
        for (int i = 0; i < 15; ++i)
            if (prof[i]) atomicAdd(&g_bwd_prof[i], (unsigned long long)prof[i]);
    if (threadIdx.x == 0) {
        atomicAdd(&g_bwd_prof[15], (unsigned long long)(clock64() - tstart));
        __threadfence();
        if (atomicAdd(&g_bwd_done, 1u) == gridDim.x - 1) {
            __threadfence();
            const char* nm[16] = {"k_empty", "v_empty",  "qg_empty", "q_empty", "p_ready", "ds_ready",
                                  "acc_empty", "k_full",  "qg_full", "s_full",  "dp_full", "acc_full",
                                  "v_full",   "-",        "-",       "total"};
            for (int i = 0; i < 16; ++i)
                printf("bwdprof %-10s %12.0f\n", nm[i], (double)atomicExch(&g_bwd_prof[i], 0ull) / gridDim.x);
            g_bwd_done = 0;
        }
    }
#endif
}
}  // namespace kv

// ============================================================================ pass 2: dQ
namespace dq {
constexpr int kQOff = 0, kGOff = kTileB, kKOff = 2 * kTileB, kVOff = kKOff + 2 * kTileB;
constexpr int kBarOff = kVOff + 2 * kTileB;
constexpr int kSmem = kBarOff + 256 + 1024;
constexpr int kThreads = 384;  // 0 TMA, 1 MMA, 4-11 row softmax (two key halves) + dQ epilogue

struct Bars {
    uint64_t q_full, q_empty, k_full[2], k_empty[2], v_full[2], v_empty[2];
    uint64_t s_full, dp_full, p_ready, ds_ready, dq_full, dq_empty;
    uint32_t tmem_base;
};

struct Params {
    const int64_t* offsets;
    const int64_t* uts;
    int* slot_unit;
    float* slot_o;   // [2 C][128][128]
    float* dqbuf;    // [B, H, S, d] (unit-major rows)
    const float* lse;
    const float* dd;
    int B, S, H, G;
    float scale_log2, scale;
    int q_per_user;
};

// TMEM: S of key tile n in buffer n % 2 (cols [128 b, 128 b + 128); the softmax writes bf16 dS over
// [128 b + 64 sg, 128 b + 64 sg + 32) for key half sg), dP [256,384), dQ [384,512).
// S = Q_g K^T -> buffer b;  dP = dO_g V^T -> [256,384)   (SS, all K-major)
__device__ __forceinline__ void issue_s(uint32_t ts, uint32_t base, int st) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t ka = base + kKOff + st * kTileB;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
        ptx::mma_ss_w(ts, ptx::sdesc_sw128(base + kQOff + off, 16, 1024), ptx::sdesc_sw128(ka + off, 16, 1024), id,
                      kk > 0);
    }
}
__device__ __forceinline__ void issue_dp(uint32_t tmem, uint32_t base, int st) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t va = base + kVOff + st * kTileB;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
        ptx::mma_ss_w(tmem + 256, ptx::sdesc_sw128(base + kGOff + off, 16, 1024), ptx::sdesc_sw128(va + off, 16, 1024),
                      id, kk > 0);
    }
}
// dQ += dS K: A = dS (bf16 in buffer ts: K steps 0-3 at +0..31, 4-7 at +64..95), B = K tile MN-major
__device__ __forceinline__ void issue_dq(uint32_t tmem, uint32_t ts, uint32_t base, int st, bool acc) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 1);
    const uint32_t ka = base + kKOff + st * kTileB;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma_ts_w(tmem + 384, ts + kk * 8 + (kk >> 2) * 32, ptx::sdesc_sw128(ka + kk * 2048, kHalf, 1024), id,
                      (acc || kk > 0) ? 1u : 0u);
}

__global__ void __launch_bounds__(kThreads, 1)
    sm100_softmax_bwd_dq_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapG,
                                const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                                const Params P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = ptx::smem_u32(smem);
    Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cta = blockIdx.x, num_ctas = gridDim.x;
    const int HG = P.H * P.G;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars->q_full, 1);
        ptx::mbar_init(&bars->q_empty, 1);
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&bars->k_full[s], 1);
            ptx::mbar_init(&bars->k_empty[s], 1);
            ptx::mbar_init(&bars->v_full[s], 1);
            ptx::mbar_init(&bars->v_empty[s], 1);
        }
        ptx::mbar_init(&bars->s_full, 1);
        ptx::mbar_init(&bars->dp_full, 1);
        ptx::mbar_init(&bars->p_ready, 256);
        ptx::mbar_init(&bars->ds_ready, 256);
        ptx::mbar_init(&bars->dq_full, 1);
        ptx::mbar_init(&bars->dq_empty, 256);
        ptx::fence_mbar_init();
        int s0, s1;
        partial_slots_g(P.uts, P.B, HG, cta, num_ctas, s0, s1, gmajor_groups(P.G, num_ctas));
        P.slot_unit[2 * cta] = s0;
        P.slot_unit[2 * cta + 1] = s1;
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);
    ItemIterG iter;
    iter.init(P.uts, P.B, HG, cta, num_ctas, gmajor_groups(P.G, num_ctas));
    Item it;
    if (warp == 0) {
        ptx::tma_prefetch(&mapQ);
        ptx::tma_prefetch(&mapG);
        ptx::tma_prefetch(&mapK);
        ptx::tma_prefetch(&mapV);
        const uint64_t pol = ptx::policy_evict_first(), pol_q = ptx::policy_evict_last();
        int st = 0;
        uint32_t ph = 0;
        int k = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int h = it.hg / P.G, g = it.hg % P.G;
            if (k > 0) ptx::mbar_wait(&bars->q_empty, (k - 1) & 1);
            ptx::mbar_arrive_expect_tx_w(&bars->q_full, 2 * kTileB);
            for (int half = 0; half < 2; ++half) {
                ptx::tma_load_4d_w(smem + kQOff + half * kHalf, &mapQ, &bars->q_full, half * 64, h, g * 128,
                                   P.q_per_user ? it.u : 0, pol_q);
                ptx::tma_load_4d_w(smem + kGOff + half * kHalf, &mapG, &bars->q_full, half * 64, h, g * 128, it.u, pol);
            }
            const int64_t row0 = P.offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                const int32_t row = (int32_t)(row0 + (int64_t)t * 128);
                ptx::mbar_wait(&bars->k_empty[st], ph ^ 1);
                ptx::mbar_arrive_expect_tx_w(&bars->k_full[st], kTileB);
                for (int half = 0; half < 2; ++half)
                    ptx::tma_load_3d_w(smem + kKOff + st * kTileB + half * kHalf, &mapK, &bars->k_full[st], half * 64, h,
                                       row, pol);
                ptx::mbar_wait(&bars->v_empty[st], ph ^ 1);
                ptx::mbar_arrive_expect_tx_w(&bars->v_full[st], kTileB);
                for (int half = 0; half < 2; ++half)
                    ptx::tma_load_3d_w(smem + kVOff + st * kTileB + half * kHalf, &mapV, &bars->v_full[st], half * 64, h,
                                       row, pol);
                if (++st == 2) { st = 0; ph ^= 1; }
            }
            ++k;
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer, software-pipelined over the key tiles n of all items:
        //   S(n) dP(n) | P(n) ready: S(n+1) | dS(n) ready: dQ(n) dP(n+1) | ...
        // S alternates between two TMEM buffers, so S(n+1) runs while the softmax computes P(n) -> dS(n);
        // S(n+2) reuses dS(n)'s buffer only after dQ(n) (MMAs execute in order).
        int st = 0, sb = 0;
        uint32_t ph = 0, pph = 0, dsph = 0, qeph = 0;
        int k = 0;
        bool pend = false, p_first = false, p_last = false;
        int p_st = 0, p_sb = 0;
        auto pend_dq = [&]() {
            ptx::mbar_wait(&bars->ds_ready, dsph);
            dsph ^= 1;
            if (p_first) {  // dQ accumulator drained by the previous item's epilogue
                ptx::mbar_wait(&bars->dq_empty, qeph ^ 1);
                qeph ^= 1;
            }
            ptx::tc_fence_after();
            issue_dq(tmem, tmem + p_sb * 128, base, p_st, !p_first);
            ptx::mma_commit_w(&bars->k_empty[p_st]);  // K feeds S and dQ
            if (p_last) ptx::mma_commit_w(&bars->dq_full);
            pend = false;
        };
        while (iter.next(it, P.uts, P.B, HG)) {
            ptx::mbar_wait(&bars->q_full, k & 1);
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->k_full[st], ph);
                if (pend) {
                    ptx::mbar_wait(&bars->p_ready, pph);
                    pph ^= 1;
                }
                ptx::tc_fence_after();
                issue_s(tmem + sb * 128, base, st);
                ptx::mma_commit_w(&bars->s_full);
                if (pend) pend_dq();
                ptx::mbar_wait(&bars->v_full[st], ph);
                ptx::tc_fence_after();
                issue_dp(tmem, base, st);
                ptx::mma_commit_w(&bars->dp_full);
                ptx::mma_commit_w(&bars->v_empty[st]);                  // V only feeds dP
                if (t + 1 == it.t1) ptx::mma_commit_w(&bars->q_empty);  // Q_g, dO_g feed only S, dP
                pend = true;
                p_first = t == it.t0;
                p_last = t + 1 == it.t1;
                p_st = st;
                p_sb = sb;
                sb ^= 1;
                if (++st == 2) { st = 0; ph ^= 1; }
            }
            ++k;
        }
        if (pend) {
            ptx::mbar_wait(&bars->p_ready, pph);
            pend_dq();
        }
    } else if (warp >= 4) {
        // ---------------- row softmax: P = exp2(S scale log2e - lse_i log2e), dS = P (dP - D_i); epilogue dQ.
        // Warpgroup sg handles keys [64 sg, 64 sg + 64) of each tile and dQ columns [64 sg, 64 sg + 64).
        const int wq = warp % 4, sg = (warp - 4) / 4;
        const int r = wq * 32 + lane;  // query row within the block = TMEM lane
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        uint32_t sph = 0, dph = 0, qph = 0;
        int sb = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int h = it.hg / P.G, g = it.hg % P.G;
            const int64_t L = P.offsets[it.u + 1] - P.offsets[it.u];
            const size_t li = ((size_t)it.u * P.H + h) * P.S + g * 128 + r;
            const float lse2 = __ldg(P.lse + li) * kLog2e, dd = __ldg(P.dd + li);
            const uint64_t sl2x2 = ptx::f2_pack(P.scale_log2, P.scale_log2), nlse2x2 = ptx::f2_pack(-lse2, -lse2),
                           ndd2 = ptx::f2_pack(-dd, -dd), zero2 = ptx::f2_pack(0.f, 0.f);
            for (int t = it.t0; t < it.t1; ++t) {
                const int64_t remv = L - (int64_t)t * 128 - sg * 64;
                const int valid = remv < 64 ? (int)remv : 64;  // keys of this half (may be <= 0)
                const uint32_t tsb = tmem + lane_bits + sb * 128 + sg * 64, tdp = tmem + lane_bits + 256 + sg * 64;
                uint32_t pk[32];
                ptx::mbar_wait(&bars->s_full, sph);
                sph ^= 1;
                ptx::tc_fence_after();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t sr[32];
                    ptx::tmem_ld32(tsb + c * 32, sr);
                    ptx::tmem_wait_ld();
                    ptx::reg_fence(sr);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {  // x = s scale log2e - lse log2e (FFMA2), p = 2^x
                        const int col = c * 32 + 2 * j;
                        float x0, x1;
                        ptx::f2_unpack(ptx::f2_fma(ptx::f2_pack(__uint_as_float(sr[2 * j]), __uint_as_float(sr[2 * j + 1])),
                                                   sl2x2, nlse2x2),
                                       x0, x1);
                        const float p0 = col < valid ? ptx::ex2(x0) : 0.f;
                        const float p1 = col + 1 < valid ? ptx::ex2(x1) : 0.f;
                        pk[16 * c + j] = ptx::pack_bf16x2(p0, p1);
                    }
                }
                ptx::tc_fence_before();  // S read: the buffer may take S(n+2) after dQ(n)
                ptx::mbar_arrive(&bars->p_ready);
                ptx::mbar_wait(&bars->dp_full, dph);
                dph ^= 1;
                ptx::tc_fence_after();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t dr[32];
                    ptx::tmem_ld32(tdp + c * 32, dr);
                    ptx::tmem_wait_ld();
                    ptx::reg_fence(dr);
                    uint32_t sw[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint32_t pw = pk[16 * c + j];  // dS = P (dP - D): FADD2 then FFMA2 (+0)
                        const uint64_t t2 =
                            ptx::f2_add(ptx::f2_pack(__uint_as_float(dr[2 * j]), __uint_as_float(dr[2 * j + 1])), ndd2);
                        float d0, d1;
                        ptx::f2_unpack(ptx::f2_fma(ptx::f2_pack(__uint_as_float(pw << 16), __uint_as_float(pw & 0xffff0000u)),
                                                   t2, zero2),
                                       d0, d1);
                        sw[j] = ptx::pack_bf16x2(d0, d1);
                    }
                    ptx::tmem_st16(tsb + c * 16, sw);
                }
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&bars->ds_ready);
                sb ^= 1;
            }
            // epilogue: dQ rows x scale (this warpgroup's 64 columns) -> final [B,H,S,d] row or a slot
            ptx::mbar_wait(&bars->dq_full, qph);
            qph ^= 1;
            ptx::tc_fence_after();
            float* dst = (item_complete(it) ? P.dqbuf + ((size_t)(it.u * HG + it.hg) * 128 + r) * 128
                                            : P.slot_o + ((size_t)item_slot(it, cta) * 128 + r) * 128) +
                         sg * 64;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t o[32];
                ptx::tmem_ld32_sync(tmem + lane_bits + 384 + sg * 64 + c * 32, o);
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + c * 32 + j) =
                        make_float4(__uint_as_float(o[j]) * P.scale, __uint_as_float(o[j + 1]) * P.scale,
                                    __uint_as_float(o[j + 2]) * P.scale, __uint_as_float(o[j + 3]) * P.scale);
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bars->dq_empty);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}
}  // namespace dq

// D[u,h,i] = sum_c dO[u,i,h,c] O[u,i,h,c]   (one warp per row; 4 consecutive channels per lane)
template <typename TO>
__global__ void softmax_bwd_d_kernel(const TO* __restrict__ out, const TO* __restrict__ dout, int B, int S, int H,
                                     float* __restrict__ dd) {
    const int64_t rrow = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;  // over (u, h, i)
    const int lane = threadIdx.x % 32;
    if (rrow >= (int64_t)B * H * S) return;
    const int u = (int)(rrow / ((int64_t)H * S)), h = (int)((rrow / S) % H), i = (int)(rrow % S);
    const size_t idx = (((size_t)u * S + i) * H + h) * 128 + 4 * lane;
    float s = 0.f;
    if constexpr (sizeof(TO) == 2) {
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(out + idx));
        const uint2 b = __ldg(reinterpret_cast<const uint2*>(dout + idx));
        const uint32_t aw[2] = {a.x, a.y}, bw[2] = {b.x, b.y};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            s = fmaf(__uint_as_float(aw[e] << 16), __uint_as_float(bw[e] << 16), s);
            s = fmaf(__uint_as_float(aw[e] & 0xffff0000u), __uint_as_float(bw[e] & 0xffff0000u), s);
        }
    } else {
        const float4 a = __ldg(reinterpret_cast<const float4*>(out + idx));
        const float4 b = __ldg(reinterpret_cast<const float4*>(dout + idx));
        s = a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) dd[rrow] = s;
}

// dq (final): shared seeds [S,H,d] = sum_u dqbuf[u,h,i,:] (ascending u); per-user [B,S,H,d].
// Four columns per thread; the loads of 8 users are issued before their (in-order) additions.
__global__ void softmax_bwd_dq_final_kernel(const float* __restrict__ dqbuf, int B, int S, int H, int per_user,
                                            float* __restrict__ dq) {
    const int64_t n4 = (per_user ? (int64_t)B * S * H * 128 : (int64_t)S * H * 128) / 4;
    const size_t ustride = (size_t)H * S * 128 / 4;  // one user's rows, in float4
    const float4* src = reinterpret_cast<const float4*>(dqbuf);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
        const int c4 = (int)(e % 32);
        const int h = (int)((e / 32) % H);
        const int i = (int)((e / (32 * H)) % S);
        const size_t hi = ((size_t)h * S + i) * 32 + c4;  // within a user
        if (per_user) {
            const int u = (int)(e / ((int64_t)32 * H * S));
            reinterpret_cast<float4*>(dq)[e] = src[(size_t)u * ustride + hi];
        } else {
            float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
            int u = 0;
            for (; u + 8 <= B; u += 8) {
                float4 v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = __ldg(src + (size_t)(u + j) * ustride + hi);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    s.x += v[j].x;
                    s.y += v[j].y;
                    s.z += v[j].z;
                    s.w += v[j].w;
                }
            }
            for (; u < B; ++u) {
                const float4 v = __ldg(src + (size_t)u * ustride + hi);
                s.x += v.x;
                s.y += v.y;
                s.z += v.z;
                s.w += v.w;
            }
            reinterpret_cast<float4*>(dq)[e] = s;
        }
    }
}

}  // namespace

bool softmax_bwd_supported(const Problem& p, bool dout_bf16) {
    return p.in_bf16 && dout_bf16 && p.d == 128 && p.S % 128 == 0 && p.S <= kv::kMaxS &&
           p.total_len < (int64_t(1) << 31) && (p.q_user_stride % 8) == 0;
}

size_t softmax_bwd_workspace(const Problem& p) {
    const size_t C = (size_t)p.num_sms;
    size_t off = 0;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    off = al(off + (size_t)(p.B + 1) * 8);           // uts
    off = al(off + 2 * C * sizeof(int));             // slot_unit
    off = al(off + 2 * C * 128 * 128 * 4);           // slots
    off = al(off + (size_t)p.B * p.H * p.S * 4);     // D
    off = al(off + (size_t)p.B * p.H * p.S * 128 * 4);  // dq buffer
    return off;
}

cudaError_t launch_softmax_bwd(const Problem& p, const void* out, const float* lse, const void* dout, float* dq_out,
                               void* dk, void* dv, char* ws, int* nlaunch, cudaEvent_t ev_a, cudaEvent_t ev_b) {
    const size_t C = (size_t)p.num_sms;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t off = 0;
    int64_t* uts = reinterpret_cast<int64_t*>(ws + off);
    off = al(off + (size_t)(p.B + 1) * 8);
    int* slot_unit = reinterpret_cast<int*>(ws + off);
    off = al(off + 2 * C * sizeof(int));
    float* slots = reinterpret_cast<float*>(ws + off);
    off = al(off + 2 * C * 128 * 128 * 4);
    float* dd = reinterpret_cast<float*>(ws + off);
    off = al(off + (size_t)p.B * p.H * p.S * 4);
    float* dqbuf = reinterpret_cast<float*>(ws + off);
    cudaError_t e;
    int nl = 0;
    // tile prefix (no output fill: nothing is written for empty users here)
    Problem ps = p;
    ps.outs = OutSpec{OUT_PARTIAL, 0, nullptr, nullptr};
    ps.attn = VISTA_QLA;  // no softmax empty-fill
    if ((e = launch_user_tiles(ps, uts, nullptr)) != cudaSuccess) return e;
    ++nl;
    // D
    {
        const int64_t rows = (int64_t)p.B * p.H * p.S;
        const unsigned grid = (unsigned)((rows + 7) / 8);
        softmax_bwd_d_kernel<__nv_bfloat16><<<grid, 256, 0, p.stream>>>(
            reinterpret_cast<const __nv_bfloat16*>(out), reinterpret_cast<const __nv_bfloat16*>(dout), p.B, p.S, p.H, dd);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        ++nl;
    }
    CUtensorMap mq, mg, mk, mv;
    if (!make_q_map(&mq, p.q, p.S, p.H, p.B, p.q_user_stride) ||
        !make_q_map(&mg, dout, p.S, p.H, p.B, (int64_t)p.S * p.H * 128) || !make_kv_map(&mk, p.k, p.total_len, p.H) ||
        !make_kv_map(&mv, p.v, p.total_len, p.H))
        return cudaErrorInvalidValue;
    // pass 1: dK, dV
    {
        kv::Params P;
        P.offsets = p.offsets;
        P.uts = uts;
        P.lse = lse;
        P.dd = dd;
        P.dk = reinterpret_cast<__nv_bfloat16*>(dk);
        P.dv = reinterpret_cast<__nv_bfloat16*>(dv);
        P.B = p.B;
        P.S = p.S;
        P.H = p.H;
        P.scale_log2 = p.scale * kLog2e;
        P.scale = p.scale;
        P.q_per_user = p.q_user_stride != 0;
        const bool stream = p.S > kv::kResidentMaxS;
        const cudaError_t attr0 = set_smem_attr(reinterpret_cast<const void*>(kv::sm100_softmax_bwd_kv_kernel<false>), kv::kSmem);
        const cudaError_t attr1 = set_smem_attr(reinterpret_cast<const void*>(kv::sm100_softmax_bwd_kv_kernel<true>), kv::kSmem);
        if (attr0 != cudaSuccess) return attr0;
        if (attr1 != cudaSuccess) return attr1;
        if (ev_a && (e = cudaEventRecord(ev_a, p.stream)) != cudaSuccess) return e;
        if (stream)
            kv::sm100_softmax_bwd_kv_kernel<true><<<(unsigned)C, kv::kThreads, kv::kSmem, p.stream>>>(mq, mg, mk, mv, P);
        else
            kv::sm100_softmax_bwd_kv_kernel<false><<<(unsigned)C, kv::kThreads, kv::kSmem, p.stream>>>(mq, mg, mk, mv, P);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (ev_b && (e = cudaEventRecord(ev_b, p.stream)) != cudaSuccess) return e;
        ++nl;
    }
    // pass 2: dQ (stream-K over (u, h, g) units, partial slots summed into dqbuf)
    {
        if ((e = cudaMemsetAsync(dqbuf, 0, (size_t)p.B * p.H * p.S * 128 * 4, p.stream)) != cudaSuccess) return e;
        dq::Params P;
        P.offsets = p.offsets;
        P.uts = uts;
        P.slot_unit = slot_unit;
        P.slot_o = slots;
        P.dqbuf = dqbuf;
        P.lse = lse;
        P.dd = dd;
        P.B = p.B;
        P.S = p.S;
        P.H = p.H;
        P.G = p.S / 128;
        P.scale_log2 = p.scale * kLog2e;
        P.scale = p.scale;
        P.q_per_user = p.q_user_stride != 0;
        const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(dq::sm100_softmax_bwd_dq_kernel), dq::kSmem);
        if (attr != cudaSuccess) return attr;
        dq::sm100_softmax_bwd_dq_kernel<<<(unsigned)C, dq::kThreads, dq::kSmem, p.stream>>>(mq, mg, mk, mv, P);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        ++nl;
        // split units: sum the run of slots (the QLA slot merge; units of 128 rows)
        Workspace w{};
        w.num_ctas = (int)C;
        w.slot_unit_off = (size_t)(reinterpret_cast<char*>(slot_unit) - ws);
        w.slot_o_off = (size_t)(reinterpret_cast<char*>(slots) - ws);
        if ((e = launch_merge_qla_slots(p, w, ws, dqbuf)) != cudaSuccess) return e;
        ++nl;
    }
    {
        const bool per_user = p.q_user_stride != 0;
        const int64_t n = per_user ? (int64_t)p.B * p.S * p.H * 128 : (int64_t)p.S * p.H * 128;
        softmax_bwd_dq_final_kernel<<<(unsigned)std::min<int64_t>((n / 4 + 255) / 256, 4096), 256, 0, p.stream>>>(
            dqbuf, p.B, p.S, p.H, per_user, dq_out);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        ++nl;
    }
    *nlaunch = nl;
    return cudaSuccess;
}

}  // namespace vista
