// sm100_softmax2.cu -- seed-row softmax summarization on a CTA PAIR (cta_group::2), S % 256 == 0.
//
// Same math as sm100_softmax.cu (O = RowSoftmax(scale Q K^T) V, lse; PAPER.md:158-163 at the seed
// rows PAPER.md:148-149), different machine mapping.  A 2-CTA cluster owns one work unit
// (user, head, 256 seed rows); CTA r holds query rows [128 r, 128 r + 128) and the MMAs are
// M = 256 tcgen05.mma.cta_group::2 issued by the leader:
//   S = Q K^T   A = Q (each CTA its 128 rows), B = K tile split along N: CTA r loads keys
//               [64 r, 64 r + 64) of every 128-key tile
//   O += P V    A = P from TMEM (each CTA its rows), B = V tile split along N = d: CTA r loads
//               channels [64 r, 64 r + 64) of all 128 keys
// so each SM streams half of every K/V tile (HBM and L2->SM traffic stay 1x) while holding only
// one Q tile, which frees TMEM for TWO score buffers and TWO output accumulators per SM:
//   cols [0,128) S_A   [128,256) S_B   [256,384) O_A   [384,512) O_B
// Two softmax warpgroups per CTA take alternate key tiles (A: even, B: odd), each with its own
// running max / sum and its own O accumulator; the epilogue merges (m_A, l_A, O_A) and
// (m_B, l_B, O_B) exactly (the same identity as the split-L LSE merge).  While warpgroup A
// exponentiates tile t, the tensor core runs S(t+1) for B and PV(t-1) -- the serial
// softmax -> PV -> S chain of the single-CTA kernel is gone.
//
// Roles per CTA (384 threads): warp 0 TMA producer (its halves of Q/K/V, completion signalled on
// the leader's barriers); warp 1 MMA issuer (leader CTA only); warps 4-7 softmax WG A, warps 8-11
// softmax WG B (one thread per query row = TMEM lane; warp % 4 = lane quarter).
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>

#include "internal.h"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

bool make_map_bf16(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                   const cuuint32_t* box);
bool make_kv_map(CUtensorMap* map, const void* base, int64_t total_len, int H);
bool make_q_map(CUtensorMap* map, const void* base, int S, int H, int B, int64_t q_user_stride);

#ifdef VISTA_TRACE  // debug timeline of pair 0, first item: clock64 per (event, tile, slot)
__device__ unsigned long long g_vista_trace2[16][64][4];
#define VTRACE2(ev, t, q) \
    do { if (blockIdx.x < 2 && (t) < 64) g_vista_trace2[ev][t][q] = clock64(); } while (0)
#else
#define VTRACE2(ev, t, q) do { } while (0)
#endif

namespace {

constexpr int kQBytes = 128 * 128 * 2;       // this CTA's 128 query rows (two 64-channel halves)
constexpr int kQHalf = kQBytes / 2;
constexpr int kKBytes = 64 * 128 * 2;        // 64 keys x 128 channels (two 8 KB channel halves)
constexpr int kKHalf = kKBytes / 2;
constexpr int kVBytes = 128 * 64 * 2;        // 128 keys x 64 channels
constexpr int kStageBytes = kKBytes + kVBytes;
constexpr int kStages = 5;
constexpr int kStageOff = kQBytes;
constexpr int kBarOff = kStageOff + kStages * kStageBytes;
constexpr int kThreads = 384;
constexpr int kTmemCols = 512;
constexpr float kRescaleThreshold = 8.0f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
#ifndef VISTA_CTL_REGS2
#define VISTA_CTL_REGS2 152
#endif
constexpr int kCtlRegs = VISTA_CTL_REGS2;
constexpr int kSoftmaxRegs = ((64512 - 128 * kCtlRegs) / 256) & ~7;

struct Bars {
    uint64_t q_full, q_empty;
    uint64_t st_full[kStages], st_empty[kStages];
    uint64_t s_full[2], p_full[2], o_full[2];
    uint32_t tmem_base;
    float ml[2][2][128];  // [warpgroup][m | l][row] exchanged in the epilogue
};
constexpr int kSmem = kBarOff + (int)sizeof(Bars) + 1024;

struct Params {
    const int64_t* offsets;
    const int64_t* uts;
    int* slot_unit;
    float* slot_o;
    float* slot_lse;
    OutSpec outs;
    int B, S, H, G;
    float scale_log2;
    int q_per_user;
};

// ---- MMA issue with compile-time geometry (uniform descriptors) ----
template <int BUF, int ST>
__device__ __forceinline__ void issue_S2(uint32_t tmem, uint32_t sQ, uint32_t sSt) {
    // S_BUF = Q K^T: M = 256 (both CTAs' rows), N = 128 keys (this CTA supplies 64), K = 128 channels
    constexpr uint32_t id = ptx::idesc_bf16_f32(256, 128, 0, 0);
    const uint32_t k = sSt + ST * kStageBytes;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma2_ss_w(tmem + BUF * 128, ptx::sdesc_sw128(sQ + (kk >> 2) * kQHalf + (kk & 3) * 32, 16, 1024),
                       ptx::sdesc_sw128(k + (kk >> 2) * kKHalf + (kk & 3) * 32, 16, 1024), id, kk > 0);
}
template <int BUF, int ST, bool ACC>
__device__ __forceinline__ void issue_PV2(uint32_t tmem, uint32_t sSt) {
    // O_BUF += P_BUF V: M = 256, N = 128 channels (this CTA supplies 64), K = 128 keys; P from TMEM
    constexpr uint32_t id = ptx::idesc_bf16_f32(256, 128, 0, 1);
    const uint32_t v = sSt + ST * kStageBytes + kKBytes;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma2_ts_w(tmem + 256 + BUF * 128, tmem + BUF * 128 + kk * 8, ptx::sdesc_sw128(v + kk * 2048, 16384, 1024),
                       id, (ACC || kk > 0) ? 1u : 0u);
}
template <int BUF>
__device__ __forceinline__ void issue_S2_d(int st, uint32_t tmem, uint32_t sQ, uint32_t sSt) {
    switch (st) {
        case 0: issue_S2<BUF, 0>(tmem, sQ, sSt); break;
        case 1: issue_S2<BUF, 1>(tmem, sQ, sSt); break;
        case 2: issue_S2<BUF, 2>(tmem, sQ, sSt); break;
        case 3: issue_S2<BUF, 3>(tmem, sQ, sSt); break;
        default: issue_S2<BUF, 4>(tmem, sQ, sSt); break;
    }
}
template <int BUF, bool ACC>
__device__ __forceinline__ void issue_PV2_d(int st, uint32_t tmem, uint32_t sSt) {
    switch (st) {
        case 0: issue_PV2<BUF, 0, ACC>(tmem, sSt); break;
        case 1: issue_PV2<BUF, 1, ACC>(tmem, sSt); break;
        case 2: issue_PV2<BUF, 2, ACC>(tmem, sSt); break;
        case 3: issue_PV2<BUF, 3, ACC>(tmem, sSt); break;
        default: issue_PV2<BUF, 4, ACC>(tmem, sSt); break;
    }
}

struct Cursor {  // ring position (stage index + phase bit)
    int idx = 0;
    uint32_t ph = 0;
    __device__ void next() {
        if (++idx == kStages) { idx = 0; ph ^= 1; }
    }
};

// p = 2^(s scale log2e - m) for one 128-key row; P overwrites the first 64 TMEM columns of S.
__device__ __forceinline__ float exp_row(const uint32_t (&r)[4][32], float sl2, float neg, uint32_t tS) {
    const uint64_t sl2x2 = ptx::f2_pack(sl2, sl2);
    const uint64_t negx2 = ptx::f2_pack(neg, neg);
    uint64_t acc[2] = {ptx::f2_pack(0.f, 0.f), ptx::f2_pack(0.f, 0.f)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint64_t x2 = ptx::f2_fma(
                ptx::f2_pack(__uint_as_float(r[c][2 * j]), __uint_as_float(r[c][2 * j + 1])), sl2x2, negx2);
            float x0, x1;
            ptx::f2_unpack(x2, x0, x1);
            const float p0 = ptx::ex2(x0), p1 = ptx::ex2(x1);
            acc[j & 1] = ptx::f2_add(acc[j & 1], ptx::f2_pack(p0, p1));
            pk[j] = ptx::pack_bf16x2(p0, p1);
        }
        ptx::tmem_st16(tS + c * 16, pk);
    }
    float la, lb, lc, ld;
    ptx::f2_unpack(acc[0], la, lb);
    ptx::f2_unpack(acc[1], lc, ld);
    return (la + lb) + (lc + ld);
}

__device__ __forceinline__ void store_row(const Params& P, const Item& it, int pair, int row_in_unit,
                                          const float (&o)[32], int c0, float lse, bool write_lse) {
    constexpr int kRows = 256;
    const int h = it.hg / P.G, g = it.hg % P.G;
    if (!item_complete(it)) {
        const int slot = item_slot(it, pair);
        float* dst = P.slot_o + ((size_t)slot * kRows + row_in_unit) * 128 + c0;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
        if (write_lse) P.slot_lse[(size_t)slot * kRows + row_in_unit] = lse;
        return;
    }
    const int i = g * kRows + row_in_unit;
    if (P.outs.mode == OUT_PARTIAL) {
        float* dst = reinterpret_cast<float*>(P.outs.out) + (((size_t)it.u * P.H + h) * P.S + i) * 128 + c0;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
        if (write_lse) P.outs.lse[((size_t)it.u * P.H + h) * P.S + i] = lse;
        return;
    }
    const size_t base = (((size_t)it.u * P.S + i) * P.H + h) * 128 + c0;
    if (P.outs.out_bf16) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(P.outs.out) + base;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            uint4 pk;
            pk.x = ptx::pack_bf16x2(o[j], o[j + 1]);
            pk.y = ptx::pack_bf16x2(o[j + 2], o[j + 3]);
            pk.z = ptx::pack_bf16x2(o[j + 4], o[j + 5]);
            pk.w = ptx::pack_bf16x2(o[j + 6], o[j + 7]);
            *reinterpret_cast<uint4*>(dst + j) = pk;
        }
    } else {
        float* dst = reinterpret_cast<float*>(P.outs.out) + base;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
    }
    if (write_lse && P.outs.lse) P.outs.lse[((size_t)it.u * P.H + h) * P.S + i] = lse;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    sm100_softmax2_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                          const __grid_constant__ CUtensorMap mapV, const Params P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    Bars* bars = reinterpret_cast<Bars*>(smem_raw + (base - ptx::smem_u32(smem_raw)) + kBarOff);
    const uint32_t sQ = base, sSt = base + kStageOff;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int HG = P.H * P.G;

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars->q_full, 2);
        ptx::mbar_init(&bars->q_empty, 1);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bars->st_full[s], 2);
            ptx::mbar_init(&bars->st_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->s_full[b], 1);
            ptx::mbar_init(&bars->p_full[b], 8);  // 4 warps here + 4 warps in the peer CTA
            ptx::mbar_init(&bars->o_full[b], 1);
        }
        ptx::fence_mbar_init();
        if (rank == 0) {
            int s0, s1;
            partial_slots(P.uts, P.B, HG, pair, npairs, s0, s1);
            P.slot_unit[2 * pair] = s0;
            P.slot_unit[2 * pair + 1] = s1;
        }
    }
    if (warp == 1) ptx::tmem_alloc2(&bars->tmem_base, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // peer barriers are initialized before any remote arrive / TMA signal
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);

    ItemIter iter;
    iter.init(P.uts, P.B, HG, pair, npairs);
    Item it;

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
        if (warp == 0) {
            // ============================ TMA producer (both CTAs) ============================
            ptx::tma_prefetch(&mapQ);
            ptx::tma_prefetch(&mapK);
            ptx::tma_prefetch(&mapV);
            const uint64_t pol_kv = ptx::policy_evict_first();
            const uint64_t pol_q = ptx::policy_evict_last();
            const uint32_t q_full_L = ptx::mapa(ptx::smem_u32(&bars->q_full), 0);
            Cursor cs;
            int k = 0;
            while (iter.next(it, P.uts, P.B, HG)) {
                const int h = it.hg / P.G, g = it.hg % P.G;
                if (k > 0) ptx::mbar_wait(&bars->q_empty, (k - 1) & 1);
                ptx::mbar_arrive_expect_tx_cluster_w(q_full_L, kQBytes);
                for (int half = 0; half < 2; ++half)
                    ptx::tma_load_4d_2sm_w(sQ + half * kQHalf, &mapQ, q_full_L, half * 64, h, g * 256 + (int)rank * 128,
                                           P.q_per_user ? it.u : 0, pol_q);
                const int64_t row0 = P.offsets[it.u];
                for (int t = it.t0; t < it.t1; ++t) {
                    ptx::mbar_wait(&bars->st_empty[cs.idx], cs.ph ^ 1);
                    if (k == 0 && lane == 0) VTRACE2(8, t - it.t0, rank);
                    const uint32_t full_L = ptx::mapa(ptx::smem_u32(&bars->st_full[cs.idx]), 0);
                    ptx::mbar_arrive_expect_tx_cluster_w(full_L, kStageBytes);
                    const int32_t row = (int32_t)(row0 + (int64_t)t * kTile);
                    const uint32_t st = sSt + cs.idx * kStageBytes;
                    for (int half = 0; half < 2; ++half)  // keys [64 rank, +64), channel half
                        ptx::tma_load_3d_2sm_w(st + half * kKHalf, &mapK, full_L, half * 64, h, row + (int)rank * 64, pol_kv);
                    // all 128 keys, channels [64 rank, +64)
                    ptx::tma_load_3d_2sm_w(st + kKBytes, &mapV, full_L, (int)rank * 64, h, row, pol_kv);
                    cs.next();
                }
                ++k;
            }
        } else if (warp == 1 && rank == 0) {
            // ============================ MMA issuer (leader CTA) ============================
            Cursor cload, cfree;  // stage of the next S to issue / of the next PV to retire
            bool first = true;
            uint32_t q_phase = 0;
            uint32_t p_phase[2] = {0, 0};
            while (iter.next(it, P.uts, P.B, HG)) {
                const int n = it.t1 - it.t0;
                ptx::mbar_wait(&bars->q_full, q_phase);
                q_phase ^= 1;
                ptx::mbar_wait(&bars->st_full[cload.idx], cload.ph);
                ptx::tc_fence_after();
                issue_S2_d<0>(cload.idx, tmem, sQ, sSt);
                ptx::mma2_commit_mc_w(&bars->s_full[0]);
                cload.next();
                if (n > 1) {
                    ptx::mbar_wait(&bars->st_full[cload.idx], cload.ph);
                    ptx::tc_fence_after();
                    issue_S2_d<1>(cload.idx, tmem, sQ, sSt);
                    ptx::mma2_commit_mc_w(&bars->s_full[1]);
                    cload.next();
                }
                for (int t = 0; t < n; ++t) {
                    const int b = t & 1;
                    if (first && lane == 0) VTRACE2(0, t, 0);
                    ptx::mbar_wait(&bars->p_full[b], p_phase[b]);
                    if (first && lane == 0) VTRACE2(1, t, 0);
                    p_phase[b] ^= 1;
                    ptx::tc_fence_after();
                    if (b == 0) {
                        if (t >= 2) issue_PV2_d<0, true>(cfree.idx, tmem, sSt); else issue_PV2_d<0, false>(cfree.idx, tmem, sSt);
                    } else {
                        if (t >= 2) issue_PV2_d<1, true>(cfree.idx, tmem, sSt); else issue_PV2_d<1, false>(cfree.idx, tmem, sSt);
                    }
                    ptx::mma2_commit_mc_w(&bars->st_empty[cfree.idx]);
                    cfree.next();
                    if (first && lane == 0) VTRACE2(9, t, 0);
                    if (t + 2 < n) {
                        ptx::mbar_wait(&bars->st_full[cload.idx], cload.ph);
                        if (first && lane == 0) VTRACE2(10, t, 0);
                        ptx::tc_fence_after();
                        if (b == 0) issue_S2_d<0>(cload.idx, tmem, sQ, sSt); else issue_S2_d<1>(cload.idx, tmem, sQ, sSt);
                        ptx::mma2_commit_mc_w(&bars->s_full[b]);
                        cload.next();
                    }
                    if (first && lane == 0) VTRACE2(2, t, 0);
                }
                first = false;
                ptx::mma2_commit_mc_w(&bars->o_full[0]);
                ptx::mma2_commit_mc_w(&bars->o_full[1]);
                ptx::mma2_commit_mc_w(&bars->q_empty);
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
        // ============================ softmax warpgroups (both CTAs) ============================
        const int wg = (warp - 4) / 4;  // 0: even key tiles (S_A, O_A); 1: odd (S_B, O_B)
        const int wq = warp % 4;
        const int row = wq * 32 + lane;
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_bits + wg * 128;
        const uint32_t tOA = tmem + lane_bits + 256, tOB = tmem + lane_bits + 384;
        const uint32_t tO = wg ? tOB : tOA;
        const uint32_t p_full_L = ptx::mapa(ptx::smem_u32(&bars->p_full[wg]), 0);
        const float sl2 = P.scale_log2;
        uint32_t s_phase = 0, o_phase = 0;
        bool first = true;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int64_t L = P.offsets[it.u + 1] - P.offsets[it.u];
            const int n = it.t1 - it.t0;
            float m_used = -INFINITY, l = 0.f;
            for (int t = wg; t < n; t += 2) {
                const bool tr = first && row == 0;
                if (tr) VTRACE2(3, t, rank * 2 + wg);
                ptx::mbar_wait(&bars->s_full[wg], s_phase);
                if (tr) VTRACE2(4, t, rank * 2 + wg);
                s_phase ^= 1;
                ptx::tc_fence_after();
                uint32_t r[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tS + c * 32, r[c]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::reg_fence(r[c]);
                const int64_t valid = L - (int64_t)(it.t0 + t) * kTile;
                if (valid < kTile) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c * 32 + j >= valid) r[c][j] = __float_as_uint(-INFINITY);
                }
                float m8[8];
#pragma unroll
                for (int a = 0; a < 8; ++a) {
                    const int c = a >> 1, o = (a & 1) * 16;
                    float m = ptx::max3(__uint_as_float(r[c][o]), __uint_as_float(r[c][o + 1]),
                                        __uint_as_float(r[c][o + 2]));
#pragma unroll
                    for (int j = 3; j < 15; j += 2)
                        m = ptx::max3(m, __uint_as_float(r[c][o + j]), __uint_as_float(r[c][o + j + 1]));
                    m8[a] = fmaxf(m, __uint_as_float(r[c][o + 15]));
                }
                const float mxs = ptx::max3(ptx::max3(m8[0], m8[1], m8[2]), ptx::max3(m8[3], m8[4], m8[5]),
                                            fmaxf(m8[6], m8[7])) * sl2;
                const bool any = __any_sync(0xffffffffu, mxs > m_used + kRescaleThreshold);
                const float m_old = m_used;
                if (any) m_used = fmaxf(m_used, mxs);
                if (tr) VTRACE2(5, t, rank * 2 + wg);
                const float lt = exp_row(r, sl2, -m_used, tS);
                if (tr) VTRACE2(6, t, rank * 2 + wg);
                if (any && t >= 2) {
                    // O_wg holds PV(t-2): S(t) was issued after it, so s_full(t) covered its completion
                    const float f = ptx::ex2(m_old - m_used);
                    l *= f;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        ptx::tmem_ld32_sync(tO + c * 32, o);
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
                        ptx::tmem_st32(tO + c * 32, o);
                    }
                }
                l += lt;
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0) ptx::mbar_arrive(&bars->p_full[wg]);
                    else ptx::mbar_arrive_cluster(p_full_L, 1);
                }
                if (tr) VTRACE2(7, t, rank * 2 + wg);
            }
            // ---- epilogue: merge the two warpgroups' (m, l, O) exactly, write O / l and lse
            bars->ml[wg][0][row] = m_used;
            bars->ml[wg][1][row] = l;
            ptx::named_bar_sync(1, 256);
            const float m_o = bars->ml[wg ^ 1][0][row], l_o = bars->ml[wg ^ 1][1][row];
            ptx::mbar_wait(&bars->o_full[0], o_phase);
            ptx::mbar_wait(&bars->o_full[1], o_phase);
            o_phase ^= 1;
            ptx::tc_fence_after();
            const float M = fmaxf(m_used, m_o);
            const float w_self = m_used == -INFINITY ? 0.f : ptx::ex2(m_used - M);
            const float w_oth = m_o == -INFINITY ? 0.f : ptx::ex2(m_o - M);
            const float Lsum = w_self * l + w_oth * l_o;
            const float inv = 1.f / Lsum;
            const float lse = (M + __log2f(Lsum)) * kLn2;
            const float wA = (wg ? w_oth : w_self) * inv, wB = (wg ? w_self : w_oth) * inv;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int c = wg * 2 + cc;  // WG A writes channels [0, 64), WG B [64, 128)
                uint32_t oa[32];
                ptx::tmem_ld32_sync(tOA + c * 32, oa);
                float of[32];
                if (n > 1) {
                    uint32_t ob[32];
                    ptx::tmem_ld32_sync(tOB + c * 32, ob);
#pragma unroll
                    for (int j = 0; j < 32; ++j) of[j] = wA * __uint_as_float(oa[j]) + wB * __uint_as_float(ob[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) of[j] = wA * __uint_as_float(oa[j]);
                }
                store_row(P, it, pair, (int)rank * 128 + row, of, c * 32, lse, c == 0);
            }
            ptx::tc_fence_before();
            ptx::named_bar_sync(2, 256);  // both warpgroups done with O_A / O_B before the next item's PVs
            first = false;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    if (warp == 1) ptx::tmem_dealloc2(tmem, kTmemCols);
}

}  // namespace

static bool make_k_half_map(CUtensorMap* map, const void* base, int64_t total_len, int H) {
    const cuuint64_t dims[3] = {128, (cuuint64_t)H, (cuuint64_t)(total_len > 0 ? total_len : 1)};
    const cuuint64_t strides[2] = {128 * 2, (cuuint64_t)H * 128 * 2};
    const cuuint32_t box[3] = {64, 1, 64};
    return make_map_bf16(map, base, 3, dims, strides, box);
}

#ifdef VISTA_TRACE
extern "C" int vista_debug_trace2(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_vista_trace2, bytes < sizeof(g_vista_trace2) ? bytes : sizeof(g_vista_trace2));
}
#endif

cudaError_t launch_sm100_softmax2(const Problem& p, const Workspace& w, char* ws) {
    CUtensorMap mq, mk, mv;
    if (!make_q_map(&mq, p.q, p.S, p.H, p.B, p.q_user_stride) || !make_k_half_map(&mk, p.k, p.total_len, p.H) ||
        !make_kv_map(&mv, p.v, p.total_len, p.H))
        return cudaErrorInvalidValue;
    Params P;
    P.offsets = p.offsets;
    P.uts = reinterpret_cast<const int64_t*>(ws + w.uts_off);
    P.slot_unit = reinterpret_cast<int*>(ws + w.slot_unit_off);
    P.slot_o = reinterpret_cast<float*>(ws + w.slot_o_off);
    P.slot_lse = reinterpret_cast<float*>(ws + w.slot_lse_off);
    P.outs = p.outs;
    P.B = p.B;
    P.S = p.S;
    P.H = p.H;
    P.G = p.S / 256;
    P.scale_log2 = p.scale * kLog2e;
    P.q_per_user = p.q_user_stride != 0;
    static const cudaError_t attr =
        cudaFuncSetAttribute(sm100_softmax2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (attr != cudaSuccess) return attr;
    sm100_softmax2_kernel<<<2 * w.num_ctas, kThreads, kSmem, p.stream>>>(mq, mk, mv, P);
    return cudaGetLastError();
}

}  // namespace vista
