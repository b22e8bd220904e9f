// sm100_softmax.cu -- seed-row softmax summarization on B200: TMA + tcgen05 (TMEM accumulators).
//
// Computes, for every work unit (user u, head h, group of NQ*128 seed rows):
//   O = RowSoftmax(scale * Q K^T) V,  lse = ln sum_j exp(scale q.k_j)
// over the user's jagged history rows [offsets[u], offsets[u+1]) -- the seed-row outputs of
// self-attention with virtual seeds.  The S x L score matrix never exists:
// keys stream through shared memory 128 at a time with an online softmax (flash style).
//
// Per CTA (persistent, one per SM, stream-K flat tile ranges, see work.cuh):
//   warp 0      TMA producer: Q tiles once per item, K/V 128x128 bf16 tiles into an smem ring
//   warp 1      MMA issuer (one thread): S_q = Q_q K^T (SS), O_q += P_q V (TS, P read from TMEM)
//   warps 4..   NQ softmax warpgroups (warp % 4 = TMEM lane quarter), one thread per query row (= TMEM lane): online softmax,
//               P (bf16) written back into the S columns of TMEM, epilogue
// Every K/V tile is read from HBM once and used by all NQ query tiles (S = 256 -> NQ = 2).
// TMEM: S/P_q at columns [128 q, 128 q + 128), O_q at [128 NQ + 128 q, ...) -> 512 cols at NQ=2.
// Ping-pong: the MMA warp issues PV_0(t), S_0(t+1), PV_1(t), S_1(t+1), ... so one warpgroup's
// exponentials overlap the other's GEMMs.  A commit after S_q(t+1) also covers PV_q(t), which is
// why a softmax thread may rescale O_q right after s_full fires.
// Conditional rescale (threshold 2^8): the running max used for the exponent only moves when a
// row max exceeds it by more than 8 (log2 units); otherwise p <= 256 and O is left alone.
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>

#include "internal.h"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

namespace {

constexpr int kHalfBytes = 128 * 128;       // 128 rows x 64 bf16 (one 128-B swizzle column block)
constexpr int kTileBytes = 2 * kHalfBytes;  // 128 x 128 bf16
constexpr float kRescaleThreshold = 8.0f;   // log2 units
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

template <int NQ>
struct Cfg {
    static constexpr int kStages = NQ == 2 ? 2 : 3;
    static constexpr int kQOff = 0;
    static constexpr int kKVOff = NQ * kTileBytes;
    static constexpr int kStageBytes = 2 * kTileBytes;  // K + V
    static constexpr int kBarOff = kKVOff + kStages * kStageBytes;
    static constexpr int kSmem = kBarOff + 256 + 1024;  // + alignment slack
    static constexpr int kThreads = 128 + NQ * 128;  // control warpgroup + NQ softmax warpgroups
    static constexpr int kTmemCols = NQ == 2 ? 512 : 256;
};

struct Bars {
    uint64_t q_full, q_empty;
    uint64_t kv_full[3], kv_empty[3];
    uint64_t s_full[2], p_full[2], o_full[2];
    uint32_t tmem_base;
};

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

__device__ __forceinline__ void store_row(const Params& P, const Item& it, int cta, int row_in_unit,
                                          const float (&o)[32], int c0, float lse, bool write_lse, int NQrows) {
    // writes 32 consecutive channels [c0, c0+32) of one normalized output row (+ lse once)
    const int h = it.hg / P.G, g = it.hg % P.G;
    if (!item_complete(it)) {
        const int slot = item_slot(it, cta);
        float* dst = P.slot_o + ((size_t)slot * NQrows + row_in_unit) * 128 + c0;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
        if (write_lse) P.slot_lse[(size_t)slot * NQrows + row_in_unit] = lse;
        return;
    }
    const int i = g * NQrows + row_in_unit;
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

template <int NQ>
__global__ void __launch_bounds__(Cfg<NQ>::kThreads, 1)
    sm100_softmax_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                         const __grid_constant__ CUtensorMap mapV, const Params P) {
    using C = Cfg<NQ>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem + C::kQOff;
    uint8_t* sKV = smem + C::kKVOff;
    Bars* bars = reinterpret_cast<Bars*>(smem + C::kBarOff);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cta = blockIdx.x, num_ctas = gridDim.x;
    const int HG = P.H * P.G;
    constexpr int kRows = NQ * 128;

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars->q_full, 1);
        ptx::mbar_init(&bars->q_empty, 1);
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&bars->kv_full[s], 1);
            ptx::mbar_init(&bars->kv_empty[s], 1);
        }
        for (int q = 0; q < NQ; ++q) {
            ptx::mbar_init(&bars->s_full[q], 1);
            ptx::mbar_init(&bars->p_full[q], 128);
            ptx::mbar_init(&bars->o_full[q], 1);
        }
        ptx::fence_mbar_init();
        // record which units this CTA's partial slots will hold (read by the merge kernel)
        ItemIter itr;
        itr.init(P.uts, P.B, HG, cta, num_ctas);
        Item it;
        int s0 = -1, s1 = -1;
        while (itr.next(it)) {
            if (!item_complete(it)) {
                if (it.first) s0 = it.u * HG + it.hg; else s1 = it.u * HG + it.hg;
            }
        }
        P.slot_unit[2 * cta] = s0;
        P.slot_unit[2 * cta + 1] = s1;
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, C::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    ItemIter iter;
    iter.init(P.uts, P.B, HG, cta, num_ctas);
    Item it;

    if (warp < 4) {
        // register split: the launch grants 168 x 384 = 64512 registers; 128 x 88 + 256 x 208 = 64512
        // (setmaxnreg.inc blocks forever if the pool cannot cover it).  Softmax rows hold 128 fp32 scores.
        if constexpr (NQ == 2) asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            ptx::tma_prefetch(&mapQ);
            ptx::tma_prefetch(&mapK);
            ptx::tma_prefetch(&mapV);
            const uint64_t pol_kv = ptx::policy_evict_first();
            const uint64_t pol_q = ptx::policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            int k = 0;
            while (iter.next(it)) {
                const int h = it.hg / P.G, g = it.hg % P.G;
                if (k > 0) ptx::mbar_wait(&bars->q_empty, (k - 1) & 1);
                ptx::mbar_arrive_expect_tx(&bars->q_full, NQ * kTileBytes);
                for (int q = 0; q < NQ; ++q)
                    for (int half = 0; half < 2; ++half)
                        ptx::tma_load_4d(sQ + q * kTileBytes + half * kHalfBytes, &mapQ, &bars->q_full, half * 64, h,
                                         g * kRows + q * 128, P.q_per_user ? it.u : 0, pol_q);
                const int64_t row0 = P.offsets[it.u];
                for (int t = it.t0; t < it.t1; ++t) {
                    ptx::mbar_wait(&bars->kv_empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&bars->kv_full[stage], C::kStageBytes);
                    uint8_t* sk = sKV + stage * C::kStageBytes;
                    uint8_t* sv = sk + kTileBytes;
                    const int32_t row = (int32_t)(row0 + (int64_t)t * kTile);
                    for (int half = 0; half < 2; ++half) {
                        ptx::tma_load_3d(sk + half * kHalfBytes, &mapK, &bars->kv_full[stage], half * 64, h, row, pol_kv);
                        ptx::tma_load_3d(sv + half * kHalfBytes, &mapV, &bars->kv_full[stage], half * 64, h, row, pol_kv);
                    }
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                }
                ++k;
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ============================ MMA issuer ============================
        if (lane == 0) {
            constexpr uint32_t idS = ptx::idesc_bf16_f32(128, 128, 0, 0);  // Q, K both K-major
            constexpr uint32_t idP = ptx::idesc_bf16_f32(128, 128, 0, 1);  // P (TMEM), V MN-major
            const uint32_t sQa = ptx::smem_u32(sQ), sKVa = ptx::smem_u32(sKV);
            int stage = 0;
            uint32_t kv_phase = 0, q_phase = 0;
            uint32_t p_phase[2] = {0, 0};
            auto issue_S = [&](int q, int st) {
                const uint32_t qa = sQa + q * kTileBytes;
                const uint32_t ka = sKVa + st * C::kStageBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
                    ptx::mma_ss(tmem + q * 128, ptx::sdesc_sw128(qa + off, 16, 1024),
                                ptx::sdesc_sw128(ka + off, 16, 1024), idS, kk > 0);
                }
            };
            auto issue_PV = [&](int q, int st, bool acc) {
                const uint32_t va = sKVa + st * C::kStageBytes + kTileBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    ptx::mma_ts(tmem + NQ * 128 + q * 128, tmem + q * 128 + kk * 8,
                                ptx::sdesc_sw128(va + kk * 2048, kHalfBytes, 1024), idP, (acc || kk > 0) ? 1u : 0u);
                }
            };
            while (iter.next(it)) {
                const int n = it.t1 - it.t0;
                ptx::mbar_wait(&bars->q_full, q_phase);
                q_phase ^= 1;
                ptx::mbar_wait(&bars->kv_full[stage], kv_phase);
                ptx::tc_fence_after();
                for (int q = 0; q < NQ; ++q) {
                    issue_S(q, stage);
                    ptx::mma_commit(&bars->s_full[q]);
                }
                for (int i = 0; i < n; ++i) {
                    const int cur = stage;
                    int nst = stage + 1;
                    uint32_t nph = kv_phase;
                    if (nst == C::kStages) { nst = 0; nph ^= 1; }
                    for (int q = 0; q < NQ; ++q) {
                        ptx::mbar_wait(&bars->p_full[q], p_phase[q]);
                        p_phase[q] ^= 1;
                        ptx::tc_fence_after();
                        issue_PV(q, cur, i > 0);
                        if (q == NQ - 1) ptx::mma_commit(&bars->kv_empty[cur]);
                        if (i == n - 1) {
                            ptx::mma_commit(&bars->o_full[q]);
                            if (q == NQ - 1) ptx::mma_commit(&bars->q_empty);
                        } else {
                            if (q == 0) {
                                ptx::mbar_wait(&bars->kv_full[nst], nph);
                                ptx::tc_fence_after();
                            }
                            issue_S(q, nst);
                            ptx::mma_commit(&bars->s_full[q]);
                        }
                    }
                    stage = nst;
                    kv_phase = nph;
                }
            }
        }
        __syncwarp();
    }
    } else {
        if constexpr (NQ == 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
        // ============================ softmax warpgroups ============================
        const int wg = (warp - 4) / 4;  // warps 4..7 -> Q tile 0, 8..11 -> Q tile 1
        const int wq = warp % 4;
        const int row = wq * 32 + lane;  // row within Q tile = TMEM lane
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_bits + wg * 128;
        const uint32_t tO = tmem + lane_bits + NQ * 128 + wg * 128;
        const float sl2 = P.scale_log2;
        uint32_t s_phase = 0, o_phase = 0;
        while (iter.next(it)) {
            const int64_t L = P.offsets[it.u + 1] - P.offsets[it.u];
            float m_used = -INFINITY, l = 0.f;
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->s_full[wg], s_phase);
                s_phase ^= 1;
                ptx::tc_fence_after();
                uint32_t r[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tS + c * 32, r[c]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::reg_fence(r[c]);
                const int64_t valid = L - (int64_t)t * kTile;
                if (valid < kTile) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c * 32 + j >= valid) r[c][j] = __float_as_uint(-INFINITY);
                }
                float mx = -INFINITY;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r[c][j]));
                const float mxs = mx * sl2;
                const bool need = mxs > m_used + kRescaleThreshold;
                const bool any = __any_sync(0xffffffffu, need);
                const float m_old = m_used;
                if (any) m_used = fmaxf(m_used, mxs);
                const float neg = -m_used;
                float lt = 0.f;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t pk[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int col = hf * 64 + 2 * j;
                        const float p0 = ptx::ex2(fmaf(__uint_as_float(r[col >> 5][col & 31]), sl2, neg));
                        const float p1 = ptx::ex2(fmaf(__uint_as_float(r[(col + 1) >> 5][(col + 1) & 31]), sl2, neg));
                        lt += p0 + p1;
                        pk[j] = ptx::pack_bf16x2(p0, p1);
                    }
                    ptx::tmem_st32(tS + hf * 32, pk);
                }
                if (any && t > it.t0) {
                    // O_q holds this item's sum so far (PV_q(t-1) completed: covered by s_full(t))
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
                ptx::mbar_arrive(&bars->p_full[wg]);
            }
            // epilogue: O / l, lse
            ptx::mbar_wait(&bars->o_full[wg], o_phase);
            o_phase ^= 1;
            ptx::tc_fence_after();
            const float inv_l = 1.f / l;
            const float lse = (m_used + __log2f(l)) * kLn2;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t o[32];
                ptx::tmem_ld32_sync(tO + c * 32, o);
                float of[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) of[j] = __uint_as_float(o[j]) * inv_l;
                store_row(P, it, cta, wg * 128 + row, of, c * 32, lse, c == 0, kRows);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode_tiled() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

// bf16 tensor [outer..., d=128 inner] as a TMA map with box {64, 1, 128(, 1)} and 128-B swizzle.
bool make_map_bf16(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                   const cuuint32_t* box) {
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return false;
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_kv_map(CUtensorMap* map, const void* base, int64_t total_len, int H) {
    const cuuint64_t dims[3] = {128, (cuuint64_t)H, (cuuint64_t)(total_len > 0 ? total_len : 1)};
    const cuuint64_t strides[2] = {128 * 2, (cuuint64_t)H * 128 * 2};
    const cuuint32_t box[3] = {64, 1, 128};
    return make_map_bf16(map, base, 3, dims, strides, box);
}

bool make_q_map(CUtensorMap* map, const void* base, int S, int H, int B, int64_t q_user_stride) {
    const int Bq = q_user_stride ? (B > 0 ? B : 1) : 1;
    const cuuint64_t dims[4] = {128, (cuuint64_t)H, (cuuint64_t)S, (cuuint64_t)Bq};
    const cuuint64_t ustride = q_user_stride ? (cuuint64_t)q_user_stride * 2 : (cuuint64_t)S * H * 128 * 2;
    const cuuint64_t strides[3] = {128 * 2, (cuuint64_t)H * 128 * 2, ustride};
    const cuuint32_t box[4] = {64, 1, 128, 1};
    return make_map_bf16(map, base, 4, dims, strides, box);
}

template <int NQ>
static cudaError_t launch_nq(const Problem& p, const Workspace& w, char* ws) {
    using C = Cfg<NQ>;
    CUtensorMap mq, mk, mv;
    if (!make_q_map(&mq, p.q, p.S, p.H, p.B, p.q_user_stride) || !make_kv_map(&mk, p.k, p.total_len, p.H) ||
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
    P.G = p.S / (NQ * 128);
    P.scale_log2 = p.scale * kLog2e;
    P.q_per_user = p.q_user_stride != 0;
    static const cudaError_t attr =
        cudaFuncSetAttribute(sm100_softmax_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (attr != cudaSuccess) return attr;
    sm100_softmax_kernel<NQ><<<w.num_ctas, C::kThreads, C::kSmem, p.stream>>>(mq, mk, mv, P);
    return cudaGetLastError();
}

int sm100_softmax_nq(int S) { return (S % 256 == 0) ? 2 : 1; }

cudaError_t launch_sm100_softmax(const Problem& p, const Workspace& w, char* ws) {
    return sm100_softmax_nq(p.S) == 2 ? launch_nq<2>(p, w, ws) : launch_nq<1>(p, w, ws);
}

}  // namespace vista
