// sm100_qla_rows.cu -- QLA at arbitrary per-user query rows on B200 (NEXT-3 / NEXT-4):
//   history rows   O[S] = phi(Q[S]) phi(phi(K[S])^T V[S])
//   target rows    O[T] = phi(Q[T]) phi(phi(K[S])^T V[S]) + Delta(phi(Q[T]), phi(K[T])) V[T]
//                  Delta(X, Y)_ij = sum_k X_ik Y_ik delta_ij
// Row r of user u (r in [row_offsets[u], row_offsets[u+1])):
//   o_r = phi1(q_r) W_u  [+ (phi1(q_r) . phi1(k_self_r)) v_self_r / N_u],   W_u = phi2(Z_u / N_u)
// with Z_u the user's state (the forward state kernel, partial mode) and W_u its bf16 MN-major
// operand (qla_prep_w_kernel).  DESIGN.md readings R10 (1/N) and R20: with normalization the Delta
// term is divided by the same N_u (App. B, O = (Q K^T (.) M) V / N).
//
// sm100_qla_rows_kernel: persistent, one CTA per SM, stream-K over the flat 128-row tiles of the
// rows' jagged layout (work.cuh), one 128x128x128 tcgen05 GEMM per tile with W_u as the B operand.
// HBM-bound: per row-head 256 B of q read and 256 B (bf16) of o written (+ 512 B of k_self, v_self
// with the Delta term), 2 d^2 = 32,768 flop.
//   warp 0        TMA producer: q tiles (history rows: 3 stages of 32 KB) or q, k_self tiles
//                 (target rows: 2 stages of 64 KB); W_u (bulk copy) per unit into one of two buffers
//   warp 1        MMA issuer; O double-buffered in TMEM
//   warps 4..7    transform: phi1(Q) in place (bf16), one row per thread; with Delta also the row dot
//                 phi1(q) . phi1(k_self) (/ N_u) from the staged k tile, into shared memory
//   warps 8..15   epilogue: TMEM (+ d_r v_self_r, the v_self row prefetched) -> rows (bf16 coalesced
//                 through a TMEM round trip, or f32); two warps per TMEM lane quarter, 64 columns each
// qla_rows_simt_kernel: CUDA-core path for f32 inputs or d in {32, 64} (one block per (row, head)).
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "qla_common.cuh"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

bool make_kv_map(CUtensorMap* map, const void* base, int64_t total_len, int H);

namespace {

constexpr int kHalf = 128 * 128;  // one 64-column half of a 128 x 128 bf16 tile
constexpr int kTile = 2 * kHalf;  // 32 KB
constexpr int kThreads = 512;
constexpr int kXform = 128;
constexpr int kEpi = 256;

// Shared-memory geometry: history rows stage q only (3 x 32 KB); target rows stage q and k_self of
// a tile together (2 x 64 KB) for the Delta dot, and the epilogue reads its v_self row from global
// memory (prefetched ahead of the accumulator).  W_u is double-buffered (2 x 32 KB), so the next
// unit's operand loads while the current unit's tiles run.
template <bool DELTA>
struct Geo {
    static constexpr int kStages = DELTA ? 2 : 3;
    static constexpr int kStageBytes = DELTA ? 2 * kTile : kTile;
    static constexpr int kWOff = kStages * kStageBytes;
    static constexpr int kBarOff = kWOff + 2 * kTile;
    static constexpr int kDrOff = kBarOff + 256;  // float [stage][128 rows]: the Delta dot of each row
    static constexpr int kSmem = kDrOff + kStages * 128 * 4 + 1024;
    static_assert(kSmem <= 232448, "shared memory");
};

struct Bars {
    uint64_t q_full[3], q_ready[3], q_empty[3];
    uint64_t acc_full[2], acc_empty[2];
    uint64_t w_full[2], w_empty[2];
    uint32_t tmem_base;
};

struct Params {
    const int64_t* row_offsets;
    const int64_t* uts;           // tile starts of the rows' layout
    const uint8_t* w_op;          // [B*H][32 KB] W_u operands
    void* out;                    // [R, H, 128] bf16 or f32
    const int64_t* offsets;       // history offsets [B+1]: N_u for the Delta term's 1/N ...
    const int64_t* user_len;      // ... or N_u given directly ([B], may be NULL)
    const __nv_bfloat16* gate;    // [R, H, 128] or NULL: out = o (.) sigmoid(gate) (the summarizer's SGLU gate)
    const __nv_bfloat16* v_self;  // Delta: [R, H, 128], read by the epilogue
    int out_bf16;
    int normalize;
    int B, H;
};

template <int PHI>
__device__ __forceinline__ float phi(float x) {
    if constexpr (PHI == VISTA_ACT_SILU) {
        float t;
        asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
        return x * fmaf(0.5f, t, 0.5f);  // x sigma(x), sigma(x) = (1 + tanh(x/2)) / 2
    } else if constexpr (PHI == VISTA_ACT_SHIFTED_ELU) {
        return x >= 1.f ? x : ptx::ex2((x - 1.f) * 1.4426950408889634f);
    } else {
        return x;
    }
}

// phi on a packed bf16x2 pair -> packed bf16x2 (SiLU in packed bf16 math, one MUFU op per pair)
template <int PHI>
__device__ __forceinline__ uint32_t phi2x(uint32_t w) {
    if constexpr (PHI == VISTA_ACT_SILU) {
        return qla_silu_bf16x2(w);
    } else if constexpr (PHI == VISTA_ACT_SHIFTED_ELU) {
        return ptx::pack_bf16x2(phi<PHI>(__uint_as_float(w << 16)), phi<PHI>(__uint_as_float(w & 0xFFFF0000u)));
    } else {
        return w;
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
__device__ __forceinline__ void st_v8(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
// byte offset of 16-B chunk c (of 8) of row r in a 128-row, 128-B-row SWIZZLE_128B half tile
__device__ __forceinline__ uint32_t swz_chunk(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// phi1 in place over a q tile, one row per thread (16 chunks of 8 values); with DELTA also the row
// dot phi1(q_r) . phi1(k_self_r) from the k tile of the stage.  Returns the dot (0 without DELTA).
template <int PHI, bool DELTA>
__device__ __forceinline__ float xform_row(uint32_t qbuf, uint32_t kbuf, int r) {
    float dot = 0.f;
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll 4
        for (int c = 0; c < 8; ++c) {
            const uint32_t off = half * kHalf + swz_chunk(r, c);
            const uint4 raw = lds128(qbuf + off);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
            uint32_t ph[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) ph[e] = phi2x<PHI>(w[e]);
            sts128(qbuf + off, make_uint4(ph[0], ph[1], ph[2], ph[3]));
            if constexpr (DELTA) {
                const uint4 kr = lds128(kbuf + off);
                const uint32_t kw[4] = {kr.x, kr.y, kr.z, kr.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {  // the dot of the bf16 phi1 values (those the MMA sees), in f32
                    const uint32_t pk = phi2x<PHI>(kw[e]);
                    dot = fmaf(__uint_as_float(ph[e] << 16), __uint_as_float(pk << 16), dot);
                    dot = fmaf(__uint_as_float(ph[e] & 0xFFFF0000u), __uint_as_float(pk & 0xFFFF0000u), dot);
                }
            }
        }
    return dot;
}

// phi1(Q) in place without the Delta dot, 16-B chunk by chunk (the swizzle only permutes chunks
// within a row): consecutive threads take consecutive chunks
template <int PHI>
__device__ __forceinline__ void xform_tile(uint32_t qbuf, int xt) {
#pragma unroll 4
    for (int i = 0; i < (kTile / 16) / kXform; ++i) {
        const uint32_t off = (uint32_t)(xt + i * kXform) * 16;
        const uint4 raw = lds128(qbuf + off);
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
        uint32_t ph[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) ph[e] = phi2x<PHI>(w[e]);
        sts128(qbuf + off, make_uint4(ph[0], ph[1], ph[2], ph[3]));
    }
}

// O = phi1(Q) W: A = phi1(Q) [row][c1] K-major, B = W [K = c1][N = c2] MN-major
template <int SB, int ST, int WOFF>
__device__ __forceinline__ void issue_tile(uint32_t tacc, uint32_t base, uint32_t wsel) {
    const uint32_t qb = base + ST * SB, wb = base + WOFF + wsel;
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 1);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma_ss_w(tacc, ptx::sdesc_sw128(qb + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024),
                      ptx::sdesc_sw128(wb + kk * 2048, kHalf, 1024), id, kk > 0);
}

template <bool DELTA>
__device__ __forceinline__ void issue_tile_d(int stage, uint32_t tacc, uint32_t base, uint32_t wsel) {
    using G = Geo<DELTA>;
    switch (stage) {
        case 0: issue_tile<G::kStageBytes, 0, G::kWOff>(tacc, base, wsel); break;
        case 1: issue_tile<G::kStageBytes, 1 % G::kStages, G::kWOff>(tacc, base, wsel); break;
        default: issue_tile<G::kStageBytes, 2 % G::kStages, G::kWOff>(tacc, base, wsel); break;
    }
}

#ifdef VISTA_TRACE  // per CTA (globaltimer): start, after the PDL wait, first W ready, first tile's MMA
                    // issued, first tile stored, end
__device__ unsigned long long g_rows_cta[160][8];
__device__ __forceinline__ unsigned long long rows_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define RTRACE(slot, cond) \
    do { if ((cond) && blockIdx.x < 160) g_rows_cta[blockIdx.x][slot] = rows_gtime(); } while (0)
#else
#define RTRACE(slot, cond) do { } while (0)
#endif

template <int PHI1, bool DELTA>
__global__ void __launch_bounds__(kThreads, 1)
    sm100_qla_rows_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                          const Params P) {
    using G = Geo<DELTA>;
    constexpr int kStages = G::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t base = ptx::smem_u32(smem);
    Bars* bars = reinterpret_cast<Bars*>(smem + G::kBarOff);
    float* dr_smem = reinterpret_cast<float*>(smem + G::kDrOff);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cta = blockIdx.x, num_ctas = gridDim.x;
    const int HG = P.H;
    RTRACE(0, threadIdx.x == 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bars->q_full[s], 1);
            ptx::mbar_init(&bars->q_ready[s], kXform);
            // freed by the MMA commit (q consumed) and, with DELTA, by the epilogue (v_self consumed)
            ptx::mbar_init(&bars->q_empty[s], DELTA ? 1 + kEpi : 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->acc_full[b], 1);
            ptx::mbar_init(&bars->acc_empty[b], kEpi);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->w_full[b], 1);
            ptx::mbar_init(&bars->w_empty[b], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);
    // PDL: the prologue above overlapped the tile scan; its results (uts) and everything before it
    // on the stream are visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    RTRACE(1, threadIdx.x == 0);

    ItemIter iter;
    iter.init(P.uts, P.B, HG, cta, num_ctas, true);  // every role walks with full warps
    Item it;
    if (warp == 0) {
        // ---------------- TMA producer: q tiles (+ k_self, v_self tiles); W_u per unit
        ptx::tma_prefetch(&mapQ);
        if constexpr (DELTA) {
            ptx::tma_prefetch(&mapK);
        }
        const uint64_t pol = ptx::policy_evict_first();
        int stage = 0;
        uint32_t phase = 0;
        int k = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            // W buffer k % 2: free once unit k - 2's GEMMs are done with it
            if (k >= 2) ptx::mbar_wait(&bars->w_empty[k & 1], (uint32_t)((k >> 1) - 1) & 1u);
            ptx::mbar_arrive_expect_tx_w(&bars->w_full[k & 1], kTile);
            ptx::bulk_g2s_w(base + G::kWOff + (k & 1) * kTile, P.w_op + (size_t)(it.u * HG + it.hg) * kTile, kTile,
                            &bars->w_full[k & 1]);
            const int64_t row0 = P.row_offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->q_empty[stage], phase ^ 1);
                ptx::mbar_arrive_expect_tx_w(&bars->q_full[stage], G::kStageBytes);
                const int32_t row = (int32_t)(row0 + (int64_t)t * 128);
                uint8_t* st = smem + stage * G::kStageBytes;
                for (int half = 0; half < 2; ++half) {
                    ptx::tma_load_3d_w(st + half * kHalf, &mapQ, &bars->q_full[stage], half * 64, it.hg, row, pol);
                    if constexpr (DELTA)
                        ptx::tma_load_3d_w(st + kTile + half * kHalf, &mapK, &bars->q_full[stage], half * 64, it.hg,
                                           row, pol);
                }
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            ++k;
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        int stage = 0, ab = 0;
        uint32_t phase = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        int k = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            ptx::mbar_wait(&bars->w_full[k & 1], (uint32_t)(k >> 1) & 1u);
            RTRACE(2, k == 0 && lane == 0);
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->q_ready[stage], phase);
                RTRACE(3, k == 0 && t == it.t0 && lane == 0);
                ptx::mbar_wait(&bars->acc_empty[ab], ((aphm >> ab) & 1u) ^ 1);
                aphm ^= 1u << ab;
                ptx::tc_fence_after();
                const uint32_t tacc = tmem + ab * 128;
                issue_tile_d<DELTA>(stage, tacc, base, (k & 1) * kTile);
                ptx::mma_commit_w(&bars->acc_full[ab]);
                ptx::mma_commit_w(&bars->q_empty[stage]);
                ab ^= 1;
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            ptx::mma_commit_w(&bars->w_empty[k & 1]);
            ++k;
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- transform: phi1(Q) in place, one row per thread (+ the Delta dot)
        const int r = threadIdx.x - 128;
        int stage = 0;
        uint32_t phase = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            float inv_n = 1.f;  // App. B: the Delta term under the state's 1/N_u (reading R20)
            if (DELTA && P.normalize) {
                const int64_t N = P.user_len ? P.user_len[it.u] : P.offsets[it.u + 1] - P.offsets[it.u];
                if (N > 0) inv_n = 1.f / (float)N;
            }
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->q_full[stage], phase);
                RTRACE(6, threadIdx.x == 128 && t == it.t0 && stage == 0 && phase == 0);
                const uint32_t sb = base + stage * G::kStageBytes;
                if constexpr (DELTA) dr_smem[stage * 128 + r] = xform_row<PHI1, true>(sb, sb + kTile, r) * inv_n;
                else xform_tile<PHI1>(sb, r);
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&bars->q_ready[stage]);
                RTRACE(7, threadIdx.x == 128 && t == it.t0 && stage == 0 && phase == 0);
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp >= 8) {
        // ---------------- epilogue
        const int wq = warp % 4;
        const int chalf = (warp - 8) / 4;  // columns [64 chalf, 64 chalf + 64)
        const int row = wq * 32 + lane;    // row within the tile = TMEM lane
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const size_t rstride = (size_t)P.H * 128;  // elements between rows
#ifdef VISTA_TRACE
        bool g_first = true;
#endif
        int ab = 0, stage = 0;
        uint32_t aphm = 0;  // accumulator phases, bit b for buffer b (no local-memory array)
        uint32_t phase = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int64_t R = P.row_offsets[it.u + 1] - P.row_offsets[it.u];
            const int64_t row0 = P.row_offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                const int64_t rem = R - (int64_t)t * 128;
                const int valid = rem < 128 ? (int)rem : 128;
                const int64_t grow0 = row0 + (int64_t)t * 128;
                const size_t e0 = ((size_t)grow0 * P.H + it.hg) * 128;  // element (row 0, col 0) of the tile
                uint4 vrow[8];  // Delta: this thread's 64 v_self values, in flight while the GEMM runs
                if constexpr (DELTA) {
                    const int vr = row < valid ? row : valid - 1;
                    const uint4* vs = reinterpret_cast<const uint4*>(P.v_self + e0 + (size_t)vr * rstride + chalf * 64);
#pragma unroll
                    for (int c = 0; c < 8; ++c) vrow[c] = __ldg(vs + c);
                }
                ptx::mbar_wait(&bars->acc_full[ab], ((aphm >> ab) & 1u));
                aphm ^= 1u << ab;
                ptx::tc_fence_after();
                const uint32_t tc = tmem + lane_bits + ab * 128 + chalf * 64;
                float o[64];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t r[32];
                    ptx::tmem_ld32_sync(tc + c * 32, r);
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[32 * c + j] = __uint_as_float(r[j]);
                }
                if constexpr (DELTA) {  // + d_r v_self_r (d_r from shared memory, v_self prefetched)
                    ptx::mbar_wait(&bars->q_ready[stage], phase);  // orders the transform's d_r writes
                    const float dr = dr_smem[stage * 128 + row];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 b = vrow[c];
                        const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            o[8 * c + 2 * e] = fmaf(dr, __uint_as_float(bw[e] << 16), o[8 * c + 2 * e]);
                            o[8 * c + 2 * e + 1] = fmaf(dr, __uint_as_float(bw[e] & 0xFFFF0000u), o[8 * c + 2 * e + 1]);
                        }
                    }
                    ptx::mbar_arrive(&bars->q_empty[stage]);  // d_r read: the stage's transform may run again
                }
                if (P.gate && row < valid) {  // SGLU gate (reading R23): o (.) sigmoid(g), sigmoid via one tanh
                    const uint4* gs = reinterpret_cast<const uint4*>(P.gate + e0 + (size_t)row * rstride + chalf * 64);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 b = __ldg(gs + c);
                        const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float t0, t1;
                            asm("tanh.approx.f32 %0, %1;" : "=f"(t0) : "f"(0.5f * __uint_as_float(bw[e] << 16)));
                            asm("tanh.approx.f32 %0, %1;" : "=f"(t1) : "f"(0.5f * __uint_as_float(bw[e] & 0xFFFF0000u)));
                            o[8 * c + 2 * e] *= fmaf(0.5f, t0, 0.5f);
                            o[8 * c + 2 * e + 1] *= fmaf(0.5f, t1, 0.5f);
                        }
                    }
                }
                if (P.out_bf16) {
                    // coalesced: permuted 32x32b store into the (read) accumulator columns, 16x256b load
                    // back, so a quad of threads holds 128 contiguous bytes of one row
                    uint32_t a[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const int g = c >> 3, p = (c & 7) >> 1, e = c & 1;
                        const int j = 8 * p + 2 * g + e;  // packed word j = columns 2j, 2j+1
                        a[c] = ptx::pack_bf16x2(o[2 * j], o[2 * j + 1]);
                    }
                    ptx::tmem_st32(tc, a);
                    ptx::tmem_wait_st();
                    __nv_bfloat16* gbase = reinterpret_cast<__nv_bfloat16*>(P.out) + e0 + chalf * 64;
                    const int p = lane & 3;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        uint32_t r[16];
                        ptx::tmem_ld16x256b_x4(tc + ((uint32_t)(16 * half) << 16), r);
                        ptx::tmem_wait_ld();
                        ptx::reg_fence(r);
                        const int ra = wq * 32 + 16 * half + (lane >> 2);
                        const uint32_t v0[8] = {r[0], r[1], r[4], r[5], r[8], r[9], r[12], r[13]};
                        const uint32_t v1[8] = {r[2], r[3], r[6], r[7], r[10], r[11], r[14], r[15]};
                        if (ra < valid) st_v8(gbase + (size_t)ra * rstride + 16 * p, v0);
                        if (ra + 8 < valid) st_v8(gbase + (size_t)(ra + 8) * rstride + 16 * p, v1);
                    }
                } else if (row < valid) {
                    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(P.out) + e0 + (size_t)row * rstride +
                                                            chalf * 64);
#pragma unroll
                    for (int j = 0; j < 16; ++j) dst[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&bars->acc_empty[ab]);
                RTRACE(4, threadIdx.x == 256 && g_first);
#ifdef VISTA_TRACE
                g_first = false;
#endif
                ab ^= 1;
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    RTRACE(5, threadIdx.x == 0);
    if (warp == 1) ptx::tmem_dealloc(tmem, 256);
}

template <int PHI1, bool DELTA>
cudaError_t launch_phi(const Problem& p, const CUtensorMap& mq, const CUtensorMap& mk,
                       const Params& P) {
    using G = Geo<DELTA>;
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(sm100_qla_rows_kernel<PHI1, DELTA>), G::kSmem);
    if (attr != cudaSuccess) return attr;
    // PDL: the prologue overlaps the tile scan launched just before (griddepcontrol.wait in the kernel)
    return launch_pdl(sm100_qla_rows_kernel<PHI1, DELTA>, dim3(p.num_sms), dim3(kThreads), G::kSmem, p.stream, mq, mk, P);
}

// ---------------------------------------------------------------- SIMT: one block per (row, head)
template <typename T>
__device__ __forceinline__ float ldf(const T* p, size_t i);
template <>
__device__ __forceinline__ float ldf<float>(const float* p, size_t i) { return p[i]; }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p, size_t i) { return __bfloat162float(p[i]); }

template <typename T>
__global__ void qla_rows_simt_kernel(const float* __restrict__ z, const int64_t* __restrict__ offsets,
                                     const int64_t* __restrict__ user_len, const int64_t* __restrict__ row_offsets, int B, int H, int d, int phi1, int phi2,
                                     int normalize, const T* __restrict__ q, const T* __restrict__ k_self,
                                     const T* __restrict__ v_self, int out_bf16, void* __restrict__ out) {
    __shared__ float fq[128];
    __shared__ float red[4];
    const int64_t r = blockIdx.x / H;
    const int h = blockIdx.x % H, c = threadIdx.x;
    int lo = 0, hi = B;  // user u: row_offsets[u] <= r < row_offsets[u+1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (row_offsets[mid] <= r) lo = mid; else hi = mid;
    }
    const int u = lo;
    const size_t e0 = ((size_t)r * H + h) * d;
    const float fqc = c < d ? qla_act(phi1, ldf(q, e0 + c)) : 0.f;
    if (c < d) fq[c] = fqc;
    float dr = 0.f;
    if (k_self) {  // Delta: phi1(q_r) . phi1(k_self_r)
        float part = c < d ? fqc * qla_act(phi1, ldf(k_self, e0 + c)) : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (c % 32 == 0) red[c / 32] = part;
    }
    __syncthreads();
    if (k_self)
        for (int w = 0; w < (d + 31) / 32; ++w) dr += red[w];
    if (c >= d) return;
    const int64_t N = user_len ? user_len[u] : offsets[u + 1] - offsets[u];
    const float inv = (normalize && N > 0) ? 1.f / (float)N : 1.f;
    dr *= inv;  // App. B: the Delta term under the same 1/N_u (reading R20)
    const float* zu = z + (size_t)(u * H + h) * d * d;
    float acc = 0.f;
    for (int c1 = 0; c1 < d; ++c1) acc = fmaf(fq[c1], qla_act(phi2, zu[(size_t)c1 * d + c] * inv), acc);
    if (k_self) acc = fmaf(dr, ldf(v_self, e0 + c), acc);
    if (out_bf16) reinterpret_cast<__nv_bfloat16*>(out)[e0 + c] = __float2bfloat16_rn(acc);
    else reinterpret_cast<float*>(out)[e0 + c] = acc;
}

}  // namespace

bool qla_rows_uses_tc(const Problem& p, int64_t total_rows) {
    return p.in_bf16 && p.d == 128 && p.total_len < (int64_t(1) << 31) && total_rows < (int64_t(1) << 31);
}

// p: the history problem (B, H, d, phi, normalize, stream); uts: tile starts of the rows' layout;
// w_op: the W_u operands (qla_prep_w); user_len: N_u per user (NULL: from p.offsets)
cudaError_t launch_sm100_qla_rows(const Problem& p, const int64_t* row_offsets, int64_t total_rows, const int64_t* uts,
                                  const uint8_t* w_op, const void* q, const void* k_self, const void* v_self,
                                  int out_bf16, void* out, const int64_t* user_len, const void* gate) {
    CUtensorMap mq, mk;  // (v_self rows are read by the epilogue threads directly)
    if (!make_kv_map(&mq, q, total_rows, p.H)) return cudaErrorInvalidValue;
    const bool delta = k_self != nullptr;
    if (delta && !make_kv_map(&mk, k_self, total_rows, p.H)) return cudaErrorInvalidValue;
    if (!delta) mk = mq;
    Params P;
    P.row_offsets = row_offsets;
    P.uts = uts;
    P.w_op = w_op;
    P.out = out;
    P.offsets = p.offsets;
    P.user_len = user_len;
    P.gate = reinterpret_cast<const __nv_bfloat16*>(gate);
    P.v_self = reinterpret_cast<const __nv_bfloat16*>(v_self);
    P.normalize = p.normalize;
    P.out_bf16 = out_bf16;
    P.B = p.B;
    P.H = p.H;
    if (delta)
        return p.phi1 == VISTA_ACT_SILU ? launch_phi<VISTA_ACT_SILU, true>(p, mq, mk, P)
             : p.phi1 == VISTA_ACT_SHIFTED_ELU ? launch_phi<VISTA_ACT_SHIFTED_ELU, true>(p, mq, mk, P)
                                               : launch_phi<VISTA_ACT_IDENTITY, true>(p, mq, mk, P);
    return p.phi1 == VISTA_ACT_SILU ? launch_phi<VISTA_ACT_SILU, false>(p, mq, mk, P)
         : p.phi1 == VISTA_ACT_SHIFTED_ELU ? launch_phi<VISTA_ACT_SHIFTED_ELU, false>(p, mq, mk, P)
                                           : launch_phi<VISTA_ACT_IDENTITY, false>(p, mq, mk, P);
}

cudaError_t launch_qla_rows_simt(const Problem& p, const float* z, const int64_t* row_offsets, int64_t total_rows,
                                 const void* q, const void* k_self, const void* v_self, int out_bf16, void* out,
                                 const int64_t* user_len) {
    if (total_rows == 0) return cudaSuccess;
    const unsigned grid = (unsigned)(total_rows * p.H);
    const int threads = p.d < 32 ? 32 : p.d;
    if (p.in_bf16)
        qla_rows_simt_kernel<__nv_bfloat16><<<grid, threads, 0, p.stream>>>(
            z, p.offsets, user_len, row_offsets, p.B, p.H, p.d, p.phi1, p.phi2, p.normalize,
            reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k_self),
            reinterpret_cast<const __nv_bfloat16*>(v_self), out_bf16, out);
    else
        qla_rows_simt_kernel<float><<<grid, threads, 0, p.stream>>>(
            z, p.offsets, user_len, row_offsets, p.B, p.H, p.d, p.phi1, p.phi2, p.normalize, reinterpret_cast<const float*>(q),
            reinterpret_cast<const float*>(k_self), reinterpret_cast<const float*>(v_self), out_bf16, out);
    return cudaGetLastError();
}

}  // namespace vista

#ifdef VISTA_TRACE
extern "C" int vista_debug_rows_cta(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, vista::g_rows_cta, bytes < sizeof(vista::g_rows_cta) ? bytes : sizeof(vista::g_rows_cta));
}
#endif

