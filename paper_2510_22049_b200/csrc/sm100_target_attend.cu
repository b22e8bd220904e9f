// sm100_target_attend.cu -- stage-2 target-aware attention over the cached summary tokens (NEXT-4).
//
// "any attention network can technically be used for the target-aware attention stage ... we selected
// a standard O(N^2) transformer block, which delivers excellent performance on the compact summary
// sequences" (Sec. 3.3).  The stage-1 summary tokens are "retrieved from the cache
// and dequantized": this kernel reads the int8 export of vista_summarize_fwd_int8
// directly and dequantizes it in the load path.  Reading R22: candidate c of user u
// attends to [the S tokens of u; itself] and never to another candidate:
//   t_i = code * scale + zp,  s_i = scale q_c . t_i,  s_self = scale q_c . k_c
//   out_c = (sum_i e^{s_i} t_i + e^{s_self} v_c) / (sum_i e^{s_i} + e^{s_self})  [+ resid_c]
//
// sm100_target_attend_kernel (bf16, d = 128, S in {128, 256}): persistent, stream-K over the flat
// 128-candidate tiles of the candidates' jagged layout (work.cuh).  Per item (user, head) the S x 128
// tokens are dequantized once into shared memory (bf16, 128-B swizzle) and serve as the B operand of
// both GEMMs: K-major for S = Q T^T, MN-major for O = P T.  TMEM: S [0, S), P (bf16) [256, 256 + S/2),
// O [384, 512) -- P has its own columns, so the score GEMM of tile t + 1 runs while the softmax of
// tile t is still exponentiating.  Warp roles:
//   warp 0       TMA: q and k_self tiles (2-stage ring)
//   warp 1       score GEMMs S(t) = Q_t T^T (as N = 128 halves), as soon as the softmax has read S(t-1)
//   warp 3       PV GEMM O(t) = P(t) T once P(t) is written and the epilogue has read O(t - 1)
//   warps 4-11   softmax, two threads per candidate row (tokens [0, S/2) / [S/2, S), the 16x32bx2
//                TMEM shape): the self logit q_c . k_c from the staged tiles, a two-pass softmax over
//                [tokens; self] (1 of every 4 exponential pairs on the FMA pipe); also dequantize each
//                item's tokens once its predecessor's last PV is done (int8 -> f32 by PRMT + FADD2, no
//                I2F) and pull the next item's codes into L2
//   warps 12-15  epilogue, one thread per row: (O + p_self v_c) / l [+ resid] -> bf16 / f32 rows, lse;
//                v_c in and the bf16 row out by per-row 256-B bulk copies through a staging tile
//                (272-B row stride: bank-conflict free; the row pad carries 1/l, p_self/l, lse);
//                O released after its last TMEM load
// Registers (setmaxnreg): control warps 64, softmax 144, epilogue 160 -- the epilogue has its own role
// branch so the iterator state stays in registers.
// (Measured slower and not kept: staging the jagged tables in shared memory, 0.0370 vs 0.0354 ms at
// c2; one 2-D TMA load / store of the whole staging tile instead of per-row bulk copies, 0.0328 vs
// 0.0316 ms.)
// simt_target_attend_kernel: CUDA cores, one warp per (candidate, head), any S >= 1, d <= 128, f32 or
// bf16 -- the shapes the tcgen05 kernel does not take.
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>

#include "internal.h"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

bool make_kv_map(CUtensorMap* map, const void* base, int64_t total_len, int H);

#ifdef VISTA_TRACE  // debug timeline of CTA 0: clock64 per (event, tile)
__device__ unsigned long long g_ta_trace[16][64];
__device__ unsigned long long g_ta_cta[160][3];  // per CTA: globaltimer at start, after the PDL wait, at the end
#define TTRACE(ev, g) \
    do { if (blockIdx.x == 0 && (g) < 64) g_ta_trace[ev][g] = clock64(); } while (0)
__device__ __forceinline__ unsigned long long ta_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define CTRACE(slot) \
    do { if (threadIdx.x == 0 && blockIdx.x < 160) g_ta_cta[blockIdx.x][slot] = ta_gtime(); } while (0)
#else
#define TTRACE(ev, g) do { } while (0)
#define CTRACE(slot) do { } while (0)
#endif

namespace {

constexpr int kHalf = 128 * 128;  // one 64-column half of a 128-row bf16 tile
constexpr int kTileB = 2 * kHalf;  // 32 KB
constexpr int kThreads = 512;
#ifndef VISTA_TA_EMU  // pairs out of every 4 whose exponentials run on the FMA pipe (A/B: 1 beats 0 and 2)
#define VISTA_TA_EMU 1
#endif
constexpr int kTaEmu = VISTA_TA_EMU;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
// smem: tokens T (S x 128 bf16, two 64-column halves; 64 KB at S = 256), a 2-stage ring of (q, k_self)
// tiles (128 KB), barriers and the per-row statistics
constexpr int kTOff = 0;
constexpr int kQKOff = 2 * kTileB;  // stage s: q at kQKOff + 2 s kTileB, k_self at + kTileB
// output staging (epilogue): 128 rows of 256 B (v_c in by bulk copy, the bf16 result out by bulk
// copy, one row per epilogue thread), row stride 272 B so that 8 lanes reading / writing the same
// 16-B chunk of their rows hit distinct banks; the 16-B pad of row r holds the softmax's
// (1 / l, p_self / l, lse) of row r
constexpr int kStgStride = 272;
constexpr int kStgOff = kQKOff + 4 * kTileB;
constexpr int kBarOff = kStgOff + 128 * kStgStride;

struct TABars {
    uint64_t qk_full[2], qk_empty[2];
    uint64_t t_full, t_free;    // the item's tokens in smem / its last PV done (T reusable)
    uint64_t s_full, s_free;    // S(t) computed / read by the softmax
    uint64_t p_full, p_free;    // P(t) written / read by PV(t)
    uint64_t o_full, o_empty;   // O(t) computed / read by the epilogue
    uint64_t ml_full, ml_empty;  // the row statistics of tile t, softmax -> epilogue
    uint64_t v_full;             // the tile's v_c rows in the staging rows (bulk copies)
    uint32_t tmem_base, pad;
};
// no alignment slack: the dynamic shared memory is declared 1024-B aligned (checked at run time)
constexpr int kSmem = kBarOff + (int)sizeof(TABars);
static_assert(kSmem <= 232448, "shared memory");

struct TAParams {
    const int64_t* row_offsets;
    const int64_t* uts;
    const int8_t* codes;  // [B, S, H, 128]
    const float* tscale;  // [B, S, H]
    const float* tzp;
    const void* v;      // v_self [R, H, 128] bf16
    const void* resid;  // [R, H, 128] (in dtype bf16) or NULL
    void* out;          // [R, H, 128]
    float* lse;         // [R, H] or NULL
    int B, S, H, out_bf16;
    float scale_log2;
};

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// 16-B chunk c (of 8) of row r in a SWIZZLE_128B half tile of 128-B rows
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

template <int NS>  // N = S tokens, issued as N = 128 halves (the B operand T is one 128-B swizzle column wide)
__device__ __forceinline__ void issue_scores(uint32_t tS, uint32_t sQ, uint32_t sT) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 0);  // Q, T both K-major
    constexpr int halfT = NS * 128;
#pragma unroll
    for (int n = 0; n < NS / 128; ++n)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
            ptx::mma_ss_w(tS + n * 128, ptx::sdesc_sw128(sQ + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024),
                          ptx::sdesc_sw128(sT + (kk >> 2) * halfT + n * 128 * 128 + (kk & 3) * 32, 16, 1024), id,
                          kk > 0);
}
template <int NS>
__device__ __forceinline__ void issue_pv(uint32_t tO, uint32_t tP, uint32_t sT) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, 128, 0, 1);  // P (TMEM, 8 columns per 16 tokens) x T (MN-major)
    constexpr int halfT = NS * 128;
#pragma unroll
    for (int kk = 0; kk < NS / 16; ++kk)
        ptx::mma_ts_w(tO, tP + kk * 8, ptx::sdesc_sw128(sT + kk * 2048, halfT, 1024), id, kk > 0);
}

template <int NS>
__global__ void __launch_bounds__(kThreads, 1)
    sm100_target_attend_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                               const TAParams P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if (ptx::smem_u32(smem) & 1023u) __trap();  // the SWIZZLE_128B operand tiles need 1024-B alignment
    const uint32_t base = ptx::smem_u32(smem);
    TABars* bars = reinterpret_cast<TABars*>(smem + kBarOff);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) TTRACE(14, 0);
    CTRACE(0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&bars->qk_full[s], 1);
            ptx::mbar_init(&bars->qk_empty[s], 256);  // the softmax threads: self dot done, S(t) done
        }
        ptx::mbar_init(&bars->t_full, 256);  // warps 4-11 dequantized their share
        ptx::mbar_init(&bars->t_free, 1);
        ptx::mbar_init(&bars->s_full, 1);
        ptx::mbar_init(&bars->s_free, 256);
        ptx::mbar_init(&bars->p_full, 256);
        ptx::mbar_init(&bars->p_free, 1);
        ptx::mbar_init(&bars->o_full, 1);
        ptx::mbar_init(&bars->o_empty, 128);
        ptx::mbar_init(&bars->ml_full, 256);
        ptx::mbar_init(&bars->ml_empty, 128);
        ptx::mbar_init(&bars->v_full, 128);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    // PDL: the prologue above overlapped the tile scan; its results (uts) and everything before it
    // on the stream are visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    CTRACE(1);
    const uint32_t tmem = bars->tmem_base;
    const int64_t* uts = P.uts;
    const int64_t* roff = P.row_offsets;
    const uint32_t tS = tmem, tP = tmem + 256, tO = tmem + 384;
    const int H = P.H;
    // registers: the control warpgroup (warps 0-3) gives 64 per thread back; the epilogue warpgroup
    // (v_c rows prefetched: 64 registers live across its waits) takes 32 and the two softmax
    // warpgroups (the dequantization's loads in flight) 16 each
    if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    ItemIter iter;
    iter.init(uts, P.B, H, blockIdx.x, gridDim.x, true);  // every role walks with full warps
    Item it;
    if (warp == 0) {
        // ============================ TMA producer ============================
        const uint64_t pol = ptx::policy_evict_first();
        int g = 0;
        while (iter.next(it, uts, P.B, H)) {
            const int h = it.hg;
            for (int t = it.t0; t < it.t1; ++t, ++g) {
                const int32_t row0 = (int32_t)(roff[it.u] + (int64_t)t * 128);
                const int st = g & 1;
                if (g >= 2) ptx::mbar_wait(&bars->qk_empty[st], (uint32_t)((g >> 1) - 1) & 1u);
                if (lane == 0) TTRACE(0, g);
                ptx::mbar_arrive_expect_tx_w(&bars->qk_full[st], 2 * kTileB);
                uint8_t* sq = smem + kQKOff + st * 2 * kTileB;
                for (int half = 0; half < 2; ++half) {
                    ptx::tma_load_3d_w(sq + half * kHalf, &mapQ, &bars->qk_full[st], half * 64, h, row0, pol);
                    ptx::tma_load_3d_w(sq + kTileB + half * kHalf, &mapK, &bars->qk_full[st], half * 64, h, row0, pol);
                }
            }
        }
    } else if (warp == 1) {
        // ============================ score GEMMs ============================
        int g = 0;
        for (int k = 0; iter.next(it, uts, P.B, H); ++k) {
            ptx::mbar_wait(&bars->t_full, (uint32_t)k & 1u);
            for (int t = it.t0; t < it.t1; ++t, ++g) {
                const int st = g & 1;
                ptx::mbar_wait(&bars->qk_full[st], (uint32_t)(g >> 1) & 1u);
                if (lane == 0) TTRACE(1, g);
                if (g >= 1) ptx::mbar_wait(&bars->s_free, (uint32_t)(g - 1) & 1u);  // the softmax read S(g - 1)
                ptx::tc_fence_after();
                issue_scores<NS>(tS, base + kQKOff + st * 2 * kTileB, base + kTOff);
                ptx::mma_commit_w(&bars->s_full);
                if (lane == 0) TTRACE(2, g);
            }
        }
    } else if (warp == 3) {
        // ============================ PV GEMMs ============================
        int g = 0;
        for (int k = 0; iter.next(it, uts, P.B, H); ++k) {
            for (int t = it.t0; t < it.t1; ++t, ++g) {
                ptx::mbar_wait(&bars->p_full, (uint32_t)g & 1u);
                if (lane == 0) TTRACE(3, g);
                if (g >= 1) ptx::mbar_wait(&bars->o_empty, (uint32_t)(g - 1) & 1u);  // epilogue read O(g - 1)
                ptx::tc_fence_after();
                issue_pv<NS>(tO, tP, base + kTOff);
                ptx::mma_commit_w(&bars->o_full);
                ptx::mma_commit_w(&bars->p_free);
                if (t == it.t1 - 1) ptx::mma_commit_w(&bars->t_free);
                if (lane == 0) TTRACE(4, g);
            }
        }
    } else if (warp >= 12) {
        // ============ epilogue: (O + p_self v_c) / l [+ resid], one thread per row ============
        asm volatile("setmaxnreg.inc.sync.aligned.u32 160;");
        const int wq = warp & 3;
        const int row = wq * 32 + lane;  // candidate row = TMEM lane
        const uint32_t lb = (uint32_t)(wq * 32) << 16;
        const size_t rstride = (size_t)H * 128;
        int g = 0;
        for (int k = 0; iter.next(it, uts, P.B, H); ++k) {
            const int u = it.u, h = it.hg;
            const int64_t R = roff[u + 1] - roff[u];
            for (int t = it.t0; t < it.t1; ++t, ++g) {
                    // ============ epilogue: (O + p_self v_c) / l [+ resid] ============
                    const int64_t row0 = roff[u] + (int64_t)t * 128;
                    const int64_t remr = R - (int64_t)t * 128;
                    const int valid = remr < 128 ? (int)remr : 128;
                    // v_c of this thread's row -> its staging row (bulk copy, in flight while the softmax
                    // and the PV GEMM run), once this thread's previous bulk store has read the row.
                    // (One 2-D TMA load / store per tile instead was measured slower: 0.0328 vs 0.0316 ms
                    // at c2 -- the whole tile waits for its slowest row.)
                    const uint32_t srow = base + kStgOff + row * kStgStride;
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    if (row < valid) {
                        ptx::mbar_arrive_expect_tx(&bars->v_full, 256);
                        ptx::bulk_g2s(srow, reinterpret_cast<const __nv_bfloat16*>(P.v) + (size_t)(row0 + row) * rstride +
                                                (size_t)h * 128,
                                      256, &bars->v_full);
                    } else {
                        ptx::mbar_arrive(&bars->v_full);
                    }
                    ptx::mbar_wait(&bars->ml_full, (uint32_t)g & 1u);
                    if (threadIdx.x == 384) TTRACE(9, g);
                    const float* pad = reinterpret_cast<const float*>(smem + kStgOff + row * kStgStride + 256);
                    const float inv = pad[0], wself = pad[1], lse = pad[2];
                    ptx::mbar_arrive(&bars->ml_empty);
                    ptx::mbar_wait(&bars->o_full, (uint32_t)g & 1u);
                    if (threadIdx.x == 384) TTRACE(10, g);
                    ptx::tc_fence_after();
                    ptx::mbar_wait(&bars->v_full, (uint32_t)g & 1u);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {  // 32 channels at a time
                        uint32_t r[32];
                        ptx::tmem_ld32_sync(tO + lb + q4 * 32, r);
                        if (q4 == 3) {  // O fully read: PV(g + 1) may overwrite it
                            ptx::tc_fence_before();
                            ptx::mbar_arrive(&bars->o_empty);
                        }
                        float o[32];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint4 va = lds128(srow + q4 * 64 + c * 16);
                            const uint32_t vw[4] = {va.x, va.y, va.z, va.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                o[8 * c + 2 * e] = fmaf(wself, __uint_as_float(vw[e] << 16),
                                                        __uint_as_float(r[8 * c + 2 * e]) * inv);
                                o[8 * c + 2 * e + 1] = fmaf(wself, __uint_as_float(vw[e] & 0xFFFF0000u),
                                                            __uint_as_float(r[8 * c + 2 * e + 1]) * inv);
                            }
                        }
                        const size_t eo = (size_t)(row0 + row) * rstride + (size_t)h * 128 + q4 * 32;
                        if (P.resid && row < valid) {
                            const uint4* rs = reinterpret_cast<const uint4*>(
                                reinterpret_cast<const __nv_bfloat16*>(P.resid) + eo);
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint4 ra = __ldg(rs + c);
                                const uint32_t rw[4] = {ra.x, ra.y, ra.z, ra.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    o[8 * c + 2 * e] += __uint_as_float(rw[e] << 16);
                                    o[8 * c + 2 * e + 1] += __uint_as_float(rw[e] & 0xFFFF0000u);
                                }
                            }
                        }
                        if (P.out_bf16) {  // back into the staging row (v_c of these channels is read)
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                sts128(srow + q4 * 64 + c * 16,
                                       make_uint4(ptx::pack_bf16x2(o[8 * c], o[8 * c + 1]),
                                                  ptx::pack_bf16x2(o[8 * c + 2], o[8 * c + 3]),
                                                  ptx::pack_bf16x2(o[8 * c + 4], o[8 * c + 5]),
                                                  ptx::pack_bf16x2(o[8 * c + 6], o[8 * c + 7])));
                        } else if (row < valid) {
                            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(P.out) + eo);
#pragma unroll
                            for (int c = 0; c < 8; ++c)
                                dst[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
                        }
                    }
                    if (P.out_bf16 && row < valid) {  // the row's 256 B to global in one bulk copy
                        ptx::fence_proxy_async_smem();
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;\n\t"
                                     "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<__nv_bfloat16*>(P.out) +
                                                                          (size_t)(row0 + row) * rstride + (size_t)h * 128),
                                     "r"(srow)
                                     : "memory");
                    }
                    if (P.lse && row < valid) P.lse[(size_t)(row0 + row) * H + h] = lse;
                    if (threadIdx.x == 384) TTRACE(11, g);
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // this thread's bulk stores are complete
    } else if (warp >= 4) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 144;");
        // softmax: lane quarter wq, row half rh, token half ch
        const int wq = warp & 3, rh = (warp - 4) >> 2, ch = lane >> 4;
        const int row = wq * 32 + rh * 16 + (lane & 15);  // candidate row = TMEM lane
        const uint32_t lb = (uint32_t)(wq * 32 + rh * 16) << 16;
        int g = 0;
        for (int k = 0; iter.next(it, uts, P.B, H); ++k) {
            const int u = it.u, h = it.hg;
            // ---- the item's tokens: int8 codes * scale + zero point -> bf16, swizzled, both halves
            //      (the softmax warps 4-11)
            if (threadIdx.x == 128) TTRACE(12, k);
            {
                // every thread's NS / 32 chunks: all loads first (in flight together), then convert
                constexpr int kPer = NS * 8 / 256;
                uint4 raw[kPer];
                float a[kPer], b[kPer];
#pragma unroll
                for (int n = 0; n < kPer; ++n) {
                    const int x = threadIdx.x - 128 + 256 * n;  // x = (token i, 16-B chunk cc of its codes)
                    const size_t tix = ((size_t)u * NS + (x >> 3)) * H + h;
                    raw[n] = __ldg(reinterpret_cast<const uint4*>(P.codes + tix * 128) + (x & 7));
                    a[n] = __ldg(P.tscale + tix);
                    b[n] = __ldg(P.tzp + tix);
                }
#ifdef VISTA_TRACE
                if (threadIdx.x == 128 && blockIdx.x == 0 && k < 32) {  // when this thread's loads landed
                    uint32_t acc = 0;
#pragma unroll
                    for (int n = 0; n < kPer; ++n) acc ^= raw[n].x ^ raw[n].w ^ __float_as_uint(a[n] + b[n]);
                    unsigned long long tt;
                    asm volatile("mov.u64 %0, %%clock64; // %1" : "=l"(tt) : "r"(acc));
                    g_ta_trace[13][32 + k] = tt;
                }
#endif
                // the loads overlap the previous item's last PV; T is rewritten only after it
                if (k >= 1) ptx::mbar_wait(&bars->t_free, (uint32_t)(k - 1) & 1u);
#pragma unroll
                for (int n = 0; n < kPer; ++n) {
                    const int x = threadIdx.x - 128 + 256 * n;
                    const int i = x >> 3, cc = x & 7;  // codes [16 cc, 16 cc + 16) of token i
                    const uint32_t w[4] = {raw[n].x, raw[n].y, raw[n].z, raw[n].w};
                    uint32_t o[8];
                    // int8 -> f32 without I2F: byte c ^ 0x80 = c + 128 placed in the mantissa of 2^23
                    // (PRMT), then (2^23 + c + 128) - (2^23 + 128) = c exactly (FADD2); t = c scale + zp (FFMA2)
                    const uint64_t a2 = ptx::f2_pack(a[n], a[n]), b2 = ptx::f2_pack(b[n], b[n]);
                    const uint64_t off2 = ptx::f2_pack(-8388736.f, -8388736.f);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t x = w[e] ^ 0x80808080u;
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const float f0 = __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7440u + 2 * hh));
                            const float f1 = __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7441u + 2 * hh));
                            float t0, t1;
                            ptx::f2_unpack(ptx::f2_fma(ptx::f2_add(ptx::f2_pack(f0, f1), off2), a2, b2), t0, t1);
                            o[2 * e + hh] = ptx::pack_bf16x2(t0, t1);
                        }
                    }
                    // channels 16 cc .. 16 cc + 15 = 16-B bf16 chunks 2 cc, 2 cc + 1 of the row (half = cc / 4)
                    const uint32_t hb = base + kTOff + (cc >> 2) * (NS * 128);
                    const int c0 = (2 * cc) & 7;
                    sts128(hb + swz(i, c0), make_uint4(o[0], o[1], o[2], o[3]));
                    sts128(hb + swz(i, c0 + 1), make_uint4(o[4], o[5], o[6], o[7]));
                }
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&bars->t_full);
                // the next item of this CTA (if any): walk a copy of the iterator now, while the tiles
                // run, and pull that item's codes and scale / zero-point lines into L2 (its dequant
                // then waits on L2, not HBM; the walk's uts loads are cached for the real next())
                ItemIter la = iter;
                Item nx;
                if (la.next(nx, uts, P.B, H)) {
                    const int tl = threadIdx.x - 128;  // 0..255: token tl's 128-B code line
                    if (tl < NS) {
                        const size_t tix = ((size_t)nx.u * NS + tl) * H + nx.hg;
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.codes + tix * 128));
                        if ((tl & 7) == 0) {  // scale / zp: 8 tokens per 128-B line at H = 4
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(P.tscale + tix));
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(P.tzp + tix));
                        }
                    }
                }
            }
            if (threadIdx.x == 128) TTRACE(13, k);
            for (int t = it.t0; t < it.t1; ++t, ++g) {
                const int st = g & 1;
                    // ============ softmax over [tokens; self], two threads per candidate row ============
                    ptx::mbar_wait(&bars->qk_full[st], (uint32_t)(g >> 1) & 1u);
                    if (threadIdx.x == 128) TTRACE(5, g);
                    const uint32_t sq = base + kQKOff + st * 2 * kTileB;
                    float self = 0.f;  // q_c . k_c from the staged tiles: this thread's 64 channels
#pragma unroll 4
                    for (int c = 0; c < 8; ++c) {
                        const uint4 qa = lds128(sq + ch * kHalf + swz(row, c));
                        const uint4 ka = lds128(sq + kTileB + ch * kHalf + swz(row, c));
                        const uint32_t qw[4] = {qa.x, qa.y, qa.z, qa.w}, kw[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            self = fmaf(__uint_as_float(qw[e] << 16), __uint_as_float(kw[e] << 16), self);
                            self = fmaf(__uint_as_float(qw[e] & 0xFFFF0000u), __uint_as_float(kw[e] & 0xFFFF0000u),
                                        self);
                        }
                    }
                    self += __shfl_xor_sync(0xffffffffu, self, 16);
                    self *= P.scale_log2;
                    ptx::mbar_wait(&bars->s_full, (uint32_t)g & 1u);
                    if (threadIdx.x == 128) TTRACE(6, g);
                    ptx::mbar_arrive(&bars->qk_empty[st]);  // q (S done) and k (dot done) of this stage read
                    ptx::tc_fence_after();
                    // this thread: tokens [ch NS/2, ch NS/2 + NS/2) = S columns of the same range
                    float m = self;
#pragma unroll 1
                    for (int c = 0; c < NS / 2; c += 32) {
                        uint32_t r[32];
                        ptx::tmem_ld16x32bx2_x32<NS / 2>(tS + lb + c, r);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 32; ++j) m = fmaxf(m, __uint_as_float(r[j]) * P.scale_log2);
                    }
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
                    if (threadIdx.x == 128) TTRACE(7, g);
                    // P(g) has its own columns: free once PV(g - 1) has read them
                    if (g >= 1) ptx::mbar_wait(&bars->p_free, (uint32_t)(g - 1) & 1u);
                    ptx::tc_fence_after();
                    float l = 0.f;
#pragma unroll 1
                    for (int c = 0; c < NS / 2; c += 32) {
                        uint32_t r[32], pk[16];
                        ptx::tmem_ld16x32bx2_x32<NS / 2>(tS + lb + c, r);
                        ptx::tmem_wait_ld();
                        if (c == NS / 2 - 32) {  // last S chunk of this thread loaded: S(g + 1) may overwrite S
                            ptx::tc_fence_before();
                            ptx::mbar_arrive(&bars->s_free);
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            float p0, p1;
                            if ((j & 3) < kTaEmu) {  // this pair on the FMA pipe (no masked tokens here)
                                const uint64_t x2 = ptx::f2_fma(ptx::f2_pack(__uint_as_float(r[2 * j]),
                                                                             __uint_as_float(r[2 * j + 1])),
                                                                ptx::f2_pack(P.scale_log2, P.scale_log2),
                                                                ptx::f2_pack(-m, -m));
                                ptx::f2_unpack(ptx::exp2_emu2(x2), p0, p1);
                            } else {
                                p0 = ptx::ex2(fmaf(__uint_as_float(r[2 * j]), P.scale_log2, -m));
                                p1 = ptx::ex2(fmaf(__uint_as_float(r[2 * j + 1]), P.scale_log2, -m));
                            }
                            l += p0 + p1;
                            pk[j] = ptx::pack_bf16x2(p0, p1);
                        }
                        // P of these 32 tokens: 16 columns (2 tokens per column), token order
                        ptx::tmem_st16x32bx2_x16<NS / 4>(tP + lb + c / 2, pk);
                    }
                    l += __shfl_xor_sync(0xffffffffu, l, 16);
                    const float pself = ptx::ex2(self - m);
                    l += pself;
                    const float inv = 1.f / l;
                    if (g >= 1) ptx::mbar_wait(&bars->ml_empty, (uint32_t)(g - 1) & 1u);
                    if (ch == 0) {
                        float* pad = reinterpret_cast<float*>(smem + kStgOff + row * kStgStride + 256);
                        pad[0] = inv;
                        pad[1] = pself * inv;
                        pad[2] = (m + __log2f(l)) * kLn2;
                    }
                    ptx::mbar_arrive(&bars->ml_full);
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&bars->p_full);
                    if (threadIdx.x == 128) TTRACE(8, g);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TTRACE(15, 0);
    CTRACE(2);
    if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- SIMT: one warp per (candidate, head)
template <typename T>
__device__ __forceinline__ float ldv(const T* p, size_t i);
template <>
__device__ __forceinline__ float ldv<float>(const float* p, size_t i) { return p[i]; }
template <>
__device__ __forceinline__ float ldv<__nv_bfloat16>(const __nv_bfloat16* p, size_t i) { return __bfloat162float(p[i]); }

template <typename T>
__global__ void simt_target_attend_kernel(const int64_t* __restrict__ row_offsets, const int8_t* __restrict__ codes,
                                          const float* __restrict__ tscale, const float* __restrict__ tzp,
                                          const T* __restrict__ q, const T* __restrict__ k_self,
                                          const T* __restrict__ v_self, const T* __restrict__ resid, int B, int S,
                                          int H, int d, float scale, int out_bf16, void* __restrict__ out,
                                          float* __restrict__ lse, int64_t total) {
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (gw >= total * H) return;
    const int lane = threadIdx.x % 32;
    const int64_t c = gw / H;
    const int h = (int)(gw % H);
    int lo = 0, hi = B;  // user u: row_offsets[u] <= c < row_offsets[u+1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (row_offsets[mid] <= c) lo = mid; else hi = mid;
    }
    const int u = lo;
    const size_t e0 = ((size_t)c * H + h) * d;
    float qv[4], acc[4], vv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = lane + 32 * j;
        qv[j] = e < d ? ldv(q, e0 + e) : 0.f;
        acc[j] = 0.f;
    }
    // self logit first, then the tokens, online softmax (natural-log domain, f32)
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = lane + 32 * j;
        if (e < d) s = fmaf(qv[j], ldv(k_self, e0 + e), s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    float m = s * scale, l = 1.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = lane + 32 * j;
        acc[j] = e < d ? ldv(v_self, e0 + e) : 0.f;
    }
    for (int i = 0; i < S; ++i) {
        const size_t tix = ((size_t)u * S + i) * H + h;
        const float a = tscale[tix], b = tzp[tix];
        float dot = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int e = lane + 32 * j;
            vv[j] = e < d ? fmaf((float)codes[tix * d + e], a, b) : 0.f;
            dot = fmaf(qv[j], vv[j], dot);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const float x = dot * scale;
        const float mn = fmaxf(m, x);
        const float f = __expf(m - mn), p = __expf(x - mn);
        l = l * f + p;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = fmaf(acc[j], f, p * vv[j]);
        m = mn;
    }
    const float inv = 1.f / l;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = lane + 32 * j;
        if (e >= d) continue;
        float y = acc[j] * inv;
        if (resid) y += ldv(resid, e0 + e);
        if (out_bf16) reinterpret_cast<__nv_bfloat16*>(out)[e0 + e] = __float2bfloat16_rn(y);
        else reinterpret_cast<float*>(out)[e0 + e] = y;
    }
    if (lse && lane == 0) lse[(size_t)c * H + h] = m + __logf(l);
}

}  // namespace

bool target_attend_uses_tc(const Problem& p) { return p.in_bf16 && p.d == 128 && (p.S == 128 || p.S == 256); }

cudaError_t launch_sm100_target_attend(const Problem& p, const int64_t* row_offsets, int64_t total_rows,
                                       const int64_t* uts, const int8_t* codes, const float* tscale, const float* tzp,
                                       const void* q, const void* k_self, const void* v_self, const void* resid,
                                       int out_bf16, void* out, float* lse) {
    CUtensorMap mq, mk;  // v_self rows are read by the epilogue threads directly
    if (!make_kv_map(&mq, q, total_rows, p.H) || !make_kv_map(&mk, k_self, total_rows, p.H))
        return cudaErrorInvalidValue;
    TAParams P;
    P.row_offsets = row_offsets;
    P.uts = uts;
    P.codes = codes;
    P.tscale = tscale;
    P.tzp = tzp;
    P.v = v_self;
    P.resid = resid;
    P.out = out;
    P.lse = lse;
    P.B = p.B;
    P.S = p.S;
    P.H = p.H;
    P.out_bf16 = out_bf16;
    P.scale_log2 = p.scale * kLog2e;
    const void* fn = p.S == 256 ? reinterpret_cast<const void*>(sm100_target_attend_kernel<256>)
                                : reinterpret_cast<const void*>(sm100_target_attend_kernel<128>);
    const cudaError_t attr = set_smem_attr(fn, kSmem);
    if (attr != cudaSuccess) return attr;
    // PDL: the prologue overlaps the tile scan launched just before (griddepcontrol.wait in the kernel)
    if (p.S == 256)
        return launch_pdl(sm100_target_attend_kernel<256>, dim3(p.num_sms), dim3(kThreads), kSmem, p.stream, mq, mk, P);
    return launch_pdl(sm100_target_attend_kernel<128>, dim3(p.num_sms), dim3(kThreads), kSmem, p.stream, mq, mk, P);
}

#ifdef VISTA_TRACE
extern "C" int vista_debug_ta_trace(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_ta_trace, bytes < sizeof(g_ta_trace) ? bytes : sizeof(g_ta_trace));
}
extern "C" int vista_debug_ta_cta(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_ta_cta, bytes < sizeof(g_ta_cta) ? bytes : sizeof(g_ta_cta));
}
#endif

cudaError_t launch_simt_target_attend(const Problem& p, const int64_t* row_offsets, int64_t total_rows,
                                      const int8_t* codes, const float* tscale, const float* tzp, const void* q,
                                      const void* k_self, const void* v_self, const void* resid, int out_bf16,
                                      void* out, float* lse) {
    if (total_rows == 0) return cudaSuccess;
    const int64_t warps = total_rows * p.H;
    const unsigned grid = (unsigned)((warps + 7) / 8);
    if (p.in_bf16)
        simt_target_attend_kernel<__nv_bfloat16><<<grid, 256, 0, p.stream>>>(
            row_offsets, codes, tscale, tzp, reinterpret_cast<const __nv_bfloat16*>(q),
            reinterpret_cast<const __nv_bfloat16*>(k_self), reinterpret_cast<const __nv_bfloat16*>(v_self),
            reinterpret_cast<const __nv_bfloat16*>(resid), p.B, p.S, p.H, p.d, p.scale, out_bf16, out, lse, total_rows);
    else
        simt_target_attend_kernel<float><<<grid, 256, 0, p.stream>>>(
            row_offsets, codes, tscale, tzp, reinterpret_cast<const float*>(q), reinterpret_cast<const float*>(k_self),
            reinterpret_cast<const float*>(v_self), reinterpret_cast<const float*>(resid), p.B, p.S, p.H, p.d, p.scale,
            out_bf16, out, lse, total_rows);
    return cudaGetLastError();
}

}  // namespace vista
