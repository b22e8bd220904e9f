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
#include "int8_export.cuh"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

#ifdef VISTA_TRACE  // debug timeline of CTA 0, first item: clock64 per (event, tile, q tile)
__device__ unsigned long long g_vista_trace[12][64][2];
#define VTRACE(ev, t, q) \
    do { if (blockIdx.x == 0 && (t) < 64) g_vista_trace[ev][t][q] = clock64(); } while (0)
// per-item events of CTA 0 (first 64 items), see scripts/trace_items.py
__device__ unsigned long long g_vista_itrace[12][64];
#define ITRACE(ev, i) \
    do { if (blockIdx.x == 0 && (i) < 64) g_vista_itrace[ev][i] = clock64(); } while (0)
#else
#define VTRACE(ev, t, q) do { } while (0)
#define ITRACE(ev, i) do { } while (0)
#endif

namespace {

constexpr int kHalfBytes = 128 * 128;       // 128 rows x 64 bf16 (one 128-B swizzle column block)
constexpr int kTileBytes = 2 * kHalfBytes;  // 128 x 128 bf16
constexpr float kRescaleThreshold = 8.0f;   // log2 units
#ifndef VISTA_SETMAXNREG
#define VISTA_SETMAXNREG 1
#endif
#ifndef VISTA_EMU_PER_EIGHT
#define VISTA_EMU_PER_EIGHT 0
#endif
constexpr int kEmuPerEight = VISTA_EMU_PER_EIGHT;
  // exp2 on the FMA pipe for this many of every 8 score pairs
#ifndef VISTA_CTL_REGS
#define VISTA_CTL_REGS 152
#endif
// the launch grants 168 x 384 = 64512 registers; 128 x ctl + 256 x softmax must not exceed it
constexpr int kCtlRegs = VISTA_CTL_REGS;
constexpr int kSoftmaxRegs = ((64512 - 128 * kCtlRegs) / 256) & ~7;
constexpr bool kSetMaxNReg = VISTA_SETMAXNREG;  // shift registers from the control warps to the softmax warps
#ifndef VISTA_SPLIT_P
#define VISTA_SPLIT_P 2
#endif
// P handed to the MMA in kSplitP parts of 128 / kSplitP keys (one arrive each; 1 = whole tile), so
// the PV GEMM of a part overlaps the exponentials of the next parts
constexpr int kSplitP = VISTA_SPLIT_P;
static_assert(kSplitP == 1 || kSplitP == 2 || kSplitP == 4, "P split");
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

template <int NQ>
struct Cfg {
    // smem: Q tiles, a ring of K tiles and a separate (shallower) ring of V tiles.  K is released as
    // soon as the score GEMMs of its tile have run, V only after the PV GEMMs, so splitting the
    // rings keeps ~3 tiles of HBM reads in flight per SM instead of ~2.
    static constexpr int kKStages = 3;
    static constexpr int kVStages = NQ == 2 ? 2 : 3;  // 224 KB total either way
    static constexpr int kQOff = 0;
    static constexpr int kKOff = NQ * kTileBytes;
    static constexpr int kVOff = kKOff + kKStages * kTileBytes;
    static constexpr int kBarOff = kVOff + kVStages * kTileBytes;
    static constexpr int kBarBytes = 768;
    static constexpr int kRingOff = kBarOff + kBarBytes;  // item ring (kItemRing x ItemEntry)
    static constexpr int kSmem = kRingOff + 512 + 1024;  // + alignment slack
    static_assert(kSmem <= 232448, "shared memory");
    static constexpr int kThreads = 128 + NQ * 128;     // control warpgroup + NQ softmax warpgroups
    static constexpr int kTmemCols = NQ == 2 ? 512 : 256;
};

// Item ring: the scheduler lane (warp 3) walks the CTA's tile range (ItemIter: uts / offsets
// loads) up to kItemRing items ahead and publishes each item here, so no role has a global load
// or a search on its per-item path.
constexpr int kItemRing = 16;
struct ItemEntry {
    int u, hg, t0, t1, Tu, row0, len, flags;  // flags: 1 valid, 2 first, 4 last
};
static_assert(kItemRing * sizeof(ItemEntry) <= 512, "ring region");

struct Bars {
    uint64_t it_full[kItemRing], it_empty[kItemRing];
    uint64_t q_full, q_empty;
    uint64_t k_full[4], k_empty[4], v_full[4], v_empty[4];
    uint64_t s_full[2][2], p_full[2][2];  // [q tile][P part: 0 first, 1 last]
    uint64_t p_part[2][2];                // [q tile][middle P parts] (kSplitP == 4)
    uint64_t pv_done[2], o_full[2];
    uint32_t tmem_base;
};

static_assert(sizeof(Bars) <= Cfg<2>::kBarBytes, "barrier region");

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
    int out_v8, slot_v8;  // outputs / slots 32-B aligned: 256-bit stores
};


// Next item from the ring (all lanes of the calling warp; lane 0 releases the entry).
__device__ __forceinline__ bool fetch_item(Bars* bars, const ItemEntry* ring, int k, Item& it) {
    const int s = k % kItemRing;
    ptx::mbar_wait(&bars->it_full[s], (uint32_t)(k / kItemRing) & 1u);
    const volatile int* e = reinterpret_cast<const volatile int*>(ring + s);
    it.u = e[0];
    it.hg = e[1];
    it.t0 = e[2];
    it.t1 = e[3];
    it.Tu = e[4];
    it.row0 = e[5];
    it.len = e[6];
    const int f = e[7];
    it.first = f & 2;
    it.last = f & 4;
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&bars->it_empty[s]);
    return f & 1;
}

__device__ __forceinline__ void st_v8(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
// 32 floats to global, 256-bit stores when aligned (V8), else 128-bit
__device__ __forceinline__ void st_f32x32(float* dst, const float (&o)[32], bool v8) {
    if (v8) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            const uint32_t w[8] = {__float_as_uint(o[j]),     __float_as_uint(o[j + 1]), __float_as_uint(o[j + 2]),
                                   __float_as_uint(o[j + 3]), __float_as_uint(o[j + 4]), __float_as_uint(o[j + 5]),
                                   __float_as_uint(o[j + 6]), __float_as_uint(o[j + 7])};
            st_v8(dst + j, w);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
    }
}

__device__ __forceinline__ void store_row(const Params& P, const Item& it, int cta, int row_in_unit,
                                          const float (&o)[32], int c0, float lse, bool write_lse, int NQrows) {
    // writes 32 consecutive channels [c0, c0+32) of one normalized output row (+ lse once)
    const int h = it.hg / P.G, g = it.hg % P.G;
    if (!item_complete(it)) {
        const int slot = item_slot(it, cta);
        st_f32x32(P.slot_o + ((size_t)slot * NQrows + row_in_unit) * 128 + c0, o, P.slot_v8);
        if (write_lse) P.slot_lse[(size_t)slot * NQrows + row_in_unit] = lse;
        return;
    }
    const int i = g * NQrows + row_in_unit;
    if (P.outs.mode == OUT_PARTIAL) {
        st_f32x32(reinterpret_cast<float*>(P.outs.out) + (((size_t)it.u * P.H + h) * P.S + i) * 128 + c0, o,
                  P.out_v8);
        if (write_lse) P.outs.lse[((size_t)it.u * P.H + h) * P.S + i] = lse;
        return;
    }
    const size_t base = (((size_t)it.u * P.S + i) * P.H + h) * 128 + c0;
    if (P.outs.out_bf16) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(P.outs.out) + base;
        if (P.out_v8) {
#pragma unroll
            for (int j = 0; j < 32; j += 16) {
                uint32_t w[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) w[e] = ptx::pack_bf16x2(o[j + 2 * e], o[j + 2 * e + 1]);
                st_v8(dst + j, w);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
                uint4 pk;
                pk.x = ptx::pack_bf16x2(o[j], o[j + 1]);
                pk.y = ptx::pack_bf16x2(o[j + 2], o[j + 3]);
                pk.z = ptx::pack_bf16x2(o[j + 4], o[j + 5]);
                pk.w = ptx::pack_bf16x2(o[j + 6], o[j + 7]);
                *reinterpret_cast<uint4*>(dst + j) = pk;
            }
        }
    } else {
        st_f32x32(reinterpret_cast<float*>(P.outs.out) + base, o, P.out_v8);
    }
    if (write_lse && P.outs.lse) P.outs.lse[((size_t)it.u * P.H + h) * P.S + i] = lse;
}

// lse of one row (natural log): partial slot or the caller's lse output (if any)
__device__ __forceinline__ void store_lse(const Params& P, const Item& it, int cta, int row, float lse, int NQrows) {
    if (!item_complete(it)) {
        P.slot_lse[(size_t)item_slot(it, cta) * NQrows + row] = lse;
        return;
    }
    if (!P.outs.lse) return;
    const int h = it.hg / P.G, g = it.hg % P.G;
    P.outs.lse[((size_t)it.u * P.H + h) * P.S + g * NQrows + row] = lse;
}

// Start of output row `row` (row within the unit's NQ*128 rows) of item `it`: a partial slot row
// (f32) for a split unit, else the final output row (bf16 or f32).
__device__ __forceinline__ char* out_row_ptr(const Params& P, const Item& it, int cta, int row, int NQrows) {
    if (!item_complete(it))
        return reinterpret_cast<char*>(P.slot_o + ((size_t)item_slot(it, cta) * NQrows + row) * 128);
    const int h = it.hg / P.G, g = it.hg % P.G;
    const int i = g * NQrows + row;
    if (P.outs.mode == OUT_PARTIAL)
        return reinterpret_cast<char*>(P.outs.out) + ((((size_t)it.u * P.H + h) * P.S + i) * 128) * 4;
    return reinterpret_cast<char*>(P.outs.out) +
           ((((size_t)it.u * P.S + i) * P.H + h) * 128) * (P.outs.out_bf16 ? 2 : 4);
}

// Coalesced epilogue store of 256 bytes per row (64 32-bit words v[] of the calling thread's row,
// byte offset `boff` in the row).  The row-per-thread layout of the accumulator would make every
// warp store touch 32 rows (32 lines); instead the words go back to TMEM (the O columns at tcol,
// already read) in a permuted column order and come out again with the 16x256b shape, where the 4
// threads of a quad hold 128 contiguous bytes of one row: each warp store then writes 8 full
// 128-B lines.  Column 8g + 2p + e holds word 8p + 2g + e (g < 4) or 32 + 8p + 2(g-4) + e (g >= 4).
__device__ __forceinline__ void store_rows_coalesced(const Params& P, const Item& it, int cta, int row0, int NQrows,
                                                     uint32_t tcol_warp, const uint32_t (&v)[64], int boff) {
    const int lane = threadIdx.x & 31;
    uint32_t a[32], b[32];
#pragma unroll
    for (int c = 0; c < 64; ++c) {
        const int g = c >> 3, p = (c & 7) >> 1, e = c & 1;
        const int w = g < 4 ? 8 * p + 2 * g + e : 32 + 8 * p + 2 * (g - 4) + e;
        if (c < 32) a[c] = v[w]; else b[c - 32] = v[w];
    }
    ptx::tmem_st32(tcol_warp, a);
    ptx::tmem_st32(tcol_warp + 32, b);
    ptx::tmem_wait_st();
    const int p = lane & 3;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        uint32_t r[32];
        ptx::tmem_ld16x256b_x8(tcol_warp + ((uint32_t)(16 * half) << 16), r);
        ptx::tmem_wait_ld();
        ptx::reg_fence(r);
        const int ra = row0 + 16 * half + (lane >> 2);
        char* pa = out_row_ptr(P, it, cta, ra, NQrows) + boff + 32 * p;
        char* pb = out_row_ptr(P, it, cta, ra + 8, NQrows) + boff + 32 * p;
        const uint32_t a0[8] = {r[0], r[1], r[4], r[5], r[8], r[9], r[12], r[13]};
        const uint32_t a1[8] = {r[16], r[17], r[20], r[21], r[24], r[25], r[28], r[29]};
        const uint32_t b0[8] = {r[2], r[3], r[6], r[7], r[10], r[11], r[14], r[15]};
        const uint32_t b1[8] = {r[18], r[19], r[22], r[23], r[26], r[27], r[30], r[31]};
        st_v8(pa, a0);
        st_v8(pa + 128, a1);
        st_v8(pb, b0);
        st_v8(pb + 128, b1);
    }
}

// p = 2^(s * scale * log2 e - m) for one 128-key row: packed FFMA2, exp2 on MUFU (ex2.approx) and,
// for EMU of every 8 pairs, on the FMA pipe (exp2_emu2; only for tiles without masked keys);
// bf16x2 pack; P overwrites the first 64 TMEM columns of S (16 columns per 32 keys).  Returns the
// row sum of the (unrounded) p.
template <int EMU>
__device__ __forceinline__ float exp_tile(const uint32_t (&r)[4][32], float sl2, float neg, uint32_t tS) {
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
            uint64_t p2;
            if (EMU > 0 && (j & 7) >= 8 - EMU) {
                p2 = ptx::exp2_emu2(x2);
            } else {
                float x0, x1;
                ptx::f2_unpack(x2, x0, x1);
                p2 = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
            }
            acc[j & 1] = ptx::f2_add(acc[j & 1], p2);
            float p0, p1;
            ptx::f2_unpack(p2, p0, p1);
            pk[j] = ptx::pack_bf16x2(p0, p1);
        }
        ptx::tmem_st16(tS + c * 16, pk);
    }
    float la, lb, lc, ld;
    ptx::f2_unpack(acc[0], la, lb);
    ptx::f2_unpack(acc[1], lc, ld);
    return (la + lb) + (lc + ld);
}

// exp_tile for part PART of NP equal key ranges (32-key chunks [PART 4/NP, (PART+1) 4/NP)); P into
// the matching TMEM columns
template <int PART, int NP, int EMU = 0>
__device__ __forceinline__ float exp_part(const uint32_t (&r)[4][32], float sl2, float neg, uint32_t tS) {
    const uint64_t sl2x2 = ptx::f2_pack(sl2, sl2);
    const uint64_t negx2 = ptx::f2_pack(neg, neg);
    uint64_t acc[2] = {ptx::f2_pack(0.f, 0.f), ptx::f2_pack(0.f, 0.f)};
#pragma unroll
    for (int c = PART * (4 / NP); c < (PART + 1) * (4 / NP); ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint64_t x2 = ptx::f2_fma(
                ptx::f2_pack(__uint_as_float(r[c][2 * j]), __uint_as_float(r[c][2 * j + 1])), sl2x2, negx2);
            uint64_t p2;
            if (EMU > 0 && (j & 7) >= 8 - EMU) {
                p2 = ptx::exp2_emu2(x2);
            } else {
                float x0, x1;
                ptx::f2_unpack(x2, x0, x1);
                p2 = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
            }
            acc[j & 1] = ptx::f2_add(acc[j & 1], p2);
            float p0, p1;
            ptx::f2_unpack(p2, p0, p1);
            pk[j] = ptx::pack_bf16x2(p0, p1);
        }
        ptx::tmem_st16(tS + c * 16, pk);
    }
    float la, lb, lc, ld;
    ptx::f2_unpack(acc[0], la, lb);
    ptx::f2_unpack(acc[1], lc, ld);
    return (la + lb) + (lc + ld);
}

#ifndef VISTA_MMA_SPIN
#define VISTA_MMA_SPIN 0
#endif
// The MMA warp's waits for P: optionally poll (test_wait) before the suspending try_wait.
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t phase) {
#if VISTA_MMA_SPIN > 0
#pragma unroll 1
    for (int i = 0; i < VISTA_MMA_SPIN; ++i)
        if (ptx::mbar_test_wait(bar, phase)) return;
#endif
    ptx::mbar_wait(bar, phase);
}

// ---- MMA issue with compile-time geometry (see the MMA role) ----
template <int NQ, int Q, int ST>
__device__ __forceinline__ void issue_S_t(uint32_t tmem, uint32_t sQa, uint32_t sKa) {
    // S_Q = Q_Q K^T over the 128 keys of K stage ST -> TMEM columns [128 Q, 128 Q + 128)
    constexpr uint32_t idS = ptx::idesc_bf16_f32(128, 128, 0, 0);  // Q, K both K-major
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
        ptx::mma_ss_w(tmem + Q * 128, ptx::sdesc_sw128(sQa + Q * kTileBytes + off, 16, 1024),
                      ptx::sdesc_sw128(sKa + ST * kTileBytes + off, 16, 1024), idS, kk > 0);
    }
}
template <int NQ, int Q, int ST, bool ACC, int K0 = 0, int K1 = 8>
__device__ __forceinline__ void issue_PV_t(uint32_t tmem, uint32_t sVa) {
    // O_Q += P_Q V over keys [16 K0, 16 K1) of V stage ST; P (bf16) read from TMEM columns [128 Q, 128 Q + 64)
    constexpr uint32_t idP = ptx::idesc_bf16_f32(128, 128, 0, 1);  // P (TMEM) x V (MN-major)
#pragma unroll
    for (int kk = K0; kk < K1; ++kk)
        ptx::mma_ts_w(tmem + NQ * 128 + Q * 128, tmem + Q * 128 + kk * 8,
                      ptx::sdesc_sw128(sVa + ST * kTileBytes + kk * 2048, kHalfBytes, 1024), idP,
                      (ACC || kk > 0) ? 1u : 0u);
}
template <int NQ, int Q>
__device__ __forceinline__ void issue_S_q(int st, uint32_t tmem, uint32_t sQa, uint32_t sKa) {
    switch (st) {
        case 0: issue_S_t<NQ, Q, 0>(tmem, sQa, sKa); break;
        case 1: issue_S_t<NQ, Q, 1>(tmem, sQa, sKa); break;
        default: issue_S_t<NQ, Q, 2>(tmem, sQa, sKa); break;
    }
}
template <int NQ>
__device__ __forceinline__ void issue_S_d(int q, int st, uint32_t tmem, uint32_t sQa, uint32_t sKa) {
    if (q == 0) issue_S_q<NQ, 0>(st, tmem, sQa, sKa);
    else if constexpr (NQ > 1) issue_S_q<NQ, 1>(st, tmem, sQa, sKa);
}
template <int NQ, int Q, bool ACC, int K0 = 0, int K1 = 8>
__device__ __forceinline__ void issue_PV_q(int st, uint32_t tmem, uint32_t sVa) {
    switch (st) {
        case 0: issue_PV_t<NQ, Q, 0, ACC, K0, K1>(tmem, sVa); break;
        case 1: issue_PV_t<NQ, Q, 1, ACC, K0, K1>(tmem, sVa); break;
        default: issue_PV_t<NQ, Q, 2, ACC, K0, K1>(tmem, sVa); break;
    }
}
template <int NQ, int K0 = 0, int K1 = 8>
__device__ __forceinline__ void issue_PV_d(int q, int st, bool acc, uint32_t tmem, uint32_t sVa) {
    if (q == 0) {
        if (acc) issue_PV_q<NQ, 0, true, K0, K1>(st, tmem, sVa); else issue_PV_q<NQ, 0, false, K0, K1>(st, tmem, sVa);
    } else if constexpr (NQ > 1) {
        if (acc) issue_PV_q<NQ, 1, true, K0, K1>(st, tmem, sVa); else issue_PV_q<NQ, 1, false, K0, K1>(st, tmem, sVa);
    }
}

template <int NQ>
__global__ void __launch_bounds__(Cfg<NQ>::kThreads, 1)
    sm100_softmax_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                         const __grid_constant__ CUtensorMap mapV, const Params P) {
    using C = Cfg<NQ>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem + C::kQOff;
    uint8_t* sK = smem + C::kKOff;
    uint8_t* sV = smem + C::kVOff;
    Bars* bars = reinterpret_cast<Bars*>(smem + C::kBarOff);
    ItemEntry* ring = reinterpret_cast<ItemEntry*>(smem + C::kRingOff);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cta = blockIdx.x, num_ctas = gridDim.x;
    const int HG = P.H * P.G;
    constexpr int kRows = NQ * 128;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kItemRing; ++s) {
            ptx::mbar_init(&bars->it_full[s], 1);
            ptx::mbar_init(&bars->it_empty[s], 3 + NQ * 4);
        }
        ptx::mbar_init(&bars->q_full, 1);
        ptx::mbar_init(&bars->q_empty, 1);
        for (int s = 0; s < C::kKStages; ++s) {
            ptx::mbar_init(&bars->k_full[s], 1);
            ptx::mbar_init(&bars->k_empty[s], 1);
        }
        for (int s = 0; s < C::kVStages; ++s) {
            ptx::mbar_init(&bars->v_full[s], 1);
            ptx::mbar_init(&bars->v_empty[s], 1);
        }
        for (int q = 0; q < NQ; ++q) {
            for (int b = 0; b < 2; ++b) {
                ptx::mbar_init(&bars->s_full[q][b], 1);
                ptx::mbar_init(&bars->p_full[q][b], 128);
                ptx::mbar_init(&bars->p_part[q][b], 128);
            }
            ptx::mbar_init(&bars->pv_done[q], 1);
            ptx::mbar_init(&bars->o_full[q], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, C::kTmemCols);
    // PDL: everything above overlapped the scan kernel; its results (uts) are needed from here on
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        // record which units this CTA's partial slots will hold (read by the merge kernel)
        int s0, s1;
        partial_slots(P.uts, P.B, HG, cta, num_ctas, s0, s1);
        P.slot_unit[2 * cta] = s0;
        P.slot_unit[2 * cta + 1] = s1;
    }
    asm volatile("griddepcontrol.launch_dependents;");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);

    Item it;

    if (warp < 4) {
        // register split (kCtlRegs / kSoftmaxRegs): setmaxnreg.inc blocks forever if the pool cannot
        // cover it, so the two budgets add up to exactly the launch grant.
        if constexpr (NQ == 2 && kSetMaxNReg) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
        if (warp == 0) {
            // ============================ TMA producer: Q, K ============================
            ptx::tma_prefetch(&mapQ);
            ptx::tma_prefetch(&mapK);
            const uint64_t pol_kv = ptx::policy_evict_first();
            const uint64_t pol_q = ptx::policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            int k = 0;
            while (fetch_item(bars, ring, k, it)) {
                const int h = it.hg / P.G, g = it.hg % P.G;
                if (lane == 0) ITRACE(8, k);
                if (k > 0) ptx::mbar_wait(&bars->q_empty, (k - 1) & 1);
                if (lane == 0) ITRACE(9, k);
                ptx::mbar_arrive_expect_tx_w(&bars->q_full, NQ * kTileBytes);
                for (int q = 0; q < NQ; ++q)
                    for (int half = 0; half < 2; ++half)
                        ptx::tma_load_4d_w(sQ + q * kTileBytes + half * kHalfBytes, &mapQ, &bars->q_full, half * 64, h,
                                         g * kRows + q * 128, P.q_per_user ? it.u : 0, pol_q);
                const int row0 = it.row0;
                for (int t = it.t0; t < it.t1; ++t) {
                    ptx::mbar_wait(&bars->k_empty[stage], phase ^ 1);
                    if (k == 0 && lane == 0) VTRACE(8, t - it.t0, 0);
                    if (lane == 0 && t == it.t0) ITRACE(10, k);
                    ptx::mbar_arrive_expect_tx_w(&bars->k_full[stage], kTileBytes);
                    const int32_t row = row0 + t * kTile;
                    for (int half = 0; half < 2; ++half)
                        ptx::tma_load_3d_w(sK + stage * kTileBytes + half * kHalfBytes, &mapK, &bars->k_full[stage],
                                         half * 64, h, row, pol_kv);
                    if (++stage == C::kKStages) { stage = 0; phase ^= 1; }
                }
                ++k;
            }
        } else if (warp == 2) {
            // ============================ TMA producer: V ============================
            ptx::tma_prefetch(&mapV);
            const uint64_t pol_kv = ptx::policy_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            bool first_item = true;
            int ki = 0;
            while (fetch_item(bars, ring, ki++, it)) {
                const int h = it.hg / P.G;
                const int row0 = it.row0;
                for (int t = it.t0; t < it.t1; ++t) {
                    ptx::mbar_wait(&bars->v_empty[stage], phase ^ 1);
                    if (first_item && lane == 0) VTRACE(9, t - it.t0, 0);
                    ptx::mbar_arrive_expect_tx_w(&bars->v_full[stage], kTileBytes);
                    const int32_t row = row0 + t * kTile;
                    for (int half = 0; half < 2; ++half)
                        ptx::tma_load_3d_w(sV + stage * kTileBytes + half * kHalfBytes, &mapV, &bars->v_full[stage],
                                         half * 64, h, row, pol_kv);
                    if (++stage == C::kVStages) { stage = 0; phase ^= 1; }
                }
                first_item = false;
            }
        } else if (warp == 1) {
            // ============================ MMA issuer ============================
            // Per K/V tile t and Q tile q: S_q(t) = Q_q K_t^T (TMEM cols of q), softmax writes P_q(t)
            // over it, O_q += P_q(t) V_t.  Issue order PV_0(t) S_0(t+1) PV_1(t) S_1(t+1): one Q tile's
            // exponentials overlap the other's GEMMs, and the commit after S_q(t+1) also covers
            // PV_q(t) (in-order completion), which is what lets a softmax thread rescale O_q.
            // The whole warp runs this loop and every MMA operand is a uniform base plus a
            // compile-time offset, so ptxas keeps descriptors in uniform registers.
            const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
            const uint32_t sQa = base + C::kQOff, sKa = base + C::kKOff, sVa = base + C::kVOff;
            int kst = 0, vst = 0;
            uint32_t kph = 0, vph = 0, q_phase = 0;
            uint32_t p_phase[2] = {0, 0};
            bool first_item = true;
#ifdef VISTA_TRACE
            int item_no = 0;
#endif
            int ki = 0;
            while (fetch_item(bars, ring, ki++, it)) {
                const int ntiles = it.t1 - it.t0;
#ifdef VISTA_TRACE
                if (blockIdx.x == 0 && lane == 0 && item_no < 32) {
                    g_vista_trace[10][item_no][0] = clock64();
                    g_vista_trace[10][item_no][1] = ptx::globaltimer_ns();
                    g_vista_trace[11][item_no][0] = (unsigned long long)ntiles;
                }
                ++item_no;
#endif
                if (lane == 0) ITRACE(0, item_no - 1);
                ptx::mbar_wait(&bars->q_full, q_phase);
                if (lane == 0) ITRACE(1, item_no - 1);
                q_phase ^= 1;
                ptx::mbar_wait(&bars->k_full[kst], kph);
                if (lane == 0) ITRACE(2, item_no - 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    issue_S_d<NQ>(q, kst, tmem, sQa, sKa);
                    ptx::mma_commit_w(&bars->s_full[q][0]);
                }
                ptx::mma_commit_w(&bars->k_empty[kst]);  // K tile t0 fully consumed once these complete
                if (++kst == C::kKStages) { kst = 0; kph ^= 1; }
                if (ntiles == 1) ptx::mma_commit_w(&bars->q_empty);  // last S of the item: Q free early
                for (int t = 0; t < ntiles; ++t) {
                    const bool more = t + 1 < ntiles;
                    ptx::mbar_wait(&bars->v_full[vst], vph);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        if (first_item && lane == 0) VTRACE(0, t, q);
                        mma_wait(&bars->p_full[q][0], p_phase[q]);
                        if (first_item && lane == 0) VTRACE(1, t, q);
                        ptx::tc_fence_after();
                        if constexpr (kSplitP == 2) {
                            // keys 0-63 as soon as their P is in TMEM, keys 64-127 after the rest
                            issue_PV_d<NQ, 0, 4>(q, vst, t > 0, tmem, sVa);
                            mma_wait(&bars->p_full[q][1], p_phase[q]);
                            ptx::tc_fence_after();
                            issue_PV_d<NQ, 4, 8>(q, vst, true, tmem, sVa);
                        } else if constexpr (kSplitP == 4) {
                            issue_PV_d<NQ, 0, 2>(q, vst, t > 0, tmem, sVa);
                            ptx::mbar_wait(&bars->p_part[q][0], p_phase[q]);
                            ptx::tc_fence_after();
                            issue_PV_d<NQ, 2, 4>(q, vst, true, tmem, sVa);
                            ptx::mbar_wait(&bars->p_part[q][1], p_phase[q]);
                            ptx::tc_fence_after();
                            issue_PV_d<NQ, 4, 6>(q, vst, true, tmem, sVa);
                            ptx::mbar_wait(&bars->p_full[q][1], p_phase[q]);
                            ptx::tc_fence_after();
                            issue_PV_d<NQ, 6, 8>(q, vst, true, tmem, sVa);
                        } else {
                            issue_PV_d<NQ>(q, vst, t > 0, tmem, sVa);
                        }
                        p_phase[q] ^= 1;
                        if (!more) {
                            if (lane == 0 && q == NQ - 1) ITRACE(3, item_no - 1);
                            ptx::mma_commit_w(&bars->o_full[q]);
                        } else {
                            if (q == 0) {
                                ptx::mbar_wait(&bars->k_full[kst], kph);
                                ptx::tc_fence_after();
                            }
                            issue_S_d<NQ>(q, kst, tmem, sQa, sKa);
                            ptx::mma_commit_w(&bars->s_full[q][0]);
                            if (first_item && lane == 0) VTRACE(2, t, q);
                            if (q == NQ - 1) {
                                ptx::mma_commit_w(&bars->k_empty[kst]);
                                if (++kst == C::kKStages) { kst = 0; kph ^= 1; }
                                // last S of the item: the next item's Q load overlaps the last PVs
                                if (t + 2 == ntiles) ptx::mma_commit_w(&bars->q_empty);
                            }
                        }
                    }
                    ptx::mma_commit_w(&bars->v_empty[vst]);
                    if (++vst == C::kVStages) { vst = 0; vph ^= 1; }
                }
                first_item = false;
            }
            (void)first_item;
        } else if (warp == 3) {
            // ============================ item scheduler ============================
            if (lane == 0) {
                ItemIter iter;
                iter.init(P.uts, P.B, HG, cta, num_ctas);
                for (int k = 0;; ++k) {
                    const bool ok = iter.next(it, P.uts, P.B, HG);
                    const int s = k % kItemRing;
                    if (k >= kItemRing) ptx::mbar_wait(&bars->it_empty[s], (uint32_t)(k / kItemRing - 1) & 1u);
                    volatile int* e = reinterpret_cast<volatile int*>(ring + s);
                    if (ok) {
                        const int64_t r0 = P.offsets[it.u], r1 = P.offsets[it.u + 1];
                        e[0] = it.u;
                        e[1] = it.hg;
                        e[2] = it.t0;
                        e[3] = it.t1;
                        e[4] = it.Tu;
                        e[5] = (int)r0;
                        e[6] = (int)(r1 - r0);
                    }
                    e[7] = ok ? (1 | (it.first ? 2 : 0) | (it.last ? 4 : 0)) : 0;
                    ptx::mbar_arrive(&bars->it_full[s]);  // release: the entry is visible to the waiters
                    if (!ok) break;
                }
            }
        }
        __syncwarp();
    } else {
        if constexpr (NQ == 2 && kSetMaxNReg) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
        // ============================ softmax warpgroups ============================
        const int wg = (warp - 4) / 4;  // warps 4..7 -> Q tile 0, 8..11 -> Q tile 1
        const int wq = warp % 4;
        const int row = wq * 32 + lane;  // row within Q tile = TMEM lane
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_bits + wg * 128;
        const uint32_t tO = tmem + lane_bits + NQ * 128 + wg * 128;
        const float sl2 = P.scale_log2;
        uint32_t s_phase = 0, o_phase = 0;
        bool first_item = true;
#ifdef VISTA_TRACE
        int sitem = 0;
#endif
        int ki = 0;
        while (fetch_item(bars, ring, ki++, it)) {
#ifdef VISTA_TRACE
            const bool itr = row == 0 && wg == 0;
            if (itr) ITRACE(4, sitem);
#endif
            const int L = it.len;
            float m_used = -INFINITY, l = 0.f;
            for (int t = it.t0; t < it.t1; ++t) {
                const bool tr = first_item && row == 0;
                if (tr) VTRACE(3, t - it.t0, wg);
                ptx::mbar_wait(&bars->s_full[wg][0], s_phase);
                if (tr) VTRACE(4, t - it.t0, wg);
                s_phase ^= 1;
#ifdef VISTA_TRACE
                if (itr && t == it.t0) ITRACE(5, sitem);
#endif
                ptx::tc_fence_after();
                uint32_t r[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tS + c * 32, r[c]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::reg_fence(r[c]);
                if (tr) VTRACE(5, t - it.t0, wg);
                const int valid = L - t * kTile;
                const bool full = valid >= kTile;
                if (!full) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c * 32 + j >= valid) r[c][j] = __float_as_uint(-INFINITY);
                }
                // row max: 8 independent FMNMX3 chains, then a small tree
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
                const bool need = mxs > m_used + kRescaleThreshold;
                const bool any = __any_sync(0xffffffffu, need);
                const float m_old = m_used;
                if (any) m_used = fmaxf(m_used, mxs);
                if constexpr (kSplitP > 1) {
                    const float lt0 = full ? exp_part<0, kSplitP, kEmuPerEight>(r, sl2, -m_used, tS)
                                           : exp_part<0, kSplitP>(r, sl2, -m_used, tS);
                    // O rescale before the first arrive (PV(t) accumulates into O right after it);
                    // placed after the first part so its registers are free
                    if (any && t > it.t0) {
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
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&bars->p_full[wg][0]);
                    float lt = lt0;
                    if constexpr (kSplitP == 4) {
                        lt += exp_part<1, 4>(r, sl2, -m_used, tS);
                        ptx::tmem_wait_st();
                        ptx::tc_fence_before();
                        ptx::mbar_arrive(&bars->p_part[wg][0]);
                        lt += exp_part<2, 4>(r, sl2, -m_used, tS);
                        ptx::tmem_wait_st();
                        ptx::tc_fence_before();
                        ptx::mbar_arrive(&bars->p_part[wg][1]);
                        lt += exp_part<3, 4>(r, sl2, -m_used, tS);
                    } else {
                        lt += full ? exp_part<1, 2, kEmuPerEight>(r, sl2, -m_used, tS)
                                   : exp_part<1, 2>(r, sl2, -m_used, tS);
                    }
                    if (tr) VTRACE(6, t - it.t0, wg);
                    l += lt;
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&bars->p_full[wg][1]);
                } else {
                // P = 2^(S scale log2e - m) over S_q (exp_tile); FMA-pipe exp2 only on unmasked tiles
                const float lt = full ? exp_tile<kEmuPerEight>(r, sl2, -m_used, tS) : exp_tile<0>(r, sl2, -m_used, tS);
                if (tr) VTRACE(6, t - it.t0, wg);
                if (any && t > it.t0) {
                    // O_q holds this item's sum so far: PV_q(t-1) completed (covered by s_full(t))
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
                ptx::mbar_arrive(&bars->p_full[wg][0]);
                }
                if (tr) VTRACE(7, t - it.t0, wg);
            }
            first_item = false;
            // epilogue: O / l, lse
            ptx::mbar_wait(&bars->o_full[wg], o_phase);
#ifdef VISTA_TRACE
            if (itr) ITRACE(6, sitem);
#endif
            o_phase ^= 1;
            ptx::tc_fence_after();
            const float inv_l = 1.f / l;
            const float lse = (m_used + __log2f(l)) * kLn2;
            const bool complete = item_complete(it);
            const bool coalesced = complete ? P.out_v8 : P.slot_v8;
            const bool out16 = complete && P.outs.mode != OUT_PARTIAL && P.outs.out_bf16;
            if (coalesced && out16) {
                uint32_t v[64];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[32];
                    ptx::tmem_ld32_sync(tO + c * 32, o);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        v[c * 16 + j] = ptx::pack_bf16x2(__uint_as_float(o[2 * j]) * inv_l,
                                                         __uint_as_float(o[2 * j + 1]) * inv_l);
                }
                if (P.outs.codes) {  // NEXT-1: int8 export of the row, as stored (bf16)
                    const int h = it.hg / P.G, g = it.hg % P.G;
                    const size_t orow = ((size_t)it.u * P.S + g * kRows + wg * 128 + row) * P.H + h;
                    i8_export_row_bf16(v, P.outs.codes + orow * 128, P.outs.qscale + orow, P.outs.qzp + orow);
                }
                store_rows_coalesced(P, it, cta, wg * 128 + wq * 32, kRows, tO, v, 0);
            } else if (coalesced) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    uint32_t v[64];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t o[32];
                        ptx::tmem_ld32_sync(tO + hh * 64 + c * 32, o);
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[c * 32 + j] = __float_as_uint(__uint_as_float(o[j]) * inv_l);
                    }
                    store_rows_coalesced(P, it, cta, wg * 128 + wq * 32, kRows, tO + hh * 64, v, hh * 256);
                }
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[32];
                    ptx::tmem_ld32_sync(tO + c * 32, o);
                    float of[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) of[j] = __uint_as_float(o[j]) * inv_l;
                    store_row(P, it, cta, wg * 128 + row, of, c * 32, lse, false, kRows);
                }
            }
            store_lse(P, it, cta, wg * 128 + row, lse, kRows);
#ifdef VISTA_TRACE
            if (itr) ITRACE(7, sitem);
            ++sitem;
#endif
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
#ifdef VISTA_TRACE
    if (threadIdx.x == 0) {
        g_vista_trace[11][32 + (blockIdx.x & 31)][0] = clock64();
        g_vista_trace[11][32 + (blockIdx.x & 31)][1] = ptx::globaltimer_ns();
    }
#endif
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
    P.out_v8 = (reinterpret_cast<uintptr_t>(p.outs.out) & 31) == 0;
    P.slot_v8 = (reinterpret_cast<uintptr_t>(P.slot_o) & 31) == 0;
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(sm100_softmax_kernel<NQ>), C::kSmem);
    if (attr != cudaSuccess) return attr;
    return launch_pdl(sm100_softmax_kernel<NQ>, dim3(w.num_ctas), dim3(C::kThreads), C::kSmem, p.stream, mq, mk, mv, P);
}

int sm100_softmax_nq(int S) { return (S % 256 == 0) ? 2 : 1; }

#ifdef VISTA_TRACE
extern "C" int vista_debug_itrace(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_vista_itrace, bytes < sizeof(g_vista_itrace) ? bytes : sizeof(g_vista_itrace));
}
extern "C" int vista_debug_trace(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_vista_trace, bytes < sizeof(g_vista_trace) ? bytes : sizeof(g_vista_trace));
}
#endif

cudaError_t launch_sm100_softmax(const Problem& p, const Workspace& w, char* ws) {
    return sm100_softmax_nq(p.S) == 2 ? launch_nq<2>(p, w, ws) : launch_nq<1>(p, w, ws);
}

}  // namespace vista
