// sm100_softmax.cu -- seed-row softmax summarization on B200: clusters of single-CTA tcgen05 MMAs
// sharing every K/V tile by TMA multicast, double-buffered scores in TMEM.
//
// Computes, for every work unit (user u, head h, group of C*128 seed rows):
//   O = RowSoftmax(scale * Q K^T) V,  lse = ln sum_j exp(scale q.k_j)
// over the user's jagged history rows [offsets[u], offsets[u+1]) -- the seed-row outputs of
// self-attention with virtual seeds.  The S x L score matrix never exists:
// keys stream through shared memory 128 at a time with an online softmax (flash style).
//
// Machine mapping:
//   * A cluster of C = S/128 (power of two, <= 8) CTAs owns a unit; CTA r holds query rows
//     [128 r, 128 r + 128).  Each 128-key K and V tile is fetched from L2/HBM ONCE per cluster: CTA r
//     loads rows [r 128/C, (r+1) 128/C) of it and multicasts them into every CTA's shared memory.
//   * One Q tile per CTA frees TMEM for double-buffered scores and a separate P (bf16) buffer pair:
//       cols [0,128) S_0   [128,256) S_1   [256,384) O   [384,448) P_0   [448,512) P_1
//     so S(g+2) may overwrite S buffer g % 2 as soon as the softmax has LOADED S(g), independent of
//     PV(g).  Two warps issue tcgen05 MMAs -- one the score GEMMs, one the PV GEMMs -- so one
//     warp's barrier waits overlap the other's issue and the tensor core's shallow instruction
//     queue stays fed (one issuing warp left it ~35% idle between its waits).
//   * Two softmax warpgroups split the rows: in lane quarter q, warp 4 + q owns rows 32q + [0, 16)
//     and warp 8 + q rows 32q + [16, 32), two threads per row (keys 0-63 / 64-127, the 16x32bx2
//     TMEM access shape).  Each SMSP thus runs two independent softmax warps whose max / barrier /
//     store phases overlap the other's MUFU exponentials.  A row's two threads meet with one
//     shuffle per tile.
//   * Shared memory: Q 32 KB (this CTA's rows), K ring 3 x 32 KB, V ring 2 x 32 KB.
//   * Persistent grid of clusters, stream-K flat tile ranges over clusters (work.cuh); split units
//     write fp32 partial slots merged by merge_softmax_slots_kernel.
// Roles per CTA (512 threads):
//   warp 0      item scheduler (ring of items for the other roles) + TMA: Q rows, K slices (multicast)
//   warp 1      score MMAs: S(g) = Q K_g^T (SS) into S buffer g % 2, up to two tiles ahead
//   warp 2      TMA: V slices (multicast)
//   warp 3      PV MMAs: O += P(g) V_g (TS: P from TMEM)
//   warps 4-11  softmax: two threads per query row (= TMEM lane), online softmax, P into TMEM
//   warps 12-15 epilogue: O / l, lse, coalesced stores (+ fused int8 export)
// Conditional rescale (threshold 2^8): the running max used for the exponent only moves when a
// row max exceeds it by more than 8 (log2 units); otherwise p <= 256 and O is left alone.
// Variant (VISTA_SOFTMAX_PAIR=1, clusters of two): a CTA pair issuing cta_group::2 MMAs (M = 256),
// each SM holding half of every K and V tile; parity-green but slower at c2.
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include "internal.h"
#include "int8_export.cuh"
#include "sm100_ptx.cuh"
#include "work.cuh"

namespace vista {

bool make_kv_map_rows(CUtensorMap* map, const void* base, int64_t total_len, int H, int rows);
bool make_q_map(CUtensorMap* map, const void* base, int S, int H, int B, int64_t q_user_stride);

#ifdef VISTA_TRACE  // debug timeline of CTA 0: clock64 per (event, global tile)
__device__ unsigned long long g_vista_trace[28][64];
#define VTRACE(ev, g) \
    do { if (blockIdx.x == 0 && (g) < 64) g_vista_trace[ev][g] = clock64(); } while (0)
__device__ unsigned long long g_vista_cta[256][4];  // per CTA: globaltimer start / end, clock64 start / end
__device__ int g_vista_probe[2][64];  // CTA 0 softmax: s_full / p_free already complete at the first probe
#define VPROBE(i, g, bar, par) \
    do { if (blockIdx.x == 0 && (g) < 64) g_vista_probe[i][g] = ptx::mbar_test_wait(bar, par) ? 1 : 0; } while (0)
#else
#define VPROBE(i, g, bar, par) do { } while (0)
#define VTRACE(ev, g) do { } while (0)
#endif

namespace {

constexpr int kHalfBytes = 128 * 128;       // 128 rows x 64 bf16 (one 128-B swizzle column block)
constexpr int kTileBytes = 2 * kHalfBytes;  // 128 x 128 bf16
constexpr float kRescaleThreshold = 8.0f;   // log2 units
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
#ifndef VISTA_KSTAGES
#define VISTA_KSTAGES 3
#endif
#ifndef VISTA_VSTAGES
#define VISTA_VSTAGES (5 - VISTA_KSTAGES)
#endif
constexpr int kKStages = VISTA_KSTAGES, kVStages = VISTA_VSTAGES;
// CTA-pair mode (cta_group::2): a stage holds this CTA's half of a tile (K: 64 keys x 128
// channels, V: 128 keys x 64 channels), so the same 160 KB of rings hold more stages
constexpr int kPairBytes = kTileBytes / 2;
constexpr int kPairKStages = 6, kPairVStages = 4;
constexpr int kMaxStages = 6;

constexpr int kQOff = 0;
constexpr int kKOff = kQOff + kTileBytes;
constexpr int kVOff = kKOff + kKStages * kTileBytes;
constexpr int kPairVOff = kKOff + kPairKStages * kPairBytes;
constexpr int kRingsEnd = kVOff + kVStages * kTileBytes > kPairVOff + kPairVStages * kPairBytes
                              ? kVOff + kVStages * kTileBytes
                              : kPairVOff + kPairVStages * kPairBytes;
constexpr int kThreads = 512;
constexpr int kTmemCols = 512;
#ifndef VISTA_ITEM_RING
#define VISTA_ITEM_RING 16
#endif
constexpr int kItemRing = VISTA_ITEM_RING;
constexpr int kRingConsumers = 15;  // warps 1, 2, 3 and the 12 softmax / epilogue warps
#ifndef VISTA_CTL_REGS
#define VISTA_CTL_REGS 96
#endif
// the launch grants 128 x 512 registers; the control warpgroup gives 32 per thread back
// (setmaxnreg.dec) and the softmax warpgroups take 16 each (setmaxnreg.inc blocks until the pool can
// cover it); the epilogue warpgroup keeps whatever is left (128 by default)
constexpr int kCtlRegs = VISTA_CTL_REGS;
#ifndef VISTA_SMX_REGS  // registers of the two softmax warpgroups (A/B p17: 144 beats 128, 152, 160)
#define VISTA_SMX_REGS 144
#endif
constexpr int kSmxRegs = VISTA_SMX_REGS;
constexpr int kEpiRegs = 128 + (128 - kCtlRegs) - 2 * (kSmxRegs - 128);
static_assert(kCtlRegs % 8 == 0 && kSmxRegs % 8 == 0 && kEpiRegs % 8 == 0 && kCtlRegs <= 128 && kEpiRegs >= 24 &&
                  kEpiRegs <= 256, "register split");

struct ItemEntry {
    int u, hg, t0, t1, Tu, row0, len, flags;  // flags: 1 valid, 2 first, 4 last
};

struct Bars {
    uint64_t it_full[kItemRing], it_empty[kItemRing];
    uint64_t q_full, q_empty;  // the item's Q tile in smem / its last S done
    uint64_t k_full[kMaxStages], k_empty[kMaxStages], v_full[kMaxStages], v_empty[kMaxStages];
    uint64_t s_full[2], s_free[2];  // S(g) in buffer g % 2 complete / loaded by both softmax halves
    uint64_t p_full[2], p_free[2];  // P(g) in buffer g % 2 written (256 arrivals) / read by PV(g)
    uint64_t pv_done;               // one completion per PV (the rescale waits for the previous one)
    uint64_t o_full, o_empty;        // the item's O complete / read by the epilogue
    uint64_t ml_full, ml_empty;      // the item's 1/l and lse rows, softmax -> epilogue
    uint32_t tmem_base;
    uint32_t pad;
    float ml[2][128];  // [l | m][row], the item's row statistics for the epilogue
};
constexpr int kBarOff = kRingsEnd;
constexpr int kRingOff = kBarOff + (int)((sizeof(Bars) + 15) & ~size_t(15));
constexpr int kSmemUsed = kRingOff + kItemRing * (int)sizeof(ItemEntry);
constexpr int kSmem = kSmemUsed + 1024;  // + alignment slack of the dynamic smem base
static_assert(kSmem <= 232448, "shared memory");

struct Params {
    const int64_t* offsets;
    const int64_t* uts;
    int* slot_unit;
    float* slot_o;
    float* slot_lse;
    OutSpec outs;
    int B, S, H, G;  // G: units (groups of C*128 rows) per head
    float scale_log2;
    int q_per_user;
    int groups;  // > 1: query-group-major work order (ItemIterG; the G groups of a unit run side by side)
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

// writes 32 consecutive channels [c0, c0+32) of one normalized output row (row within the unit)
template <bool PEERS>
__device__ __forceinline__ void store_row(const Params& P, const PeerSpec& pe, const Item& it, int slot_base, int row_in_unit,
                                          const float (&o)[32], int c0, int NQrows) {
    const int h = it.hg / P.G, g = it.hg % P.G;
    if (!item_complete(it)) {
        const int slot = item_slot(it, slot_base);
        st_f32x32(P.slot_o + ((size_t)slot * NQrows + row_in_unit) * 128 + c0, o, P.slot_v8);
        return;
    }
    const int i = g * NQrows + row_in_unit;
    if (P.outs.mode == OUT_PARTIAL) {
        const size_t idx = (((size_t)it.u * P.H + h) * P.S + i) * 128 + c0;
        if constexpr (PEERS) {  // fused exchange: every rank's receive buffer
#pragma unroll
            for (int r = 0; r < kMaxExchangeRanks; ++r) {
                if (r >= pe.n) break;
                st_f32x32(pe.o[r] + idx, o, P.out_v8);
            }
        } else {
            st_f32x32(reinterpret_cast<float*>(P.outs.out) + idx, o, P.out_v8);
        }
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
        st_f32x32(reinterpret_cast<float*>(P.outs.out) + base, o, P.out_v8);
    }
}

// lse of one row (natural log): partial slot, partial output or the caller's lse (if any)
template <bool PEERS>
__device__ __forceinline__ void store_lse(const Params& P, const PeerSpec& pe, const Item& it, int slot_base, int row, float lse,
                                          int NQrows) {
    if (!item_complete(it)) {
        P.slot_lse[(size_t)item_slot(it, slot_base) * NQrows + row] = lse;
        return;
    }
    const int h = it.hg / P.G, g = it.hg % P.G;
    const size_t idx = ((size_t)it.u * P.H + h) * P.S + g * NQrows + row;
    if constexpr (PEERS) {
        if (P.outs.mode == OUT_PARTIAL) {  // fused exchange: every rank's receive buffer
#pragma unroll
            for (int r = 0; r < kMaxExchangeRanks; ++r) {
                if (r >= pe.n) break;
                pe.lse[r][idx] = lse;
            }
            return;
        }
    }
    if (!P.outs.lse) return;
    P.outs.lse[idx] = lse;
}

// Start of output row `row` (row within the unit) of item `it`: a partial slot row (f32) for a
// split unit, else the final output row (bf16 or f32).
__device__ __forceinline__ char* out_row_ptr(const Params& P, const Item& it, int slot_base, int row, int NQrows) {
    if (!item_complete(it))
        return reinterpret_cast<char*>(P.slot_o + ((size_t)item_slot(it, slot_base) * NQrows + row) * 128);
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
template <bool PEERS>
__device__ __forceinline__ void store_rows_coalesced(const Params& P, const PeerSpec& pe, const Item& it, int slot_base, int row0,
                                                     int NQrows, uint32_t tcol_warp, const uint32_t (&v)[64],
                                                     int boff) {
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
        char* pa = out_row_ptr(P, it, slot_base, ra, NQrows) + boff + 32 * p;
        char* pb = out_row_ptr(P, it, slot_base, ra + 8, NQrows) + boff + 32 * p;
        const uint32_t a0[8] = {r[0], r[1], r[4], r[5], r[8], r[9], r[12], r[13]};
        const uint32_t a1[8] = {r[16], r[17], r[20], r[21], r[24], r[25], r[28], r[29]};
        const uint32_t b0[8] = {r[2], r[3], r[6], r[7], r[10], r[11], r[14], r[15]};
        const uint32_t b1[8] = {r[18], r[19], r[22], r[23], r[26], r[27], r[30], r[31]};
        if constexpr (PEERS) if (P.outs.mode == OUT_PARTIAL && item_complete(it)) {
            // fused split-L exchange: the same bytes into every rank's receive buffer (NVLink stores)
            const size_t da = (size_t)(reinterpret_cast<uintptr_t>(pa) - reinterpret_cast<uintptr_t>(P.outs.out));
            const size_t db = (size_t)(reinterpret_cast<uintptr_t>(pb) - reinterpret_cast<uintptr_t>(P.outs.out));
#pragma unroll
            for (int q = 0; q < kMaxExchangeRanks; ++q) {
                if (q >= pe.n) break;
                char* base = reinterpret_cast<char*>(pe.o[q]);
                st_v8(base + da, a0);
                st_v8(base + da + 128, a1);
                st_v8(base + db, b0);
                st_v8(base + db + 128, b1);
            }
            continue;
        }
        st_v8(pa, a0);
        st_v8(pa + 128, a1);
        st_v8(pb, b0);
        st_v8(pb + 128, b1);
    }
}

// p = 2^(s * scale * log2 e - m) for the 64 keys a thread owns of its row: packed FFMA2, exp2 on
// MUFU, bf16x2 pack; P into TMEM at tP
// with the 16x32bx2 shape (16 columns = 32 keys per store; the row's other thread writes 32 columns
// further).  Returns the sum of the (unrounded) p.
__device__ __forceinline__ float exp_half(const uint32_t (&r)[2][32], float sl2, float neg, uint32_t tP) {
    const uint64_t sl2x2 = ptx::f2_pack(sl2, sl2);
    const uint64_t negx2 = ptx::f2_pack(neg, neg);
    uint64_t acc[2] = {ptx::f2_pack(0.f, 0.f), ptx::f2_pack(0.f, 0.f)};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint64_t x2 = ptx::f2_fma(
                ptx::f2_pack(__uint_as_float(r[c][2 * j]), __uint_as_float(r[c][2 * j + 1])), sl2x2, negx2);
            float x0, x1;
            ptx::f2_unpack(x2, x0, x1);
            const uint64_t p2 = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
            acc[j & 1] = ptx::f2_add(acc[j & 1], p2);
            float p0, p1;
            ptx::f2_unpack(p2, p0, p1);
            pk[j] = ptx::pack_bf16x2(p0, p1);
        }
        ptx::tmem_st16x32bx2_x16<32>(tP + c * 16, pk);
    }
    float la, lb, lc, ld;
    ptx::f2_unpack(acc[0], la, lb);
    ptx::f2_unpack(acc[1], lc, ld);
    return (la + lb) + (lc + ld);
}

// ---- MMA issue with compile-time geometry (descriptors stay in uniform registers) ----
template <int KS>
__device__ __forceinline__ void issue_S_t(uint32_t tS, uint32_t sQa, uint32_t sKa) {
    // S = Q K^T over the 128 keys of K stage KS -> the TMEM S buffer at tS (Q, K both K-major)
    constexpr uint32_t idS = ptx::idesc_bf16_f32(128, 128, 0, 0);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
        ptx::mma_ss_w(tS, ptx::sdesc_sw128(sQa + off, 16, 1024), ptx::sdesc_sw128(sKa + KS * kTileBytes + off, 16, 1024),
                      idS, kk > 0);
    }
}
template <int VS>
__device__ __forceinline__ void issue_PV_t(uint32_t tO, uint32_t tP, uint32_t sVa, bool acc) {
    // O += P V over the 128 keys of V stage VS; P (bf16) read from TMEM at tP (8 columns per 16 keys)
    constexpr uint32_t idP = ptx::idesc_bf16_f32(128, 128, 0, 1);  // P (TMEM) x V (MN-major)
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma_ts_w(tO, tP + kk * 8, ptx::sdesc_sw128(sVa + VS * kTileBytes + kk * 2048, kHalfBytes, 1024), idP,
                      (acc || kk > 0) ? 1u : 0u);
}
__device__ __forceinline__ void issue_S(int ks, uint32_t tS, uint32_t sQa, uint32_t sKa) {
    switch (ks) {
        case 0: issue_S_t<0>(tS, sQa, sKa); break;
        case 1: issue_S_t<1 % kKStages>(tS, sQa, sKa); break;
        case 2: issue_S_t<2 % kKStages>(tS, sQa, sKa); break;
        default: issue_S_t<3 % kKStages>(tS, sQa, sKa); break;
    }
}
__device__ __forceinline__ void issue_PV(int vs, uint32_t tO, uint32_t tP, uint32_t sVa, bool acc) {
    switch (vs) {
        case 0: issue_PV_t<0>(tO, tP, sVa, acc); break;
        case 1: issue_PV_t<1 % kVStages>(tO, tP, sVa, acc); break;
        case 2: issue_PV_t<2 % kVStages>(tO, tP, sVa, acc); break;
        default: issue_PV_t<3 % kVStages>(tO, tP, sVa, acc); break;
    }
}

// ---- CTA pair (cta_group::2, M = 256; issued by the leader CTA for both) ----
template <int KS>
__device__ __forceinline__ void issue_S2_t(uint32_t tS, uint32_t sQa, uint32_t sKa) {
    // S = Q K^T: A = Q (each CTA its 128 rows), B = K tile split along N: each CTA holds 64 keys x
    // 128 channels (two 8 KB channel halves)
    constexpr uint32_t idS = ptx::idesc_bf16_f32(256, 128, 0, 0);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma2_ss_w(tS, ptx::sdesc_sw128(sQa + (kk >> 2) * kHalfBytes + (kk & 3) * 32, 16, 1024),
                       ptx::sdesc_sw128(sKa + KS * kPairBytes + (kk >> 2) * (kPairBytes / 2) + (kk & 3) * 32, 16, 1024),
                       idS, kk > 0);
}
template <int VS>
__device__ __forceinline__ void issue_PV2_t(uint32_t tO, uint32_t tP, uint32_t sVa, bool acc) {
    // O += P V: A = P from each CTA's TMEM, B = V tile split along N = channels: each CTA holds all
    // 128 keys x 64 channels (one 128-B swizzle column)
    constexpr uint32_t idP = ptx::idesc_bf16_f32(256, 128, 0, 1);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma2_ts_w(tO, tP + kk * 8, ptx::sdesc_sw128(sVa + VS * kPairBytes + kk * 2048, kHalfBytes, 1024), idP,
                       (acc || kk > 0) ? 1u : 0u);
}
__device__ __forceinline__ void issue_S2(int ks, uint32_t tS, uint32_t sQa, uint32_t sKa) {
    static_assert(kPairKStages == 6, "stage switch");
    switch (ks) {
        case 0: issue_S2_t<0>(tS, sQa, sKa); break;
        case 1: issue_S2_t<1>(tS, sQa, sKa); break;
        case 2: issue_S2_t<2>(tS, sQa, sKa); break;
        case 3: issue_S2_t<3>(tS, sQa, sKa); break;
        case 4: issue_S2_t<4>(tS, sQa, sKa); break;
        default: issue_S2_t<5>(tS, sQa, sKa); break;
    }
}
__device__ __forceinline__ void issue_PV2(int vs, uint32_t tO, uint32_t tP, uint32_t sVa, bool acc) {
    static_assert(kPairVStages == 4, "stage switch");
    switch (vs) {
        case 0: issue_PV2_t<0>(tO, tP, sVa, acc); break;
        case 1: issue_PV2_t<1>(tO, tP, sVa, acc); break;
        case 2: issue_PV2_t<2>(tO, tP, sVa, acc); break;
        default: issue_PV2_t<3>(tO, tP, sVa, acc); break;
    }
}

// arrive of one warp (lane 0, after the warp's own tcgen05 accesses are fenced) on a barrier of
// the pair's leader CTA: local for the leader, through the cluster window for the peer
__device__ __forceinline__ void warp_arrive_leader(uint64_t* bar, int rank) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        if (rank == 0) ptx::mbar_arrive(bar);
        else ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(bar), 0), 1);
    }
}

// PEERS: the fused split-L exchange (vista_summarize_partial_peers) -- partial rows to every rank's
// receive buffer; a separate instantiation so the default kernel carries none of it
template <int C, bool PAIR, bool PEERS = false>
__global__ void __launch_bounds__(kThreads, 1)
    sm100_softmax_kernel(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                         const __grid_constant__ CUtensorMap mapV, const Params P,
                         const __grid_constant__ PeerSpec peers) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem + kQOff;
    uint8_t* sK = smem + kKOff;
    uint8_t* sV = smem + (PAIR ? kPairVOff : kVOff);
    Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
    ItemEntry* ring = reinterpret_cast<ItemEntry*>(smem + kRingOff);

    static_assert(!PAIR || C == 2, "a CTA pair is a cluster of two");
    constexpr uint16_t kMask = (uint16_t)((1u << C) - 1u);
    constexpr int KST = PAIR ? kPairKStages : kKStages, VST = PAIR ? kPairVStages : kVStages;
    constexpr int kSlice = 128 / C;  // K/V rows this CTA loads (and multicasts) per tile
    constexpr int kRows = C * 128;   // query rows per unit
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rank = C > 1 ? (int)ptx::cluster_ctarank() : 0;
    const int cid = C > 1 ? (int)ptx::cluster_id_x() : (int)blockIdx.x;
    const int nclusters = C > 1 ? (int)ptx::num_clusters_x() : (int)gridDim.x;
    const int HG = P.H * P.G;
#ifdef VISTA_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 256) {
        g_vista_cta[blockIdx.x][0] = ptx::globaltimer_ns();
        g_vista_cta[blockIdx.x][2] = clock64();
    }
#endif

    if (threadIdx.x == 0) {
        for (int s = 0; s < kItemRing; ++s) {
            ptx::mbar_init(&bars->it_full[s], 1);
            ptx::mbar_init(&bars->it_empty[s], kRingConsumers);
        }
        // pair mode: the full barriers of the leader count its producer's expect_tx (both halves'
        // bytes) and the TMA completions of both CTAs; the leader's MMA commits arrive on the
        // barriers of both CTAs (count 1); the consumers of both CTAs arrive once per warp on the
        // leader's s_free / p_full / o_empty
        ptx::mbar_init(&bars->q_full, 1);
        ptx::mbar_init(&bars->q_empty, 1);
        for (int s = 0; s < KST; ++s) {
            ptx::mbar_init(&bars->k_full[s], 1);
            ptx::mbar_init(&bars->k_empty[s], PAIR ? 1 : C);  // multicast mode: released by every CTA
        }
        for (int s = 0; s < VST; ++s) {
            ptx::mbar_init(&bars->v_full[s], 1);
            ptx::mbar_init(&bars->v_empty[s], PAIR ? 1 : C);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->s_full[b], 1);
            ptx::mbar_init(&bars->s_free[b], PAIR ? 16 : 256);
            ptx::mbar_init(&bars->p_full[b], PAIR ? 16 : 256);
            ptx::mbar_init(&bars->p_free[b], 1);
        }
        ptx::mbar_init(&bars->pv_done, 1);
        ptx::mbar_init(&bars->o_full, 1);
        ptx::mbar_init(&bars->o_empty, PAIR ? 8 : 128);
        ptx::mbar_init(&bars->ml_full, 256);
        ptx::mbar_init(&bars->ml_empty, 128);
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        if constexpr (PAIR) ptx::tmem_alloc2(&bars->tmem_base, kTmemCols);
        else ptx::tmem_alloc(&bars->tmem_base, kTmemCols);
    }
    // PDL: everything above overlapped the scan kernel; its results (uts) are needed from here on
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && rank == 0) {
        // record which units this cluster's partial slots will hold (read by the merge kernel)
        int s0, s1;
        partial_slots_g(P.uts, P.B, HG, cid, nclusters, s0, s1, P.groups);
        P.slot_unit[2 * cid] = s0;
        P.slot_unit[2 * cid + 1] = s1;
    }
    asm volatile("griddepcontrol.launch_dependents;");
    ptx::tc_fence_before();
    if constexpr (C > 1) ptx::cluster_sync();  // every CTA's barriers exist before any multicast
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;

    Item it;
    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtlRegs));
        if (warp == 0) {
            // ===================== item scheduler + TMA: Q (own rows), K slices (multicast) =====================
            // Every lane walks the same items (uts loads are broadcasts); lane 0 publishes each item in
            // the ring, then the warp issues the item's Q tile and its K slices.
            ptx::tma_prefetch(&mapQ);
            ptx::tma_prefetch(&mapK);
            const uint64_t pol_kv = ptx::policy_evict_first();
            const uint64_t pol_q = ptx::policy_evict_last();
            // group-major order when a unit is several query groups (the groups of a (user, head)
            // stream the same K/V tiles at the same time: the second read hits L2)
            ItemIterG iter;
            iter.init(P.uts, P.B, HG, cid, nclusters, P.groups);
            int stage = 0, gk = 0;
            uint32_t phase = 0;
            for (int k = 0;; ++k) {
                const bool ok = iter.next(it, P.uts, P.B, HG);
                const int s = k % kItemRing;
                if (k >= kItemRing) ptx::mbar_wait(&bars->it_empty[s], (uint32_t)(k / kItemRing - 1) & 1u);
                int row0 = 0;
                if (lane == 0) {
                    volatile int* e = reinterpret_cast<volatile int*>(ring + s);
                    if (ok) {
                        const int64_t r0 = P.offsets[it.u], r1 = P.offsets[it.u + 1];
                        row0 = (int)r0;
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
                }
                __syncwarp();
                if (!ok) break;
                row0 = __shfl_sync(0xffffffffu, row0, 0);
                const int h = it.hg / P.G, g = it.hg % P.G;
                if (k >= 1) ptx::mbar_wait(&bars->q_empty, (uint32_t)(k - 1) & 1u);  // previous item's S done
                if (lane == 0) VTRACE(17, k);
                if constexpr (PAIR) {
                    // this CTA's Q rows; completion on the leader's q_full (armed for both CTAs)
                    const uint32_t qf = ptx::mapa(ptx::smem_u32(&bars->q_full), 0);
                    if (rank == 0) ptx::mbar_arrive_expect_tx_w(&bars->q_full, 2 * kTileBytes);
                    for (int half = 0; half < 2; ++half)
                        ptx::tma_load_4d_2sm_w(ptx::smem_u32(sQ + half * kHalfBytes), &mapQ, qf, half * 64, h,
                                               g * kRows + rank * 128, P.q_per_user ? it.u : 0, pol_q);
                } else {
                    ptx::mbar_arrive_expect_tx_w(&bars->q_full, kTileBytes);
                    for (int half = 0; half < 2; ++half)
                        ptx::tma_load_4d_w(sQ + half * kHalfBytes, &mapQ, &bars->q_full, half * 64, h,
                                           g * kRows + rank * 128, P.q_per_user ? it.u : 0, pol_q);
                }
                for (int t = it.t0; t < it.t1; ++t) {
                    ptx::mbar_wait(&bars->k_empty[stage], phase ^ 1);
                    if (lane == 0) VTRACE(5, gk);
                    ++gk;
                    if constexpr (PAIR) {
                        // keys [64 rank, 64 rank + 64) of the tile, both channel halves
                        const uint32_t kf = ptx::mapa(ptx::smem_u32(&bars->k_full[stage]), 0);
                        if (rank == 0) ptx::mbar_arrive_expect_tx_w(&bars->k_full[stage], 2 * kPairBytes);
                        const int32_t row = row0 + t * kTile + rank * 64;
                        for (int half = 0; half < 2; ++half)
                            ptx::tma_load_3d_2sm_w(ptx::smem_u32(sK + stage * kPairBytes + half * (kPairBytes / 2)), &mapK,
                                                   kf, half * 64, h, row, pol_kv);
                    } else {
                        ptx::mbar_arrive_expect_tx_w(&bars->k_full[stage], kTileBytes);
                        const int32_t row = row0 + t * kTile + rank * kSlice;
                        for (int half = 0; half < 2; ++half) {
                            uint8_t* dst = sK + stage * kTileBytes + half * kHalfBytes + rank * kSlice * 128;
                            if constexpr (C > 1)
                                ptx::tma_load_3d_mc_w(dst, &mapK, &bars->k_full[stage], half * 64, h, row, kMask, pol_kv);
                            else
                                ptx::tma_load_3d_w(dst, &mapK, &bars->k_full[stage], half * 64, h, row, pol_kv);
                        }
                    }
                    if (++stage == KST) { stage = 0; phase ^= 1; }
                }
            }
        } else if (warp == 2) {
            // ============================ TMA: V slices (multicast) ============================
            ptx::tma_prefetch(&mapV);
            const uint64_t pol_kv = ptx::policy_evict_first();
            int stage = 0, gv = 0;
            uint32_t phase = 0;
            for (int k = 0; fetch_item(bars, ring, k, it); ++k) {
                const int h = it.hg / P.G;
                for (int t = it.t0; t < it.t1; ++t) {
                    ptx::mbar_wait(&bars->v_empty[stage], phase ^ 1);
                    if (lane == 0) VTRACE(6, gv);
                    ++gv;
                    if constexpr (PAIR) {
                        // all 128 keys of the tile, channels [64 rank, 64 rank + 64)
                        const uint32_t vf = ptx::mapa(ptx::smem_u32(&bars->v_full[stage]), 0);
                        if (rank == 0) ptx::mbar_arrive_expect_tx_w(&bars->v_full[stage], 2 * kPairBytes);
                        ptx::tma_load_3d_2sm_w(ptx::smem_u32(sV + stage * kPairBytes), &mapV, vf, rank * 64, h,
                                               it.row0 + t * kTile, pol_kv);
                    } else {
                        ptx::mbar_arrive_expect_tx_w(&bars->v_full[stage], kTileBytes);
                        const int32_t row = it.row0 + t * kTile + rank * kSlice;
                        for (int half = 0; half < 2; ++half) {
                            uint8_t* dst = sV + stage * kTileBytes + half * kHalfBytes + rank * kSlice * 128;
                            if constexpr (C > 1)
                                ptx::tma_load_3d_mc_w(dst, &mapV, &bars->v_full[stage], half * 64, h, row, kMask, pol_kv);
                            else
                                ptx::tma_load_3d_w(dst, &mapV, &bars->v_full[stage], half * 64, h, row, pol_kv);
                        }
                    }
                    if (++stage == VST) { stage = 0; phase ^= 1; }
                }
            }
        } else if (PAIR && rank != 0) {
            // pair mode: the peer CTA's MMA warps only drain the item ring (the leader issues for both)
            for (int k = 0; fetch_item(bars, ring, k, it); ++k) {
            }
        } else if (warp == 1) {
            // ============================ score MMAs ============================
            // S(g) into buffer g % 2 as soon as K_g is in and the softmax has loaded S(g - 2).
            const uint32_t sQa = base + kQOff, sKa = base + kKOff;
            int kst = 0, g = 0;
            uint32_t kph = 0;
            for (int k = 0; fetch_item(bars, ring, k, it); ++k) {
                ptx::mbar_wait(&bars->q_full, (uint32_t)k & 1u);
                VTRACE(16, k);
                for (int t = it.t0; t < it.t1; ++t, ++g) {
                    const int b = g & 1;
                    if (g >= 2) ptx::mbar_wait(&bars->s_free[b], (uint32_t)((g >> 1) - 1) & 1u);
                    VTRACE(7, g);
                    ptx::mbar_wait(&bars->k_full[kst], kph);
                    VTRACE(8, g);
                    ptx::tc_fence_after();
                    if constexpr (PAIR) {
                        issue_S2(kst, tmem + b * 128, sQa, sKa);
                        ptx::mma2_commit_mc_w(&bars->s_full[b]);
                        ptx::mma2_commit_mc_w(&bars->k_empty[kst]);
                        if (t == it.t1 - 1) ptx::mma2_commit_mc_w(&bars->q_empty);
                    } else {
                        issue_S(kst, tmem + b * 128, sQa, sKa);
                        ptx::mma_commit_w(&bars->s_full[b]);
                        if constexpr (C > 1) ptx::mma_commit_mc_w(&bars->k_empty[kst], kMask);
                        else ptx::mma_commit_w(&bars->k_empty[kst]);
                        if (t == it.t1 - 1) ptx::mma_commit_w(&bars->q_empty);  // Q free once its last S completes
                    }
                    VTRACE(0, g);
                    if (++kst == KST) { kst = 0; kph ^= 1; }
                }
            }
        } else {
            // ============================ PV MMAs ============================
            const uint32_t sVa = base + (PAIR ? kPairVOff : kVOff);
            int vst = 0, g = 0;
            uint32_t vph = 0;
            for (int k = 0; fetch_item(bars, ring, k, it); ++k) {
                VTRACE(11, g);
                if (k >= 1) ptx::mbar_wait(&bars->o_empty, (uint32_t)(k - 1) & 1u);  // epilogue read O
                VTRACE(18, k);
                for (int t = it.t0; t < it.t1; ++t, ++g) {
                    const int b = g & 1;
                    VTRACE(9, g);
                    ptx::mbar_wait(&bars->v_full[vst], vph);
                    VTRACE(10, g);
                    ptx::mbar_wait(&bars->p_full[b], (uint32_t)(g >> 1) & 1u);
                    VTRACE(1, g);
                    ptx::tc_fence_after();
                    if constexpr (PAIR) {
                        issue_PV2(vst, tmem + 256, tmem + 384 + b * 64, sVa, t > it.t0);
                        ptx::mma2_commit_mc_w(&bars->p_free[b]);
                        ptx::mma2_commit_mc_w(&bars->pv_done);
                        ptx::mma2_commit_mc_w(&bars->v_empty[vst]);
                        if (t == it.t1 - 1) ptx::mma2_commit_mc_w(&bars->o_full);
                    } else {
                        issue_PV(vst, tmem + 256, tmem + 384 + b * 64, sVa, t > it.t0);
                        ptx::mma_commit_w(&bars->p_free[b]);
                        ptx::mma_commit_w(&bars->pv_done);
                        if constexpr (C > 1) ptx::mma_commit_mc_w(&bars->v_empty[vst], kMask);
                        else ptx::mma_commit_w(&bars->v_empty[vst]);
                        if (t == it.t1 - 1) ptx::mma_commit_w(&bars->o_full);
                    }
                    VTRACE(2, g);
                    if (++vst == VST) { vst = 0; vph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp < 12) {
        if constexpr (kSmxRegs > 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSmxRegs));
        // ============================ softmax (two threads per row) ============================
        const int wq = warp % 4;
        const int rh = (warp - 4) / 4;             // row half of the lane quarter
        const int ch = lane >> 4;                  // key half of the row: keys [64 ch, 64 ch + 64)
        const int row = wq * 32 + rh * 16 + (lane & 15);  // row within the CTA's Q tile = TMEM lane
        const uint32_t lane_bits = (uint32_t)(wq * 32 + rh * 16) << 16;
        const uint32_t tO = tmem + lane_bits + 256;
        const float sl2 = P.scale_log2;
        int g = 0;
        for (int k = 0; fetch_item(bars, ring, k, it); ++k) {
            const int L = it.len;
            float m_used = -INFINITY, l = 0.f;
            for (int t = it.t0; t < it.t1; ++t, ++g) {
                const int b = g & 1;
                const uint32_t tS = tmem + lane_bits + b * 128;
                const uint32_t tP = tmem + lane_bits + 384 + b * 64;
                if (row == 0 && ch == 0) {
                    VTRACE(26, g);
                    VPROBE(0, g, &bars->s_full[b], (uint32_t)(g >> 1) & 1u);
                }
                ptx::mbar_wait(&bars->s_full[b], (uint32_t)(g >> 1) & 1u);
                if (row == 0 && ch == 0) VTRACE(3, g);
                ptx::tc_fence_after();
                uint32_t r[2][32];
                ptx::tmem_ld16x32bx2_x32<64>(tS, r[0]);
                ptx::tmem_ld16x32bx2_x32<64>(tS + 32, r[1]);
                ptx::tmem_wait_ld();
                ptx::reg_fence(r[0]);
                ptx::reg_fence(r[1]);
                ptx::tc_fence_before();
                if constexpr (PAIR) warp_arrive_leader(&bars->s_free[b], rank);
                else ptx::mbar_arrive(&bars->s_free[b]);  // S buffer b may take S(g + 2)
                if (row == 0 && ch == 0) VTRACE(12, g);
                const int valid = L - t * kTile - ch * 64;  // valid keys among this thread's 64
                if (valid < 64) {
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c * 32 + j >= valid) r[c][j] = __float_as_uint(-INFINITY);
                }
                // row max: 4 independent FMNMX3 chains over this thread's keys, then the row's other thread
                float m4[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int c = a >> 1, o = (a & 1) * 16;
                    float m = ptx::max3(__uint_as_float(r[c][o]), __uint_as_float(r[c][o + 1]),
                                        __uint_as_float(r[c][o + 2]));
#pragma unroll
                    for (int j = 3; j < 15; j += 2)
                        m = ptx::max3(m, __uint_as_float(r[c][o + j]), __uint_as_float(r[c][o + j + 1]));
                    m4[a] = fmaxf(m, __uint_as_float(r[c][o + 15]));
                }
                float mh = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                mh = fmaxf(mh, __shfl_xor_sync(0xffffffffu, mh, 16));
                const float mxs = mh * sl2;
                if (row == 0 && ch == 0) VTRACE(13, g);
                const bool need = mxs > m_used + kRescaleThreshold;
                const bool any = __any_sync(0xffffffffu, need);
                const float m_old = m_used;
                if (any) m_used = fmaxf(m_used, mxs);
                // P buffer b is free once PV(g - 2) has read it
                if (row == 0 && ch == 0 && g >= 2) {
                    VTRACE(27, g);
                    VPROBE(1, g, &bars->p_free[b], (uint32_t)((g >> 1) - 1) & 1u);
                }
                if (g >= 2) ptx::mbar_wait(&bars->p_free[b], (uint32_t)((g >> 1) - 1) & 1u);
                if (row == 0 && ch == 0) VTRACE(14, g);
                ptx::tc_fence_after();
                if (lane == 0 && wq == 0) VTRACE(22 + 2 * rh, g);
                const float lt = exp_half(r, sl2, -m_used, tP);
                if (lane == 0 && wq == 0) VTRACE(23 + 2 * rh, g);
                if (any && t > it.t0) {
                    // O holds this item's sum up to PV(g - 1): wait for it, then rescale this row's
                    // 128 columns in place, 64 per thread (PV(g) cannot start before the p_full arrive)
                    ptx::mbar_wait(&bars->pv_done, (uint32_t)(g - 1) & 1u);
                    ptx::tc_fence_after();
                    const float f = ptx::ex2(m_old - m_used);
                    l *= f;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t o[32];
                        ptx::tmem_ld16x32bx2_x32<64>(tO + c * 32, o);
                        ptx::tmem_wait_ld();
                        ptx::reg_fence(o);
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * f);
                        ptx::tmem_st16x32bx2_x32<64>(tO + c * 32, o);
                    }
                }
                if (row == 0 && ch == 0) VTRACE(15, g);
                l += lt;
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                if constexpr (PAIR) warp_arrive_leader(&bars->p_full[b], rank);
                else ptx::mbar_arrive(&bars->p_full[b]);
                if (row == 0 && ch == 0) VTRACE(4, g);
            }
            // the row's sum (both threads) and running max to the epilogue (single buffer: wait until
            // it took the previous item's)
            l += __shfl_xor_sync(0xffffffffu, l, 16);
            if (k >= 1) ptx::mbar_wait(&bars->ml_empty, (uint32_t)(k - 1) & 1u);
            if (ch == 0) {
                bars->ml[0][row] = l;
                bars->ml[1][row] = m_used;
            }
            ptx::mbar_arrive(&bars->ml_full);
        }
    } else {
        if constexpr (kEpiRegs > 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
        else if constexpr (kEpiRegs < 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
        // ============================ epilogue ============================
        const int wq = warp % 4;
        const int row = wq * 32 + lane;
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const uint32_t tO = tmem + lane_bits + 256;
        bool have = fetch_item(bars, ring, 0, it);
        for (int k = 0; have; ++k) {
            Item nxt;  // the next item is fetched ahead (its ring entry is released early)
            const bool have_n = fetch_item(bars, ring, k + 1, nxt);
            ptx::mbar_wait(&bars->ml_full, (uint32_t)k & 1u);
            if (row == 0) VTRACE(20, k);
            const float lsum = bars->ml[0][row];
            const float inv_l = 1.f / lsum;
            const float lse = (bars->ml[1][row] + __log2f(lsum)) * kLn2;
            ptx::mbar_arrive(&bars->ml_empty);
            ptx::mbar_wait(&bars->o_full, (uint32_t)k & 1u);
            if (row == 0) VTRACE(21, k);
            ptx::tc_fence_after();
            const int urow = rank * 128 + row;  // row within the unit
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
                if (P.outs.codes) {
                    store_rows_coalesced<PEERS>(P, peers, it, cid, rank * 128 + wq * 32, kRows, tO, v, 0);
                    // O is read (and its round trip done): the next item's PV may start while this
                    // thread exports the row from registers (NEXT-1 int8 export, the row as stored)
                    ptx::tc_fence_before();
                    if constexpr (PAIR) warp_arrive_leader(&bars->o_empty, rank);
                    else ptx::mbar_arrive(&bars->o_empty);
                    const int h = it.hg / P.G, g = it.hg % P.G;
                    const size_t orow = ((size_t)it.u * P.S + g * kRows + urow) * P.H + h;
                    i8_export_row_bf16(v, P.outs.codes + orow * 128, P.outs.qscale + orow, P.outs.qzp + orow);
                } else {
                    store_rows_coalesced<PEERS>(P, peers, it, cid, rank * 128 + wq * 32, kRows, tO, v, 0);
                    ptx::tc_fence_before();
                    if constexpr (PAIR) warp_arrive_leader(&bars->o_empty, rank);
                    else ptx::mbar_arrive(&bars->o_empty);
                }
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
                    store_rows_coalesced<PEERS>(P, peers, it, cid, rank * 128 + wq * 32, kRows, tO + hh * 64, v, hh * 256);
                }
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[32];
                    ptx::tmem_ld32_sync(tO + c * 32, o);
                    float of[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) of[j] = __uint_as_float(o[j]) * inv_l;
                    store_row<PEERS>(P, peers, it, cid, urow, of, c * 32, kRows);
                }
            }
            if (!(coalesced && out16)) {  // (the bf16 coalesced path released O above)
                ptx::tc_fence_before();
                if constexpr (PAIR) warp_arrive_leader(&bars->o_empty, rank);
                else ptx::mbar_arrive(&bars->o_empty);
            }
            store_lse<PEERS>(P, peers, it, cid, urow, lse, kRows);
            if (row == 0) VTRACE(19, k);
            it = nxt;
            have = have_n;
        }
    }
    ptx::tc_fence_before();
    if constexpr (C > 1) ptx::cluster_sync();  // no CTA leaves while a peer may still multicast into it
    else __syncthreads();
#ifdef VISTA_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 256) {
        g_vista_cta[blockIdx.x][1] = ptx::globaltimer_ns();
        g_vista_cta[blockIdx.x][3] = clock64();
    }
#endif
    if (warp == 1) {
        if constexpr (PAIR) ptx::tmem_dealloc2(tmem, kTmemCols);
        else ptx::tmem_dealloc(tmem, kTmemCols);
    }
}

}  // namespace

// Cluster size for S query rows: the largest power of two <= 8 dividing S / 128 (K/V slices of
// 128 / C rows stay whole 8-row swizzle atoms).
// VISTA_SOFTMAX_CMAX caps the cluster size (A/B: a cluster of 4 fits 132 of the 148 SMs).
static int cluster_cap() {
    static const int v = [] {
        const char* e = getenv("VISTA_SOFTMAX_CMAX");
        const int c = e ? atoi(e) : 8;
        return (c == 1 || c == 2 || c == 4) ? c : 8;
    }();
    return v;
}
int sm100_softmax_cluster(int S) {
    const int tiles = S / 128;
    const int cap = cluster_cap();
    int c = 1;
    while (c < cap && tiles % (2 * c) == 0) c *= 2;
    return c;
}

template <int C>
static cudaLaunchConfig_t cluster_config(dim3 grid, cudaStream_t stream, cudaLaunchAttribute* attrs) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = stream;
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = C;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    return cfg;
}

// CTA-pair mode (cta_group::2) for clusters of two (S = 256 per unit): VISTA_SOFTMAX_PAIR=1 selects it
// instead of the multicast kernel.  Parity-green, but measured 4% slower at c2, so
// it is off by default.
static bool use_pair() {
    static const int v = [] {
        const char* e = getenv("VISTA_SOFTMAX_PAIR");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    return v != 0;
}

// Persistent grid: the number of clusters of C CTAs that can be co-resident on this device.
template <int C, bool PAIR>
static int max_clusters(int num_sms) {
    if (C == 1) return num_sms;
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        const void* fn = reinterpret_cast<const void*>(sm100_softmax_kernel<C, PAIR>);
        if (set_smem_attr(fn, kSmem) != cudaSuccess)
            return num_sms / C;  // no device (host-only sizing): the upper bound
        cudaLaunchAttribute attrs[2];
        cudaLaunchConfig_t cfg = cluster_config<C>(dim3(C * (num_sms / C)), nullptr, attrs);
        cfg.numAttrs = 1;  // cluster dimension only
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) n = num_sms / C;
        cache[dev] = std::min(n, num_sms / C);
    }
    return cache[dev];
}

int sm100_softmax_num_clusters(const Problem& p) {
    switch (sm100_softmax_cluster(p.S)) {
        case 8: return max_clusters<8, false>(p.num_sms);
        case 4: return max_clusters<4, false>(p.num_sms);
        case 2: return use_pair() ? max_clusters<2, true>(p.num_sms) : max_clusters<2, false>(p.num_sms);
        default: return max_clusters<1, false>(p.num_sms);
    }
}

template <int C, bool PAIR>
static cudaError_t launch_c(const Problem& p, const Workspace& w, char* ws) {
    CUtensorMap mq, mk, mv;
    // K / V boxes: the rows one CTA loads per tile (pair: 64 keys of K, all 128 keys of V for its
    // 64 channels; multicast: 128 / C rows of each)
    const int krows = PAIR ? 64 : 128 / C, vrows = PAIR ? 128 : 128 / C;
    if (!make_q_map(&mq, p.q, p.S, p.H, p.B, p.q_user_stride) || !make_kv_map_rows(&mk, p.k, p.total_len, p.H, krows) ||
        !make_kv_map_rows(&mv, p.v, p.total_len, p.H, vrows))
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
    P.G = p.S / (C * 128);
    P.scale_log2 = p.scale * kLog2e;
    P.q_per_user = p.q_user_stride != 0;
    P.groups = (P.G > 1 && w.num_ctas % P.G == 0) ? P.G : 1;
    P.out_v8 = (reinterpret_cast<uintptr_t>(p.outs.out) & 31) == 0;
    for (int r = 0; r < p.peers.n; ++r)  // fused exchange: the rows also go to every receive buffer
        P.out_v8 = P.out_v8 && (reinterpret_cast<uintptr_t>(p.peers.o[r]) & 31) == 0;
    P.slot_v8 = (reinterpret_cast<uintptr_t>(P.slot_o) & 31) == 0;
    // the fused-exchange instantiation only for the softmax partial with peers (not the CTA-pair mode)
    const bool peers = p.outs.mode == OUT_PARTIAL && p.peers.n > 0;
    if (PAIR && peers) return cudaErrorNotSupported;  // the CTA-pair mode (off by default) has no fused exchange
    const void* fn = peers ? reinterpret_cast<const void*>(sm100_softmax_kernel<C, PAIR, !PAIR>)
                           : reinterpret_cast<const void*>(sm100_softmax_kernel<C, PAIR>);
    const cudaError_t attr = set_smem_attr(fn, kSmem);
    if (attr != cudaSuccess) return attr;
    cudaLaunchAttribute attrs[2];
    cudaLaunchConfig_t cfg = cluster_config<C>(dim3(C * w.num_ctas), p.stream, attrs);
#ifdef VISTA_NO_PDL
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
#endif
    if (peers) return cudaLaunchKernelEx(&cfg, sm100_softmax_kernel<C, PAIR, !PAIR>, mq, mk, mv, P, p.peers);
    return cudaLaunchKernelEx(&cfg, sm100_softmax_kernel<C, PAIR>, mq, mk, mv, P, p.peers);
}

#ifdef VISTA_TRACE
extern "C" int vista_debug_trace(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_vista_trace, bytes < sizeof(g_vista_trace) ? bytes : sizeof(g_vista_trace));
}
#endif

cudaError_t launch_sm100_softmax(const Problem& p, const Workspace& w, char* ws) {
    switch (sm100_softmax_cluster(p.S)) {
        case 8: return launch_c<8, false>(p, w, ws);
        case 4: return launch_c<4, false>(p, w, ws);
        case 2: return use_pair() ? launch_c<2, true>(p, w, ws) : launch_c<2, false>(p, w, ws);
        default: return launch_c<1, false>(p, w, ws);
    }
}

}  // namespace vista

#ifdef VISTA_TRACE
extern "C" int vista_debug_probe(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, vista::g_vista_probe, bytes < sizeof(vista::g_vista_probe) ? bytes : sizeof(vista::g_vista_probe));
}
extern "C" int vista_debug_cta_times(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, vista::g_vista_cta, bytes < sizeof(vista::g_vista_cta) ? bytes : sizeof(vista::g_vista_cta));
}
extern "C" int vista_debug_softmax_clusters(int S) {
    vista::Problem p{};
    p.S = S;
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    p.num_sms = n;
    return vista::sm100_softmax_num_clusters(p);
}
#endif
