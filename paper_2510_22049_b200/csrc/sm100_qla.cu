// sm100_qla.cu -- QLA state on B200: Z_uh = sum_j phi1(k_j)^T v_j  (d x d, fp32 in TMEM).
//
// "phi(K[S])^T V[S]" (Sec. 3.2.2); App. B: "sum_j K[S]_j^T V[S]_j can be computed
// first".  The state GEMM has M = d (c1), N = d (c2), K = history items, so each
// 128-item tile is one 128x128x128 tcgen05 MMA chain with BOTH operands MN-major straight out of
// the TMA tiles (no transpose):  A[c1][j] = phi1(K)[j][c1],  B[j][c2] = V[j][c2].
// HBM-bound (2 d^2 = 32768 flop per 512 B of K+V), so the design goal is to keep the TMA ring
// full: 3 x 64 KB stages, one CTA per SM, stream-K flat tile ranges (work.cuh).
//
//   warp 0        TMA producer (K, V tiles of 128 items x 128 channels, bf16, 128-B swizzle)
//   warp 1        MMA issuer (one thread), Z double-buffered in TMEM (2 x 128 columns)
//   warps 4..11   phi1 transform of the K tile in shared memory (bf16 -> f32 -> phi1 -> bf16,
//                 rows past the user's end zeroed AFTER activation: phi1(0) != 0 for shifted ELU),
//                 then the epilogue: Z rows (TMEM lane = c1) -> zbuf[u,h] or a split slot.
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100_ptx.cuh"
#include "qla_common.cuh"
#include "work.cuh"

namespace vista {

bool make_kv_map(CUtensorMap* map, const void* base, int64_t total_len, int H);

namespace {

constexpr int kHalfBytes = 128 * 128;
constexpr int kTileBytes = 2 * kHalfBytes;
constexpr int kStages = 3;
constexpr int kStageBytes = 2 * kTileBytes;
constexpr int kBarOff = kStages * kStageBytes;
constexpr int kSmem = kBarOff + 256 + 1024;
constexpr int kXformWarps = 8;
constexpr int kThreads = 128 + kXformWarps * 32;
constexpr int kTmemCols = 256;

struct Bars {
    uint64_t kv_full[kStages], k_ready[kStages], kv_empty[kStages];
    uint64_t z_full[2], z_empty[2];
    uint32_t tmem_base;
};

struct Params {
    const int64_t* offsets;
    const int64_t* uts;
    int* slot_unit;
    float* slot_o;
    float* zbuf;      // complete units' Z (f32) -- unless wbuf is set
    uint8_t* wbuf;    // fused finalize: complete units' W = phi2(Z / N) (bf16 MMA operand) instead
    int B, H, phi1, phi2, normalize;
};

__device__ __forceinline__ float phi(int kind, float x) {
    if (kind == VISTA_ACT_SILU) {
        float t;
        asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
        return x * fmaf(0.5f, t, 0.5f);  // x * sigmoid(x)
    }
    if (kind == VISTA_ACT_SHIFTED_ELU) return x >= 1.f ? x : ptx::ex2((x - 1.f) * 1.4426950408889634f);
    return x;
}

__device__ __forceinline__ uint32_t phi_bf16x2(int kind, uint32_t w) {
    const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xFFFF0000u);
    return ptx::pack_bf16x2(phi(kind, lo), phi(kind, hi));
}

template <int PHI>
__device__ __forceinline__ uint32_t phi2x(uint32_t w) {
    if constexpr (PHI == VISTA_ACT_SILU) return qla_silu_bf16x2(w);
    else if constexpr (PHI == VISTA_ACT_SHIFTED_ELU) return phi_bf16x2(VISTA_ACT_SHIFTED_ELU, w);
    else return w;
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

// phi1 over one 128 x 128 bf16 K tile in shared memory (in place, layout-agnostic: the 128-B
// swizzle only permutes 16-B chunks within a row), rows >= valid zeroed AFTER activation.
// 256 threads x 8 chunks of 16 B; all loads first for ILP.
template <int PHI>
__device__ __forceinline__ void phi_tile(uint32_t tile, int xt, int64_t valid) {
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = lds128(tile + (uint32_t)(xt + i * 256) * 16);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int c = xt + i * 256;
        const int j = (c & 1023) >> 3;  // 128-B line = history row within the tile
        if (j >= valid) {
            v[i] = make_uint4(0, 0, 0, 0);
        } else if constexpr (PHI != VISTA_ACT_IDENTITY) {
            v[i].x = phi2x<PHI>(v[i].x);
            v[i].y = phi2x<PHI>(v[i].y);
            v[i].z = phi2x<PHI>(v[i].z);
            v[i].w = phi2x<PHI>(v[i].w);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) sts128(tile + (uint32_t)(xt + i * 256) * 16, v[i]);
}

// Z (+)= phi1(K)^T V for one staged tile: A = phi1(K) [j][c1] read as MN-major (M = c1),
// B = V [j][c2] MN-major (N = c2); 8 k-steps of 16 history rows.  Compile-time stage / buffer so
// the descriptors stay in uniform registers (see sm100_softmax.cu).
template <int ZB, int ST>
__device__ __forceinline__ void issue_Z_t(uint32_t tmem, uint32_t base, bool acc) {
    constexpr uint32_t idZ = ptx::idesc_bf16_f32(128, 128, 1, 1);
    const uint32_t ka = base + ST * kStageBytes, va = ka + kTileBytes;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
        ptx::mma_ss_w(tmem + ZB * 128, ptx::sdesc_sw128(ka + kk * 2048, kHalfBytes, 1024),
                      ptx::sdesc_sw128(va + kk * 2048, kHalfBytes, 1024), idZ, (acc || kk > 0) ? 1u : 0u);
}
template <int ZB>
__device__ __forceinline__ void issue_Z_s(int st, uint32_t tmem, uint32_t base, bool acc) {
    switch (st) {
        case 0: issue_Z_t<ZB, 0>(tmem, base, acc); break;
        case 1: issue_Z_t<ZB, 1>(tmem, base, acc); break;
        default: issue_Z_t<ZB, 2>(tmem, base, acc); break;
    }
}

// PEERS: the fused split-L exchange (vista_summarize_partial_peers, QLA) -- complete units' Z to every
// rank's receive buffer; a separate instantiation so the default kernel carries none of it
template <int PHI1, bool PEERS = false>
__global__ void __launch_bounds__(kThreads, 1)
    sm100_qla_state_kernel(const __grid_constant__ CUtensorMap mapK, const __grid_constant__ CUtensorMap mapV,
                           const Params P, const __grid_constant__ PeerSpec peers) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int cta = blockIdx.x, num_ctas = gridDim.x;
    const int HG = P.H;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bars->kv_full[s], 1);
            ptx::mbar_init(&bars->k_ready[s], kXformWarps * 32);
            ptx::mbar_init(&bars->kv_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bars->z_full[b], 1);
            ptx::mbar_init(&bars->z_empty[b], kXformWarps * 32);
        }
        ptx::fence_mbar_init();
        int s0, s1;
        partial_slots(P.uts, P.B, HG, cta, num_ctas, s0, s1);
        P.slot_unit[2 * cta] = s0;
        P.slot_unit[2 * cta + 1] = s1;
    }
    if (warp == 1) ptx::tmem_alloc(&bars->tmem_base, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;");  // PDL: the slot merge may start its prologue
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, bars->tmem_base, 0);

    ItemIter iter;
    iter.init(P.uts, P.B, HG, cta, num_ctas);
    Item it;

    if (warp == 0) {
        // ============================ TMA producer (warp-wide, one elected lane issues) ============
        ptx::tma_prefetch(&mapK);
        ptx::tma_prefetch(&mapV);
        const uint64_t pol = ptx::policy_evict_first();
        int stage = 0;
        uint32_t phase = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int h = it.hg;
            const int64_t row0 = P.offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->kv_empty[stage], phase ^ 1);
                ptx::mbar_arrive_expect_tx_w(&bars->kv_full[stage], kStageBytes);
                uint8_t* sk = smem + stage * kStageBytes;
                const int32_t row = (int32_t)(row0 + (int64_t)t * kTile);
                for (int half = 0; half < 2; ++half) {
                    ptx::tma_load_3d_w(sk + half * kHalfBytes, &mapK, &bars->kv_full[stage], half * 64, h, row, pol);
                    ptx::tma_load_3d_w(sk + kTileBytes + half * kHalfBytes, &mapV, &bars->kv_full[stage], half * 64,
                                       h, row, pol);
                }
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer (warp-wide) ============================
        const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
        int stage = 0;
        uint32_t phase = 0;
        uint32_t zuse[2] = {0, 0};
        int k = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int zb = k & 1;
            ptx::mbar_wait(&bars->z_empty[zb], (zuse[zb] & 1) ^ 1);
            ++zuse[zb];
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->k_ready[stage], phase);
                ptx::tc_fence_after();
#ifndef VISTA_EXP_QLA_NOMMA
                if (zb == 0) issue_Z_s<0>(stage, tmem, base, t > it.t0);
                else issue_Z_s<1>(stage, tmem, base, t > it.t0);
#endif
                ptx::mma_commit_w(&bars->kv_empty[stage]);
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            ptx::mma_commit_w(&bars->z_full[zb]);
            ++k;
        }
    } else if (warp >= 4) {
        const int xt = threadIdx.x - 128;  // 0 .. 255
        const int wq = warp % 4;
        const int chalf = (warp - 4) / 4;  // epilogue: columns [64*chalf, 64*chalf + 64)
        const uint32_t lane_bits = (uint32_t)(wq * 32) << 16;
        const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
        int stage = 0;
        uint32_t phase = 0;
        uint32_t zphase[2] = {0, 0};
        int k = 0;
        while (iter.next(it, P.uts, P.B, HG)) {
            const int64_t L = P.offsets[it.u + 1] - P.offsets[it.u];
            for (int t = it.t0; t < it.t1; ++t) {
                ptx::mbar_wait(&bars->kv_full[stage], phase);
                const int64_t valid = L - (int64_t)t * kTile;
#ifdef VISTA_EXP_QLA_NOXFORM
                if (false) {
#else
                if (PHI1 != VISTA_ACT_IDENTITY || valid < kTile) {
#endif
                    phi_tile<PHI1>(base + stage * kStageBytes, xt, valid);
                    ptx::fence_proxy_async_smem();
                }
                ptx::mbar_arrive(&bars->k_ready[stage]);
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            // epilogue
            const int zb = k & 1;
            ptx::mbar_wait(&bars->z_full[zb], zphase[zb]);
            zphase[zb] ^= 1;
            ptx::tc_fence_after();
            const int c1 = wq * 32 + lane;
            if (P.wbuf && item_complete(it)) {
                // W[c1][c2] = phi2(Z[c1][c2] / N) as the bf16 B operand of the finalize GEMM
                // (MN-major, 128-B swizzled halves of 64 columns: qla_w_swz)
                const float inv = (P.normalize && L > 0) ? 1.f / (float)L : 1.f;
                uint8_t* wdst = P.wbuf + (size_t)(it.u * HG + it.hg) * kTileBytes;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t r[32];
                    ptx::tmem_ld32_sync(tmem + lane_bits + zb * 128 + chalf * 64 + c * 32, r);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 pk;
                        uint32_t* pw = &pk.x;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            // same packed activation as the K transform (phi2x): W is a bf16 operand
                            const uint32_t zz = ptx::pack_bf16x2(__uint_as_float(r[8 * q + 2 * e]) * inv,
                                                                 __uint_as_float(r[8 * q + 2 * e + 1]) * inv);
                            pw[e] = P.phi2 == VISTA_ACT_SILU ? qla_silu_bf16x2(zz)
                                  : P.phi2 == VISTA_ACT_SHIFTED_ELU ? phi_bf16x2(VISTA_ACT_SHIFTED_ELU, zz)
                                                                    : zz;
                        }
                        *reinterpret_cast<uint4*>(wdst + qla_w_swz(c1, chalf * 64 + c * 32 + 8 * q)) = pk;
                    }
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&bars->z_empty[zb]);
                ++k;
                continue;
            }
            float* dst;
            const bool comp = item_complete(it);
            const size_t zoff = ((size_t)(it.u * HG + it.hg) * 128 + c1) * 128;
            if (comp) dst = P.zbuf + zoff;
            else dst = P.slot_o + ((size_t)item_slot(it, cta) * 128 + c1) * 128;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t r[32];
                ptx::tmem_ld32_sync(tmem + lane_bits + zb * 128 + chalf * 64 + c * 32, r);
                if (PEERS && comp) {  // fused exchange: the row of Z into every rank's receive buffer
#pragma unroll
                    for (int q = 0; q < kMaxExchangeRanks; ++q) {
                        if (q >= peers.n) break;
                        float4* d4 = reinterpret_cast<float4*>(peers.o[q] + zoff + chalf * 64 + c * 32);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            d4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                                __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
                    }
                    continue;
                }
                float4* d4 = reinterpret_cast<float4*>(dst + chalf * 64 + c * 32);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    d4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                        __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bars->z_empty[zb]);
            ++k;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace

template <int PHI1>
static cudaError_t launch_phi(const Problem& p, const Workspace& w, const CUtensorMap& mk, const CUtensorMap& mv,
                              const Params& P) {
    const bool peers = p.outs.mode == OUT_PARTIAL && p.peers.n > 0 && P.wbuf == nullptr;
    const void* fn = peers ? reinterpret_cast<const void*>(sm100_qla_state_kernel<PHI1, true>)
                           : reinterpret_cast<const void*>(sm100_qla_state_kernel<PHI1>);
    const cudaError_t attr = set_smem_attr(fn, kSmem);
    if (attr != cudaSuccess) return attr;
    if (peers) sm100_qla_state_kernel<PHI1, true><<<w.num_ctas, kThreads, kSmem, p.stream>>>(mk, mv, P, p.peers);
    else sm100_qla_state_kernel<PHI1><<<w.num_ctas, kThreads, kSmem, p.stream>>>(mk, mv, P, p.peers);
    return cudaGetLastError();
}

cudaError_t launch_sm100_qla_state(const Problem& p, const Workspace& w, char* ws, float* zbuf, uint8_t* wbuf) {
    CUtensorMap mk, mv;
    if (!make_kv_map(&mk, p.k, p.total_len, p.H) || !make_kv_map(&mv, p.v, p.total_len, p.H))
        return cudaErrorInvalidValue;
    Params P;
    P.offsets = p.offsets;
    P.uts = reinterpret_cast<const int64_t*>(ws + w.uts_off);
    P.slot_unit = reinterpret_cast<int*>(ws + w.slot_unit_off);
    P.slot_o = reinterpret_cast<float*>(ws + w.slot_o_off);
    P.zbuf = zbuf;
    P.wbuf = wbuf;
    P.B = p.B;
    P.H = p.H;
    P.phi1 = p.phi1;
    P.phi2 = p.phi2;
    P.normalize = p.normalize;
    return p.phi1 == VISTA_ACT_SILU ? launch_phi<VISTA_ACT_SILU>(p, w, mk, mv, P)
         : p.phi1 == VISTA_ACT_SHIFTED_ELU ? launch_phi<VISTA_ACT_SHIFTED_ELU>(p, w, mk, mv, P)
                                           : launch_phi<VISTA_ACT_IDENTITY>(p, w, mk, mv, P);
}

}  // namespace vista
