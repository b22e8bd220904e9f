// kernels_misc.cu -- the small kernels around the tiled sm100 kernels, and the SIMT path.
//
//   user_tiles_kernel        offsets -> per-user tile prefix (work decomposition), empty-user fill
//   merge_softmax_slots      split-L LSE merge of intra-GPU partial slots (flash-decoding combine)
//   merge_qla_slots          split-L sum of QLA state partials (plain sum, ascending CTA order)
//   merge_softmax_parts      LSE merge of P stacked partials (multi-GPU history-length shards)
//   qla_finalize_kernel      O = phi1(Q) phi2((sum_p Z_p) / N_u)
//   simt_softmax_kernel      fp32-accumulate SIMT seed-row softmax (f32 inputs, or d / S the tiled
//                            kernel does not cover); online softmax over 32-key chunks
//   simt_qla_state_kernel    Z = sum_j phi1(k_j)^T v_j with FFMA (f32 inputs or d != 128)
#include <cuda_bf16.h>
#include <math.h>

#include "internal.h"
#include "int8_export.cuh"
#include "qla_common.cuh"
#include "sm100_ptx.cuh"

namespace vista {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ float act(int kind, float x) {
    // phi: identity; SiLU x*sigmoid(x); shifted ELU (x >= 1 -> x)
    if (kind == VISTA_ACT_SILU) return x / (1.f + __expf(-x));
    if (kind == VISTA_ACT_SHIFTED_ELU) return x >= 1.f ? x : __expf(x - 1.f);
    return x;
}

template <typename T>
__device__ __forceinline__ float ld(const T* p);
template <>
__device__ __forceinline__ float ld<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Store one normalized output element (row i of user u, head h, channel c) per OutSpec.
__device__ __forceinline__ void out_store(const OutSpec& o, int S, int H, int d, int u, int h, int i, int c, float val) {
    if (o.mode == OUT_PARTIAL) {
        reinterpret_cast<float*>(o.out)[(((size_t)u * H + h) * S + i) * d + c] = val;
    } else {
        const size_t idx = (((size_t)u * S + i) * H + h) * d + c;
        if (o.out_bf16) reinterpret_cast<__nv_bfloat16*>(o.out)[idx] = __float2bfloat16_rn(val);
        else reinterpret_cast<float*>(o.out)[idx] = val;
    }
}
__device__ __forceinline__ void lse_store(const OutSpec& o, int S, int H, int u, int h, int i, float val) {
    if (o.lse) o.lse[((size_t)u * H + h) * S + i] = val;
}

// ---------------------------------------------------------------------------------------------
#ifdef VISTA_TRACE
__device__ unsigned long long g_scan_end;  // globaltimer when the last tile scan finished
}  // namespace
}  // namespace vista
extern "C" unsigned long long vista_debug_scan_end() {
    unsigned long long t = 0;
    cudaMemcpyFromSymbol(&t, vista::g_scan_end, sizeof(t));
    return t;
}
namespace vista {
namespace {
#endif
__global__ void user_tiles_kernel(const int64_t* __restrict__ offsets, int B, int64_t* __restrict__ uts, OutSpec outs,
                                  int S, int H, int d, int softmax, float* __restrict__ zbuf,
                                  const __grid_constant__ PeerSpec pe) {
    __shared__ int64_t wsum[32];
    __shared__ int64_t carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    asm volatile("griddepcontrol.launch_dependents;");  // PDL: the main kernel may start its prologue
    // launched with PDL itself (its launch overlaps the previous kernel's tail): uts and the outputs
    // may still be read by that kernel, so wait for it before writing anything
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0) {
        carry = 0;
        uts[0] = 0;
    }
    __syncthreads();
    for (int base = 0; base < B; base += blockDim.x) {
        const int u = base + tid;
        int64_t T = 0;
        if (u < B) T = (offsets[u + 1] - offsets[u] + kTile - 1) / kTile;
        int64_t x = T;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int64_t w = (lane < (int)(blockDim.x / 32)) ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;  // inclusive warp prefix
        }
        __syncthreads();
        const int64_t incl = x + (warp > 0 ? wsum[warp - 1] : 0) + carry;
        if (u < B) uts[u + 1] = incl;
        __syncthreads();
        if (tid == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
    // empty users: softmax out = 0, lse = -inf (identity of the LSE merge); QLA Z = 0.
    // One warp per empty user (found with a block-wide ballot scan; no serial pass over B).
    const size_t n_sm = (size_t)S * H * d, n_z = (size_t)H * d * d;
    for (int base = 0; base < B; base += blockDim.x) {
        const int u = base + tid;
        const bool empty = u < B && offsets[u + 1] == offsets[u];
        if (!__syncthreads_or(empty)) continue;
        unsigned m = __ballot_sync(0xffffffffu, empty);
        while (m) {  // this warp fills its own empty users
            const int uu = base + warp * 32 + __ffs(m) - 1;
            m &= m - 1;
            if (softmax) {
                if (outs.mode == OUT_PARTIAL && pe.n > 0) {  // fused exchange: every receive buffer
#pragma unroll
                    for (int r = 0; r < kMaxExchangeRanks; ++r) {
                        if (r >= pe.n) break;
                        for (size_t e = lane; e < n_sm; e += 32) pe.o[r][(size_t)uu * n_sm + e] = 0.f;
                        for (int e = lane; e < H * S; e += 32) pe.lse[r][(size_t)uu * H * S + e] = -INFINITY;
                    }
                    continue;
                }
                if (outs.mode == OUT_PARTIAL) {
                    float* o = reinterpret_cast<float*>(outs.out) + (size_t)uu * n_sm;
                    for (size_t e = lane; e < n_sm; e += 32) o[e] = 0.f;
                } else if (outs.out_bf16) {
                    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(outs.out) + (size_t)uu * n_sm;
                    for (size_t e = lane; e < n_sm; e += 32) o[e] = __float2bfloat16_rn(0.f);
                } else {
                    float* o = reinterpret_cast<float*>(outs.out) + (size_t)uu * n_sm;
                    for (size_t e = lane; e < n_sm; e += 32) o[e] = 0.f;
                }
                if (outs.lse)
                    for (int e = lane; e < H * S; e += 32) outs.lse[(size_t)uu * H * S + e] = -INFINITY;
                if (outs.codes) {  // zero rows export as code 0, scale 1e-12, zero point 0
                    for (size_t e = lane; e < n_sm; e += 32) outs.codes[(size_t)uu * n_sm + e] = 0;
                    for (int e = lane; e < S * H; e += 32) {
                        outs.qscale[(size_t)uu * S * H + e] = 1e-12f;
                        outs.qzp[(size_t)uu * S * H + e] = 0.f;
                    }
                }
            } else if (pe.n > 0 && outs.mode == OUT_PARTIAL) {  // fused exchange: every receive buffer
#pragma unroll
                for (int r = 0; r < kMaxExchangeRanks; ++r) {
                    if (r >= pe.n) break;
                    for (size_t e = lane; e < n_z; e += 32) pe.o[r][(size_t)uu * n_z + e] = 0.f;
                }
            } else if (zbuf) {
                for (size_t e = lane; e < n_z; e += 32) zbuf[(size_t)uu * n_z + e] = 0.f;
            }
        }
    }
#ifdef VISTA_TRACE
    __syncthreads();
    if (tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_scan_end = t;
    }
#endif
}

// ---------------------------------------------------------------------------------------------
// Is slot s the first slot of its unit's run?  (units are non-decreasing over valid slots)
__device__ __forceinline__ bool slot_is_head(const int* slot_unit, int s, int n) {
    for (int p = s - 1; p >= 0; --p) {
        const int m = slot_unit[p];
        if (m >= 0) return m != n;
    }
    return true;
}

// Vectorized store of 4 consecutive channels [c, c+4) of one output row.
__device__ __forceinline__ void out_store4(const OutSpec& o, int S, int H, int u, int h, int i, int c, float4 v) {
    if (o.mode == OUT_PARTIAL) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(o.out) + (((size_t)u * H + h) * S + i) * 128 + c) = v;
        return;
    }
    const size_t idx = (((size_t)u * S + i) * H + h) * 128 + c;
    if (o.out_bf16) {
        uint2 pk;
        pk.x = ptx::pack_bf16x2(v.x, v.y);
        pk.y = ptx::pack_bf16x2(v.z, v.w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(o.out) + idx) = pk;
    } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(o.out) + idx) = v;
    }
}

// The fused split-L exchange (PeerSpec, vista_summarize_partial_peers): a partial-mode row / lse to
// every rank's receive buffer instead of outs.
__device__ __forceinline__ void out_store4_p(const OutSpec& o, const PeerSpec& pe, int S, int H, int u, int h, int i,
                                             int c, float4 v) {
    if (o.mode == OUT_PARTIAL && pe.n > 0) {
        const size_t idx = (((size_t)u * H + h) * S + i) * 128 + c;
#pragma unroll
        for (int r = 0; r < kMaxExchangeRanks; ++r) {
            if (r >= pe.n) break;
            *reinterpret_cast<float4*>(pe.o[r] + idx) = v;
        }
        return;
    }
    out_store4(o, S, H, u, h, i, c, v);
}
__device__ __forceinline__ void lse_store_p(const OutSpec& o, const PeerSpec& pe, int S, int H, int u, int h, int i,
                                            float val) {
    if (o.mode == OUT_PARTIAL && pe.n > 0) {
#pragma unroll
        for (int r = 0; r < kMaxExchangeRanks; ++r) {
            if (r >= pe.n) break;
            pe.lse[r][((size_t)u * H + h) * S + i] = val;
        }
        return;
    }
    lse_store(o, S, H, u, h, i, val);
}

// LSE merge of the run of partial slots of each split unit.  Block = (slot s, 32 rows), 8 warps x
// 4 rows, lanes over 128 channels (float4); blocks whose slot does not start a run exit at once.
// Warp 0 lists the run's slots (lane-parallel over 32 positions at a time: a run ends at the first
// slot holding another unit, -1 slots are unused); then the members' 32-row slabs of o (16 KB
// each, contiguous) and lse stream into shared memory by bulk copy, two members per group, and
// the rows are combined with an online max (any run length).  One stage (33 KB of smem) keeps six
// blocks per SM resident, so the split units of a step merge in one wave; runs longer than two
// members (very long users) load their groups one after the other.
constexpr int kMergeRows = 32;
constexpr int kMergeMaxRun = 320;  // >= 2 * max CTAs a unit can span + 2
static_assert(kMergeMaxRun >= 2 * kMaxPersistentCtas + 2, "merge run list");
#ifndef VISTA_MERGE_STAGES
#define VISTA_MERGE_STAGES 1
#endif
constexpr int kMergeStages = VISTA_MERGE_STAGES;
struct MergeSmem {
    float o[kMergeStages][2][kMergeRows * 128];  // [stage][member][row * 128 + channel]
    float lse[kMergeStages][2][kMergeRows];
    uint64_t full[kMergeStages];
    int list[kMergeMaxRun];
    int count, n, head;
};

__global__ void __launch_bounds__(256) merge_softmax_slots_kernel(const int* __restrict__ slot_unit, int num_slots,
                                                                  const float* __restrict__ slot_o,
                                                                  const float* __restrict__ slot_lse, int rows,
                                                                  OutSpec outs, int S, int H, int G,
                                                                  const __grid_constant__ PeerSpec pe) {
    extern __shared__ __align__(128) uint8_t merge_smem_raw[];
    MergeSmem& sm = *reinterpret_cast<MergeSmem*>(merge_smem_raw);
    // PDL: launched while the summarization kernel runs; its slots are complete after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int s = blockIdx.x;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int row0 = blockIdx.y * kMergeRows;
    if (warp == 0) {
        // positions s-1 .. s+30 (lane 0 = the slot before s, for the run-head test)
        const int x = s - 1 + lane;
        int m = (x >= 0 && x < num_slots) ? slot_unit[x] : -2;
        const int n = __shfl_sync(0xffffffffu, m, 1);
        int prev = __shfl_sync(0xffffffffu, m, 0);
        if (prev == -1) {  // walk back over unused slots (rare)
            for (int p = s - 2; p >= 0; --p) {
                prev = slot_unit[p];
                if (prev >= 0) break;
            }
        }
        const bool head = n >= 0 && prev != n;
        int count = 0;
        if (head) {
            bool own = lane >= 1;
            for (int c0 = s - 1;; c0 += 32) {
                if (c0 != s - 1) {
                    const int xx = c0 + lane;
                    m = xx < num_slots ? slot_unit[xx] : -2;
                    own = true;
                }
                const unsigned stop = __ballot_sync(0xffffffffu, own && (m == -2 || (m >= 0 && m != n)));
                const int lim = stop ? __ffs(stop) - 1 : 32;
                const bool mem = own && lane < lim && m == n;
                const unsigned mask = __ballot_sync(0xffffffffu, mem);
                if (mem && count + __popc(mask & ((1u << lane) - 1)) < kMergeMaxRun)
                    sm.list[count + __popc(mask & ((1u << lane) - 1))] = c0 + lane;
                count = min(count + __popc(mask), kMergeMaxRun);
                if (stop) break;
            }
        }
        if (lane == 0) {
            sm.n = n;
            sm.head = head && row0 < rows;
            sm.count = count;
            for (int st = 0; st < kMergeStages; ++st) ptx::mbar_init(&sm.full[st], 1);
            ptx::fence_mbar_init();
        }
    }
    __syncthreads();
    if (!sm.head) return;
    const int n = sm.n, R = sm.count;
    const int ngroups = (R + 1) / 2;
    auto issue = [&](int gi) {  // thread 0: bulk copies of group gi (members 2 gi, 2 gi + 1)
        const int st = gi % kMergeStages;
        const int k = min(2, R - 2 * gi);
        ptx::mbar_arrive_expect_tx(&sm.full[st], (uint32_t)k * (kMergeRows * 128 * 4 + kMergeRows * 4));
        for (int j = 0; j < k; ++j) {
            const int slot = sm.list[2 * gi + j];
            ptx::bulk_g2s(ptx::smem_u32(sm.o[st][j]), slot_o + ((size_t)slot * rows + row0) * 128,
                          kMergeRows * 128 * 4, &sm.full[st]);
            ptx::bulk_g2s(ptx::smem_u32(sm.lse[st][j]), slot_lse + (size_t)slot * rows + row0, kMergeRows * 4,
                          &sm.full[st]);
        }
    };
    if (threadIdx.x == 0)
        for (int gi = 0; gi < kMergeStages && gi < ngroups; ++gi) issue(gi);
    float M[4], l[4];
    float4 acc[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        M[r] = -INFINITY;
        l[r] = 0.f;
        acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int gi = 0; gi < ngroups; ++gi) {
        const int st = gi % kMergeStages;
        const int k = min(2, R - 2 * gi);
        ptx::mbar_wait(&sm.full[st], (uint32_t)(gi / kMergeStages) & 1u);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int rl = warp * 4 + r;  // row within the block's 32
            const float l0 = sm.lse[st][0][rl];
            const float l1 = k > 1 ? sm.lse[st][1][rl] : -INFINITY;
            const float Mn = fmaxf(M[r], fmaxf(l0, l1));
            const float sc = __expf(M[r] - Mn);
            const float w0 = __expf(l0 - Mn), w1 = k > 1 ? __expf(l1 - Mn) : 0.f;
            const float4 o0 = reinterpret_cast<const float4*>(sm.o[st][0] + rl * 128)[lane];
            const float4 o1 = k > 1 ? reinterpret_cast<const float4*>(sm.o[st][1] + rl * 128)[lane]
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            acc[r].x = acc[r].x * sc + w0 * o0.x + w1 * o1.x;
            acc[r].y = acc[r].y * sc + w0 * o0.y + w1 * o1.y;
            acc[r].z = acc[r].z * sc + w0 * o0.z + w1 * o1.z;
            acc[r].w = acc[r].w * sc + w0 * o0.w + w1 * o1.w;
            l[r] = l[r] * sc + w0 + w1;
            M[r] = Mn;
        }
        __syncthreads();  // stage st free again
        if (threadIdx.x == 0 && gi + kMergeStages < ngroups) issue(gi + kMergeStages);
    }
    const int HG = H * G;
    const int u = n / HG, hg = n % HG, h = hg / G, g = hg % G;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int row = row0 + warp * 4 + r;
        if (row >= rows) break;
        const float inv = 1.f / l[r];
        const float4 v = make_float4(acc[r].x * inv, acc[r].y * inv, acc[r].z * inv, acc[r].w * inv);
        const int i = g * rows + row;
        out_store4_p(outs, pe, S, H, u, h, i, lane * 4, v);
        if (outs.codes) {  // NEXT-1 fused int8 export of the merged row, as stored
            float x[4] = {v.x, v.y, v.z, v.w};
            if (outs.out_bf16)
#pragma unroll
                for (int e = 0; e < 4; ++e) x[e] = __bfloat162float(__float2bfloat16_rn(x[e]));
            float mx = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3])), mn = fminf(fminf(x[0], x[1]), fminf(x[2], x[3]));
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            }
            float sc, z;
            i8_scale_zp(mx, mn, sc, z);
            const size_t orow = ((size_t)u * S + i) * H + h;
            reinterpret_cast<uint32_t*>(outs.codes + orow * 128)[lane] =
                i8_pack4(x[0], x[1], x[2], x[3], sc, z, i8_recip(sc));
            if (lane == 0) {
                outs.qscale[orow] = sc;
                outs.qzp[orow] = z;
            }
        }
        if (lane == 0) lse_store_p(outs, pe, S, H, u, h, i, M[r] + logf(l[r]));
    }
}

// Sum the run of QLA state slots of each split unit into zbuf[unit] (d = 128 rows of 128).
__global__ void merge_qla_slots_kernel(const int* __restrict__ slot_unit, int num_slots, const float* __restrict__ slot_o,
                                       float* __restrict__ zbuf, const __grid_constant__ PeerSpec pe) {
    const int s = blockIdx.x;
    const int n = slot_unit[s];
    if (n < 0 || !slot_is_head(slot_unit, s, n)) return;
    const int row = blockIdx.y * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int x = s; x < num_slots; ++x) {
        const int m = slot_unit[x];
        if (m < 0) continue;
        if (m != n) break;
        const float4 o = reinterpret_cast<const float4*>(slot_o + ((size_t)x * 128 + row) * 128)[lane];
        acc.x += o.x;
        acc.y += o.y;
        acc.z += o.z;
        acc.w += o.w;
    }
    if (pe.n > 0) {  // fused exchange: every rank's receive buffer
#pragma unroll
        for (int r = 0; r < kMaxExchangeRanks; ++r) {
            if (r >= pe.n) break;
            reinterpret_cast<float4*>(pe.o[r] + ((size_t)n * 128 + row) * 128)[lane] = acc;
        }
        return;
    }
    reinterpret_cast<float4*>(zbuf + ((size_t)n * 128 + row) * 128)[lane] = acc;
}

// Fused-finalize variant: W[n] = phi2((sum of the run's Z) / N_u) as the bf16 swizzled operand.
__global__ void merge_qla_slots_w_kernel(const int* __restrict__ slot_unit, int num_slots, const float* __restrict__ slot_o,
                                         const int64_t* __restrict__ offsets, int H, int phi2, int normalize,
                                         uint8_t* __restrict__ wbuf) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the state kernel's slots are complete
    asm volatile("griddepcontrol.launch_dependents;");
    const int s = blockIdx.x;
    const int n = slot_unit[s];
    if (n < 0 || !slot_is_head(slot_unit, s, n)) return;
    const int row = blockIdx.y * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int x = s; x < num_slots; ++x) {
        const int m = slot_unit[x];
        if (m < 0) continue;
        if (m != n) break;
        const float4 o = reinterpret_cast<const float4*>(slot_o + ((size_t)x * 128 + row) * 128)[lane];
        acc.x += o.x;
        acc.y += o.y;
        acc.z += o.z;
        acc.w += o.w;
    }
    const int u = n / H;
    const int64_t N = offsets[u + 1] - offsets[u];
    const float inv = (normalize && N > 0) ? 1.f / (float)N : 1.f;
    uint2 pk;
    pk.x = ptx::pack_bf16x2(qla_act(phi2, acc.x * inv), qla_act(phi2, acc.y * inv));
    pk.y = ptx::pack_bf16x2(qla_act(phi2, acc.z * inv), qla_act(phi2, acc.w * inv));
    const int col = lane * 4;
    *reinterpret_cast<uint2*>(wbuf + (size_t)n * (2 * 128 * 128) + qla_w_swz(row, col) + (col & 7) * 2) = pk;
}

// P stacked partials part_o [P,B,H,S,d] / part_lse [P,B,H,S] -> outs (FINAL).  One warp per row.
template <int D>
__global__ void merge_softmax_parts_kernel(int P, int B, int H, int S, const float* __restrict__ part_o,
                                           const float* __restrict__ part_lse, OutSpec outs) {
    const int64_t r = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;  // row index over (u, h, i)
    const int lane = threadIdx.x % 32;
    const int64_t nrows = (int64_t)B * H * S;
    if (r >= nrows) return;
    float M = -INFINITY;
    for (int p = 0; p < P; ++p) M = fmaxf(M, part_lse[p * nrows + r]);
    constexpr int V = D / 32;
    float acc[V];
#pragma unroll
    for (int t = 0; t < V; ++t) acc[t] = 0.f;
    float lse = -INFINITY;
    if (M != -INFINITY) {
        float l = 0.f;
        for (int p = 0; p < P; ++p) l += expf(part_lse[p * nrows + r] - M);
        lse = M + logf(l);
        for (int p = 0; p < P; ++p) {
            const float w = expf(part_lse[p * nrows + r] - lse);
#pragma unroll
            for (int t = 0; t < V; ++t) acc[t] += w * part_o[(p * nrows + r) * D + lane + 32 * t];
        }
    }
    const int u = (int)(r / ((int64_t)H * S)), h = (int)((r / S) % H), i = (int)(r % S);
#pragma unroll
    for (int t = 0; t < V; ++t) out_store(outs, S, H, D, u, h, i, lane + 32 * t, acc[t]);
    if (lane == 0) lse_store(outs, S, H, u, h, i, lse);
}

// Shared key prefix (softmax): LSE merge of each user's history result (o [B,H,S,D], lse [B,H,S])
// with the prefix-only result of the same seeds (opre [H,S,D], lpre [H,S]) -> outs (FINAL or
// PARTIAL layout).  Attention over the union of the two key sets (reading R18).
template <int D>
__global__ void merge_prefix_kernel(int B, int H, int S, const float* __restrict__ o, const float* __restrict__ lse,
                                    const float* __restrict__ opre, const float* __restrict__ lpre, OutSpec outs) {
    const int64_t r = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;  // row over (u, h, i)
    const int lane = threadIdx.x % 32;
    if (r >= (int64_t)B * H * S) return;
    const int64_t rp = r % ((int64_t)H * S);  // (h, i) of the prefix row
    const float l1 = lse[r], l2 = lpre[rp];
    const float M = fmaxf(l1, l2);
    constexpr int V = D / 32;
    float acc[V];
    float L = -INFINITY;
    if (M == -INFINITY) {
#pragma unroll
        for (int t = 0; t < V; ++t) acc[t] = 0.f;
    } else {
        const float w1 = expf(l1 - M), w2 = expf(l2 - M);
        const float inv = 1.f / (w1 + w2);
        L = M + logf(w1 + w2);
#pragma unroll
        for (int t = 0; t < V; ++t)
            acc[t] = (w1 * o[r * D + lane + 32 * t] + w2 * opre[rp * D + lane + 32 * t]) * inv;
    }
    const int u = (int)(r / ((int64_t)H * S)), h = (int)((r / S) % H), i = (int)(r % S);
#pragma unroll
    for (int t = 0; t < V; ++t) out_store(outs, S, H, D, u, h, i, lane + 32 * t, acc[t]);
    if (lane == 0) lse_store(outs, S, H, u, h, i, L);
}

// Shared key prefix (QLA): Z[u,h] += Zpre[h] and user_len[u] = L_u + P (the prefix counts in N_u).
__global__ void add_prefix_state_kernel(int B, int H, int D, float* __restrict__ z, const float* __restrict__ zpre,
                                        const int64_t* __restrict__ offsets, int64_t P, int64_t* __restrict__ user_len) {
    const int64_t n = (int64_t)B * H * D * D;
    const int64_t per = (int64_t)H * D * D;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        z[e] += zpre[e % per];
    if (user_len)
        for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < B; u += (int64_t)gridDim.x * blockDim.x)
            user_len[u] = offsets[u + 1] - offsets[u] + P;
}

__global__ void write_prefix_offsets_kernel(int64_t* off, int64_t P) {
    off[0] = 0;
    off[1] = P;
}

// ---------------------------------------------------------------------------------------------
// O[u, i, h, :] = phi1(q_i) W,  W = phi2((sum_p Z_p[u,h]) * inv_N).  Block: 64 rows x D cols,
// 256 threads, thread tile RT rows x 4 cols.
template <int D, typename TQ>
__global__ void __launch_bounds__(256) qla_finalize_kernel(const TQ* __restrict__ q, int64_t q_user_stride,
                                                           const float* __restrict__ zparts, int P, int64_t part_stride,
                                                           const int64_t* __restrict__ offsets,
                                                           const int64_t* __restrict__ user_len, int S, int H, int phi1,
                                                           int phi2, int normalize, OutSpec outs) {
    constexpr int CT = D / 4;          // column-threads
    constexpr int RTH = 256 / CT;      // row-threads
    constexpr int RT = 64 / RTH;       // rows per thread
    extern __shared__ float sm[];
    float* W = sm;                     // [D][D]
    float* Qt = sm + D * D;            // [D][64] phi1(q) transposed
    const int unit = blockIdx.y;       // u * H + h
    const int u = unit / H, h = unit % H;
    const int i0 = blockIdx.x * 64;
    const int64_t N = user_len ? user_len[u] : (offsets[u + 1] - offsets[u]);
    const float inv = (normalize && N > 0) ? 1.f / (float)N : 1.f;
    for (int e = threadIdx.x; e < D * D; e += 256) {
        float z = 0.f;
        for (int p = 0; p < P; ++p) z += zparts[(size_t)p * part_stride + (size_t)unit * D * D + e];
        W[e] = act(phi2, z * inv);
    }
    const TQ* qb = q + (size_t)u * q_user_stride;
    for (int e = threadIdx.x; e < 64 * D; e += 256) {
        const int r = e / D, c = e % D;
        const int i = i0 + r;
        Qt[c * 64 + r] = (i < S) ? act(phi1, ld<TQ>(qb + ((size_t)i * H + h) * D + c)) : 0.f;
    }
    __syncthreads();
    const int ct = threadIdx.x % CT, rt = threadIdx.x / CT;
    float acc[RT][4];
#pragma unroll
    for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
#pragma unroll 4
    for (int c1 = 0; c1 < D; ++c1) {
        const float4 w = *reinterpret_cast<const float4*>(W + c1 * D + ct * 4);
        float qv[RT];
#pragma unroll
        for (int a = 0; a < RT; ++a) qv[a] = Qt[c1 * 64 + rt * RT + a];
#pragma unroll
        for (int a = 0; a < RT; ++a) {
            acc[a][0] = fmaf(qv[a], w.x, acc[a][0]);
            acc[a][1] = fmaf(qv[a], w.y, acc[a][1]);
            acc[a][2] = fmaf(qv[a], w.z, acc[a][2]);
            acc[a][3] = fmaf(qv[a], w.w, acc[a][3]);
        }
    }
#pragma unroll
    for (int a = 0; a < RT; ++a) {
        const int i = i0 + rt * RT + a;
        if (i >= S) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) out_store(outs, S, H, D, u, h, i, ct * 4 + b, acc[a][b]);
    }
}

// ---------------------------------------------------------------------------------------------
// SIMT softmax: block = 8 warps = 8 query rows of one (user, head); 32-key chunks in smem.
template <int D, typename T>
__global__ void __launch_bounds__(256) simt_softmax_kernel(const T* __restrict__ q, int64_t q_user_stride,
                                                           const T* __restrict__ k, const T* __restrict__ v,
                                                           const int64_t* __restrict__ offsets, int S, int H,
                                                           float scale_log2, OutSpec outs) {
    __shared__ float Ks[32][D + 1];
    __shared__ float Vs[32][D];
    __shared__ float Qs[8][D];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int unit = blockIdx.y, u = unit / H, h = unit % H;
    const int i = blockIdx.x * 8 + warp;
    const bool active = i < S;
    const int64_t j0 = offsets[u], L = offsets[u + 1] - offsets[u];
    for (int c = lane; c < D; c += 32)
        Qs[warp][c] = active ? ld<T>(q + (size_t)u * q_user_stride + ((size_t)i * H + h) * D + c) * scale_log2 : 0.f;
    constexpr int V = D / 32;
    float o[V];
#pragma unroll
    for (int t = 0; t < V; ++t) o[t] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int64_t kb = 0; kb < L; kb += 32) {
        __syncthreads();
        for (int e = threadIdx.x; e < 32 * D; e += 256) {
            const int jj = e / D, c = e % D;
            const int64_t j = kb + jj;
            float kv = 0.f, vv = 0.f;
            if (j < L) {
                const size_t idx = ((size_t)(j0 + j) * H + h) * D + c;
                kv = ld<T>(k + idx);
                vv = ld<T>(v + idx);
            }
            Ks[jj][c] = kv;
            Vs[jj][c] = vv;
        }
        __syncthreads();
        if (!active) continue;
        float s = 0.f;
#pragma unroll 8
        for (int c = 0; c < D; ++c) s = fmaf(Qs[warp][c], Ks[lane][c], s);
        if (kb + lane >= L) s = -INFINITY;
        const float m_new = fmaxf(m, warp_max(s));
        const float corr = exp2f(m - m_new);
        const float p = exp2f(s - m_new);
        l = l * corr + warp_sum(p);
#pragma unroll
        for (int t = 0; t < V; ++t) o[t] *= corr;
#pragma unroll 4
        for (int jj = 0; jj < 32; ++jj) {
            const float pj = __shfl_sync(0xffffffffu, p, jj);
#pragma unroll
            for (int t = 0; t < V; ++t) o[t] = fmaf(pj, Vs[jj][lane + 32 * t], o[t]);
        }
        m = m_new;
    }
    if (!active) return;
    const float inv = L > 0 ? 1.f / l : 0.f;
#pragma unroll
    for (int t = 0; t < V; ++t) out_store(outs, S, H, D, u, h, i, lane + 32 * t, o[t] * inv);
    if (lane == 0) {
        const float lse = L > 0 ? (m + log2f(l)) * kLn2 : -INFINITY;
        if (outs.mode == OUT_PARTIAL) outs.lse[((size_t)u * H + h) * S + i] = lse;
        else lse_store(outs, S, H, u, h, i, lse);
    }
}

// SIMT QLA state: block per (user, head); thread owns column c2 = t % D and rows c1 = t / D + k * (256 / D).
template <int D, typename T>
__global__ void __launch_bounds__(256) simt_qla_state_kernel(const T* __restrict__ k, const T* __restrict__ v,
                                                             const int64_t* __restrict__ offsets, int H, int phi1,
                                                             float* __restrict__ zbuf) {
    constexpr int RSTEP = 256 / D;
    constexpr int NR = D / RSTEP;  // accumulators per thread = D*D/256
    __shared__ float Ks[32][D];
    __shared__ float Vs[32][D];
    const int unit = blockIdx.x, u = unit / H, h = unit % H;
    const int c2 = threadIdx.x % D, r0 = threadIdx.x / D;
    const int64_t j0 = offsets[u], L = offsets[u + 1] - offsets[u];
    float acc[NR];
#pragma unroll
    for (int a = 0; a < NR; ++a) acc[a] = 0.f;
    for (int64_t kb = 0; kb < L; kb += 32) {
        __syncthreads();
        for (int e = threadIdx.x; e < 32 * D; e += 256) {
            const int jj = e / D, c = e % D;
            const int64_t j = kb + jj;
            float kv = 0.f, vv = 0.f;
            if (j < L) {
                const size_t idx = ((size_t)(j0 + j) * H + h) * D + c;
                kv = act(phi1, ld<T>(k + idx));  // phi1 applied, then rows past L stay 0
                vv = ld<T>(v + idx);
            }
            Ks[jj][c] = kv;
            Vs[jj][c] = vv;
        }
        __syncthreads();
        const int jn = (L - kb) < 32 ? (int)(L - kb) : 32;
        for (int jj = 0; jj < jn; ++jj) {
            const float vv = Vs[jj][c2];
#pragma unroll
            for (int a = 0; a < NR; ++a) acc[a] = fmaf(Ks[jj][r0 + a * RSTEP], vv, acc[a]);
        }
    }
#pragma unroll
    for (int a = 0; a < NR; ++a) zbuf[((size_t)unit * D + r0 + a * RSTEP) * D + c2] = acc[a];
}

// Int8 export (NEXT-1): one warp per row; float32 arithmetic without contraction (matches the
// oracle's decisions bit for bit): scale = max((mx - mn) / 254, 1e-12), zp = (mx + mn) / 2,
// code = clamp(rint((x - zp) / scale), -127, 127).
template <typename T>
__global__ void quantize_rows_kernel(int64_t n, int d, const T* __restrict__ x, int8_t* __restrict__ codes,
                                     float* __restrict__ scale, float* __restrict__ zp) {
    const int64_t r = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (r >= n) return;
    const T* xr = x + r * d;
    float mx = -INFINITY, mn = INFINITY;
    for (int c = lane; c < d; c += 32) {
        const float v = ld<T>(xr + c);
        mx = fmaxf(mx, v);
        mn = fminf(mn, v);
    }
    mx = warp_max(mx);
    mn = -warp_max(-mn);
    float s = __fdiv_rn(__fsub_rn(mx, mn), 254.0f);
    if (!(s > 1e-12f)) s = 1e-12f;
    const float z = __fmul_rn(0.5f, __fadd_rn(mx, mn));
    if (lane == 0) {
        scale[r] = s;
        zp[r] = z;
    }
    for (int c = lane; c < d; c += 32) {
        float q = rintf(__fdiv_rn(__fsub_rn(ld<T>(xr + c), z), s));
        q = fminf(fmaxf(q, -127.f), 127.f);
        codes[r * d + c] = (int8_t)q;
    }
}

// Vectorized variant for d = 128: 16 threads per row, 8 consecutive values per thread (one 16-B
// load for bf16), 8-byte code stores; same float32 arithmetic as quantize_rows_kernel.
template <typename T>
__global__ void __launch_bounds__(256) quantize_rows128_kernel(int64_t n, const T* __restrict__ x,
                                                               int8_t* __restrict__ codes, float* __restrict__ scale,
                                                               float* __restrict__ zp) {
    const int64_t r = (int64_t)blockIdx.x * 16 + threadIdx.x / 16;
    const int sub = threadIdx.x % 16;
    const bool ok = r < n;
    float v[8];
    if (ok) {
        const T* xr = x + r * 128 + sub * 8;
        if constexpr (sizeof(T) == 2) {
            const uint4 raw = *reinterpret_cast<const uint4*>(xr);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                v[2 * e] = __uint_as_float(w[e] << 16);
                v[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
            }
        } else {
            const float4 a = *reinterpret_cast<const float4*>(xr), b = *reinterpret_cast<const float4*>(xr + 4);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        }
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = 0.f;
    }
    float mx = v[0], mn = v[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) {
        mx = fmaxf(mx, v[e]);
        mn = fminf(mn, v[e]);
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (!ok) return;
    float s = __fdiv_rn(__fsub_rn(mx, mn), 254.0f);
    if (!(s > 1e-12f)) s = 1e-12f;
    const float z = __fmul_rn(0.5f, __fadd_rn(mx, mn));
    if (sub == 0) {
        scale[r] = s;
        zp[r] = z;
    }
    uint32_t pk[2] = {0, 0};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float q = fminf(fmaxf(rintf(__fdiv_rn(__fsub_rn(v[e], z), s)), -127.f), 127.f);
        pk[e >> 2] |= ((uint32_t)(uint8_t)(int8_t)q) << (8 * (e & 3));
    }
    *reinterpret_cast<uint2*>(codes + r * 128 + sub * 8) = make_uint2(pk[0], pk[1]);
}

}  // namespace

cudaError_t launch_quantize_rows(int64_t n, int d, int in_bf16, const void* x, int8_t* codes, float* scale, float* zp,
                                 cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(codes)) & 15) == 0;
    if (d == 128 && aligned) {
        const unsigned g = (unsigned)((n + 15) / 16);
        if (in_bf16)
            quantize_rows128_kernel<__nv_bfloat16><<<g, 256, 0, stream>>>(n, reinterpret_cast<const __nv_bfloat16*>(x),
                                                                          codes, scale, zp);
        else
            quantize_rows128_kernel<float><<<g, 256, 0, stream>>>(n, reinterpret_cast<const float*>(x), codes, scale, zp);
        return cudaGetLastError();
    }
    const unsigned grid = (unsigned)((n + 7) / 8);
    if (in_bf16)
        quantize_rows_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(n, d, reinterpret_cast<const __nv_bfloat16*>(x),
                                                                      codes, scale, zp);
    else
        quantize_rows_kernel<float><<<grid, 256, 0, stream>>>(n, d, reinterpret_cast<const float*>(x), codes, scale, zp);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Summary tokens of the multi-layer summarizer: the first S rows of every user's segment of x
// [R, D] (bf16) -> tokens [B, S, D] (bf16 or f32).  One block per (user, seed row).
__global__ void gather_seed_rows_kernel(const __nv_bfloat16* __restrict__ x, const int64_t* __restrict__ x_offsets,
                                        int S, int D, int out_bf16, void* __restrict__ tokens) {
    const int u = blockIdx.x / S, i = blockIdx.x % S;
    const __nv_bfloat16* src = x + (size_t)(x_offsets[u] + i) * D;
    const size_t dst = ((size_t)u * S + i) * D;
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        if (out_bf16) reinterpret_cast<__nv_bfloat16*>(tokens)[dst + c] = src[c];
        else reinterpret_cast<float*>(tokens)[dst + c] = __bfloat162float(src[c]);
    }
}

// ============================================================================== launchers
cudaError_t launch_user_tiles(const Problem& p, int64_t* uts, float* zbuf) {
    return launch_pdl(user_tiles_kernel, dim3(1), dim3(1024), 0, p.stream, p.offsets, p.B, uts, p.outs, p.S, p.H,
                      p.d, (int)(p.attn == VISTA_SOFTMAX), zbuf, p.peers);
}

cudaError_t launch_merge_softmax_slots(const Problem& p, const Workspace& w, char* ws) {
    const int num_slots = 2 * w.num_ctas;
    dim3 grid(num_slots, (w.rows_per_unit + kMergeRows - 1) / kMergeRows);
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(merge_softmax_slots_kernel), (int)sizeof(MergeSmem));
    if (attr != cudaSuccess) return attr;
    return launch_pdl(merge_softmax_slots_kernel, grid, dim3(256), sizeof(MergeSmem), p.stream,
                      reinterpret_cast<const int*>(ws + w.slot_unit_off), num_slots,
                      reinterpret_cast<const float*>(ws + w.slot_o_off),
                      reinterpret_cast<const float*>(ws + w.slot_lse_off), w.rows_per_unit, p.outs, p.S, p.H,
                      p.S / w.rows_per_unit, p.peers);
}

cudaError_t launch_merge_qla_slots_w(const Problem& p, const Workspace& w, char* ws, uint8_t* wbuf) {
    const int num_slots = 2 * w.num_ctas;
    dim3 grid(num_slots, 128 / 8);
    return launch_pdl(merge_qla_slots_w_kernel, grid, dim3(256), 0, p.stream,
                      reinterpret_cast<const int*>(ws + w.slot_unit_off), num_slots,
                      reinterpret_cast<const float*>(ws + w.slot_o_off), p.offsets, p.H, p.phi2, p.normalize, wbuf);
}

cudaError_t launch_merge_qla_slots(const Problem& p, const Workspace& w, char* ws, float* zbuf) {
    const int num_slots = 2 * w.num_ctas;
    dim3 grid(num_slots, 128 / 8);
    merge_qla_slots_kernel<<<grid, 256, 0, p.stream>>>(reinterpret_cast<const int*>(ws + w.slot_unit_off), num_slots,
                                                       reinterpret_cast<const float*>(ws + w.slot_o_off), zbuf,
                                                       p.outs.mode == OUT_PARTIAL ? p.peers : PeerSpec{});
    return cudaGetLastError();
}

template <int D>
static cudaError_t merge_parts_d(const Problem& p, int P, const float* po, const float* pl) {
    const int64_t nrows = (int64_t)p.B * p.H * p.S;
    if (nrows == 0) return cudaSuccess;
    merge_softmax_parts_kernel<D><<<(unsigned)((nrows + 7) / 8), 256, 0, p.stream>>>(P, p.B, p.H, p.S, po, pl, p.outs);
    return cudaGetLastError();
}
cudaError_t launch_merge_softmax_parts(const Problem& p, int P, const float* po, const float* pl) {
    switch (p.d) {
        case 32: return merge_parts_d<32>(p, P, po, pl);
        case 64: return merge_parts_d<64>(p, P, po, pl);
        case 128: return merge_parts_d<128>(p, P, po, pl);
    }
    return cudaErrorInvalidValue;
}

template <int D, typename TQ>
static cudaError_t finalize_d(const Problem& p, const float* zparts, int P, int64_t part_stride, const int64_t* user_len) {
    if (p.B == 0) return cudaSuccess;
    const size_t smem = (size_t)(D * D + D * 64) * sizeof(float);
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(qla_finalize_kernel<D, TQ>), (int)smem);
    if (attr != cudaSuccess) return attr;
    dim3 grid((p.S + 63) / 64, p.B * p.H);
    qla_finalize_kernel<D, TQ><<<grid, 256, smem, p.stream>>>(
        reinterpret_cast<const TQ*>(p.q), p.q_user_stride, zparts, P, part_stride, p.offsets, user_len, p.S, p.H, p.phi1,
        p.phi2, p.normalize, p.outs);
    return cudaGetLastError();
}
bool qla_finalize_uses_tc(const Problem& p) { return p.in_bf16 && p.d == 128 && (p.q_user_stride % 8) == 0; }

cudaError_t launch_qla_finalize(const Problem& p, const float* zparts, int P, int64_t part_stride,
                                const int64_t* user_len, void* ws) {
    if (qla_finalize_uses_tc(p))  // tensor-core finalize (sm100_qla_finalize.cu)
        return launch_sm100_qla_finalize(p, zparts, P, part_stride, user_len, ws);
    if (p.in_bf16) {
        switch (p.d) {
            case 32: return finalize_d<32, __nv_bfloat16>(p, zparts, P, part_stride, user_len);
            case 64: return finalize_d<64, __nv_bfloat16>(p, zparts, P, part_stride, user_len);
            case 128: return finalize_d<128, __nv_bfloat16>(p, zparts, P, part_stride, user_len);
        }
    } else {
        switch (p.d) {
            case 32: return finalize_d<32, float>(p, zparts, P, part_stride, user_len);
            case 64: return finalize_d<64, float>(p, zparts, P, part_stride, user_len);
            case 128: return finalize_d<128, float>(p, zparts, P, part_stride, user_len);
        }
    }
    return cudaErrorInvalidValue;
}

template <int D, typename T>
static cudaError_t simt_softmax_d(const Problem& p) {
    if (p.B == 0) return cudaSuccess;
    dim3 grid((p.S + 7) / 8, p.B * p.H);
    simt_softmax_kernel<D, T><<<grid, 256, 0, p.stream>>>(reinterpret_cast<const T*>(p.q), p.q_user_stride,
                                                           reinterpret_cast<const T*>(p.k), reinterpret_cast<const T*>(p.v),
                                                           p.offsets, p.S, p.H, p.scale * kLog2e, p.outs);
    return cudaGetLastError();
}
cudaError_t launch_simt_softmax(const Problem& p) {
    if (p.in_bf16) {
        switch (p.d) {
            case 32: return simt_softmax_d<32, __nv_bfloat16>(p);
            case 64: return simt_softmax_d<64, __nv_bfloat16>(p);
            case 128: return simt_softmax_d<128, __nv_bfloat16>(p);
        }
    } else {
        switch (p.d) {
            case 32: return simt_softmax_d<32, float>(p);
            case 64: return simt_softmax_d<64, float>(p);
            case 128: return simt_softmax_d<128, float>(p);
        }
    }
    return cudaErrorInvalidValue;
}

template <int D, typename T>
static cudaError_t simt_qla_d(const Problem& p, float* zbuf) {
    if (p.B == 0) return cudaSuccess;
    simt_qla_state_kernel<D, T><<<p.B * p.H, 256, 0, p.stream>>>(reinterpret_cast<const T*>(p.k),
                                                                  reinterpret_cast<const T*>(p.v), p.offsets, p.H, p.phi1,
                                                                  zbuf);
    return cudaGetLastError();
}
cudaError_t launch_simt_qla_state(const Problem& p, float* zbuf) {
    if (p.in_bf16) {
        switch (p.d) {
            case 32: return simt_qla_d<32, __nv_bfloat16>(p, zbuf);
            case 64: return simt_qla_d<64, __nv_bfloat16>(p, zbuf);
            case 128: return simt_qla_d<128, __nv_bfloat16>(p, zbuf);
        }
    } else {
        switch (p.d) {
            case 32: return simt_qla_d<32, float>(p, zbuf);
            case 64: return simt_qla_d<64, float>(p, zbuf);
            case 128: return simt_qla_d<128, float>(p, zbuf);
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_write_prefix_offsets(int64_t* off, int64_t P, cudaStream_t st) {
    write_prefix_offsets_kernel<<<1, 1, 0, st>>>(off, P);
    return cudaGetLastError();
}

cudaError_t launch_merge_prefix(const Problem& p, const float* o, const float* lse, const float* opre,
                                const float* lpre) {
    const int64_t nrows = (int64_t)p.B * p.H * p.S;
    if (nrows == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((nrows + 7) / 8);
    switch (p.d) {
        case 32: merge_prefix_kernel<32><<<grid, 256, 0, p.stream>>>(p.B, p.H, p.S, o, lse, opre, lpre, p.outs); break;
        case 64: merge_prefix_kernel<64><<<grid, 256, 0, p.stream>>>(p.B, p.H, p.S, o, lse, opre, lpre, p.outs); break;
        case 128: merge_prefix_kernel<128><<<grid, 256, 0, p.stream>>>(p.B, p.H, p.S, o, lse, opre, lpre, p.outs); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_add_prefix_state(const Problem& p, float* z, const float* zpre, int64_t P, int64_t* user_len) {
    if (p.B == 0) return cudaSuccess;
    add_prefix_state_kernel<<<p.num_sms * 4, 256, 0, p.stream>>>(p.B, p.H, p.d, z, zpre, p.offsets, P, user_len);
    return cudaGetLastError();
}

}  // namespace vista

namespace vista {
cudaError_t launch_gather_seed_rows(const void* x, const int64_t* x_offsets, int B, int S, int D, int out_bf16,
                                    void* tokens, cudaStream_t stream) {
    if (B == 0) return cudaSuccess;
    gather_seed_rows_kernel<<<B * S, 128, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(x), x_offsets, S, D,
                                                       out_bf16, tokens);
    return cudaGetLastError();
}
}  // namespace vista
