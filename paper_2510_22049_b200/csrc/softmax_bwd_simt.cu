// softmax_bwd_simt.cu -- softmax backward on CUDA cores for the shapes the tcgen05 kernels do not
// take (f32 inputs, d in {32, 64}, S % 128 != 0, S > 1024, f32 dout).  Same math as
// sm100_softmax_bwd.cu (gradients of o_i = sum_j p_ij v_j, p_ij = softmax_j(scale q_i . k_j),
// PAPER.md:158-163), fp32 throughout:
//   D_i = sum_c dO_ic O_ic;  p_ij = exp(scale q_i . k_j - lse_i);  ds_ij = p_ij (dO_i . v_j - D_i)
//   dV_j = sum_i p_ij dO_i;  dK_j = scale sum_i ds_ij q_i;  dQ_i = scale sum_j ds_ij k_j
// One warp per (key, head) for dK / dV and one warp per (query row, head) for dQ (looping over the
// users in ascending order for shared seeds); lanes stride over the d channels.
#include <cuda_bf16.h>

#include "internal.h"

namespace vista {

namespace {

template <typename T>
__device__ __forceinline__ float ld(const T* p, size_t i);
template <>
__device__ __forceinline__ float ld<float>(const float* p, size_t i) { return p[i]; }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p, size_t i) { return __bfloat162float(p[i]); }
template <typename T>
__device__ __forceinline__ void st(T* p, size_t i, float x);
template <>
__device__ __forceinline__ void st<float>(float* p, size_t i, float x) { p[i] = x; }
template <>
__device__ __forceinline__ void st<__nv_bfloat16>(__nv_bfloat16* p, size_t i, float x) { p[i] = __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

constexpr int kMaxPer = 4;  // d / 32 channels per lane (d <= 128)

// D[u,h,i] = sum_c dO[u,i,h,c] O[u,i,h,c]
template <typename TO>
__global__ void d_kernel(const TO* __restrict__ out, const TO* __restrict__ dout, int64_t rows, int S, int H, int d,
                         float* __restrict__ dd) {
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // over (u, h, i)
    const int lane = threadIdx.x % 32;
    if (r >= rows) return;
    const int64_t u = r / ((int64_t)H * S);
    const int h = (int)((r / S) % H), i = (int)(r % S);
    const size_t e0 = (((size_t)u * S + i) * H + h) * d;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s += ld(out, e0 + c) * ld(dout, e0 + c);
    s = warp_sum(s);
    if (lane == 0) dd[r] = s;
}

// dK, dV of key j (one warp per (j, h))
template <typename TI, typename TO>
__global__ void kv_kernel(const TI* __restrict__ q, int64_t q_user_stride, const TI* __restrict__ k,
                          const TI* __restrict__ v, const int64_t* __restrict__ offsets, int B, int S, int H, int d,
                          int64_t total_len, float scale, const float* __restrict__ lse, const TO* __restrict__ dout,
                          const float* __restrict__ dd, TI* __restrict__ dk, TI* __restrict__ dv) {
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // over (j, h)
    const int lane = threadIdx.x % 32;
    if (w >= total_len * H) return;
    const int64_t j = w / H;
    const int h = (int)(w % H);
    int lo = 0, hi = B;  // user of key j: offsets[u] <= j < offsets[u+1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (offsets[mid] <= j) lo = mid; else hi = mid;
    }
    const int u = lo;
    const int per = d / 32;
    float kj[kMaxPer], vj[kMaxPer], akk[kMaxPer] = {0.f, 0.f, 0.f, 0.f}, avv[kMaxPer] = {0.f, 0.f, 0.f, 0.f};
    const size_t kv0 = ((size_t)j * H + h) * d;
    for (int e = 0; e < per; ++e) {
        kj[e] = ld(k, kv0 + lane + 32 * e);
        vj[e] = ld(v, kv0 + lane + 32 * e);
    }
    for (int i = 0; i < S; ++i) {
        const size_t q0 = (size_t)u * q_user_stride + ((size_t)i * H + h) * d;
        const size_t g0 = (((size_t)u * S + i) * H + h) * d;
        float qi[kMaxPer], gi[kMaxPer], sq = 0.f, sg = 0.f;
        for (int e = 0; e < per; ++e) {
            qi[e] = ld(q, q0 + lane + 32 * e);
            gi[e] = ld(dout, g0 + lane + 32 * e);
            sq += qi[e] * kj[e];
            sg += gi[e] * vj[e];
        }
        sq = warp_sum(sq);
        sg = warp_sum(sg);
        const size_t li = ((size_t)u * H + h) * S + i;
        const float p = __expf(scale * sq - lse[li]);
        const float ds = p * (sg - dd[li]);
        for (int e = 0; e < per; ++e) {
            avv[e] += p * gi[e];
            akk[e] += ds * qi[e];
        }
    }
    for (int e = 0; e < per; ++e) {
        st(dv, kv0 + lane + 32 * e, avv[e]);
        st(dk, kv0 + lane + 32 * e, scale * akk[e]);
    }
}

// dQ of row i (one warp per (u, i, h) for per-user Q; per (i, h) summing over users for shared seeds)
template <typename TI, typename TO>
__global__ void q_kernel(const TI* __restrict__ q, int64_t q_user_stride, const TI* __restrict__ k,
                         const TI* __restrict__ v, const int64_t* __restrict__ offsets, int B, int S, int H, int d,
                         float scale, const float* __restrict__ lse, const TO* __restrict__ dout,
                         const float* __restrict__ dd, float* __restrict__ dq) {
    const bool per_user = q_user_stride != 0;
    const int64_t nw = (per_user ? (int64_t)B : 1) * S * H;
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (w >= nw) return;
    const int h = (int)(w % H), i = (int)((w / H) % S);
    const int u0 = per_user ? (int)(w / ((int64_t)H * S)) : 0, u1 = per_user ? u0 + 1 : B;
    const int per = d / 32;
    float acc[kMaxPer] = {0.f, 0.f, 0.f, 0.f};
    for (int u = u0; u < u1; ++u) {
        const size_t q0 = (size_t)u * q_user_stride + ((size_t)i * H + h) * d;
        const size_t g0 = (((size_t)u * S + i) * H + h) * d;
        const size_t li = ((size_t)u * H + h) * S + i;
        const float l = lse[li], D = dd[li];
        float qi[kMaxPer], gi[kMaxPer];
        for (int e = 0; e < per; ++e) {
            qi[e] = ld(q, q0 + lane + 32 * e);
            gi[e] = ld(dout, g0 + lane + 32 * e);
        }
        for (int64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
            const size_t kv0 = ((size_t)j * H + h) * d;
            float kj[kMaxPer], sq = 0.f, sg = 0.f;
            for (int e = 0; e < per; ++e) {
                kj[e] = ld(k, kv0 + lane + 32 * e);
                sq += qi[e] * kj[e];
                sg += gi[e] * ld(v, kv0 + lane + 32 * e);
            }
            sq = warp_sum(sq);
            sg = warp_sum(sg);
            const float ds = __expf(scale * sq - l) * (sg - D);
            for (int e = 0; e < per; ++e) acc[e] += ds * kj[e];
        }
    }
    const size_t o0 = (size_t)w * d;  // [B|1, S, H, d] row (u, i, h) = w
    for (int e = 0; e < per; ++e) dq[o0 + lane + 32 * e] = scale * acc[e];
}

template <typename TI, typename TO>
cudaError_t launch_typed(const Problem& p, const void* out, const float* lse, const void* dout, float* dq, void* dk,
                         void* dv, float* dd) {
    const int64_t rows = (int64_t)p.B * p.H * p.S;
    d_kernel<TO><<<(unsigned)((rows + 7) / 8), 256, 0, p.stream>>>(
        reinterpret_cast<const TO*>(out), reinterpret_cast<const TO*>(dout), rows, p.S, p.H, p.d, dd);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const TI* q = reinterpret_cast<const TI*>(p.q);
    const TI* k = reinterpret_cast<const TI*>(p.k);
    const TI* v = reinterpret_cast<const TI*>(p.v);
    if (p.total_len > 0) {
        const int64_t nw = p.total_len * p.H;
        kv_kernel<TI, TO><<<(unsigned)((nw + 7) / 8), 256, 0, p.stream>>>(
            q, p.q_user_stride, k, v, p.offsets, p.B, p.S, p.H, p.d, p.total_len, p.scale, lse,
            reinterpret_cast<const TO*>(dout), dd, reinterpret_cast<TI*>(dk), reinterpret_cast<TI*>(dv));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    const int64_t nq = (p.q_user_stride ? (int64_t)p.B : 1) * p.S * p.H;
    q_kernel<TI, TO><<<(unsigned)((nq + 7) / 8), 256, 0, p.stream>>>(q, p.q_user_stride, k, v, p.offsets, p.B, p.S,
                                                                     p.H, p.d, p.scale, lse,
                                                                     reinterpret_cast<const TO*>(dout), dd, dq);
    return cudaGetLastError();
}

}  // namespace

size_t softmax_bwd_simt_workspace(const Problem& p) { return ((size_t)p.B * p.H * p.S * 4 + 255) & ~size_t(255); }

cudaError_t launch_softmax_bwd_simt(const Problem& p, bool dout_bf16, const void* out, const float* lse,
                                    const void* dout, float* dq, void* dk, void* dv, char* ws) {
    float* dd = reinterpret_cast<float*>(ws);
    if (p.in_bf16)
        return dout_bf16 ? launch_typed<__nv_bfloat16, __nv_bfloat16>(p, out, lse, dout, dq, dk, dv, dd)
                         : launch_typed<__nv_bfloat16, float>(p, out, lse, dout, dq, dk, dv, dd);
    return dout_bf16 ? launch_typed<float, __nv_bfloat16>(p, out, lse, dout, dq, dk, dv, dd)
                     : launch_typed<float, float>(p, out, lse, dout, dq, dk, dv, dd);
}

}  // namespace vista
