// qla_bwd.cu -- QLA backward (NEXT-2, stage-1 training), the CUDA-core kernels.
//
// Forward per (user u, head h) (two activations PAPER.md:831-836; 1/N
// PAPER.md:646-649):  A = phi1(Q), Z = sum_j phi1(k_j)^T v_j, Zbar = Z / N_u, W = phi2(Zbar),
// O = A W.  Backward (appendix gradients PAPER.md:776-783 / 817-829 for phi2 = identity, composed
// through phi2 and 1/N by the chain rule; reading R19):
//   dW = A^T dO;   dZ = (dW . phi2'(Zbar)) / N_u;   dA = dO W^T;   dQ = dA . phi1'(Q)
//   dV_j = phi1(k_j) dZ;   dK_j = (v_j dZ^T) . phi1'(k_j)
// ("W := Q^T dL/dO ... d x d first".)
//
//   qla_bwd_unit_kernel    one block per (u, h): dW, dZ (f32, and optionally the bf16 MMA
//                          operand for sm100_qla_bwd.cu), dA -> per-user dQ
//   qla_bwd_kv_kernel      SIMT dK / dV (f32 inputs or d != 128)
//   qla_bwd_dq_sum_kernel  shared seeds: dQ = sum_u dQ_u in ascending u (deterministic)
#include <cuda_bf16.h>
#include <math.h>

#include <algorithm>

#include "internal.h"
#include "qla_common.cuh"
#include "sm100_ptx.cuh"

namespace vista {

namespace {

__device__ __forceinline__ float act_f(int kind, float x) {
    if (kind == VISTA_ACT_SILU) return x / (1.f + expf(-x));
    if (kind == VISTA_ACT_SHIFTED_ELU) return x >= 1.f ? x : expf(x - 1.f);
    return x;
}
__device__ __forceinline__ float act_prime_f(int kind, float x) {
    if (kind == VISTA_ACT_SILU) {
        const float s = 1.f / (1.f + expf(-x));
        return s * (1.f + x * (1.f - s));
    }
    if (kind == VISTA_ACT_SHIFTED_ELU) return x >= 1.f ? 1.f : expf(x - 1.f);
    return 1.f;
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T>
__device__ __forceinline__ void stf(T* p, float v);
template <>
__device__ __forceinline__ void stf<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void stf<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

constexpr int kChunk = 32;  // rows of Q / dO per smem chunk

// One block (256 threads) per unit (u, h).  Dynamic smem: W [D][D+1] + A, G chunks [32][D] (f32).
template <int D, typename TQ, typename TO>
__global__ void __launch_bounds__(256) qla_bwd_unit_kernel(const TQ* __restrict__ q, int64_t q_user_stride,
                                                           const TO* __restrict__ dout, const float* __restrict__ z,
                                                           const int64_t* __restrict__ offsets, int S, int H,
                                                           int phi1, int phi2, int normalize,
                                                           float* __restrict__ dz, uint8_t* __restrict__ dz_op,
                                                           float* __restrict__ dqu) {
    extern __shared__ float sm[];
    float* Ws = sm;                        // [D][D+1]
    float* As = Ws + D * (D + 1);          // [kChunk][D]
    float* Gs = As + kChunk * D;           // [kChunk][D]
    constexpr int RSTEP = 256 / D;
    constexpr int NR = D / RSTEP;          // dW accumulators per thread
    const int unit = blockIdx.x, u = unit / H, h = unit % H;
    const int t = threadIdx.x;
    const int64_t N = offsets[u + 1] - offsets[u];
    const float inv = (normalize && N > 0) ? 1.f / (float)N : 1.f;
    const float* zu = z + (size_t)unit * D * D;
    for (int e = t; e < D * D; e += 256) Ws[(e / D) * (D + 1) + e % D] = act_f(phi2, zu[e] * inv);
    const TQ* qu = q + (size_t)(q_user_stride ? u : 0) * q_user_stride;
    const TO* gu = dout + (size_t)u * S * H * D;
    const int c2 = t % D, r0 = t / D;
    float acc[NR];
#pragma unroll
    for (int a = 0; a < NR; ++a) acc[a] = 0.f;
    // dW = A^T dO over the S rows
    for (int i0 = 0; i0 < S; i0 += kChunk) {
        __syncthreads();
        for (int e = t; e < kChunk * D; e += 256) {
            const int ii = e / D, c = e % D, i = i0 + ii;
            float a = 0.f, g = 0.f;
            if (i < S) {
                a = act_f(phi1, ldf<TQ>(qu + ((size_t)i * H + h) * D + c));
                g = ldf<TO>(gu + ((size_t)i * H + h) * D + c);
            }
            As[e] = a;
            Gs[e] = g;
        }
        __syncthreads();
#pragma unroll 4
        for (int ii = 0; ii < kChunk; ++ii) {
            const float g = Gs[ii * D + c2];
#pragma unroll
            for (int a = 0; a < NR; ++a) acc[a] += As[ii * D + r0 + a * RSTEP] * g;
        }
    }
    // dZ = dW . phi2'(Zbar) / N
#pragma unroll
    for (int a = 0; a < NR; ++a) {
        const int c1 = r0 + a * RSTEP;
        const float zb = zu[c1 * D + c2] * inv;
        const float g = acc[a] * act_prime_f(phi2, zb) * inv;
        dz[(size_t)unit * D * D + c1 * D + c2] = g;
        if (dz_op) {  // bf16 operand [c1][c2], 128-B swizzled halves (qla_w_swz), D = 128 only
            *reinterpret_cast<__nv_bfloat16*>(dz_op + (size_t)unit * (2 * 128 * 128) + qla_w_swz(c1, c2) +
                                              (c2 & 7) * 2) = __float2bfloat16_rn(g);
        }
    }
    // dA = dO W^T, dQ_u = dA . phi1'(Q)
    constexpr int OPT = kChunk * D / 256;  // outputs per thread per chunk
    for (int i0 = 0; i0 < S; i0 += kChunk) {
        __syncthreads();
        for (int e = t; e < kChunk * D; e += 256) {
            const int ii = e / D, c = e % D, i = i0 + ii;
            Gs[e] = i < S ? ldf<TO>(gu + ((size_t)i * H + h) * D + c) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int o = 0; o < OPT; ++o) {
            const int e = t + o * 256;
            const int ii = e / D, c1 = e % D, i = i0 + ii;
            float s = 0.f;
            for (int cc = 0; cc < D; ++cc) s += Gs[ii * D + cc] * Ws[c1 * (D + 1) + cc];
            if (i < S) {
                const float qv = ldf<TQ>(qu + ((size_t)i * H + h) * D + c1);
                dqu[(((size_t)u * S + i) * H + h) * D + c1] = s * act_prime_f(phi1, qv);
            }
        }
    }
}

// dQ[i,h,c] = sum_u dQ_u[u,i,h,c], ascending u.
__global__ void qla_bwd_dq_sum_kernel(const float* __restrict__ dqu, int B, int64_t n, float* __restrict__ dq) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int u = 0; u < B; ++u) s += dqu[(size_t)u * n + e];
        dq[e] = s;
    }
}

// SIMT dK / dV: one block per unit, items in chunks of 32.  Dynamic smem: dZ [D][D+1], K, V
// chunks [32][D] (f32).
template <int D, typename T>
__global__ void __launch_bounds__(256) qla_bwd_kv_kernel(const T* __restrict__ k, const T* __restrict__ v,
                                                         const int64_t* __restrict__ offsets, int H, int phi1,
                                                         const float* __restrict__ dz, T* __restrict__ dk,
                                                         T* __restrict__ dv) {
    extern __shared__ float sm[];
    float* Zs = sm;                // [D][D+1]
    float* Ks = Zs + D * (D + 1);  // raw k [32][D]
    float* Vs = Ks + kChunk * D;   // [32][D]
    const int unit = blockIdx.x, u = unit / H, h = unit % H;
    const int t = threadIdx.x;
    const int64_t j0 = offsets[u], L = offsets[u + 1] - offsets[u];
    for (int e = t; e < D * D; e += 256) Zs[(e / D) * (D + 1) + e % D] = dz[(size_t)unit * D * D + e];
    constexpr int OPT = kChunk * D / 256;
    for (int64_t jb = 0; jb < L; jb += kChunk) {
        __syncthreads();
        for (int e = t; e < kChunk * D; e += 256) {
            const int jj = e / D, c = e % D;
            const int64_t j = jb + jj;
            float kv = 0.f, vv = 0.f;
            if (j < L) {
                const size_t idx = ((size_t)(j0 + j) * H + h) * D + c;
                kv = ldf<T>(k + idx);
                vv = ldf<T>(v + idx);
            }
            Ks[e] = kv;
            Vs[e] = vv;
        }
        __syncthreads();
#pragma unroll
        for (int o = 0; o < OPT; ++o) {
            const int e = t + o * 256;
            const int jj = e / D, c = e % D;
            const int64_t j = jb + jj;
            float sv = 0.f, sk = 0.f;
            for (int cc = 0; cc < D; ++cc) {
                sv += act_f(phi1, Ks[jj * D + cc]) * Zs[cc * (D + 1) + c];  // dV[j][c2=c]
                sk += Vs[jj * D + cc] * Zs[c * (D + 1) + cc];               // (v dZ^T)[j][c1=c]
            }
            if (j < L) {
                const size_t idx = ((size_t)(j0 + j) * H + h) * D + c;
                stf<T>(dv + idx, sv);
                stf<T>(dk + idx, sk * act_prime_f(phi1, Ks[jj * D + c]));
            }
        }
    }
}

template <int D, typename TQ, typename TO>
cudaError_t unit_launch(const Problem& p, const void* dout, const float* z, float* dz, uint8_t* dz_op, float* dqu) {
    const size_t smem = (size_t)(D * (D + 1) + 2 * kChunk * D) * sizeof(float);
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(qla_bwd_unit_kernel<D, TQ, TO>), (int)smem);
    if (attr != cudaSuccess) return attr;
    qla_bwd_unit_kernel<D, TQ, TO><<<p.B * p.H, 256, smem, p.stream>>>(
        reinterpret_cast<const TQ*>(p.q), p.q_user_stride, reinterpret_cast<const TO*>(dout), z, p.offsets, p.S, p.H,
        p.phi1, p.phi2, p.normalize, dz, dz_op, dqu);
    return cudaGetLastError();
}

template <int D, typename T>
cudaError_t kv_launch(const Problem& p, const float* dz, void* dk, void* dv) {
    const size_t smem = (size_t)(D * (D + 1) + 2 * kChunk * D) * sizeof(float);
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(qla_bwd_kv_kernel<D, T>), (int)smem);
    if (attr != cudaSuccess) return attr;
    qla_bwd_kv_kernel<D, T><<<p.B * p.H, 256, smem, p.stream>>>(reinterpret_cast<const T*>(p.k),
                                                                reinterpret_cast<const T*>(p.v), p.offsets, p.H,
                                                                p.phi1, dz, reinterpret_cast<T*>(dk),
                                                                reinterpret_cast<T*>(dv));
    return cudaGetLastError();
}

template <int D>
cudaError_t unit_d(const Problem& p, bool out_bf16, const void* dout, const float* z, float* dz, uint8_t* dz_op,
                   float* dqu) {
    if (p.in_bf16)
        return out_bf16 ? unit_launch<D, __nv_bfloat16, __nv_bfloat16>(p, dout, z, dz, dz_op, dqu)
                        : unit_launch<D, __nv_bfloat16, float>(p, dout, z, dz, dz_op, dqu);
    return out_bf16 ? unit_launch<D, float, __nv_bfloat16>(p, dout, z, dz, dz_op, dqu)
                    : unit_launch<D, float, float>(p, dout, z, dz, dz_op, dqu);
}

}  // namespace

cudaError_t launch_qla_bwd_unit(const Problem& p, bool dout_bf16, const void* dout, const float* z, float* dz,
                                uint8_t* dz_op, float* dqu) {
    if (p.B == 0) return cudaSuccess;
    switch (p.d) {
        case 32: return unit_d<32>(p, dout_bf16, dout, z, dz, nullptr, dqu);
        case 64: return unit_d<64>(p, dout_bf16, dout, z, dz, nullptr, dqu);
        case 128: return unit_d<128>(p, dout_bf16, dout, z, dz, dz_op, dqu);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_qla_bwd_dq_sum(const Problem& p, const float* dqu, float* dq) {
    const int64_t n = (int64_t)p.S * p.H * p.d;
    if (n == 0) return cudaSuccess;
    qla_bwd_dq_sum_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, p.stream>>>(dqu, p.B, n, dq);
    return cudaGetLastError();
}

cudaError_t launch_qla_bwd_kv_simt(const Problem& p, const float* dz, void* dk, void* dv) {
    if (p.B == 0) return cudaSuccess;
    if (p.in_bf16) {
        switch (p.d) {
            case 32: return kv_launch<32, __nv_bfloat16>(p, dz, dk, dv);
            case 64: return kv_launch<64, __nv_bfloat16>(p, dz, dk, dv);
            case 128: return kv_launch<128, __nv_bfloat16>(p, dz, dk, dv);
        }
    } else {
        switch (p.d) {
            case 32: return kv_launch<32, float>(p, dz, dk, dv);
            case 64: return kv_launch<64, float>(p, dz, dk, dv);
            case 128: return kv_launch<128, float>(p, dz, dk, dv);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace vista
