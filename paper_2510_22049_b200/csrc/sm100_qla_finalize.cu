// sm100_qla_finalize.cu -- QLA output on the tensor cores:
//     O[u, i, h, :] = phi1(q_i) . phi2( (sum_p Z_p[u, h]) / N_u )
// with N_u = L_u when normalizing (the 1/N of App. B; reading R10).
// One CTA per (128 query rows, user, head): the CTA builds both MMA operands in shared memory
// (A = phi1(Q) rows, K-major; B = W = phi2(Zbar), MN-major; both bf16 with the 128-B swizzle),
// issues one 128x128x128 tcgen05 MMA chain into TMEM and writes the rows out.
// bf16 operands: W is rounded to bf16 (rel. 2^-9), like P in the softmax path (reading R13).
#include <cuda_bf16.h>

#include "internal.h"
#include "qla_common.cuh"
#include "sm100_ptx.cuh"

namespace vista {

namespace {

constexpr int kHalf = 128 * 128;  // bytes of one [128 rows][64 bf16] swizzled half
constexpr int kOp = 2 * kHalf;    // one 128 x 128 bf16 operand

__device__ __forceinline__ float act(int kind, float x) { return qla_act(kind, x); }
__device__ __forceinline__ uint32_t swz(int row, int col) { return qla_w_swz(row, col); }

// Prep 1 (grid = units x 4): W[unit] = phi2((sum_p Z_p) / N_u) as a bf16 [128][128] MN-major
// operand (B[K = c1][N = c2], c2 contiguous), pre-swizzled so the MMA kernel can bulk-copy it.
// 256 threads per block, each 8 consecutive values of one row (block = 32 rows).
__global__ void __launch_bounds__(256) qla_prep_w_kernel(const float* __restrict__ zparts, int P, int64_t part_stride,
                                                         const int64_t* __restrict__ offsets,
                                                         const int64_t* __restrict__ user_len, int H, int phi2,
                                                         int normalize, uint8_t* __restrict__ wbuf) {
    // PDL (rows path): the launch overlaps the previous kernel's tail; Z may come from it and W may
    // still be read by it
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int unit = blockIdx.x >> 2, u = unit / H;
    const int r = (blockIdx.x & 3) * 32 + threadIdx.x / 8, c = (threadIdx.x % 8) * 16;
    const int64_t N = user_len ? user_len[u] : (offsets[u + 1] - offsets[u]);
    const float inv = (normalize && N > 0) ? 1.f / (float)N : 1.f;
    const float* z0 = zparts + ((size_t)unit * 128 + r) * 128;
    uint8_t* dst = wbuf + (size_t)unit * kOp;
#pragma unroll
    for (int cc = c; cc < c + 16; cc += 8) {
        float4 a = *reinterpret_cast<const float4*>(z0 + cc), b = *reinterpret_cast<const float4*>(z0 + cc + 4);
        for (int p = 1; p < P; ++p) {
            const float* zp = z0 + (size_t)p * part_stride;
            const float4 a2 = *reinterpret_cast<const float4*>(zp + cc), b2 = *reinterpret_cast<const float4*>(zp + cc + 4);
            a.x += a2.x; a.y += a2.y; a.z += a2.z; a.w += a2.w;
            b.x += b2.x; b.y += b2.y; b.z += b2.z; b.w += b2.w;
        }
        uint4 pk;
        pk.x = ptx::pack_bf16x2(act(phi2, a.x * inv), act(phi2, a.y * inv));
        pk.y = ptx::pack_bf16x2(act(phi2, a.z * inv), act(phi2, a.w * inv));
        pk.z = ptx::pack_bf16x2(act(phi2, b.x * inv), act(phi2, b.y * inv));
        pk.w = ptx::pack_bf16x2(act(phi2, b.z * inv), act(phi2, b.w * inv));
        *reinterpret_cast<uint4*>(dst + swz(r, cc)) = pk;
    }
}

// Prep 2 (grid = Bq * H * ceil(S/128) * 4): A block = phi1(Q rows) as a bf16 [128][128] K-major
// operand (rows past S zero), pre-swizzled.  Bq = 1 for shared seeds, so this runs once per call.
__global__ void __launch_bounds__(256) qla_prep_q_kernel(const __nv_bfloat16* __restrict__ q, int64_t q_user_stride,
                                                         int S, int H, int phi1, uint8_t* __restrict__ abuf) {
    const int nblk = (S + 127) / 128;
    const int op = blockIdx.x >> 2;
    const int blk = op % nblk, h = (op / nblk) % H, uq = op / (nblk * H);
    const int r = (blockIdx.x & 3) * 32 + threadIdx.x / 8, c = (threadIdx.x % 8) * 16;
    const int i = blk * 128 + r;
    const __nv_bfloat16* qi = q + (size_t)uq * q_user_stride + ((size_t)i * H + h) * 128;
    uint8_t* dst = abuf + (size_t)op * kOp;
#pragma unroll
    for (int cc = c; cc < c + 16; cc += 8) {
        uint4 pk = make_uint4(0, 0, 0, 0);
        if (i < S) {
            const uint4 raw = *reinterpret_cast<const uint4*>(qi + cc);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                o[e] = ptx::pack_bf16x2(act(phi1, __uint_as_float(w[e] << 16)), act(phi1, __uint_as_float(w[e] & 0xFFFF0000u)));
            pk = make_uint4(o[0], o[1], o[2], o[3]);
        }
        *reinterpret_cast<uint4*>(dst + swz(r, cc)) = pk;
    }
    // PDL (fused path): this kernel needs nothing from its predecessor (the slot merge) and may run
    // beside it, but the finalize after it relies on this grid's completion implying the merge's:
    // let the finalize start its prologue, then wait for the merge before completing
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// One CTA per (128 query rows, user, head): bulk-copy the two prepared operands, one 128x128x128
// tcgen05 MMA chain into TMEM, rows out.
// offsets != NULL (fused path, W written by the state kernel / slot merge): an empty user has no
// W in wbuf and uses the constant W = phi2(0), the value the Z = 0 path gives.
__global__ void __launch_bounds__(128) sm100_qla_finalize_kernel(const uint8_t* __restrict__ abuf,
                                                                 const uint8_t* __restrict__ wbuf, int q_per_user,
                                                                 int S, int H, OutSpec outs,
                                                                 const int64_t* __restrict__ offsets, int phi2) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    __shared__ uint64_t bar_in, bar_mma;
    __shared__ uint32_t tmem_slot;
    const uint32_t sA = base, sB = base + kOp;
    const int r = threadIdx.x, warp = r / 32;
    const int nblk = (S + 127) / 128;
    const int blk = blockIdx.x, unit = blockIdx.y, u = unit / H, h = unit % H;
    const int i = blk * 128 + r;
    const bool empty = offsets && offsets[u + 1] == offsets[u];
    if (warp == 0) ptx::tmem_alloc(&tmem_slot, 128);
    if (r == 0) {
        ptx::mbar_init(&bar_in, 1);
        ptx::mbar_init(&bar_mma, 1);
        ptx::fence_mbar_init();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_slot, 0);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: W and phi1(Q) are complete after this
    if (empty) {  // W = phi2(0) everywhere (a constant: layout-free)
        uint8_t* sm = smem_raw + (base - ptx::smem_u32(smem_raw));
        const uint32_t c2 = ptx::pack_bf16x2(act(phi2, 0.f), act(phi2, 0.f));
        for (int e = r; e < kOp / 16; e += 128) *reinterpret_cast<uint4*>(sm + kOp + e * 16) = make_uint4(c2, c2, c2, c2);
        ptx::fence_proxy_async_smem();
        __syncthreads();
    }
    if (warp == 0) {
        const uint8_t* a = abuf + ((size_t)((q_per_user ? u : 0) * H + h) * nblk + blk) * kOp;
        const uint8_t* w = wbuf + (size_t)unit * kOp;
        ptx::mbar_arrive_expect_tx_w(&bar_in, empty ? kOp : 2 * kOp);
        ptx::bulk_g2s_w(sA, a, kOp, &bar_in);
        if (!empty) ptx::bulk_g2s_w(sB, w, kOp, &bar_in);
        ptx::mbar_wait(&bar_in, 0);
        ptx::tc_fence_after();
        constexpr uint32_t idO = ptx::idesc_bf16_f32(128, 128, 0, 1);  // A K-major, B MN-major
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
            ptx::mma_ss_w(tmem, ptx::sdesc_sw128(sA + (kk >> 2) * kHalf + (kk & 3) * 32, 16, 1024),
                          ptx::sdesc_sw128(sB + kk * 2048, kHalf, 1024), idO, kk > 0);
        ptx::mma_commit_w(&bar_mma);
    }
    ptx::mbar_wait(&bar_mma, 0);
    ptx::tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        ptx::tmem_ld32_sync(trow + c * 32, o);
        if (i < S) {
            const size_t idx = (((size_t)u * S + i) * H + h) * 128 + c * 32;
            if (outs.out_bf16) {
                __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(outs.out) + idx;
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                    uint4 pk;
                    pk.x = ptx::pack_bf16x2(__uint_as_float(o[j]), __uint_as_float(o[j + 1]));
                    pk.y = ptx::pack_bf16x2(__uint_as_float(o[j + 2]), __uint_as_float(o[j + 3]));
                    pk.z = ptx::pack_bf16x2(__uint_as_float(o[j + 4]), __uint_as_float(o[j + 5]));
                    pk.w = ptx::pack_bf16x2(__uint_as_float(o[j + 6]), __uint_as_float(o[j + 7]));
                    *reinterpret_cast<uint4*>(dst + j) = pk;
                }
            } else {
                float* dst = reinterpret_cast<float*>(outs.out) + idx;
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(o[j]), __uint_as_float(o[j + 1]),
                                                                      __uint_as_float(o[j + 2]), __uint_as_float(o[j + 3]));
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 128);
}

}  // namespace

// W_u operands for the rows path (sm100_qla_rows.cu): W = phi2(Z / N_u) from one state [B,H,d,d]
cudaError_t launch_qla_prep_w(const Problem& p, const float* z, uint8_t* wbuf, const int64_t* user_len) {
    return launch_pdl(qla_prep_w_kernel, dim3(p.B * p.H * 4), dim3(256), 0, p.stream, z, 1, (int64_t)0, p.offsets,
                      user_len, p.H, p.phi2, p.normalize, wbuf);
}

size_t sm100_qla_finalize_workspace(const Problem& p) {
    const int nblk = (p.S + 127) / 128;
    const size_t bq = p.q_user_stride ? (size_t)p.B : 1;
    return (size_t)p.B * p.H * kOp + bq * p.H * nblk * kOp;
}

cudaError_t launch_sm100_qla_finalize(const Problem& p, const float* zparts, int P, int64_t part_stride,
                                      const int64_t* user_len, void* ws) {
    if (p.B == 0) return cudaSuccess;
    const int nblk = (p.S + 127) / 128;
    const int bq = p.q_user_stride ? p.B : 1;
    uint8_t* wbuf = reinterpret_cast<uint8_t*>(ws);
    uint8_t* abuf = wbuf + (size_t)p.B * p.H * kOp;
    qla_prep_w_kernel<<<p.B * p.H * 4, 256, 0, p.stream>>>(zparts, P, part_stride, p.offsets, user_len, p.H, p.phi2,
                                                           p.normalize, wbuf);
    qla_prep_q_kernel<<<bq * p.H * nblk * 4, 256, 0, p.stream>>>(reinterpret_cast<const __nv_bfloat16*>(p.q),
                                                                 p.q_user_stride, p.S, p.H, p.phi1, abuf);
    const int smem = 2 * kOp + 1024;
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(sm100_qla_finalize_kernel), smem);
    if (attr != cudaSuccess) return attr;
    dim3 grid(nblk, p.B * p.H);
    sm100_qla_finalize_kernel<<<grid, 128, smem, p.stream>>>(abuf, wbuf, p.q_user_stride != 0, p.S, p.H, p.outs,
                                                             nullptr, p.phi2);
    return cudaGetLastError();
}

cudaError_t launch_sm100_qla_finalize_fused(const Problem& p, uint8_t* ws) {
    if (p.B == 0) return cudaSuccess;
    const int nblk = (p.S + 127) / 128;
    const int bq = p.q_user_stride ? p.B : 1;
    uint8_t* wbuf = ws;
    uint8_t* abuf = wbuf + (size_t)p.B * p.H * kOp;
    // both with PDL: phi1(Q) runs beside the slot merge, the finalize's prologue beside phi1(Q)
    cudaError_t e = launch_pdl(qla_prep_q_kernel, dim3(bq * p.H * nblk * 4), dim3(256), 0, p.stream,
                               reinterpret_cast<const __nv_bfloat16*>(p.q), p.q_user_stride, p.S, p.H, p.phi1, abuf);
    if (e != cudaSuccess) return e;
    const int smem = 2 * kOp + 1024;
    const cudaError_t attr = set_smem_attr(reinterpret_cast<const void*>(sm100_qla_finalize_kernel), smem);
    if (attr != cudaSuccess) return attr;
    dim3 grid(nblk, p.B * p.H);
    return launch_pdl(sm100_qla_finalize_kernel, grid, dim3(128), smem, p.stream, (const uint8_t*)abuf,
                      (const uint8_t*)wbuf, (int)(p.q_user_stride != 0), p.S, p.H, p.outs, p.offsets, p.phi2);
}

size_t qla_prep_q_bytes(const Problem& p) {
    const int nblk = (p.S + 127) / 128;
    const size_t bq = p.q_user_stride ? (size_t)p.B : 1;
    return bq * p.H * nblk * kOp;
}

cudaError_t launch_qla_prep_q(const Problem& p, uint8_t* abuf) {
    const int nblk = (p.S + 127) / 128;
    const int bq = p.q_user_stride ? p.B : 1;
    qla_prep_q_kernel<<<bq * p.H * nblk * 4, 256, 0, p.stream>>>(reinterpret_cast<const __nv_bfloat16*>(p.q),
                                                                 p.q_user_stride, p.S, p.H, p.phi1, abuf);
    return cudaGetLastError();
}

}  // namespace vista
