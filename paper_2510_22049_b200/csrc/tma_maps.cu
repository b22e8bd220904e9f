// tma_maps.cu -- TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point)
// for the bf16 operands the kernels stream: K / V / rows [total, H, 128] and seeds Q [B?, S, H, 128].
#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace vista {

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

// K / V [total_len, H, 128] with a box of `rows` history rows (TMA multicast slices: 128 / C rows).
bool make_kv_map_rows(CUtensorMap* map, const void* base, int64_t total_len, int H, int rows) {
    const cuuint64_t dims[3] = {128, (cuuint64_t)H, (cuuint64_t)(total_len > 0 ? total_len : 1)};
    const cuuint64_t strides[2] = {128 * 2, (cuuint64_t)H * 128 * 2};
    const cuuint32_t box[3] = {64, 1, (cuuint32_t)rows};
    return make_map_bf16(map, base, 3, dims, strides, box);
}

}  // namespace vista
