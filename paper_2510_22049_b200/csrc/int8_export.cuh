// int8_export.cuh -- NEXT-1 int8 export of summary rows, fused into the epilogues (
// "quantized and exported to a large key-value cache").  The float32 arithmetic
// is exactly that of quantize_rows_kernel (kernels_misc.cu) and of the oracle (no contraction):
//   scale = max((max - min) / 254, 1e-12), zp = (max + min) / 2, code = clamp(rint((x - zp) / scale))
// applied to the row as it is stored (bf16-rounded for a bf16 output), so the fused export equals
// vista_quantize_rows_int8 of the output bit for bit.
#pragma once
#include <cstdint>

namespace vista {

__device__ __forceinline__ void i8_scale_zp(float mx, float mn, float& s, float& z) {
    s = __fdiv_rn(__fsub_rn(mx, mn), 254.0f);
    if (!(s > 1e-12f)) s = 1e-12f;
    z = __fmul_rn(0.5f, __fadd_rn(mx, mn));
}
// rint((x - z) / s) with the division correctly rounded, as the reference does.  Fast path: y =
// (x - z) * (1/s) is within 2 ulp of the exact quotient (|y| <= ~127.5, ulp <= 2^-16), so rint(y)
// equals the reference unless y lies within 1e-4 of a half-integer; only then divide exactly.
__device__ __forceinline__ uint32_t i8_code(float x, float s, float z, float rs) {
    const float d = __fsub_rn(x, z);
    float y = __fmul_rn(d, rs);
    const float fr = y - floorf(y);
    if (fabsf(fr - 0.5f) < 1e-4f) y = __fdiv_rn(d, s);
    float q = rintf(y);
    q = fminf(fmaxf(q, -127.f), 127.f);
    return (uint32_t)(uint8_t)(int8_t)q;
}
// four codes packed little-endian (column order); rs = 1 / s (round to nearest)
__device__ __forceinline__ uint32_t i8_pack4(float a, float b, float c, float d, float s, float z, float rs) {
    return i8_code(a, s, z, rs) | (i8_code(b, s, z, rs) << 8) | (i8_code(c, s, z, rs) << 16) |
           (i8_code(d, s, z, rs) << 24);
}
__device__ __forceinline__ float i8_recip(float s) { return __frcp_rn(s); }

// One thread holds a whole d = 128 row as 64 packed bf16x2 words (column order): codes (128 B),
// scale, zp of that row.
__device__ __forceinline__ void i8_export_row_bf16(const uint32_t (&v)[64], int8_t* codes_row, float* scale,
                                                   float* zp) {
    float mx = -INFINITY, mn = INFINITY;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
        const float a = __uint_as_float(v[j] << 16), b = __uint_as_float(v[j] & 0xFFFF0000u);
        mx = fmaxf(mx, fmaxf(a, b));
        mn = fminf(mn, fminf(a, b));
    }
    float s, z;
    i8_scale_zp(mx, mn, s, z);
    const float rs = i8_recip(s);
    *scale = s;
    *zp = z;
    uint4* dst = reinterpret_cast<uint4*>(codes_row);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t lo = v[8 * q + 2 * e], hi = v[8 * q + 2 * e + 1];
            w[e] = i8_pack4(__uint_as_float(lo << 16), __uint_as_float(lo & 0xFFFF0000u), __uint_as_float(hi << 16),
                            __uint_as_float(hi & 0xFFFF0000u), s, z, rs);
        }
        dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

}  // namespace vista
