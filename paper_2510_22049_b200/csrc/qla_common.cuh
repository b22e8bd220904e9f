// qla_common.cuh -- device helpers shared by the QLA state epilogue, the slot merge and the
// finalize GEMM: the activation phi (readings R8-R10) in the
// form used for W = phi2(Zbar) and phi1(Q), and the byte layout of a 128 x 128 bf16 MMA operand
// stored as two 128-B-swizzled halves of 64 columns.
#pragma once
#include <cstdint>

#include "internal.h"

namespace vista {

__device__ __forceinline__ float qla_act(int kind, float x) {
    if (kind == VISTA_ACT_SILU) return x * __frcp_rn(1.f + __expf(-x));
    if (kind == VISTA_ACT_SHIFTED_ELU) return x >= 1.f ? x : __expf(x - 1.f);
    return x;
}

// SiLU on a bf16x2 pair with packed bf16 math: x * (0.5 + 0.5 tanh(x / 2)) -- 4 instructions per
// pair (HMUL2, MUFU.TANH bf16x2, HFMA2, HMUL2), one MUFU op for two values.  Used where the result is
// a bf16 MMA operand anyway (phi1 of K and of query rows).
__device__ __forceinline__ uint32_t qla_silu_bf16x2(uint32_t x) {
    uint32_t h, t, s, y;
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(h) : "r"(x), "r"(0x3F003F00u));
    asm("tanh.approx.bf16x2 %0, %1;" : "=r"(t) : "r"(h));
    asm("fma.rn.bf16x2 %0, %1, %2, %2;" : "=r"(s) : "r"(t), "r"(0x3F003F00u));
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(y) : "r"(x), "r"(s));
    return y;
}

// byte offset of element (row, col) of a [128][128] bf16 operand in two swizzled halves: 16-B chunk
// index XOR (row mod 8) within each 128-B row
__device__ __forceinline__ uint32_t qla_w_swz(int row, int col) {
    const int half = col >> 6, chunk = (col & 63) >> 3;
    return half * (128 * 128) + row * 128 + ((chunk ^ (row & 7)) << 4);
}

}  // namespace vista
