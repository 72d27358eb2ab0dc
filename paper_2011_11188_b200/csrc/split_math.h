// split_math.h — the per-element arithmetic of steps a1 (scale exponent) and a2 (Eq. A_1),
// shared by the split kernels (split_kernels.cu) and the fused-B converter warps of the GEMM
// (gemm3.cu), so both produce the same plane bits by construction.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace split3 {

// Scale exponent from the max-abs (reading R1): s = max(floor(log2 m) - 14, -127), s(0) = 0.
__device__ __forceinline__ int scale_exp_dev(float m) {
    unsigned b = __float_as_uint(m);
    if (b == 0u) return 0;
    int E = (b >= 0x00800000u) ? (int)(b >> 23) - 127 : (31 - __clz(b)) - 149;
    int s = E - 14;
    return s < -127 ? -127 : s;
}

// 2^-s as an fp32 (s in [-127, 113] -> exponent field 127 - s in [14, 254]: always normal).
__device__ __forceinline__ float pow2_neg(int s) { return __uint_as_float((unsigned)(127 - s) << 23); }

// Eq. A_1 for one value: returns (A1 bits, A2 bits).  __fmul_rn/__fsub_rn forbid contraction.
__device__ __forceinline__ void split1(float x, float f, unsigned short& h1, unsigned short& h2) {
    float xs = __fmul_rn(x, f);                       // exact: power-of-two scaling
    __half a1 = __float2half_rn(xs);                  // cvt.rn.f16.f32
    float r = __fsub_rn(xs, __half2float(a1));        // exact (DESIGN.md §3 R5)
    __half a2 = __float2half_rn(__fmul_rn(r, 2048.0f));
    h1 = __half_as_ushort(a1);
    h2 = __half_as_ushort(a2);
}

// Packed fp32 pair arithmetic (sm_100 FMUL2 / FADD2): each lane rounds exactly as the scalar op.
__device__ __forceinline__ float2 mul2_rn(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 A, B, D;\n\tmov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\t"
        "mul.rn.f32x2 D, A, B;\n\tmov.b64 {%0, %1}, D;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 sub2_rn(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 A, B, D;\n\tmov.b64 A, {%2, %3};\n\tmov.b64 B, {%4, %5};\n\t"
        "sub.rn.f32x2 D, A, B;\n\tmov.b64 {%0, %1}, D;}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

// split1 for four consecutive values, packed: hi = (A1 of v.x, .y, .z, .w) as 4 fp16 in 8 bytes,
// likewise lo.  Same operations and roundings as split1 per element (cvt.rn.f16x2.f32 rounds
// each element as cvt.rn.f16.f32; the f32x2 ops round each lane as the scalar op).
__device__ __forceinline__ void split4(float4 v, float f, uint2& hi, uint2& lo) {
    const float2 ff = make_float2(f, f), k11 = make_float2(2048.0f, 2048.0f);
    const float2 x01 = mul2_rn(make_float2(v.x, v.y), ff), x23 = mul2_rn(make_float2(v.z, v.w), ff);
    const __half2 h01 = __floats2half2_rn(x01.x, x01.y), h23 = __floats2half2_rn(x23.x, x23.y);
    const float2 r01 = mul2_rn(sub2_rn(x01, __half22float2(h01)), k11);
    const float2 r23 = mul2_rn(sub2_rn(x23, __half22float2(h23)), k11);
    const __half2 l01 = __floats2half2_rn(r01.x, r01.y), l23 = __floats2half2_rn(r23.x, r23.y);
    hi = make_uint2(*reinterpret_cast<const unsigned*>(&h01), *reinterpret_cast<const unsigned*>(&h23));
    lo = make_uint2(*reinterpret_cast<const unsigned*>(&l01), *reinterpret_cast<const unsigned*>(&l23));
}

}  // namespace split3
