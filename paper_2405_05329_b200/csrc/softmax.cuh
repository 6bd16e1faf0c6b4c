// softmax.cuh -- per-element arithmetic of the flash-attention softmax on sm_100a: packed
// f32x2 FMA/ADD (FFMA2 / FADD2), three-input max (FMNMX3), exp2 on the MUFU pipe and a
// degree-3 polynomial exp2 on the FMA pipe.  Shared by attn_tc.cu and attn_pair.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace kvp {
namespace smx {

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
// MUFU.EX2 (ex2(-inf) = +0 exactly)
__device__ __forceinline__ float ex2_mufu(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// two scalar FFMA.SAT (the f32x2 FMA has no .sat form)
__device__ __forceinline__ float2 ffma2_sat(float2 a, float2 b, float2 c) {
    float2 d;
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d.x) : "f"(a.x), "f"(b.x), "f"(c.x));
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d.y) : "f"(a.y), "f"(b.y), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {  // FMNMX3 (sm_100)
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// 2^x on the FMA pipe for x = 256 y - POLY_BIAS, where y = sat(x / 256 + POLY_BIAS / 256) came
// out of the (saturating) scale FFMA2 -- the clamp to x in [-125, 131] is free.  With
// M = 1.5 * 2^23: t = 256 y + (M - 125) rounds to M + n, n = rint(x); r = (M - 125) - t =
// -(n + 125) exactly; f = 256 y + r = x - n in [-1/2, 1/2]; 2^f by a degree-3 minimax polynomial
// (max rel. error 1.0e-4, far below bf16's 3.9e-3); 2^n enters the exponent bits with one IMAD
// (t's low mantissa bits hold n).  2 FFMA.SAT + 6 FFMA2-class + 2 IMAD per pair of elements.
constexpr float POLY_BIAS = 125.f;
__device__ __forceinline__ float2 ex2_poly_sat(float2 y) {
    const float2 k256 = make_float2(256.f, 256.f), mb = make_float2(12582912.f - POLY_BIAS, 12582912.f - POLY_BIAS);
    const float2 t = ffma2(y, k256, mb);
    const float2 r = fsub2(mb, t);
    const float2 f = ffma2(y, k256, r);
    float2 p = ffma2(make_float2(0.055008821f, 0.055008821f), f, make_float2(0.24221078f, 0.24221078f));
    p = ffma2(p, f, make_float2(0.6932829f, 0.6932829f));
    p = ffma2(p, f, make_float2(1.f, 1.f));
    float2 o;
    o.x = __uint_as_float(__float_as_uint(t.x) * (1u << 23) + __float_as_uint(p.x));
    o.y = __uint_as_float(__float_as_uint(t.y) * (1u << 23) + __float_as_uint(p.y));
    return o;
}

}  // namespace smx
}  // namespace kvp
