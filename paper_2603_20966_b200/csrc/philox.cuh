// philox.cuh -- device-side Omega generator (reading O1).
//
// The paper regenerates Omega on every processor from a counter-based Philox stream with a
// shared seed instead of communicating it (sec. 6.3) and sketches with
// Gaussian matrices.  The counter layout and the Box-Muller variant are our
// reading O1:
//   key = (seed lo, seed hi);
//   tag 0 (Gaussian / uniform): element (j,k) <- Philox4x32-10((j>>2) lo, (j>>2) hi, k, 0),
//     word x[j&3];  Gaussian pairs (x0,x1) -> rows 4q, 4q+1 and (x2,x3) -> rows 4q+2, 4q+3:
//     u1 = ((w1>>8)+1) 2^-24, u2 = (w2>>8) 2^-24, R = sqrt(-2 ln u1),
//     z_even = R cos(2 pi u2), z_odd = R sin(2 pi u2);
//   tag 1 (Rademacher): element (j,k) <- bit (j&31) of word (j>>5)&3 of
//     Philox4x32-10((j>>7) lo, (j>>7) hi, k, 1); bit 1 -> -1, bit 0 -> +1.
// Every entry is a pure function of (seed, dist, j, k): any tiling, split or rank reproduces it.
#pragma once
#include <cstdint>

namespace sk {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// Philox4x32-10 (Salmon et al. SC'11). The key schedule k + i*W is uniform across the CTA,
// so the compiler keeps it in uniform registers; each round is 2 IMAD.WIDE + 2 LOP3.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c.x;
        const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c.z;
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return c;
}

__device__ __forceinline__ uint4 philox_gauss_call(uint64_t q, uint32_t col, uint32_t k0,
                                                   uint32_t k1) {
    return philox4x32_10(make_uint4(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), col, 0u),
                         k0, k1);
}
__device__ __forceinline__ uint4 philox_rade_call(uint64_t g, uint32_t col, uint32_t k0,
                                                  uint32_t k1) {
    return philox4x32_10(make_uint4(static_cast<uint32_t>(g), static_cast<uint32_t>(g >> 32), col, 1u),
                         k0, k1);
}

// ---------------------------------------------------------------------------------------------
// Box-Muller, accurate fp32: logf (<=1 ulp), correctly rounded sqrtf, sincospif with exact
// argument reduction (2 u2 is exact), one rounding per product.  Exact zeros at u2 in
// {0, 1/4, 1/2, 3/4} and R = 0 at u1 = 1 (reading R14).
__device__ __forceinline__ float2 box_muller_accurate(uint32_t w1, uint32_t w2) {
    const float u1 = __uint2float_rn((w1 >> 8) + 1u) * 0x1p-24f;  // (0,1], exact
    const float t = __uint2float_rn(w2 >> 8) * 0x1p-23f;          // 2 u2 in [0,2), exact
    const float R = sqrtf(-2.0f * logf(u1));
    float s, c;
    sincospif(t, &s, &c);
    return make_float2(R * c, R * s);
}

// Box-Muller on the MUFU special-function unit (lg2 / sqrt / sin / cos .approx); allowed only
// in the tf32 / bf16 modes, whose operand rounding (2^-11 / 2^-8) dominates its error
// (reading R5).  The angle is centred to [-pi, pi) before sin/cos.approx.
__device__ __forceinline__ float2 box_muller_fast(uint32_t w1, uint32_t w2) {
    const uint32_t m = w1 >> 8;
    const float u1 = __uint2float_rn(m + 1u) * 0x1p-24f;
    const float v = __uint2float_rn(0xFFFFFFu - m) * 0x1p-24f;    // 1 - u1, exact
    int32_t a = static_cast<int32_t>(w2 >> 8);
    a = (a >= (1 << 23)) ? a - (1 << 24) : a;                      // u2 - round(u2), exact
    const float th = __int2float_rn(a) * (6.28318530717958647692f * 0x1p-24f);
    float lg, R, s, c;
    asm("lg2.approx.f32 %0, %1;" : "=f"(lg) : "f"(u1));
    // lg2.approx has ~2^-22 ABSOLUTE error, which dominates -ln u1 when u1 -> 1; there use the
    // series -ln(1 - v) = v + v^2/2 + v^3/3 + v^4/4 (truncation < v^5/5 relative, v < 2^-5).
    const float series = v * fmaf(v, fmaf(v, fmaf(v, 0.25f, 0.333333343f), 0.5f), 1.0f);
    const float mln = (v < 0.03125f) ? series : lg * -0.693147180559945309f;  // -ln u1
    asm("sqrt.approx.f32 %0, %1;" : "=f"(R) : "f"(mln + mln));
    asm("sin.approx.f32 %0, %1;" : "=f"(s) : "f"(th));
    asm("cos.approx.f32 %0, %1;" : "=f"(c) : "f"(th));
    return make_float2(R * c, R * s);
}

template <bool kFast>
__device__ __forceinline__ float4 gauss4(uint4 x) {
    const float2 a = kFast ? box_muller_fast(x.x, x.y) : box_muller_accurate(x.x, x.y);
    const float2 b = kFast ? box_muller_fast(x.z, x.w) : box_muller_accurate(x.z, x.w);
    return make_float4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ float uniform_from_word(uint32_t w) {
    return __uint2float_rn(w >> 8) * 0x1p-24f;
}

// +1 / -1 from a bit (bit set -> -1.0f): sign-bit OR into 1.0f.
__device__ __forceinline__ float rade_from_bit(uint32_t word, uint32_t bit) {
    return __uint_as_float(0x3F800000u | (((word >> bit) & 1u) << 31));
}

// Round-to-nearest (ties away) fp32 -> tf32, kept in fp32 storage (low 13 bits zero).
__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

}  // namespace sk
