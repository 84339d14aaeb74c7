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
// Box-Muller, accurate fp32 (<= 2 ulp against the correctly rounded value, checked exhaustively
// over every u1 and every u2 by tests/test_gpu_parity.py).  Exact zeros at u2 in {0, 1/4, 1/2,
// 3/4} and R = 0 at u1 = 1 (reading R14).
// -ln(u1) for u1 = M 2^-24, M in [1, 2^24] (exact fp32).  Reduction u1 = 2^k f, f in
// [sqrt(2)/2, sqrt(2)) by integer ops on the bit pattern; ln f = log1p(t), t = f - 1 (exact), via
// s = t / (2 + t) and the minimax series of FreeBSD's e_logf.c (< 1 ulp); the reciprocal is the
// approximate MUFU.RCP, whose 2^-22 error only reaches the small correction term s*(hfsq + R).
// The Lg1..Lg4 coefficients and the k / f reduction follow FreeBSD msun's e_logf.c, which carries:
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this software is freely granted, provided
//   that this notice is preserved.
__device__ __forceinline__ float neg_log_u1(float u1) {
    const uint32_t ix = __float_as_uint(u1) - 0x3F3504F3u;
    const int k = static_cast<int>(ix) >> 23;                      // exponent after reduction
    const float f = __uint_as_float((ix & 0x007FFFFFu) + 0x3F3504F3u) - 1.0f;
    float r2;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(2.0f + f));
    const float s = f * r2;
    const float z = s * s;
    const float w = z * z;
    const float t1 = w * fmaf(w, 0xf89e26.0p-26f, 0xccce13.0p-25f);
    const float t2 = z * fmaf(w, 0x91e9ee.0p-25f, 0xaaaaaa.0p-24f);
    const float R = t2 + t1;
    const float hfsq = 0.5f * f * f;
    const float dk = static_cast<float>(k);
    // ln u1 = k ln2_hi + (f - hfsq + s (hfsq + R) + k ln2_lo)
    const float lnf = fmaf(s, hfsq + R, fmaf(dk, 9.0580006145e-06f, -hfsq)) + f;
    return -fmaf(dk, 6.9313812256e-01f, lnf);
}

// (cos 2 pi u2, sin 2 pi u2) for u2 = a 2^-24: exact quadrant reduction in integers
// (a = q 2^22 + rem, rem in [-2^21, 2^21)), y = rem / 2^22 in [-1/2, 1/2] (exact), then
// sin(pi y / 2) and cos(pi y / 2) by their Taylor series to y^9 / y^10 (truncation < 2^-28) with
// the leading sine coefficient split hi + lo, and finally the rotation by q quarter turns.
__device__ __forceinline__ float2 cos_sin_2pi(uint32_t a) {
    const uint32_t qa = (a + (1u << 21)) >> 22;
    const uint32_t q = qa & 3u;
    const int32_t rem = static_cast<int32_t>(a) - static_cast<int32_t>(qa << 22);
    const float y = __int2float_rn(rem) * 0x1p-22f;
    const float y2 = y * y;
    float sp = fmaf(y2, 1.60441185e-04f, -4.68175413e-03f);
    sp = fmaf(y2, sp, 7.96926262e-02f);
    sp = fmaf(y2, sp, -6.45964098e-01f);
    const float sn = fmaf(y, 1.57079637e+00f, fmaf(y, -4.37113883e-08f, (y * y2) * sp));
    float cp = fmaf(y2, -2.52020424e-05f, 9.19260275e-04f);
    cp = fmaf(y2, cp, -2.08634808e-02f);
    cp = fmaf(y2, cp, 2.53669508e-01f);
    cp = fmaf(y2, cp, -1.23370055e+00f);
    const float cs = fmaf(y2, cp, 1.0f);
    // rotate by q quarter turns: (c, s) -> (c,s), (-s,c), (-c,-s), (s,-c)
    const float c0 = (q & 1u) ? sn : cs;
    const float s0 = (q & 1u) ? cs : sn;
    const uint32_t negc = ((q + 1u) & 2u) << 30;  // q = 1, 2
    const uint32_t negs = (q & 2u) << 30;         // q = 2, 3
    return make_float2(__uint_as_float(__float_as_uint(c0) ^ negc),
                       __uint_as_float(__float_as_uint(s0) ^ negs));
}

__device__ __forceinline__ float2 box_muller_accurate(uint32_t w1, uint32_t w2) {
    const float u1 = __uint2float_rn((w1 >> 8) + 1u) * 0x1p-24f;  // (0,1], exact
    // sqrt.rn (correctly rounded) with flush-to-zero: the argument is >= 2^-23 (never subnormal), so
    // the result is bit-identical to sqrtf without the subnormal-input slow path
    float R;
    asm("sqrt.rn.ftz.f32 %0, %1;" : "=f"(R) : "f"(2.0f * neg_log_u1(u1)));
    const float2 cs = cos_sin_2pi(w2 >> 8);
    return make_float2(R * cs.x, R * cs.y);
}

// (cos 2 pi u2, sin 2 pi u2) on the MUFU special-function unit: the same exact quarter-turn
// reduction in integers as cos_sin_2pi (rem in [-2^21, 2^21), exact), so the MUFU only ever sees
// |theta| <= pi/4 and the rotation by q quarter turns is exact -- sin/cos of 0 are exactly 0 / 1,
// which gives the exact zeros at u2 in {0, 1/4, 1/2, 3/4} (reading R14).  theta = rem * pi 2^-23
// is rounded once (relative 2^-24).
__device__ __forceinline__ float2 cos_sin_2pi_fast(uint32_t a) {
    const uint32_t qa = (a + (1u << 21)) >> 22;
    const uint32_t q = qa & 3u;
    const int32_t rem = static_cast<int32_t>(a) - static_cast<int32_t>(qa << 22);
    const float th = __int2float_rn(rem) * (3.14159265358979323846f * 0x1p-23f);
    float sn, cs;
    asm("sin.approx.f32 %0, %1;" : "=f"(sn) : "f"(th));
    asm("cos.approx.f32 %0, %1;" : "=f"(cs) : "f"(th));
    const float c0 = (q & 1u) ? sn : cs;
    const float s0 = (q & 1u) ? cs : sn;
    const uint32_t negc = ((q + 1u) & 2u) << 30;  // q = 1, 2
    const uint32_t negs = (q & 2u) << 30;         // q = 2, 3
    return make_float2(__uint_as_float(__float_as_uint(c0) ^ negc),
                       __uint_as_float(__float_as_uint(s0) ^ negs));
}

// Box-Muller on the MUFU (lg2 / sqrt / sin / cos .approx); allowed only in the tf32 / bf16 modes,
// whose operand rounding (2^-11 / 2^-8) dominates its error (reading R5: |fast - exact| <=
// 2^-18 max(|z|, 1), checked exhaustively over every u1 and every u2 by tests/test_gpu_parity.py).
__device__ __forceinline__ float2 box_muller_fast(uint32_t w1, uint32_t w2) {
    const uint32_t m = w1 >> 8;
    const float u1 = __uint2float_rn(m + 1u) * 0x1p-24f;
    const float v = __uint2float_rn(0xFFFFFFu - m) * 0x1p-24f;    // 1 - u1, exact
    float lg, R;
    asm("lg2.approx.f32 %0, %1;" : "=f"(lg) : "f"(u1));
    // lg2.approx has ~2^-22 ABSOLUTE error, which dominates -ln u1 when u1 -> 1; there use the
    // series -ln(1 - v) = v + v^2/2 + v^3/3 + v^4/4 (truncation < v^5/5 relative, v < 2^-5).
    const float series = v * fmaf(v, fmaf(v, fmaf(v, 0.25f, 0.333333343f), 0.5f), 1.0f);
    const float mln = (v < 0.03125f) ? series : lg * -0.693147180559945309f;  // -ln u1
    asm("sqrt.approx.f32 %0, %1;" : "=f"(R) : "f"(mln + mln));
    const float2 cs = cos_sin_2pi_fast(w2 >> 8);
    return make_float2(R * cs.x, R * cs.y);
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
