// omega_tile.cuh -- writes one 32-row K-step of Omega (or Omega^T) into shared memory as a K-major
// SWIZZLE_128B tcgen05 operand: row n (an Omega COLUMN, c0 + n) holds 32 consecutive Omega rows
// (K values) in 128 B; 16-byte chunk j4 of row n lives at n*128 + ((j4 ^ (n & 7)) << 4).
// Used by the sketch GEMM (Omega tile = B operand, N = Omega columns) and by the core GEMM
// (Omega^T tile = A operand, M = Omega columns): the same bits either way (reading O1).
#pragma once
#include <cstdint>

#include "kernels.cuh"
#include "philox.cuh"
#include "ptx.cuh"

namespace sk {

// Omega tile for K-iteration `kit`: rows n in [0, npad) (Omega column c0+n), 32 K-values
// (Omega rows kglob0 .. kglob0+31), K-major SW128: byte n*128 + ((j4 ^ (n&7)) << 4) + 4*e.
// kglob0 = 128-aligned base + 32*kit + roff, roff in {0,1,2,3} (roff != 0 only for block calls
// whose k0 is not a multiple of 4: then each 4-row chunk straddles two Philox calls).
// SWIZZLE_128B phase of the 128-B row at shared address `row`: address bits 7..9 (the tiles are
// 1024-B aligned, so this is n & 7 of the tile row; it also holds for a writer whose share of the
// tile starts at a row that is not a multiple of 8, as with clusters of 3 pairs)
__device__ __forceinline__ uint32_t sw128_phase(uint32_t row) { return (row >> 7) & 7u; }

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// tf32 mode: Omega rounded RN to tf32.  tf32x3 mode: Omega_hi = tf32_rn(w) at addr and
// Omega_lo = w - Omega_hi (exact in fp32) at addr + lo_off (Rademacher: +-1 is exact, no lo tile).
template <int DIST, int MODE, bool FAST>
__device__ __forceinline__ void store_chunk(uint32_t addr, float4 v, uint32_t lo_off = 0) {
    if constexpr (MODE == kTF32 || MODE == kTF32x3) {
        const float4 h = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
        st_shared_v4(addr, h);
        if constexpr (MODE == kTF32x3 && DIST != kRademacher)
            st_shared_v4(addr + lo_off, make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
    } else {
        st_shared_v4(addr, v);
    }
}

template <int DIST, bool FAST>
__device__ __forceinline__ float4 values4(uint4 x) {
    if constexpr (DIST == kUniform)
        return make_float4(uniform_from_word(x.x), uniform_from_word(x.y), uniform_from_word(x.z),
                           uniform_from_word(x.w));
    else
        return gauss4<FAST>(x);
}

__device__ __forceinline__ uint32_t pick_word(uint4 x, uint32_t sel) {
    return sel == 0 ? x.x : sel == 1 ? x.y : sel == 2 ? x.z : x.w;
}

// Rademacher tile: one Philox call per column n = t serves all 32 K-values of the tile.
template <int DIST, int MODE, bool FAST>
__device__ __forceinline__ void produce_omega_tile_r(uint8_t* tile, int64_t kglob0, int roff,
                                                     int npad, int c0, uint32_t key0,
                                                     uint32_t key1, int t, uint32_t lo_off = 0) {
    if (t >= npad) return;
    const int n = t;
    const uint32_t col = static_cast<uint32_t>(c0 + n);
    const uint32_t row_base = smem_u32(tile) + static_cast<uint32_t>(n) * 128u;
    const uint32_t sw = sw128_phase(row_base);
    {
        // bits for tile rows kk = 0..31: global rows kglob0 + kk
        const uint64_t g = static_cast<uint64_t>(kglob0);
        const uint4 x = philox_rade_call(g >> 7, col, key0, key1);
        uint32_t w = pick_word(x, static_cast<uint32_t>(g >> 5) & 3u);
        if (roff != 0) {
            const uint64_t g2 = g + 32;  // next word: same call unless it crosses 128 rows
            const uint4 x2 = ((g2 >> 7) == (g >> 7)) ? x : philox_rade_call(g2 >> 7, col, key0, key1);
            const uint32_t w2 = pick_word(x2, static_cast<uint32_t>(g2 >> 5) & 3u);
            w = __funnelshift_r(w, w2, static_cast<uint32_t>(g & 31));
        }
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
            const float4 v = make_float4(rade_from_bit(w, 4 * j4 + 0), rade_from_bit(w, 4 * j4 + 1),
                                         rade_from_bit(w, 4 * j4 + 2), rade_from_bit(w, 4 * j4 + 3));
            store_chunk<DIST, MODE, FAST>(row_base + ((static_cast<uint32_t>(j4) ^ sw) << 4), v, lo_off);
        }
    }
}

// Gaussian / uniform tile: the npad x 8 chunks (one Philox call -> 4 K-values each) are dealt to
// the kRngThreads producers as c = t + kRngThreads * i, n = c % npad, j4 = c / npad, so a warp
// stores 32 consecutive rows n at one j4 (conflict-free under the 128-B swizzle).
template <int DIST, int MODE, bool FAST>
__device__ __forceinline__ void produce_omega_tile_g(uint8_t* tile, int64_t kglob0, int roff,
                                                     int npad, int c0, uint32_t key0,
                                                     uint32_t key1, int n_start, int j_start,
                                                     int tq, int tr, uint32_t lo_off = 0) {
    const uint64_t q0 = static_cast<uint64_t>(kglob0) >> 2;
    const uint32_t tile_base = smem_u32(tile);
    int n = n_start, j4 = j_start;
    if (roff == 0) {
        // two independent chunks per iteration: their Philox / Box-Muller chains interleave
#pragma unroll 1
        while (j4 < 8) {
            int n2 = n + tr, j2 = j4 + tq;
            if (n2 >= npad) { n2 -= npad; ++j2; }
            const bool two = j2 < 8;
            const int n2c = two ? n2 : n, j2c = two ? j2 : j4;
            const uint4 xa = philox_gauss_call(q0 + j4, static_cast<uint32_t>(c0 + n), key0, key1);
            const uint4 xb = philox_gauss_call(q0 + j2c, static_cast<uint32_t>(c0 + n2c), key0, key1);
            const float4 va = values4<DIST, FAST>(xa);
            const float4 vb = values4<DIST, FAST>(xb);
            const uint32_t ra = tile_base + static_cast<uint32_t>(n) * 128u;
            store_chunk<DIST, MODE, FAST>(ra + ((static_cast<uint32_t>(j4) ^ sw128_phase(ra)) << 4), va, lo_off);
            if (two) {
                const uint32_t rb = tile_base + static_cast<uint32_t>(n2) * 128u;
                store_chunk<DIST, MODE, FAST>(rb + ((static_cast<uint32_t>(j2) ^ sw128_phase(rb)) << 4), vb, lo_off);
            }
            n = n2 + tr;
            j4 = j2 + tq;
            if (n >= npad) { n -= npad; ++j4; }
        }
        return;
    }
#pragma unroll 1
    for (; j4 < 8;) {
        const uint32_t col = static_cast<uint32_t>(c0 + n);
        const uint32_t ra = tile_base + static_cast<uint32_t>(n) * 128u;
        const uint32_t addr = ra + ((static_cast<uint32_t>(j4) ^ sw128_phase(ra)) << 4);
        // rows 4(q0+j4)+roff .. +3: tail of call q0+j4, head of call q0+j4+1
        const float4 a0 = values4<DIST, FAST>(philox_gauss_call(q0 + j4, col, key0, key1));
        const float4 a1 = values4<DIST, FAST>(philox_gauss_call(q0 + j4 + 1, col, key0, key1));
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float4 v;
        v.x = roff == 1 ? a[1] : roff == 2 ? a[2] : a[3];
        v.y = roff == 1 ? a[2] : roff == 2 ? a[3] : a[4];
        v.z = roff == 1 ? a[3] : roff == 2 ? a[4] : a[5];
        v.w = roff == 1 ? a[4] : roff == 2 ? a[5] : a[6];
        store_chunk<DIST, MODE, FAST>(addr, v, lo_off);
        n += tr;
        j4 += tq;
        if (n >= npad) { n -= npad; ++j4; }
    }
}

// ------------------------------------------------------------------------------------------
// bf16 tiles: one 64-row K-step, row n (Omega column c0 + n) = 64 bf16 = 128 B, 16-byte chunk
// j8 (K-values 8 j8 .. 8 j8 + 7) at n*128 + ((j8 ^ (n & 7)) << 4); values rounded RN to bf16.
// kglob0 = 128-aligned base + 64 * kit + roff.
template <int DIST, bool FAST>
__device__ __forceinline__ void produce_omega_tile_bf16_r(uint8_t* tile, int64_t kglob0, int roff,
                                                          int npad, int c0, uint32_t key0,
                                                          uint32_t key1, int t) {
    (void)roff;
    if (t >= npad) return;
    const int n = t;
    const uint32_t col = static_cast<uint32_t>(c0 + n);
    const uint32_t row_base = smem_u32(tile) + static_cast<uint32_t>(n) * 128u;
    const uint32_t sw = sw128_phase(row_base);
    // 64 bits for rows kglob0 .. kglob0 + 63, bit b of the 64 = row kglob0 + b
    const uint64_t g = static_cast<uint64_t>(kglob0);
    const uint4 x = philox_rade_call(g >> 7, col, key0, key1);
    const uint32_t sel = static_cast<uint32_t>(g >> 5) & 3u;
    uint32_t w0 = pick_word(x, sel), w1, w2;
    if (sel < 3) {
        w1 = pick_word(x, sel + 1);
        w2 = (sel < 2) ? pick_word(x, sel + 2) : pick_word(philox_rade_call((g >> 7) + 1, col, key0, key1), 0);
    } else {
        const uint4 x2 = philox_rade_call((g >> 7) + 1, col, key0, key1);
        w1 = x2.x;
        w2 = x2.y;
    }
    const uint32_t sh = static_cast<uint32_t>(g & 31);
    const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
#pragma unroll
    for (int j8 = 0; j8 < 8; ++j8) {
        const uint32_t w = (j8 < 4) ? lo : hi;
        const int b0 = (j8 & 3) * 8;
        // bf16 +1 = 0x3F80, -1 = 0xBF80
        uint32_t q[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t s0 = (w >> (b0 + 2 * e)) & 1u, s1 = (w >> (b0 + 2 * e + 1)) & 1u;
            q[e] = (0x3F80u | (s0 << 15)) | ((0x3F80u | (s1 << 15)) << 16);
        }
        st_shared_v4_u32(row_base + ((static_cast<uint32_t>(j8) ^ sw) << 4), q[0], q[1], q[2], q[3]);
    }
}

// Items of 8 K-values (two Philox calls, one 16-B chunk) dealt as n = c % npad, j8 = c / npad;
// HALF: items of 4 K-values (one call, 8 B), so that a small tile (npad * 8 items < producer
// threads, e.g. 32 rows per CTA with clusters of 4 pairs) still keeps every producer busy.
template <int DIST, bool FAST, bool HALF = false>
__device__ __forceinline__ void produce_omega_tile_bf16_g(uint8_t* tile, int64_t kglob0, int roff,
                                                          int npad, int c0, uint32_t key0,
                                                          uint32_t key1, int n_start, int j_start,
                                                          int tq, int tr) {
    const uint64_t q0 = static_cast<uint64_t>(kglob0) >> 2;  // call holding row kglob0 - roff
    const uint32_t tile_base = smem_u32(tile);
    int n = n_start, j = j_start;
    constexpr int kJ = HALF ? 16 : 8;
#pragma unroll 1
    while (j < kJ) {
        const uint32_t col = static_cast<uint32_t>(c0 + n);
        const uint32_t row = tile_base + static_cast<uint32_t>(n) * 128u;
        const uint32_t sw = sw128_phase(row);
        if constexpr (HALF) {
            const float4 a = values4<DIST, FAST>(philox_gauss_call(q0 + j, col, key0, key1));
            float v[4] = {a.x, a.y, a.z, a.w};
            if (roff != 0) {
                const float4 b = values4<DIST, FAST>(philox_gauss_call(q0 + j + 1, col, key0, key1));
                const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = roff == 1 ? x[e + 1] : roff == 2 ? x[e + 2] : x[e + 3];
            }
            const uint32_t addr = row + (((static_cast<uint32_t>(j) >> 1) ^ sw) << 4) + (static_cast<uint32_t>(j) & 1u) * 8u;
            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(pack_bf16x2(v[0], v[1])),
                         "r"(pack_bf16x2(v[2], v[3]))
                         : "memory");
        } else {
            const float4 a = values4<DIST, FAST>(philox_gauss_call(q0 + 2 * j, col, key0, key1));
            const float4 b = values4<DIST, FAST>(philox_gauss_call(q0 + 2 * j + 1, col, key0, key1));
            float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            if (roff != 0) {
                const float4 c = values4<DIST, FAST>(philox_gauss_call(q0 + 2 * j + 2, col, key0, key1));
                const float x[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = roff == 1 ? x[e + 1] : roff == 2 ? x[e + 2] : x[e + 3];
            }
            st_shared_v4_u32(row + ((static_cast<uint32_t>(j) ^ sw) << 4), pack_bf16x2(v[0], v[1]),
                             pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
        }
        n += tr;
        j += tq;
        if (n >= npad) { n -= npad; ++j; }
    }
}

}  // namespace sk
