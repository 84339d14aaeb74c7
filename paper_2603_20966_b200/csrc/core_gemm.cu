// core_gemm.cu -- C_part = Omega[i0:i0+m, :r]^T * B_blk (Alg. 2 line
// "C-bar_j'k' = Omega^T_i'j' * B_i'k'"), with the Omega rows REGENERATED bit-identically to the
// ones the sketch GEMM used (Alg. 2 regenerates rather than reuses; reading R16).
//
// Two implementations: core_gemm_tc_kernel (tcgen05, below: kind::tf32 in the tf32 / bf16 modes,
// 3xTF32 in tf32x3) is the product path; core_gemm_simt_kernel (fp32 FMA tiles, 64 x 64 outputs per
// CTA, 32-row K steps through shared memory) is kept for B blocks TMA cannot address (unaligned
// base or row stride) and as sketch_set_core_impl(h, 1).  Both split K into contiguous row chunks,
// one r x r partial per chunk, reduced in fixed order by core_reduce_kernel.
#include <algorithm>

#include "kernels.cuh"
#include "philox.cuh"

namespace sk {

constexpr int kCT = 64;   // output tile (a and b)
constexpr int kCK = 32;   // rows per K step

template <int DIST, bool FAST>
__global__ void __launch_bounds__(256)
    core_gemm_simt_kernel(const CoreGemmParams p) {
    __shared__ float sOm[kCK][kCT + 4];
    __shared__ float sB[kCK][kCT + 4];
    const int a0 = blockIdx.x * kCT, b0 = blockIdx.y * kCT, chunk = blockIdx.z;
    const int rbeg = chunk * p.chunk_rows;
    const int rend = min(rbeg + p.chunk_rows, p.m);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[4][4] = {};
    for (int rb = rbeg; rb < rend; rb += kCK) {
        const int nr = min(kCK, rend - rb);
        // B rows rb..rb+31, cols b0..b0+63
        for (int e = threadIdx.x; e < kCK * kCT; e += 256) {
            const int i = e / kCT, c = e % kCT;
            sB[i][c] = (i < nr && b0 + c < p.nb) ? p.B[static_cast<int64_t>(rb + i) * p.ldb + b0 + c] : 0.f;
        }
        // Omega rows (global) g0..g0+nr-1, cols a0..a0+63
        const int64_t g0 = p.i0 + rb;
        if constexpr (DIST == kRademacher) {
            const int64_t first = g0 >> 7, last = (g0 + nr - 1) >> 7;
            const int ncall = static_cast<int>(last - first + 1);
            for (int e = threadIdx.x; e < ncall * kCT; e += 256) {
                const int c = e % kCT;
                const int64_t call = first + e / kCT;
                const uint4 x = philox_rade_call(static_cast<uint64_t>(call), static_cast<uint32_t>(a0 + c),
                                                 p.key0, p.key1);
                const uint32_t w[4] = {x.x, x.y, x.z, x.w};
                for (int i = 0; i < nr; ++i) {
                    const int64_t j = g0 + i;
                    if ((j >> 7) != call) continue;
                    sOm[i][c] = (a0 + c < p.r) ? rade_from_bit(w[(j >> 5) & 3], j & 31) : 0.f;
                }
            }
        } else {
            const int64_t first = g0 >> 2, last = (g0 + nr - 1) >> 2;
            const int ncall = static_cast<int>(last - first + 1);
            for (int e = threadIdx.x; e < ncall * kCT; e += 256) {
                const int c = e % kCT;
                const int64_t call = first + e / kCT;
                const uint4 x = philox_gauss_call(static_cast<uint64_t>(call), static_cast<uint32_t>(a0 + c),
                                                  p.key0, p.key1);
                float4 v;
                if constexpr (DIST == kUniform)
                    v = make_float4(uniform_from_word(x.x), uniform_from_word(x.y),
                                    uniform_from_word(x.z), uniform_from_word(x.w));
                else
                    v = gauss4<FAST>(x);
                const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int64_t i = call * 4 + q - g0;
                    if (i >= 0 && i < nr) sOm[i][c] = (a0 + c < p.r) ? f[q] : 0.f;
                }
            }
        }
        for (int e = threadIdx.x; e < (kCK - nr) * kCT; e += 256) sOm[nr + e / kCT][e % kCT] = 0.f;
        __syncthreads();
#pragma unroll 8
        for (int i = 0; i < kCK; ++i) {
            float om[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { om[u] = sOm[i][ty * 4 + u]; bv[u] = sB[i][tx * 4 + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(om[u], bv[v], acc[u][v]);
        }
        __syncthreads();
    }
    float* out = p.part + static_cast<int64_t>(chunk) * p.r * p.ldp;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int a = a0 + ty * 4 + u;
        if (a >= p.r) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int b = b0 + tx * 4 + v;
            if (b < p.nb) out[static_cast<int64_t>(a) * p.ldp + b] = acc[u][v];
        }
    }
}

cudaError_t launch_core_gemm(const CoreGemmParams& p, int dist, bool fast, cudaStream_t s) {
    dim3 grid((p.r + kCT - 1) / kCT, (p.nb + kCT - 1) / kCT, p.chunks);
    if (dist == kRademacher) core_gemm_simt_kernel<kRademacher, false><<<grid, 256, 0, s>>>(p);
    else if (dist == kUniform) core_gemm_simt_kernel<kUniform, false><<<grid, 256, 0, s>>>(p);
    else if (fast) core_gemm_simt_kernel<kGaussian, true><<<grid, 256, 0, s>>>(p);
    else core_gemm_simt_kernel<kGaussian, false><<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace sk

// =============================================================================================
// tcgen05 core GEMM: CTA (chunk, ablk, bblk) computes the 256 x 256 block (ablk, bblk) of the r x nb
// partial of its K-chunk of B rows (one block when r, nb <= 256).
//   D[a, b] += OmegaT[a, i] * B[i, b]:  M = Omega columns a (NACC blocks of 128), N = npad (b),
//   K = rows i in 32-row steps, kind::tf32, fp32 accumulators in TMEM.
//   * tf32x3 (MODE == kTF32x3): Omega^T = hi + lo and B = hi + lo (hi = tf32 RN, lo = x - hi exact),
//     three MMAs per K step (lo*hi, hi*lo, hi*hi; Rademacher Omega is exact: two); one 128 x 128
//     block per CTA (the doubled operands fill the ring) and <= 1024 rows of K per chunk, because the
//     TMEM accumulation truncates: C stays fp32-accurate.
//   * Omega^T tile (A operand, K-major SW128) is regenerated by 16 producer warps with the sketch
//     GEMM's tile writer (bit-identical Omega).
//   * B tile: TMA loads row-major B (boxes of 32 rows x 32 columns, no swizzle) into a raw ring;
//     the producer warps transpose it into a K-major SW128 tile (row b = 32 K-values), rounding to
//     tf32 (RN) on the way.  (A transposed/MN-major tf32 operand produced zeros on sm_100a in
//     tools/umma_test.cu, so B is made K-major in shared memory instead.)
//   Chunks start at 128-aligned global Omega rows (the first may start before i0: those B rows
//   are TMA zero-filled), so the generator always runs its aligned path.
// =============================================================================================
#include <cstdio>

#include "omega_tile.cuh"
#include "ptx.cuh"

namespace sk {

constexpr int kCoreCtl = 4, kCoreRng = 16;
constexpr int kCoreThreads = (kCoreCtl + kCoreRng) * 32;
constexpr int kCoreStages = 2;     // operand (Omega^T + B^T) ring
constexpr int kCoreRawStages = 2;  // raw B ring (TMA)

struct CoreSmem {
    uint32_t raw_stage, o_stage, bt_stage, raw_off, o_off, bt_off, epi_off, bar_off, total;
};
// x3: Omega^T and B^T tiles each followed by their lo tile (olo: Omega_lo present)
__host__ __device__ inline CoreSmem core_smem(int nacc, int npad, bool x3 = false, bool olo = false) {
    CoreSmem L;
    L.raw_stage = static_cast<uint32_t>((npad + 31) / 32) * 4096u;
    L.o_stage = static_cast<uint32_t>(nacc) * 16384u * (olo ? 2u : 1u);
    L.bt_stage = static_cast<uint32_t>(npad) * 128u * (x3 ? 2u : 1u);
    L.raw_off = 0;
    L.o_off = L.raw_off + kCoreRawStages * L.raw_stage;
    L.bt_off = L.o_off + kCoreStages * L.o_stage;
    L.epi_off = L.bt_off + kCoreStages * L.bt_stage;  // 4 warps x 2 x 4 KB TMA-store staging
    L.bar_off = L.epi_off + 4 * 8192;
    L.total = L.bar_off + (2 * kCoreRawStages + 2 * kCoreStages + 2) * 8 + 16;
    return L;
}

template <int NACC, int DIST, int MODE, bool FAST>
__global__ void __launch_bounds__(kCoreThreads, 1)
    core_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmOut,
                        const CoreTcParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    constexpr bool X3 = (MODE == kTF32x3);
    constexpr bool OLO = X3 && (DIST != kRademacher);  // +-1 is exact in tf32: no Omega_lo
    const CoreSmem L = core_smem(NACC, p.npad, X3, OLO);
    const uint32_t o_lo = NACC * 16384u;                               // Omega_lo tile offset
    const uint32_t b_lo = static_cast<uint32_t>(p.npad) * 128u;        // B_lo tile offset
    uint8_t* sRaw = smem + L.raw_off;
    uint8_t* sO = smem + L.o_off;
    uint8_t* sBt = smem + L.bt_off;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* full_raw = bars;
    uint64_t* empty_raw = bars + kCoreRawStages;
    uint64_t* full_op = bars + 2 * kCoreRawStages;
    uint64_t* empty_op = full_op + kCoreStages;
    uint64_t* done = empty_op + kCoreStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const uint32_t warp = warp_id(), lane = lane_id();
    const int chunk = blockIdx.x;
    const int a_off = static_cast<int>(blockIdx.y) * 128 * NACC;  // first Omega column (row of C) of this block
    const int b_off = static_cast<int>(blockIdx.z) * p.npad;      // first column of B / C of this block
    const int64_t g0 = p.base + static_cast<int64_t>(chunk) * p.step;  // aligned global row
    const int64_t gend = min(p.i0 + static_cast<int64_t>(p.m), g0 + p.step);
    const int ksteps = static_cast<int>((gend - g0 + 31) / 32);
    uint32_t tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(NACC * p.npad)) tmem_cols <<= 1;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kCoreRawStages; ++s) { mbar_init(&full_raw[s], 1); mbar_init(&empty_raw[s], kCoreRng); }
        for (int s = 0; s < kCoreStages; ++s) { mbar_init(&full_op[s], kCoreRng); mbar_init(&empty_op[s], 1); }
        mbar_init(done, 1);
        fence_barrier_init();
        tma_prefetch_desc(&tmB);
    }
    if (warp == 2) tmem_alloc_rt(tmem_slot, tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            uint32_t st = 0, ph = 0;
            const uint64_t pol = l2_policy_evict_first();
            const int ngrp = (p.npad + 31) / 32;
            for (int t = 0; t < ksteps; ++t) {
                mbar_wait(&empty_raw[st], ph ^ 1);
                mbar_arrive_expect_tx(&full_raw[st], L.raw_stage);
                const int32_t row = static_cast<int32_t>(g0 - p.i0) + 32 * t;  // may be < 0: zero fill
                for (int gcol = 0; gcol < ngrp; ++gcol)
                    tma_load_2d(sRaw + st * L.raw_stage + gcol * 4096, &tmB, &full_raw[st], b_off + gcol * 32, row, pol);
                if (++st == kCoreRawStages) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            const uint32_t idesc = make_idesc(kFmtTF32, 128, static_cast<uint32_t>(p.npad), 0, 0);
            uint32_t so = 0, po = 0;
            for (int t = 0; t < ksteps; ++t) {
                mbar_wait(&full_op[so], po);
                tc_fence_after();
                const uint32_t bt_base = smem_u32(sBt + so * L.bt_stage);
                const uint32_t o_base = smem_u32(sO + so * L.o_stage);
#pragma unroll
                for (int k8 = 0; k8 < 4; ++k8) {
                    const uint64_t bdesc = sw128_desc(bt_base + k8 * 32, 16, 1024);
#pragma unroll
                    for (int a = 0; a < NACC; ++a) {
                        const uint64_t adesc = sw128_desc(o_base + a * 16384 + k8 * 32, 16, 1024);
                        const uint32_t d = tmem_base + a * p.npad;
                        uint32_t acc = (t > 0 || k8 > 0) ? 1u : 0u;
                        if constexpr (X3) {
                            // small terms first: Omega_lo * B_hi, Omega_hi * B_lo, then hi * hi
                            if constexpr (OLO) {
                                mma_tf32(d, sw128_desc(o_base + o_lo + a * 16384 + k8 * 32, 16, 1024), bdesc, idesc, acc);
                                acc = 1u;
                            }
                            mma_tf32(d, adesc, sw128_desc(bt_base + b_lo + k8 * 32, 16, 1024), idesc, acc);
                            acc = 1u;
                        }
                        mma_tf32(d, adesc, bdesc, idesc, acc);
                    }
                }
                mma_commit(&empty_op[so]);
                if (++so == kCoreStages) { so = 0; po ^= 1; }
            }
            mma_commit(done);
        }
    } else if (warp >= kCoreCtl) {
        const int tt = static_cast<int>(threadIdx.x) - kCoreCtl * 32;
        const int nrows = 128 * NACC;  // Omega columns generated (a = 0 .. nrows-1)
        const int n_start = tt % nrows, j_start = tt / nrows;
        const int tq = (kCoreRng * 32) / nrows, tr = (kCoreRng * 32) % nrows;
        uint32_t so = 0, po = 0, sr = 0, pr = 0;
        for (int t = 0; t < ksteps; ++t) {
            mbar_wait(&empty_op[so], po ^ 1);
            uint8_t* o_tile = sO + so * L.o_stage;
            if constexpr (DIST == kRademacher)
                produce_omega_tile_r<DIST, MODE, FAST>(o_tile, g0 + 32 * t, 0, nrows, a_off, p.key0, p.key1, tt, o_lo);
            else
                produce_omega_tile_g<DIST, MODE, FAST>(o_tile, g0 + 32 * t, 0, nrows, a_off, p.key0, p.key1,
                                                       n_start, j_start, tq, tr, o_lo);
            // transpose the raw B tile (32 rows i x npad cols b, 128-B rows per 32-col group) into
            // the K-major SW128 tile: row b, chunk j4 = rows 4 j4 .. 4 j4 + 3
            mbar_wait(&full_raw[sr], pr);
            const uint8_t* raw = sRaw + sr * L.raw_stage;
            const uint32_t bt = smem_u32(sBt + so * L.bt_stage);
            for (int c = tt; c < p.npad * 8; c += kCoreRng * 32) {
                const int b = c % p.npad, j4 = c / p.npad;
                const float* col = reinterpret_cast<const float*>(raw + (b >> 5) * 4096) + (b & 31);
                const float4 v = make_float4(col[(4 * j4 + 0) * 32], col[(4 * j4 + 1) * 32],
                                             col[(4 * j4 + 2) * 32], col[(4 * j4 + 3) * 32]);
                const float4 h = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
                const uint32_t addr = bt + static_cast<uint32_t>(b) * 128u +
                                      ((static_cast<uint32_t>(j4) ^ static_cast<uint32_t>(b & 7)) << 4);
                st_shared_v4(addr, h);
                if constexpr (X3)  // B_lo = B - B_hi (exact in fp32)
                    st_shared_v4(addr + b_lo, make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty_raw[sr]);
                mbar_arrive(&full_op[so]);
            }
            if (++so == kCoreStages) { so = 0; po ^= 1; }
            if (++sr == kCoreRawStages) { sr = 0; pr ^= 1; }
        }
        if (tt < 128) {
            const int q = tt >> 5;
            mbar_wait(done, 0);
            tc_fence_after();
            float* out = p.part + static_cast<int64_t>(chunk) * p.r * p.ldp;
            uint8_t* epi = smem + L.epi_off + q * 8192;
            int ebuf = 0;
#pragma unroll 1
            for (int a = 0; a < NACC; ++a) {
                const int row = a_off + a * 128 + q * 32 + static_cast<int>(lane);  // Omega column a
                float* orow = out + static_cast<int64_t>(row) * p.ldp + b_off;
                if ((p.tma_store || p.mc_out) && a_off + a * 128 + q * 32 >= p.r) continue;  // padding rows
#pragma unroll 1
                for (int cc = 0; cc < p.npad; cc += 32) {
                    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                           static_cast<uint32_t>(a * p.npad + cc);
                    uint32_t v[32];
                    if (cc + 32 <= p.npad) {
                        tmem_ld_32x32b_x32(taddr, v);
                    } else {
                        uint32_t h[16];
                        tmem_ld_32x32b_x16(taddr, h);
#pragma unroll
                        for (int i = 0; i < 16; ++i) { v[i] = h[i]; v[16 + i] = 0u; }
                    }
                    tmem_ld_wait();
                    if (p.mc_out != nullptr) {
                        // the AllReduce issued from the epilogue: add this partial into C on every
                        // rank of the multicast group, reduced inside the NVSwitch
                        if (row < p.r) {
                            float* dst = p.mc_out + static_cast<int64_t>(row) * p.ldc_mc + b_off + cc;
                            if (b_off + cc + 32 <= p.nb) {
#pragma unroll
                                for (int i = 0; i < 32; i += 4)
                                    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + i),
                                                 "f"(__uint_as_float(v[i])), "f"(__uint_as_float(v[i + 1])),
                                                 "f"(__uint_as_float(v[i + 2])), "f"(__uint_as_float(v[i + 3]))
                                                 : "memory");
                            } else {
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    if (b_off + cc + i < p.nb)
                                        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(dst + i),
                                                     "f"(__uint_as_float(v[i]))
                                                     : "memory");
                            }
                        }
                    } else if (p.tma_store) {
                        epi_store_tile(&tmOut, epi, ebuf, v, b_off + cc, chunk * p.r + a_off + a * 128 + q * 32);
                    } else if (row < p.r) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (b_off + cc + i < p.nb) orow[cc + i] = __uint_as_float(v[i]);
                    }
                }
            }
            if (p.tma_store && lane == 0) bulk_wait_group<0>();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_rt(tmem_base, tmem_cols);
    }
}

size_t core_gemm_tc_smem_bytes(int nacc, int npad, bool x3, bool olo) {
    return core_smem(nacc, npad, x3, olo).total + 1024;
}

template <int NACC, int DIST, int MODE, bool FAST>
static cudaError_t launch_core_tc_one(const CUtensorMap& tmB, const CUtensorMap& tmOut, const CoreTcParams& p,
                                      cudaStream_t s) {
    auto kern = core_gemm_tc_kernel<NACC, DIST, MODE, FAST>;
    const size_t smem = core_gemm_tc_smem_bytes(NACC, p.npad, MODE == kTF32x3, MODE == kTF32x3 && DIST != kRademacher);
    if (cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(kern), smem)) return e;
    const dim3 grid(p.nchunks, (p.r + 128 * NACC - 1) / (128 * NACC), (p.nb + p.npad - 1) / p.npad);
    kern<<<grid, kCoreThreads, smem, s>>>(tmB, tmOut, p);
    return cudaGetLastError();
}

template <int NACC>
static cudaError_t core_tc_dist(const CUtensorMap& tmB, const CUtensorMap& tmOut, const CoreTcParams& p,
                                int dist, bool fast, bool x3, cudaStream_t s) {
    if (x3) {  // 3xTF32, accurate Omega only (the fast transform is refused in tf32x3)
        if constexpr (NACC == 1) {
            if (dist == kRademacher) return launch_core_tc_one<1, kRademacher, kTF32x3, false>(tmB, tmOut, p, s);
            if (dist == kUniform) return launch_core_tc_one<1, kUniform, kTF32x3, false>(tmB, tmOut, p, s);
            return launch_core_tc_one<1, kGaussian, kTF32x3, false>(tmB, tmOut, p, s);
        }
        return cudaErrorNotSupported;
    }
    if (dist == kRademacher) return launch_core_tc_one<NACC, kRademacher, kTF32, false>(tmB, tmOut, p, s);
    if (dist == kUniform) return launch_core_tc_one<NACC, kUniform, kTF32, false>(tmB, tmOut, p, s);
    if (fast) return launch_core_tc_one<NACC, kGaussian, kTF32, true>(tmB, tmOut, p, s);
    return launch_core_tc_one<NACC, kGaussian, kTF32, false>(tmB, tmOut, p, s);
}

cudaError_t launch_core_gemm_tc(const CUtensorMap& tmB, const CUtensorMap& tmOut, const CoreTcParams& p,
                                int nacc, int dist, bool fast, bool x3, cudaStream_t s) {
    if (nacc == 1) return core_tc_dist<1>(tmB, tmOut, p, dist, fast, x3, s);
    if (nacc == 2) return core_tc_dist<2>(tmB, tmOut, p, dist, fast, x3, s);
    return cudaErrorNotSupported;
}

}  // namespace sk
