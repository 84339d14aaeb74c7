// sketch_gemm.cu -- fused "generate Omega tile + tcgen05 GEMM" for B = A * Omega,
// the local product of Alg. 1 ("B-bar_ik = A_ij * Omega_jk") with Omega_jk
// regenerated in the kernel instead of communicated.
//
// One persistent CTA per SM, warp-specialised:
//   warp 0      TMA producer: 128-row x 32-col fp32 tiles of A, SWIZZLE_128B (K-major), into an
//               a_stages-deep ring; L2 evict-first (A is streamed exactly once).
//   warp 1      MMA issuer (one elected thread): tcgen05.mma kind::tf32, M=128, N=npad, K=8,
//               NACC accumulators of 128 x npad fp32 in TMEM (NACC*npad <= 512 columns).
//   warp 2      TMEM allocator.
//   warps 4-11  Omega producers: Philox4x32-10 + transform, written as the K-major SWIZZLE_128B
//               B operand (row n = Omega column c0+n, 32 K-values = 128 B per row), then
//               fence.proxy.async + mbarrier arrive.  Warps 4-7 also run the epilogue
//               (tcgen05.ld 32x32b -> st.global of B or of a split-K partial).
// Work unit = (m-block of 128*NACC rows, K split s); units are dealt round-robin to CTAs.
#include "kernels.cuh"
#include "philox.cuh"
#include "ptx.cuh"

namespace sk {

constexpr int kCtlWarps = 4;
constexpr int kRngWarps = 8;
constexpr int kThreads = (kCtlWarps + kRngWarps) * 32;
constexpr int kRngThreads = kRngWarps * 32;
constexpr uint32_t kATileBytes = 128 * 32 * 4;  // one 128-row x 32-fp32 TMA box
constexpr int kMaxStages = 8;

struct SmemLayout {
    uint32_t a_stage, o_stage, a_off, o_off, bar_off, total;
};

__host__ __device__ inline SmemLayout make_layout(int nacc, int npad, int a_stages, int o_stages) {
    SmemLayout L;
    L.a_stage = static_cast<uint32_t>(nacc) * kATileBytes;
    L.o_stage = static_cast<uint32_t>(npad) * 128u;
    L.a_off = 0;
    L.o_off = L.a_off + L.a_stage * a_stages;
    L.bar_off = L.o_off + L.o_stage * o_stages;
    L.total = L.bar_off + (4 * kMaxStages + 4) * 8 + 16;
    return L;
}

// Omega tile for K-iteration `kit`: rows n in [0, npad) (Omega column c0+n), 32 K-values
// (Omega rows kglob0 .. kglob0+31), K-major SW128: byte n*128 + ((j4 ^ (n&7)) << 4) + 4*e.
// kglob0 = 128-aligned base + 32*kit + roff, roff in {0,1,2,3} (roff != 0 only for block calls
// whose k0 is not a multiple of 4: then each 4-row chunk straddles two Philox calls).
template <int DIST, int MODE, bool FAST>
__device__ __forceinline__ void store_chunk(uint32_t addr, float4 v) {
    if constexpr (MODE == kTF32) {
        v.x = to_tf32(v.x); v.y = to_tf32(v.y); v.z = to_tf32(v.z); v.w = to_tf32(v.w);
    }
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
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

template <int DIST, int MODE, bool FAST>
__device__ __forceinline__ void produce_omega_tile(uint8_t* tile, int64_t kglob0, int roff,
                                                   int npad, int c0, uint32_t key0,
                                                   uint32_t key1, int t) {
    if (t >= npad) return;
    const int n = t;
    const uint32_t col = static_cast<uint32_t>(c0 + n);
    const uint32_t row_base = smem_u32(tile) + static_cast<uint32_t>(n) * 128u;
    const uint32_t sw = static_cast<uint32_t>(n & 7);
    if constexpr (DIST == kRademacher) {
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
            store_chunk<DIST, MODE, FAST>(row_base + ((static_cast<uint32_t>(j4) ^ sw) << 4), v);
        }
    } else {
        const uint64_t q0 = static_cast<uint64_t>(kglob0) >> 2;
        if (roff == 0) {
#pragma unroll 2
            for (int j4 = 0; j4 < 8; ++j4) {
                const float4 v = values4<DIST, FAST>(philox_gauss_call(q0 + j4, col, key0, key1));
                store_chunk<DIST, MODE, FAST>(row_base + ((static_cast<uint32_t>(j4) ^ sw) << 4), v);
            }
        } else {
            // chunk j4 = rows 4(q0+j4)+roff .. +3: last 4-roff values of call q0+j4, first roff of
            // call q0+j4+1
            float4 prev = values4<DIST, FAST>(philox_gauss_call(q0, col, key0, key1));
#pragma unroll 1
            for (int j4 = 0; j4 < 8; ++j4) {
                const float4 next = values4<DIST, FAST>(philox_gauss_call(q0 + j4 + 1, col, key0, key1));
                const float a[8] = {prev.x, prev.y, prev.z, prev.w, next.x, next.y, next.z, next.w};
                float4 v;
                v.x = roff == 1 ? a[1] : roff == 2 ? a[2] : a[3];
                v.y = roff == 1 ? a[2] : roff == 2 ? a[3] : a[4];
                v.z = roff == 1 ? a[3] : roff == 2 ? a[4] : a[5];
                v.w = roff == 1 ? a[4] : roff == 2 ? a[5] : a[6];
                store_chunk<DIST, MODE, FAST>(row_base + ((static_cast<uint32_t>(j4) ^ sw) << 4), v);
                prev = next;
            }
        }
    }
}

template <int NACC, int DIST, int MODE, bool FAST>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const SketchGemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    const SmemLayout L = make_layout(NACC, p.npad, p.a_stages, p.o_stages);
    uint8_t* sA = smem + L.a_off;
    uint8_t* sO = smem + L.o_off;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* full_a = bars;
    uint64_t* empty_a = bars + kMaxStages;
    uint64_t* full_o = bars + 2 * kMaxStages;
    uint64_t* empty_o = bars + 3 * kMaxStages;
    uint64_t* tmem_full = bars + 4 * kMaxStages;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 2);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    uint32_t tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(NACC * p.npad)) tmem_cols <<= 1;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < p.a_stages; ++s) { mbar_init(&full_a[s], 1); mbar_init(&empty_a[s], 1); }
        for (int s = 0; s < p.o_stages; ++s) {
            mbar_init(&full_o[s], kRngThreads);
            mbar_init(&empty_o[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 128);
        fence_barrier_init();
        tma_prefetch_desc(&tmA);
    }
    if (warp == 2) tmem_alloc_rt(tmem_slot, tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int total_units = p.num_mblk * p.split;

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint64_t pol = l2_policy_evict_first();
            uint32_t st = 0, ph = 0;
            for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
                const int mb = u / p.split, s = u - (u / p.split) * p.split;
                const int kb = s * p.kper, ke = min(kb + p.kper, p.kiters);
                for (int kit = kb; kit < ke; ++kit) {
                    mbar_wait(&empty_a[st], ph ^ 1);
                    mbar_arrive_expect_tx(&full_a[st], L.a_stage);
#pragma unroll
                    for (int a = 0; a < NACC; ++a)
                        tma_load_2d(sA + st * L.a_stage + a * kATileBytes, &tmA, &full_a[st],
                                    kit * 32 - p.kshift, (mb * NACC + a) * 128, pol);
                    if (++st == static_cast<uint32_t>(p.a_stages)) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        if (elect_one()) {
            const uint32_t idesc = make_idesc(kFmtTF32, 128, static_cast<uint32_t>(p.npad), 0, 0);
            uint32_t sa = 0, pa = 0, so = 0, po = 0, local = 0;
            for (int u = blockIdx.x; u < total_units; u += gridDim.x, ++local) {
                const int s = u - (u / p.split) * p.split;
                const int kb = s * p.kper, ke = min(kb + p.kper, p.kiters);
                mbar_wait(tmem_empty, (local & 1) ^ 1);
                tc_fence_after();
                for (int kit = kb; kit < ke; ++kit) {
                    mbar_wait(&full_a[sa], pa);
                    mbar_wait(&full_o[so], po);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + sa * L.a_stage);
                    const uint32_t o_base = smem_u32(sO + so * L.o_stage);
#pragma unroll
                    for (int k8 = 0; k8 < 4; ++k8) {
                        const uint64_t bdesc = sw128_desc(o_base + k8 * 32, 16, 1024);
#pragma unroll
                        for (int a = 0; a < NACC; ++a) {
                            const uint64_t adesc = sw128_desc(a_base + a * kATileBytes + k8 * 32, 16, 1024);
                            mma_tf32(tmem_base + a * p.npad, adesc, bdesc, idesc,
                                     (kit > kb || k8 > 0) ? 1u : 0u);
                        }
                    }
                    mma_commit(&empty_a[sa]);
                    mma_commit(&empty_o[so]);
                    if (++sa == static_cast<uint32_t>(p.a_stages)) { sa = 0; pa ^= 1; }
                    if (++so == static_cast<uint32_t>(p.o_stages)) { so = 0; po ^= 1; }
                }
                mma_commit(tmem_full);
            }
        }
    } else if (warp >= kCtlWarps) {
        // ------------------------------------------------------------------ Omega producers + epilogue
        const int t = static_cast<int>(threadIdx.x) - kCtlWarps * 32;
        uint32_t so = 0, po = 0, local = 0;
        for (int u = blockIdx.x; u < total_units; u += gridDim.x, ++local) {
            const int mb = u / p.split, s = u - (u / p.split) * p.split;
            const int kb = s * p.kper, ke = min(kb + p.kper, p.kiters);
            for (int kit = kb; kit < ke; ++kit) {
                mbar_wait(&empty_o[so], po ^ 1);
                produce_omega_tile<DIST, MODE, FAST>(sO + so * L.o_stage,
                                                     p.k0a + static_cast<int64_t>(kit) * 32,
                                                     p.roff, p.npad, p.c0, p.key0, p.key1, t);
                fence_proxy_async_smem();
                mbar_arrive(&full_o[so]);
                if (++so == static_cast<uint32_t>(p.o_stages)) { so = 0; po ^= 1; }
            }
            if (t < 128) {
                // epilogue: warp (4+q) reads TMEM lanes 32q..32q+31
                const int q = t >> 5;
                mbar_wait(tmem_full, local & 1);
                tc_fence_after();
                float* out = p.out + (p.split > 1 ? static_cast<int64_t>(s) * p.part_stride : 0);
#pragma unroll 1
                for (int a = 0; a < NACC; ++a) {
                    const int row = (mb * NACC + a) * 128 + q * 32 + static_cast<int>(lane);
                    float* orow = out + static_cast<int64_t>(row) * p.ldo;
                    const bool vec_ok = ((p.ldo & 3) == 0) &&
                                        ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
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
                        if (row < p.n1) {
                            if (vec_ok && cc + 32 <= p.r_valid) {
#pragma unroll
                                for (int i = 0; i < 32; i += 4)
                                    *reinterpret_cast<float4*>(orow + cc + i) =
                                        make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                                    __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                            } else {
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    if (cc + i < p.r_valid) orow[cc + i] = __uint_as_float(v[i]);
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(tmem_empty);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_rt(tmem_base, tmem_cols);
    }
}

size_t sketch_gemm_smem_bytes(int nacc, int npad, int a_stages, int o_stages) {
    return make_layout(nacc, npad, a_stages, o_stages).total + 1024;
}

int sketch_gemm_max_smem() { return 227 * 1024; }

template <int NACC, int DIST, int MODE, bool FAST>
static cudaError_t launch_one(const CUtensorMap& tmA, const SketchGemmParams& p, int grid,
                              size_t smem, cudaStream_t s) {
    auto kern = sketch_gemm_kernel<NACC, DIST, MODE, FAST>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, s>>>(tmA, p);
    return cudaGetLastError();
}

template <int NACC, int DIST>
static cudaError_t dispatch_mode(const CUtensorMap& tmA, const SketchGemmParams& p, int mode,
                                 bool fast, int grid, size_t smem, cudaStream_t s) {
    if (mode == kTF32) {
        if (DIST == kGaussian && fast) return launch_one<NACC, DIST, kTF32, true>(tmA, p, grid, smem, s);
        return launch_one<NACC, DIST, kTF32, false>(tmA, p, grid, smem, s);
    }
    return cudaErrorNotSupported;
}

cudaError_t launch_sketch_gemm(const CUtensorMap& tmA, const SketchGemmParams& p, int nacc,
                               int dist, int mode, bool fast, int grid, size_t smem,
                               cudaStream_t s) {
    if (nacc == 1) {
        if (dist == kGaussian) return dispatch_mode<1, kGaussian>(tmA, p, mode, fast, grid, smem, s);
        if (dist == kRademacher) return dispatch_mode<1, kRademacher>(tmA, p, mode, fast, grid, smem, s);
        return dispatch_mode<1, kUniform>(tmA, p, mode, fast, grid, smem, s);
    }
    if (nacc == 2) {
        if (dist == kGaussian) return dispatch_mode<2, kGaussian>(tmA, p, mode, fast, grid, smem, s);
        if (dist == kRademacher) return dispatch_mode<2, kRademacher>(tmA, p, mode, fast, grid, smem, s);
        return dispatch_mode<2, kUniform>(tmA, p, mode, fast, grid, smem, s);
    }
    return cudaErrorNotSupported;
}

}  // namespace sk
