// core_gemm.cu -- C_part = Omega[i0:i0+m, :r]^T * B_blk (Alg. 2 line
// "C-bar_j'k' = Omega^T_i'j' * B_i'k'"), with the Omega rows REGENERATED bit-identically to the
// ones the sketch GEMM used (Alg. 2 regenerates rather than reuses; reading R16).
//
// v1: fp32 SIMT tiles (64 x 64 outputs per CTA, 32-row K steps through shared memory), K split
// into `chunks` contiguous row ranges, one r x r partial per chunk, reduced in fixed order by
// core_reduce_kernel.  fp32 FMA accumulation makes C at least as accurate as B in every mode.
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
            sB[i][c] = (i < nr && b0 + c < p.r) ? p.B[static_cast<int64_t>(rb + i) * p.ldb + b0 + c] : 0.f;
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
            if (b < p.r) out[static_cast<int64_t>(a) * p.ldp + b] = acc[u][v];
        }
    }
}

cudaError_t launch_core_gemm(const CoreGemmParams& p, int dist, bool fast, cudaStream_t s) {
    const int t = (p.r + kCT - 1) / kCT;
    dim3 grid(t, t, p.chunks);
    if (dist == kRademacher) core_gemm_simt_kernel<kRademacher, false><<<grid, 256, 0, s>>>(p);
    else if (dist == kUniform) core_gemm_simt_kernel<kUniform, false><<<grid, 256, 0, s>>>(p);
    else if (fast) core_gemm_simt_kernel<kGaussian, true><<<grid, 256, 0, s>>>(p);
    else core_gemm_simt_kernel<kGaussian, false><<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace sk
