// omega.cu -- materialise Omega (or its raw Philox words) for tests / debugging
// (sketch_generate / sketch_generate_bits), and the Box-Muller debug evaluator.
// The hot path never calls these: the GEMM kernels generate Omega tiles in shared memory.
#include <algorithm>

#include "kernels.cuh"
#include "philox.cuh"

namespace sk {

// One thread per (Philox call, column). Gaussian / uniform: a call covers 4 rows (q = j >> 2);
// Rademacher: a call covers 128 rows (g = j >> 7).
template <int DIST, bool BITS>
__global__ void generate_kernel(uint32_t key0, uint32_t key1, int64_t row0, int64_t nrows,
                                int64_t col0, int64_t ncols, void* out, int64_t ld) {
    const int rows_per_call = (DIST == kRademacher) ? 128 : 4;
    const int64_t first = row0 / rows_per_call;
    const int64_t last = (row0 + nrows - 1) / rows_per_call;
    const int64_t ncalls = last - first + 1;
    const int64_t total = ncalls * ncols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = idx % ncols;
        const int64_t call = first + idx / ncols;
        const uint32_t col = static_cast<uint32_t>(col0 + c);
        if constexpr (DIST == kRademacher) {
            const uint4 x = philox_rade_call(static_cast<uint64_t>(call), col, key0, key1);
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
            for (int e = 0; e < 128; ++e) {
                const int64_t j = call * 128 + e;
                if (j < row0 || j >= row0 + nrows) continue;
                const uint32_t word = w[e >> 5];
                if (BITS) {
                    static_cast<uint32_t*>(out)[(j - row0) * ld + c] = word;
                } else {
                    static_cast<float*>(out)[(j - row0) * ld + c] = rade_from_bit(word, e & 31);
                }
            }
        } else {
            const uint4 x = philox_gauss_call(static_cast<uint64_t>(call), col, key0, key1);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!BITS) {
                if (DIST == kUniform)
                    v = make_float4(uniform_from_word(x.x), uniform_from_word(x.y),
                                    uniform_from_word(x.z), uniform_from_word(x.w));
                else
                    v = gauss4<false>(x);
            }
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
            const float f[4] = {v.x, v.y, v.z, v.w};
            for (int e = 0; e < 4; ++e) {
                const int64_t j = call * 4 + e;
                if (j < row0 || j >= row0 + nrows) continue;
                if (BITS) static_cast<uint32_t*>(out)[(j - row0) * ld + c] = w[e];
                else static_cast<float*>(out)[(j - row0) * ld + c] = f[e];
            }
        }
    }
}

cudaError_t launch_generate(uint64_t seed, int dist, int64_t row0, int64_t nrows, int64_t col0,
                            int64_t ncols, void* out, int64_t ld, bool bits, cudaStream_t s) {
    if (nrows <= 0 || ncols <= 0) return cudaSuccess;
    const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
    const int per = (dist == kRademacher) ? 128 : 4;
    const int64_t calls = ((row0 + nrows - 1) / per - row0 / per + 1) * ncols;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((calls + threads - 1) / threads, 148 * 32);
    const int g = static_cast<int>(blocks);
#define SK_GEN(D, B) generate_kernel<D, B><<<g, threads, 0, s>>>(k0, k1, row0, nrows, col0, ncols, out, ld)
    if (dist == kGaussian) { if (bits) SK_GEN(kGaussian, true); else SK_GEN(kGaussian, false); }
    else if (dist == kRademacher) { if (bits) SK_GEN(kRademacher, true); else SK_GEN(kRademacher, false); }
    else { if (bits) SK_GEN(kUniform, true); else SK_GEN(kUniform, false); }
#undef SK_GEN
    return cudaGetLastError();
}

template <bool FAST>
__global__ void debug_box_muller_kernel(const uint32_t* w1, const uint32_t* w2, int64_t n,
                                        float* oe, float* oo) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float2 z = FAST ? box_muller_fast(w1[i], w2[i]) : box_muller_accurate(w1[i], w2[i]);
        oe[i] = z.x;
        oo[i] = z.y;
    }
}

cudaError_t launch_debug_box_muller(const uint32_t* w1, const uint32_t* w2, int64_t n, bool fast,
                                    float* oe, float* oo, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
    if (fast) debug_box_muller_kernel<true><<<blocks, 256, 0, s>>>(w1, w2, n, oe, oo);
    else debug_box_muller_kernel<false><<<blocks, 256, 0, s>>>(w1, w2, n, oe, oo);
    return cudaGetLastError();
}

}  // namespace sk
