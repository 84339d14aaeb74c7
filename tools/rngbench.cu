// Standalone throughput benchmark of the in-kernel Omega tile generator variants (no TMA / MMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_20966_b200/csrc tools/rngbench.cu -o tools/rngbench
#include <cstdio>
#include <cstdint>
#include "philox.cuh"
using namespace sk;

template <int VARIANT, int NW, int ILP>
__global__ void __launch_bounds__(NW * 32, 1) bench(int tiles, int npad, uint32_t k0, uint32_t k1, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int T = NW * 32;
    const int t = threadIdx.x;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const int chunks = npad * 8;
    float acc = 0.f;
    for (int tile = 0; tile < tiles; ++tile) {
        const uint64_t q0 = (static_cast<uint64_t>(blockIdx.x) * tiles + tile) * 8;
        #pragma unroll 1
        for (int c = t; c < chunks; c += T * ILP) {
            float4 v[ILP];
            int nn[ILP], jj[ILP];
            #pragma unroll
            for (int i = 0; i < ILP; ++i) {
                int cc = c + i * T; if (cc >= chunks) cc = c;
                nn[i] = cc % npad; jj[i] = cc / npad;
                uint4 x = philox_gauss_call(q0 + jj[i], nn[i], k0, k1);
                if (VARIANT == 0) v[i] = gauss4<false>(x);
                else if (VARIANT == 1) v[i] = gauss4<true>(x);
                else v[i] = make_float4(__uint_as_float(x.x), __uint_as_float(x.y), __uint_as_float(x.z), __uint_as_float(x.w));
            }
            #pragma unroll
            for (int i = 0; i < ILP; ++i) {
                const uint32_t addr = base + nn[i] * 128u + ((jj[i] ^ (nn[i] & 7)) << 4);
                asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" :: "r"(addr), "f"(v[i].x), "f"(v[i].y), "f"(v[i].z), "f"(v[i].w) : "memory");
            }
        }
        __syncthreads();
    }
    if (t == 0) sink[blockIdx.x] = acc + __uint_as_float(*reinterpret_cast<uint32_t*>(sm));
}

template <int V, int NW, int ILP>
void run(const char* name, int npad) {
    float* sink; cudaMalloc(&sink, 4096 * 4);
    int tiles = 400;
    size_t smem = npad * 128;
    auto k = bench<V, NW, ILP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<148, NW * 32, smem>>>(4, npad, 1, 2, sink);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, NW * 32, smem>>>(tiles, npad, 1, 2, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double g = 148.0 * tiles * npad * 32;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s npad=%3d NW=%2d ILP=%d: %.3f ms  %.1f G/s  %.2f /clk/SM(@1.9GHz)  err=%s\n", name, npad, NW, ILP, ms,
           g / ms / 1e6, g / (ms * 1e-3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
}

int main() {
    run<2, 16, 1>("philox only", 128);
    run<2, 16, 2>("philox only", 128);
    run<1, 16, 1>("fast", 128);
    run<1, 16, 2>("fast", 128);
    run<1, 16, 4>("fast", 128);
    run<1, 8, 2>("fast", 128);
    run<1, 24, 2>("fast", 128);
    run<0, 16, 1>("accurate", 128);
    run<0, 16, 2>("accurate", 128);
    run<0, 16, 4>("accurate", 128);
    run<0, 24, 2>("accurate", 128);
    run<1, 16, 2>("fast", 256);
    run<0, 16, 2>("accurate", 256);
    return 0;
}
