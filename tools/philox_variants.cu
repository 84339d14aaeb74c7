// Throughput of Philox4x32-10 round implementations on the SM's integer pipes (no smem / MMA):
// V0 = 64-bit product (IMAD.WIDE.U32), V1 = __umulhi + 32-bit multiply (IMAD.HI.U32 + IMAD),
// V2 = V1 with the low product as a shift-add chain where ptxas picks it.  Results must be identical.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/philox_variants.cu -o /tmp/pv/pv
#include <cstdint>
#include <cstdio>

constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;

template <int V>
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        uint32_t hi0, lo0, hi1, lo1;
        if (V == 0) {
            const uint64_t p0 = static_cast<uint64_t>(M0) * c.x, p1 = static_cast<uint64_t>(M1) * c.z;
            hi0 = p0 >> 32; lo0 = static_cast<uint32_t>(p0); hi1 = p1 >> 32; lo1 = static_cast<uint32_t>(p1);
        } else if (V == 1) {
            hi0 = __umulhi(M0, c.x); lo0 = M0 * c.x; hi1 = __umulhi(M1, c.z); lo1 = M1 * c.z;
        } else {
            asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi0) : "r"(c.x), "n"(M0));
            asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo0) : "r"(c.x), "n"(M0));
            asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi1) : "r"(c.z), "n"(M1));
            asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo1) : "r"(c.z), "n"(M1));
        }
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += W0; k1 += W1;
    }
    return c;
}

template <int V, int ILP>
__global__ void __launch_bounds__(512, 1) bench(int iters, uint32_t k0, uint32_t k1, uint32_t* sink) {
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        uint4 x[ILP];
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = philox<V>(make_uint4(it * ILP + i, 0, t, 0), k0, k1);
#pragma unroll
        for (int i = 0; i < ILP; ++i) acc ^= x[i].x ^ x[i].y ^ x[i].z ^ x[i].w;
    }
    sink[t] = acc;
}

template <int V, int ILP>
void run(const char* name, int threads) {
    uint32_t* sink;
    cudaMalloc(&sink, 148 * 1024 * 4);
    const int iters = 2000;
    bench<V, ILP><<<148, threads>>>(10, 1, 2, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<V, ILP><<<148, threads>>>(iters, 1, 2, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    uint32_t h[4];
    cudaMemcpy(h, sink, 16, cudaMemcpyDeviceToHost);
    const double calls = 148.0 * threads * iters * ILP;
    printf("%-12s thr=%4d ILP=%d: %.3f ms  %.2f calls/clk/SM (@1.9 GHz)  sink=%08x %s\n", name, threads, ILP, ms,
           calls / (ms * 1e-3) / 148 / 1.9e9, h[1], cudaGetErrorString(cudaGetLastError()));
    cudaFree(sink);
}

int main() {
    for (int thr : {256, 512}) {
        run<0, 1>("wide", thr);
        run<1, 1>("hi+lo", thr);
        run<0, 2>("wide", thr);
        run<1, 2>("hi+lo", thr);
        run<2, 1>("asm hi,lo", thr);
        run<2, 2>("asm hi,lo", thr);
    }
    return 0;
}
