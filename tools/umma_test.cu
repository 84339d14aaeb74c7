// Microtest: one CTA, D[128 x N] = A[128 x 32] * B[32 x N] with tcgen05.mma kind::tf32.
// A: K-major SW128 (known good). B: K-major SW128 or MN-major SW128 with a chosen (LBO, SBO).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2603_20966_b200/csrc tools/umma_test.cu -o tools/umma_test
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "ptx.cuh"
using namespace sk;

constexpr int M = 128, K = 32;

__global__ void umma_kernel(const float* A, const float* B, float* D, int N, int b_mn, uint32_t lbo, uint32_t sbo,
                            int swap_ls, int a_mn) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = sm;              // 128 rows x 128 B = 16 KB
    uint8_t* sB = sm + 16384;      // up to 256 x 128 B = 32 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    // A K-major SW128: row m at m*128, chunk j (4 fp32) at ((j ^ (m&7))<<4)
    for (int e = t; e < M * K; e += blockDim.x) {
        int m = e / K, k = e % K;
        uint32_t off;
        if (!a_mn) off = m * 128 + (((k >> 2) ^ (m & 7)) << 4) + (k & 3) * 4;
        else { int g = m / 32, mm = m % 32; off = g * 4096 + k * 128 + (((mm >> 2) ^ (k & 7)) << 4) + (mm & 3) * 4; }
        *(float*)(sA + off) = A[m * K + k];
    }
    for (int e = t; e < K * N; e += blockDim.x) {
        int k = e / N, n = e % N;
        uint32_t off;
        if (!b_mn) {  // K-major: row n, 32 K values
            off = n * 128 + (((k >> 2) ^ (n & 7)) << 4) + (k & 3) * 4;
        } else {      // MN-major: column group g = n/32 of 32 K-rows x 128 B at g*4096; row k at k*128
            int g = n / 32, nn = n % 32;
            off = g * 4096 + k * 128 + (((nn >> 2) ^ (k & 7)) << 4) + (nn & 3) * 4;
        }
        *(float*)(sB + off) = B[k * N + n];
    }
    fence_proxy_async_smem();
    if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (t < 32) tmem_alloc_rt(&tslot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tm = tslot;
    if (t == 0) {
        uint32_t idesc = make_idesc(kFmtTF32, 128, N, a_mn, b_mn);
        for (int k8 = 0; k8 < 4; ++k8) {
            uint64_t ad = a_mn ? sw128_desc(smem_u32(sA) + k8 * 1024, lbo, sbo) : sw128_desc(smem_u32(sA) + k8 * 32, 16, 1024);
            uint64_t bd;
            if (!b_mn) bd = sw128_desc(smem_u32(sB) + k8 * 32, 16, 1024);
            else bd = swap_ls ? sw128_desc(smem_u32(sB) + k8 * 1024, sbo, lbo) : sw128_desc(smem_u32(sB) + k8 * 1024, lbo, sbo);
            mma_tf32(tm, ad, bd, idesc, k8 > 0);
        }
        mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (t < 128) {
        int w = t / 32;
        for (int c = 0; c < N; c += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tm + ((w * 32) << 16) + c, v);
            tmem_ld_wait();
            for (int i = 0; i < 32 && c + i < N; ++i) D[t * N + c + i] = __uint_as_float(v[i]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (t < 32) { tc_fence_after(); tmem_dealloc_rt(tm, 256); }
}

int run(int N, int b_mn, uint32_t lbo, uint32_t sbo, int swap, int a_mn = 0) {
    float *A, *B, *D;
    cudaMallocManaged(&A, M * K * 4); cudaMallocManaged(&B, K * N * 4); cudaMallocManaged(&D, M * N * 4);
    for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7 % 13) - 6);
    for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 5 % 11) - 5);
    for (int i = 0; i < M * N; ++i) D[i] = -999.f;
    umma_kernel<<<1, 128, 64 * 1024>>>(A, B, D, N, b_mn, lbo, sbo, swap, a_mn);
    cudaError_t e = cudaDeviceSynchronize();
    double maxerr = 0; int bad = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double ref = 0; for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[k * N + n];
        double err = fabs(ref - D[m * N + n]); if (err > maxerr) maxerr = err; if (err > 1e-3) ++bad;
    }
    printf("a_mn=%d N=%3d b_mn=%d lbo=%5u sbo=%5u swap=%d: %s maxerr=%g bad=%d D[0]=%g\n", a_mn, N, b_mn, lbo, sbo, swap,
           cudaGetErrorString(e), maxerr, bad, D[0]);
    cudaFree(A); cudaFree(B); cudaFree(D);
    return e != cudaSuccess;
}

int main() {
    cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    run(32, 0, 16, 1024, 0);
    run(64, 0, 16, 1024, 0);
    run(32, 1, 4096, 1024, 0);
    run(64, 1, 4096, 1024, 0);
    run(64, 1, 4096, 1024, 1);
    run(64, 1, 1024, 4096, 0);
    run(256, 1, 4096, 1024, 0);
    run(256, 1, 4096, 1024, 1);
    run(64, 0, 4096, 1024, 0, 1);
    run(64, 0, 1024, 4096, 0, 1);
    run(64, 1, 4096, 1024, 0, 1);
    // small LBO/SBO values in case the unit is not bytes
    run(64, 1, 256, 64, 0);
    run(64, 1, 64, 256, 0);
    return 0;
}
