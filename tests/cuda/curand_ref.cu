// Test infrastructure only: NVIDIA cuRAND's own Philox4x32-10 round function (curand_kernel.h,
// curand_Philox4x32_10), an implementation independent of both this library and oracle/, used to
// pin the library's device Philox bit for bit on the GPU (SURVEY §4.2 unit test).
#include <cstdint>
#include <curand_kernel.h>

__global__ void curand_words_kernel(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
    const uint2 k = make_uint2(key[2 * i], key[2 * i + 1]);
    const uint4 x = curand_Philox4x32_10(c, k);
    out[4 * i] = x.x;
    out[4 * i + 1] = x.y;
    out[4 * i + 2] = x.z;
    out[4 * i + 3] = x.w;
}

extern "C" int curand_philox_words(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
    if (n <= 0) return 0;
    curand_words_kernel<<<static_cast<unsigned>((n + 255) / 256), 256>>>(ctr, key, n, out);
    return static_cast<int>(cudaDeviceSynchronize());
}
