// reduce.cu -- deterministic fixed-order reductions (reading R9): split-K partials of B and
// per-chunk r x r partials of C.  Partial s is always added in increasing s.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace sk {

// out[i, c] = sum_{s < split} part[s][i][c]   (part row stride ldp, s stride part_stride)
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int64_t part_stride,
                                     int32_t split, int32_t n1, int32_t r_valid, int32_t ldp,
                                     float* __restrict__ out, int64_t ldo) {
    const int64_t total = static_cast<int64_t>(n1) * r_valid;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / r_valid;
        const int64_t c = idx - i * r_valid;
        const float* p = part + i * ldp + c;
        float acc = __ldg(p);
        for (int s = 1; s < split; ++s) acc += __ldg(p + s * part_stride);
        out[i * ldo + c] = acc;
    }
}

// Vectorised variant: 4 consecutive columns per thread (r_valid % 4 == 0, aligned rows).
__global__ void splitk_reduce_kernel_v4(const float4* __restrict__ part, int64_t part_stride4,
                                        int32_t split, int32_t n1, int32_t r4, int32_t ldp4,
                                        float4* __restrict__ out, int64_t ldo4) {
    const int64_t total = static_cast<int64_t>(n1) * r4;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / r4;
        const int64_t c = idx - i * r4;
        const float4* p = part + i * ldp4 + c;
        float4 acc = __ldg(p);
        for (int s = 1; s < split; ++s) {
            const float4 v = __ldg(p + s * part_stride4);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        out[i * ldo4 + c] = acc;
    }
}

cudaError_t launch_splitk_reduce(const float* part, int64_t part_stride, int32_t split,
                                 int32_t n1, int32_t r_valid, int32_t ldp, float* out,
                                 int64_t ldo, cudaStream_t s) {
    if (n1 <= 0 || r_valid <= 0) return cudaSuccess;
    const int threads = 256;
    const bool v4 = (r_valid % 4 == 0) && (ldp % 4 == 0) && (ldo % 4 == 0) &&
                    (part_stride % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(part) & 15) == 0);
    const int64_t total = static_cast<int64_t>(n1) * (v4 ? r_valid / 4 : r_valid);
    const int blocks = static_cast<int>(std::min<int64_t>((total + threads - 1) / threads, 148 * 16));
    if (v4)
        splitk_reduce_kernel_v4<<<blocks, threads, 0, s>>>(
            reinterpret_cast<const float4*>(part), part_stride / 4, split, n1, r_valid / 4,
            ldp / 4, reinterpret_cast<float4*>(out), ldo / 4);
    else
        splitk_reduce_kernel<<<blocks, threads, 0, s>>>(part, part_stride, split, n1, r_valid,
                                                        ldp, out, ldo);
    return cudaGetLastError();
}

// Stream-K partials: row i belongs to m-block mb = i / rows_per_unit, whose K iterations were cut by
// the workers' ranges into pieces 0 .. last - first (first / last = first and last worker touching
// the m-block); out[i, c] = sum of those pieces in increasing piece (= K) order.
__global__ void streamk_reduce_kernel_v4(const float4* __restrict__ part, int64_t part_stride4, int32_t n1,
                                         int32_t r4, int32_t ldp4, float4* __restrict__ out, int64_t ldo4,
                                         int32_t rows_per_unit, int32_t kiters, int64_t sk_len) {
    const int64_t total = static_cast<int64_t>(n1) * r4;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / r4;
        const int64_t c = idx - i * r4;
        const int64_t mb = i / rows_per_unit;
        const int64_t first = (mb * kiters) / sk_len, last = ((mb + 1) * kiters - 1) / sk_len;
        const float4* p = part + i * ldp4 + c;
        float4 acc = __ldg(p);
        for (int64_t s = 1; s <= last - first; ++s) {
            const float4 v = __ldg(p + s * part_stride4);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        out[i * ldo4 + c] = acc;
    }
}

__global__ void streamk_reduce_kernel(const float* __restrict__ part, int64_t part_stride, int32_t n1,
                                      int32_t r_valid, int32_t ldp, float* __restrict__ out, int64_t ldo,
                                      int32_t rows_per_unit, int32_t kiters, int64_t sk_len) {
    const int64_t total = static_cast<int64_t>(n1) * r_valid;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / r_valid;
        const int64_t c = idx - i * r_valid;
        const int64_t mb = i / rows_per_unit;
        const int64_t first = (mb * kiters) / sk_len, last = ((mb + 1) * kiters - 1) / sk_len;
        const float* p = part + i * ldp + c;
        float acc = __ldg(p);
        for (int64_t s = 1; s <= last - first; ++s) acc += __ldg(p + s * part_stride);
        out[i * ldo + c] = acc;
    }
}

cudaError_t launch_streamk_reduce(const float* part, int64_t part_stride, int32_t n1, int32_t r_valid,
                                  int32_t ldp, float* out, int64_t ldo, int32_t rows_per_unit, int32_t kiters,
                                  int64_t sk_len, cudaStream_t s) {
    if (n1 <= 0 || r_valid <= 0) return cudaSuccess;
    const int threads = 256;
    const bool v4 = (r_valid % 4 == 0) && (ldp % 4 == 0) && (ldo % 4 == 0) && (part_stride % 4 == 0) &&
                    ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((reinterpret_cast<uintptr_t>(part) & 15) == 0);
    const int64_t total = static_cast<int64_t>(n1) * (v4 ? r_valid / 4 : r_valid);
    const int blocks = static_cast<int>(std::min<int64_t>((total + threads - 1) / threads, 148 * 16));
    if (v4)
        streamk_reduce_kernel_v4<<<blocks, threads, 0, s>>>(
            reinterpret_cast<const float4*>(part), part_stride / 4, n1, r_valid / 4, ldp / 4,
            reinterpret_cast<float4*>(out), ldo / 4, rows_per_unit, kiters, sk_len);
    else
        streamk_reduce_kernel<<<blocks, threads, 0, s>>>(part, part_stride, n1, r_valid, ldp, out, ldo,
                                                         rows_per_unit, kiters, sk_len);
    return cudaGetLastError();
}

// out[i] = sum_{j < n} src[j][i] in increasing j (fixed order): the AllReduce of C's r x r partials
// read straight from every rank's symmetric-memory slot over NVLink.
struct PeerPtrs {
    const float4* p[8];
};
__global__ void sum_peers_kernel(PeerPtrs src, int32_t n, int64_t n4, float4* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float4 acc = src.p[0][i];
        for (int j = 1; j < n; ++j) {
            const float4 v = src.p[j][i];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        out[i] = acc;
    }
}

// Compile-time rank count: all N x U loads of a thread are independent and issued before the adds
// (NVLink reads need many requests in flight); the sum order stays rank 0, 1, ..., N-1.
template <int N>
__global__ void __launch_bounds__(256) sum_peers_kernel_n(PeerPtrs src, int64_t n4, float4* __restrict__ out) {
    constexpr int kU = 2;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += stride * kU) {
        float4 v[kU][N];
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
            for (int j = 0; j < N; ++j)
                if (i0 + u * stride < n4) v[u][j] = src.p[j][i0 + u * stride];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (i0 + u * stride >= n4) break;
            float4 acc = v[u][0];
#pragma unroll
            for (int j = 1; j < N; ++j) {
                acc.x += v[u][j].x; acc.y += v[u][j].y; acc.z += v[u][j].z; acc.w += v[u][j].w;
            }
            out[i0 + u * stride] = acc;
        }
    }
}

cudaError_t launch_sum_peers(const float* const* src, int32_t n, int64_t elems, float* out, cudaStream_t s) {
    if (n < 1 || n > 8 || (elems & 3)) return cudaErrorInvalidValue;
    PeerPtrs pp{};
    for (int j = 0; j < n; ++j) pp.p[j] = reinterpret_cast<const float4*>(src[j]);
    const int64_t n4 = elems / 4;
    const int blocks = std::max(1, static_cast<int>(std::min<int64_t>((n4 + 255) / 256, 148 * 4)));
    float4* o = reinterpret_cast<float4*>(out);
    if (getenv("SK_SUM_PEERS_V1") == nullptr) {  // tuning: the scalar-loop kernel
        switch (n) {
            case 2: sum_peers_kernel_n<2><<<blocks, 256, 0, s>>>(pp, n4, o); return cudaGetLastError();
            case 4: sum_peers_kernel_n<4><<<blocks, 256, 0, s>>>(pp, n4, o); return cudaGetLastError();
            case 8: sum_peers_kernel_n<8><<<blocks, 256, 0, s>>>(pp, n4, o); return cudaGetLastError();
            default: break;
        }
    }
    sum_peers_kernel<<<blocks, 256, 0, s>>>(pp, n, n4, o);
    return cudaGetLastError();
}

// NVLS (NVLink SHARP): out[i] = sum over the multicast group's ranks of their copies of mc_src[i],
// reduced inside the NVSwitch (multimem.ld_reduce, fp32 RN) -- one read per element per rank instead
// of P peer reads; optionally broadcast back through the multicast mapping (multimem.st).
__device__ __forceinline__ float4 multimem_ld_sum(const float* mc) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(mc)
                 : "memory");
    return v;
}

// 4 independent in-switch loads in flight per thread (each crosses NVLink to every rank's copy)
__global__ void multimem_sum_kernel(const float* __restrict__ mc_src, int64_t n4, float* __restrict__ out,
                                    float* __restrict__ mc_out) {
    constexpr int kU = 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i0 < n4; i0 += stride * kU) {
        float4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * stride < n4) v[u] = multimem_ld_sum(mc_src + 4 * (i0 + u * stride));
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t i = i0 + u * stride;
            if (i >= n4) break;
            if (out) reinterpret_cast<float4*>(out)[i] = v[u];
            if (mc_out)
                asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_out + 4 * i),
                             "f"(v[u].x), "f"(v[u].y), "f"(v[u].z), "f"(v[u].w)
                             : "memory");
        }
    }
}

cudaError_t launch_multimem_sum(const float* mc_src, int64_t elems, float* out, float* mc_out, cudaStream_t s) {
    const int64_t n4 = elems / 4;
    if (n4 <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<int64_t>((n4 + 1023) / 1024, 148 * 2));
    multimem_sum_kernel<<<blocks, 256, 0, s>>>(mc_src, n4, out, mc_out);
    return cudaGetLastError();
}

// Column-block pack (Redist All-to-All): out[rows * cb[j] + i * (cb[j+1] - cb[j]) + (c - cb[j])] =
// B[i, c] for c in [cb[j], cb[j+1]).  One thread per element of B, reads coalesced along c.
struct ColBounds {
    int64_t b[65];
    int32_t n;
};
__global__ void pack_cols_kernel(const float* __restrict__ B, int64_t rows, int64_t ldb, ColBounds cb,
                                 float* __restrict__ out) {
    const int64_t w = cb.b[cb.n];
    const int64_t total = rows * w;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / w, c = idx - i * w;
        int j = 0;
        while (c >= cb.b[j + 1]) ++j;
        const int64_t wj = cb.b[j + 1] - cb.b[j];
        out[rows * cb.b[j] + i * wj + (c - cb.b[j])] = B[i * ldb + c];
    }
}

cudaError_t launch_pack_cols(const float* B, int64_t rows, int64_t ldb, const int64_t* cb, int32_t nblk,
                             float* out, cudaStream_t s) {
    ColBounds c{};
    for (int j = 0; j <= nblk; ++j) c.b[j] = cb[j];
    c.n = nblk;
    const int64_t total = rows * cb[nblk];
    if (total <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8));
    pack_cols_kernel<<<blocks, 256, 0, s>>>(B, rows, ldb, c, out);
    return cudaGetLastError();
}

// C[a, b] = sum_{c < chunks} part[c][a][b], r x nb, fixed order.
__global__ void core_reduce_kernel(const float* __restrict__ part, int32_t chunks, int32_t r, int32_t nb,
                                   float* __restrict__ C, int64_t ldc) {
    const int64_t rr = static_cast<int64_t>(r) * nb;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < rr;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int c = 0; c < chunks; ++c) acc += __ldg(part + c * rr + idx);
        C[(idx / nb) * ldc + idx % nb] = acc;
    }
}

// acc[a, b] (+)= part[a, b] over an r x r block (host streaming: fixed block order).
__global__ void accumulate_kernel(float* __restrict__ acc, const float* __restrict__ part, int64_t n,
                                  int first) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        acc[i] = first ? part[i] : acc[i] + part[i];
}

cudaError_t launch_accumulate(float* acc, const float* part, int64_t n, bool first, cudaStream_t s) {
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 4));
    accumulate_kernel<<<blocks, 256, 0, s>>>(acc, part, n, first ? 1 : 0);
    return cudaGetLastError();
}

// Same sums with the chunks split over 8 thread groups (many more loads in flight: the partials are
// read from L2 right after the core GEMM wrote them).  Block = 8 groups x 32 threads over 32 float4
// (128 consecutive elements); group g sums chunks [g C / 8, (g+1) C / 8) in increasing order, then
// group 0 adds the 8 group sums in increasing g: a fixed bracketing of the chunk order, so reruns
// are bit-identical.  Needs r * nb % 4 == 0 and a 16-byte aligned `part`.
__global__ void __launch_bounds__(256) core_reduce_kernel_v4(const float* __restrict__ part, int32_t chunks,
                                                             int32_t nb, int64_t rr, float* __restrict__ C,
                                                             int64_t ldc) {
    __shared__ float4 sums[8][32];
    const int g = static_cast<int>(threadIdx.x >> 5), l = static_cast<int>(threadIdx.x & 31);
    const int64_t i4 = static_cast<int64_t>(blockIdx.x) * 32 + l;  // float4 index
    const bool valid = i4 * 4 < rr;
    const int c0 = (chunks * g) / 8, c1 = (chunks * (g + 1)) / 8;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
        const float4* p4 = reinterpret_cast<const float4*>(part) + i4;
        const int64_t cs = rr / 4;
        int c = c0;
        for (; c + 4 <= c1; c += 4) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcg(p4 + (c + u) * cs);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
            }
        }
        for (; c < c1; ++c) {
            const float4 v = __ldcg(p4 + c * cs);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    sums[g][l] = acc;
    __syncthreads();
    if (g == 0 && valid) {
        float4 t = sums[0][l];
#pragma unroll
        for (int h = 1; h < 8; ++h) {
            const float4 v = sums[h][l];
            t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
        }
        const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int64_t idx = i4 * 4 + e;
            C[(idx / nb) * ldc + idx % nb] = tv[e];
        }
    }
}

cudaError_t launch_core_reduce(const float* part, int32_t chunks, int32_t r, int32_t nb, float* C,
                               int64_t ldc, cudaStream_t s) {
    const int64_t rr = static_cast<int64_t>(r) * nb;
    if (rr % 4 == 0 && (reinterpret_cast<uintptr_t>(part) & 15) == 0 && chunks >= 16) {
        const int64_t blocks = (rr / 4 + 31) / 32;
        core_reduce_kernel_v4<<<static_cast<unsigned>(blocks), 256, 0, s>>>(part, chunks, nb, rr, C, ldc);
        return cudaGetLastError();
    }
    const int blocks = static_cast<int>(std::min<int64_t>((rr + 255) / 256, 148 * 8));
    core_reduce_kernel<<<blocks, 256, 0, s>>>(part, chunks, r, nb, C, ldc);
    return cudaGetLastError();
}

}  // namespace sk
