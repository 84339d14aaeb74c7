// kernels.cuh -- launch-side declarations shared by the kernels and the C ABI (api.cu).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sk {

enum Dist : int { kGaussian = 0, kRademacher = 1, kUniform = 2 };
enum Mode : int { kTF32x3 = 0, kTF32 = 1, kBF16 = 2 };

// One launch of the fused sketch GEMM: B_pass = A[:, kshift-aligned K range] * Omega tile,
// for accumulator columns [c0, c0 + npad) of Omega.
struct SketchGemmParams {
    float* out;           // B (split == 1) or split-K partials (split > 1)
    int64_t ldo;          // row stride of out (elements)
    int64_t part_stride;  // elements between consecutive split partials
    int64_t k0a;          // global Omega row of tile row 0 of K-iteration 0 (= aligned + roff)
    int32_t kshift;       // A column of tile row 0 is (kit*32 - kshift), kshift % 4 == 0 (TMA
                          // needs 16-byte inner coordinates); negative columns -> TMA zero fill
    int32_t roff;         // k0a % 4 (0 except for unaligned block calls)
    int32_t n1;           // rows of A
    int32_t kiters;       // number of K iterations (32 wide; 64 wide in bf16 mode)
    int32_t r_valid;      // columns of this pass to store (<= npad)
    int32_t c0;           // global Omega column of accumulator column 0
    int32_t npad;         // MMA N (multiple of 16, <= 256)
    int32_t num_mblk;     // ceil(n1 / (128 * nacc))
    int32_t split;        // split-K factor S
    int32_t kper;         // K iterations per split
    int32_t a_stages;     // A smem pipeline depth
    int32_t o_stages;     // Omega smem pipeline depth
    int32_t y_stages;     // bf16: depth of the ring holding K 32..63 of each fp32 A stage
    int32_t prefetch;     // K steps of A prefetched into L2 ahead of the TMA loads (0 = off)
    int32_t kchunk;       // > 0 (tf32x3): K iterations per TMEM accumulation; each chunk is drained
                          // and added (fp32 RN) into the unit's output, which accumulates in place
    int32_t inplace;      // 1: the split / stream-K pieces of an m-block accumulate straight into out
                          // (= B) in DESCENDING piece order (the top piece stores, each lower piece
                          // waits for the one above it, then adds): no partials, no reduce kernel
    int32_t max_pieces;   // inplace: pieces per m-block (flag array stride)
    int32_t* flags;       // inplace: [m-block][piece][CTA of the cluster] completion flags, zeroed
                          // before the launch
    int64_t sk_len;       // > 0: stream-K -- worker w runs flattened (m-block, K-iteration) indices
                          // [w sk_len, (w+1) sk_len), cut at m-block boundaries; partial `piece` =
                          // w - first worker touching the m-block (split / kper unused)
    uint32_t key0, key1;  // Philox key = (seed lo, seed hi)
    uint32_t ablate;      // 0 in production; bit 0: skip Omega generation, bit 1: skip A loads
    uint64_t* trace;      // diagnostics (SK_TRACE builds): globaltimer stamps [cta][event][stage]
    int32_t trace_stages;
    // fused reduce-scatter (f1; rs_ndst > 0): output row i goes to
    //   rs_dst[i / rs_piece] + (rs_slot * split + s) * rs_slot_elems + (i % rs_piece) * ldo + col
    // (peer receive buffers mapped over NVLink) instead of out
    float* rs_dst[8];
    int32_t rs_ndst;
    int32_t rs_slot;
    int64_t rs_piece;
    int64_t rs_slot_elems;
};

struct CoreGemmParams {
    const float* B;       // B block (m x r, ldb), device
    int64_t ldb;
    float* part;          // per-chunk r x r partials (chunks x r x r), or C if chunks == 1
    int64_t ldp;          // row stride of a partial (elements)
    int64_t i0;           // global Omega row of B row 0
    int32_t m;            // rows of B
    int32_t r;            // Omega columns = rows of C
    int32_t nb;           // columns of B = columns of C (r for the Nystrom core, r/P for Redist)
    int32_t chunk_rows;   // rows of B per CTA chunk
    int32_t chunks;
    uint32_t key0, key1;
};

// tcgen05 core GEMM (r <= 256): chunk c covers global Omega rows
// [max(i0, base + c*step), min(i0 + m, base + (c+1)*step)), base = i0 & ~127, step % 128 == 0.
struct CoreTcParams {
    float* part;          // nchunks x r x ldp partials
    int64_t ldp;          // row stride of a partial (elements)
    int64_t i0;           // global Omega row of B row 0
    int64_t base;         // i0 rounded down to 128
    int64_t step;         // rows per chunk (multiple of 128)
    int32_t m;            // rows of B
    int32_t r;            // Omega columns = rows of C
    int32_t nb;           // columns of B = columns of C
    int32_t npad;         // MMA N = columns per block (multiple of 16, <= 256; <= 128 in tf32x3)
    int32_t nchunks;
    int32_t tma_store;    // 1: epilogue stores 32x32 tiles with TMA through tmOut (r % 32 == 0)
    uint32_t key0, key1;
    float* mc_out;        // non-NULL: the epilogue ADDS each partial into C on every rank of a multicast
    int64_t ldc_mc;       // group (multimem.red at mc_out + a * ldc_mc + b), instead of storing partials
};

struct LaunchCfg {
    int nacc;
    int split;
    int grid;
    int a_stages;
    int o_stages;
    size_t smem;
};

// Host-side launchers (return cudaError_t of the launch).
cudaError_t launch_sketch_gemm(const CUtensorMap& tmA, const SketchGemmParams& p, int cg,
                               int nacc, int dist, int mode, bool fast, int grid, size_t smem,
                               cudaStream_t s, int cl = 1, int ncol = 1);
int sketch_gemm_max_clusters(int cg, int nacc, int dist, int mode, bool fast, int cl, size_t smem, int ncol = 1);
size_t sketch_gemm_smem_bytes(int cg, int nacc, int npad, int a_stages, int o_stages, bool xa,
                              bool olo, int ks, int nsubo, int y_stages);
int sketch_gemm_max_smem();
cudaError_t raise_smem_limit(const void* fn, size_t smem);

cudaError_t launch_pack_cols(const float* B, int64_t rows, int64_t ldb, const int64_t* cb, int32_t nblk,
                             float* out, cudaStream_t s);
cudaError_t launch_multimem_sum(const float* mc_src, int64_t elems, float* out, float* mc_out, cudaStream_t s);
cudaError_t launch_sum_peers(const float* const* src, int32_t n, int64_t elems, float* out, cudaStream_t s);
cudaError_t launch_streamk_reduce(const float* part, int64_t part_stride, int32_t n1, int32_t r_valid,
                                  int32_t ldp, float* out, int64_t ldo, int32_t rows_per_unit, int32_t kiters,
                                  int64_t sk_len, cudaStream_t s);
cudaError_t launch_splitk_reduce(const float* part, int64_t part_stride, int32_t split,
                                 int32_t n1, int32_t r_valid, int32_t ldp, float* out,
                                 int64_t ldo, cudaStream_t s);

cudaError_t launch_core_gemm(const CoreGemmParams& p, int dist, bool fast, cudaStream_t s);
cudaError_t launch_core_gemm_tc(const CUtensorMap& tmB, const CUtensorMap& tmOut, const CoreTcParams& p,
                                int nacc, int dist, bool fast, bool x3, cudaStream_t s);
size_t core_gemm_tc_smem_bytes(int nacc, int npad, bool x3, bool olo);
cudaError_t launch_accumulate(float* acc, const float* part, int64_t n, bool first, cudaStream_t s);
cudaError_t launch_core_reduce(const float* part, int32_t chunks, int32_t r, int32_t nb, float* C,
                               int64_t ldc, cudaStream_t s);

cudaError_t launch_generate(uint64_t seed, int dist, int64_t row0, int64_t nrows, int64_t col0,
                            int64_t ncols, void* out, int64_t ld, bool bits, cudaStream_t s);
cudaError_t launch_debug_box_muller(const uint32_t* w1, const uint32_t* w2, int64_t n, bool fast,
                                    float* oe, float* oo, cudaStream_t s);

int num_sms();

}  // namespace sk
