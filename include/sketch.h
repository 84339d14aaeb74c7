/*
 * sketch.h -- C ABI of libsketch.so, the B200 (sm_100a) hot path of arXiv 2603.20966
 * "Communication Lower Bounds and Algorithms for Sketching with Random Dense Matrices".
 *
 * Operations (PAPER.md line numbers, LaTeX source):
 *   sketch_apply   B = A * Omega,        A in R^{n1 x n2}, Omega in R^{n2 x r}   (sec. 1)
 *   nystrom_core   B = A * Omega, C = Omega^T * B  (= Omega^T A Omega)          (sec. 1)
 *   *_block        the local products of Alg. 1 line "B-bar_ik = A_ij * Omega_jk" and
 *                  Alg. 2 lines "B-hat-bar = A_ij Omega_jk" / "C-bar = Omega^T_i'j' B_i'k'"
 *                  (PAPER.md:594), with global offsets selecting the rows of Omega.
 * Omega is never stored in HBM nor communicated: every kernel regenerates the tiles it needs from
 * a counter-based Philox4x32-10 stream with a shared seed (sec. 6.3), inside
 * the GEMM, straight into swizzled shared memory.  Entry (j,k) of Omega is a pure function of
 * (seed, dist, global row j, global column k) -- reading O1 in DESIGN.md:
 *   GAUSSIAN   Box-Muller on words of Philox((j>>2), k, tag 0): rows 4q,4q+1 use (x0,x1), rows
 *              4q+2,4q+3 use (x2,x3); u1 = ((w1>>8)+1)/2^24, u2 = (w2>>8)/2^24,
 *              z = sqrt(-2 ln u1) * (cos 2 pi u2 for even j | sin 2 pi u2 for odd j).  Unscaled N(0,1).
 *   RADEMACHER bit (j&31) of word ((j>>5)&3) of Philox((j>>7), k, tag 1); set bit -> -1, else +1.
 *   UNIFORM    (x[j&3] >> 8) / 2^24 in [0,1) from the tag-0 call (the paper's experiment).
 *
 * Conventions (all entry points):
 *   - matrices are fp32, ROW-MAJOR, leading dimensions in ELEMENTS;
 *   - every matrix / workspace pointer is a DEVICE pointer (cudaMalloc / torch CUDA memory) unless
 *     stated otherwise; `stream` is a cudaStream_t (NULL = legacy default stream);
 *   - the caller owns A, B, C, the workspace and the stream; the library owns only the handle
 *     (no device allocations); A is read-only; B and C are overwritten (no beta-accumulate);
 *     outputs must not alias inputs;
 *   - all validation is synchronous and happens before any launch: an error return means nothing
 *     was enqueued.  Asynchronous device faults surface as SK_ERR_CUDA from a later call;
 *   - no exception crosses the ABI; sketch_last_error() gives a thread-local detail string;
 *   - handles are immutable after configuration (sketch_set_*) and may be used concurrently from
 *     several host threads on different streams.  A sketch launch whose split / stream-K pieces
 *     accumulate in place (2-4 pieces per m-block) has CTAs waiting on other CTAs of the same grid;
 *     such launches are cooperative (the grid is scheduled only as a whole), so concurrent launches
 *     on one device cannot deadlock;
 *   - results are deterministic: fixed-order split-K / stream-K / in-place piece and core
 *     reductions, so identical calls give bit-identical outputs (the one exception is the caller's
 *     choice of sketch_multimem_sum, whose in-switch summation order is the hardware's).
 */
#ifndef PAPER_2603_20966_B200_SKETCH_H
#define PAPER_2603_20966_B200_SKETCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sk_sketch_s* sk_sketch_t; /* opaque, library-owned */

typedef enum {
    SK_DIST_GAUSSIAN = 0,   /* default: N(0,1) entries                      */
    SK_DIST_RADEMACHER = 1, /* +-1 entries (north-star extension, c3 workload)              */
    SK_DIST_UNIFORM = 2     /* U[0,1) entries (the Philox-uniform Omega of PAPER.md:1190)   */
} sk_dist_t;

typedef enum {
    SK_MODE_TF32X3 = 0, /* default, fp32-accurate: A_hi*O_hi + A_hi*O_lo + A_lo*O_hi on tf32 MMAs */
    SK_MODE_TF32 = 1,   /* one tf32 MMA per product (A read as tf32, Omega rounded RN to tf32)   */
    SK_MODE_BF16 = 2    /* A and Omega rounded RN to bf16 on chip, fp32 accumulation             */
} sk_mode_t;

typedef enum {
    SK_OMEGA_ACCURATE = 0, /* <= 2 ulp Box-Muller (logf/sqrtf/sincospif); required for TF32X3   */
    SK_OMEGA_FAST = 1      /* MUFU lg2/sqrt/sin/cos Box-Muller; tf32/bf16 modes only (reading R5) */
} sk_omega_transform_t;

typedef enum {
    SK_SUCCESS = 0,
    SK_ERR_INVALID_VALUE = 1,  /* bad scalar argument, NULL pointer, out-of-extent block        */
    SK_ERR_SHAPE_MISMATCH = 2, /* n2 != handle n2, ld < row length, ...                          */
    SK_ERR_ALIGNMENT = 3,      /* A not 16-byte aligned or lda % 4 != 0 (TMA requirement)        */
    SK_ERR_UNSUPPORTED = 4,    /* valid request outside what this build implements              */
    SK_ERR_WORKSPACE = 5,      /* ws_bytes smaller than sketch_*_workspace_size reported         */
    SK_ERR_CUDA = 6,           /* CUDA runtime / driver error (launch or earlier async fault)    */
    SK_ERR_NCCL = 7            /* reserved for the native collective layer                       */
} sk_status_t;

/* Create a handle for Omega in R^{n2 x r} drawn from `dist` with 64-bit `seed`.
 * n2 is the global number of rows of Omega (= columns of the full A); r >= 1, r <= 4096.
 * Errors: SK_ERR_INVALID_VALUE (out == NULL, n2 < 1, r < 1, r > 4096, unknown dist). */
sk_status_t sketch_create(uint64_t seed, sk_dist_t dist, int64_t n2, int64_t r, sk_sketch_t* out);
sk_status_t sketch_destroy(sk_sketch_t h);

/* Precision mode (default SK_MODE_TF32X3).  Errors: SK_ERR_INVALID_VALUE. */
sk_status_t sketch_set_mode(sk_sketch_t h, sk_mode_t mode);
/* Gaussian transform used INSIDE the GEMMs (sketch_generate always uses the accurate one).
 * SK_OMEGA_FAST with SK_MODE_TF32X3 is rejected at apply time with SK_ERR_UNSUPPORTED. */
sk_status_t sketch_set_omega_transform(sk_sketch_t h, sk_omega_transform_t t);
/* Tuning override for the split-K factor of the sketch GEMM (0 = automatic, else 1..64).  In tf32x3
 * the accuracy does not depend on it: TMEM accumulates at most 1024 K per chunk whatever the split. */
sk_status_t sketch_set_split_k(sk_sketch_t h, int32_t split_k);

/* Tuning / ablation override of the sketch GEMM's CTA grouping: 0 = automatic (CTA pairs with
 * tcgen05 cta_group::2 for n1 > 256; Gaussian Omega in tf32 / bf16: clusters of 4 pairs sharing the
 * generated slices for n1 >= 2048, of 3 pairs with SK_OMEGA_FAST at n1 >= 6144; for
 * 256 < r <= 512 (or r a multiple of 512) with Gaussian / uniform Omega in tf32 / bf16, one pass per
 * 512 columns with two N = 256 column blocks per CTA in clusters of 8 pairs = 16 CTAs, or 4 pairs
 * where 16-CTA clusters do not fit), 1 = single-CTA tiles, 2 = CTA pairs without sharing,
 * 4 = clusters of 2 pairs sharing Omega whenever the shape allows it (any mode), 6 = clusters of 3
 * pairs (6 CTAs), 8 = clusters of 4 pairs (8 CTAs) sharing Omega.  A non-zero override also keeps
 * 256-column passes.  Any other value: SK_ERR_INVALID_VALUE. */
sk_status_t sketch_set_cta_group(sk_sketch_t h, int32_t cg);

/* Core GEMM implementation: 0 = tcgen05 (default, any r: blocks of up to 256 x 256 of C with tf32
 * operands in the tf32 / bf16 modes; 128 x 128 blocks with 3xTF32 operands (hi + lo splits of Omega
 * and B, <= 1024 rows per TMEM accumulation) in tf32x3), 1 = fp32 SIMT (used automatically for a B
 * whose rows are not 16-byte aligned). */
sk_status_t sketch_set_core_impl(sk_sketch_t h, int32_t simt);

/* Performance ablation for measurements only (results are WRONG while set): bit 0 skips the
 * in-kernel Omega generation, bit 1 skips the A tile loads, bit 2 skips the MMAs, bit 3 runs
 * single-CTA tiles in clusters of 2, bit 4 uses release (not relaxed) cluster relays, bit 5 makes
 * the producers spin instead of suspend-waiting, bit 6 skips the converter warps' A transform
 * (bf16 conversion / tf32x3 A_lo), bit 7 shrinks the cluster's Omega share copies 8x.  0 restores
 * normal operation. */
sk_status_t sketch_set_ablation(sk_sketch_t h, uint32_t flags);

/* Pipeline trace for measurements only (libraries built with SK_BUILD_TRACE=1; otherwise a non-NULL
 * buffer returns SK_ERR_UNSUPPORTED): while `dev_buf` is non-NULL, the next sketch GEMM launches
 * write %globaltimer stamps (ns, uint64) of their pipeline waits for CTAs 0..159 (layout
 * [cta][event][stage], 8 events x `stages` stages per CTA; events: 0 TMA after empty_a, 1 MMA after
 * full_a / conv, 2 MMA after full_o, 3 producer after empty_o, 4 producer share written, 5
 * producer after pfree, 6 relay after full_o, 7 converter done).  The buffer is device (or mapped
 * pinned host) memory owned by the caller, >= 160 * 8 * stages * 8 bytes.  NULL disables tracing. */
sk_status_t sketch_set_trace(sk_sketch_t h, uint64_t* dev_buf, int32_t stages);

/* Fused reduce-scatter of the partial sketch (Alg. 1, on a
 * p1 x p2 grid with p2 > 1).  B-bar = A_blk[m x k] * Omega[k0 : k0+k, 0:r] is not formed locally:
 * the GEMM epilogue stores every row i (0 <= i < m) straight into the receive buffer of the rank
 * owning row piece i / piece_rows, at
 *     dst[i / piece_rows] + (slot * split + s) * slot_elems + (i % piece_rows) * npad + c,
 * s < split the split-K index, npad = round_up(r, 16), c < r.  dst[] holds ndst (<= 8) device
 * pointers valid in this process -- typically NVLink peer mappings of symmetric-memory receive
 * buffers, so the reduce-scatter traffic leaves each SM as its tiles finish; slot = this rank's
 * index in its row group.  split must be equal on all ranks of the group (sketch_rs_split gives the
 * local choice; take the max over the group).  The owners then call sketch_reduce_slots on their
 * ndst * split slots after a cross-rank barrier.  Requires r <= 256.  Stream-ordered on `stream`.
 * Errors: as sketch_apply_block, SK_ERR_INVALID_VALUE (ndst, pieces, slot, split),
 * SK_ERR_SHAPE_MISMATCH (slot_elems), SK_ERR_ALIGNMENT (dst not 16-byte aligned),
 * SK_ERR_UNSUPPORTED (r > 256). */
sk_status_t sketch_rs_split(sk_sketch_t h, int64_t m, int64_t k, int32_t* split);
sk_status_t sketch_apply_block_rs(sk_sketch_t h, const float* A_blk, int64_t m, int64_t k, int64_t lda,
                                  int64_t k0, float* const* dst, int32_t ndst, int64_t piece_rows,
                                  int32_t slot, int64_t slot_elems, int32_t split, void* stream);

/* B[rows x r] (ldb) = sum over s < nslots of slots[s * slot_elems + i * npad + c], summed in increasing
 * s (fixed order, deterministic): the owner-side half of the fused reduce-scatter.  slots is a device
 * buffer of nslots * slot_elems floats.  Errors: SK_ERR_INVALID_VALUE, SK_ERR_SHAPE_MISMATCH. */
sk_status_t sketch_reduce_slots(sk_sketch_t h, const float* slots, int32_t nslots, int64_t slot_elems,
                                int64_t rows, float* B, int64_t ldb, void* stream);

/* out[i] = src[0][i] + src[1][i] + ... + src[n-1][i] (0 <= i < elems), summed in increasing j (fixed
 * order, deterministic): the AllReduce of the Nystrom core's r x r partials (GPU
 * variant P:1839) read straight from every rank's symmetric-memory slot over NVLink.
 * src: n <= 8 device pointers valid in this process (e.g. NVLink peer mappings), 16-byte aligned;
 * elems % 4 == 0.  Stream-ordered; the caller orders it after all ranks' writes (device barrier).
 * Errors: SK_ERR_INVALID_VALUE, SK_ERR_SHAPE_MISMATCH, SK_ERR_ALIGNMENT. */
sk_status_t sketch_sum_peers(const float* const* src, int32_t n, int64_t elems, float* out, void* stream);

/* The Nystrom core's AllReduce issued from the core GEMM's epilogue (PAPER.md:611 and
 * the GPU AllReduce of C): ADDS Omega[i0 : i0+m, :r]^T B_blk into C on every rank
 * of a multicast group -- each CTA's partial tile goes out as multimem.red.add.f32 on the multicast
 * address C_mc (row stride ldc), reduced inside the NVSwitch; no partial workspace, no reduce kernel.
 * The caller zeroes every rank's C and orders that (a barrier) before any rank calls this, and
 * barriers again before reading C.  The in-switch summation order is the hardware's: C is exact in
 * the integer regime and within fp32 rounding otherwise, but not bit-reproducible run to run.
 * B_blk: device, 16-B aligned rows; C_mc: multicast virtual address, 16-B aligned, ldc % 4 == 0.
 * Errors: as core_apply_block, SK_ERR_ALIGNMENT, SK_ERR_UNSUPPORTED (B rows not TMA-addressable). */
sk_status_t core_apply_block_mc(sk_sketch_t h, const float* B_blk, int64_t m, int64_t ldb, int64_t i0,
                                float* C_mc, int64_t ldc, void* ws, size_t ws_bytes, void* stream);

/* NVLS reduction (the AllReduce of C, and the reduce-scatter of
 * partial B, done inside the NVSwitch): out[i] = sum over the ranks of a multicast
 * group of their copies of element i, for i < elems, read through the group's multicast mapping
 * `mc_src` (multimem.ld_reduce.add.f32, round-to-nearest); if `mc_out` (a multicast address) is
 * non-NULL the sums are also stored to every rank's copy there.  mc_src / mc_out: device multicast
 * virtual addresses (e.g. torch symmetric memory's multicast_ptr + byte offset); out: local device
 * buffer or NULL.  The caller orders the ranks' writes of the inputs before the call (a barrier).
 * elems % 4 == 0, all pointers 16-byte aligned.  Stream-ordered.  Errors: SK_ERR_INVALID_VALUE,
 * SK_ERR_SHAPE_MISMATCH, SK_ERR_ALIGNMENT, SK_ERR_CUDA (e.g. no multicast support). */
sk_status_t sketch_multimem_sum(const float* mc_src, int64_t elems, float* out, float* mc_out, void* stream);

/* Launch plan of sketch_apply_block for an m x k block (workspace unlimited): rows of A per work unit
 * (rows that share each generated Omega slice: 128 x CTA group x accumulators x cluster pairs), the
 * split / stream-K pieces per m-block, the CTA pairs per cluster, and the grid.  Any output pointer
 * may be NULL.  Used by the distributed layer to cut row blocks at whole units.  Host only, no launch.
 * Errors: SK_ERR_INVALID_VALUE. */
sk_status_t sketch_plan_info(sk_sketch_t h, int64_t m, int64_t k, int32_t* rows_per_unit, int32_t* split,
                             int32_t* cluster_pairs, int32_t* grid);

/* Pack of the Redist variant's All-to-All ("unpack" step PAPER.md:1536): for column
 * bounds cb[0] = 0 < cb[1] < ... < cb[nblk] <= ldb, writes block j = B[0:rows, cb[j]:cb[j+1]]
 * row-major and contiguous at out + rows * cb[j] (out holds rows * cb[nblk] floats), so that each
 * rank's send chunk is one contiguous range.  B: device, row-major, ldb >= cb[nblk]; cb: HOST array
 * of nblk + 1 bounds; 1 <= nblk <= 64.  Pure data movement (no arithmetic).  Stream-ordered.
 * Errors: SK_ERR_INVALID_VALUE (NULL pointers, nblk, non-increasing bounds),
 * SK_ERR_SHAPE_MISMATCH (cb[nblk] > ldb). */
sk_status_t sketch_pack_cols(const float* B, int64_t rows, int64_t ldb, const int64_t* cb, int32_t nblk,
                             float* out, void* stream);

/* Bytes of device workspace needed by sketch_apply / sketch_apply_block on n1 rows and
 * nystrom_core / core_apply_block (split-K partials of B and per-CTA r x r partials of C).
 * One size covers every entry point for that n1 (n for nystrom_core). */
sk_status_t sketch_workspace_size(sk_sketch_t h, int64_t n1, size_t* bytes);

/* B[n1 x r] = A[n1 x n2] * Omega[0:n2, 0:r].  n2 must equal the handle's n2.
 * A: device, lda >= n2, lda % 4 == 0, 16-byte aligned.  B: device, ldb >= r.
 * ws: device workspace of ws_bytes >= sketch_workspace_size(h, n1). */
sk_status_t sketch_apply(sk_sketch_t h, const float* A, int64_t n1, int64_t n2, int64_t lda,
                         float* B, int64_t ldb, void* ws, size_t ws_bytes, void* stream);

/* Nystrom core: B[n x r] = A Omega and C[r x r] = Omega^T B for square A
 * (n must equal the handle's n2; symmetry of A is assumed by the method, not checked).
 * C is the raw product Omega^T B (not symmetrised, reading R10). */
sk_status_t nystrom_core(sk_sketch_t h, const float* A, int64_t n, int64_t lda, float* B,
                         int64_t ldb, float* C, int64_t ldc, void* ws, size_t ws_bytes,
                         void* stream);

/* Block forms for the distributed layouts (Alg. 1 / Alg. 2 with p3 = q3 = 1):
 *   sketch_apply_block: B_part[m x r] = A_blk[m x k] * Omega[k0 : k0+k, 0:r]
 *     (column 0 of A_blk pairs with global Omega row k0; requires k0 + k <= handle n2).
 *   core_apply_block:   C_part[r x r] = Omega[i0 : i0+m, 0:r]^T * B_blk[m x r]
 *     (row 0 of B_blk pairs with global Omega row i0; requires i0 + m <= handle n2). */
sk_status_t sketch_apply_block(sk_sketch_t h, const float* A_blk, int64_t m, int64_t k,
                               int64_t lda, int64_t k0, float* B_part, int64_t ldb, void* ws,
                               size_t ws_bytes, void* stream);
sk_status_t core_apply_block(sk_sketch_t h, const float* B_blk, int64_t m, int64_t ldb,
                             int64_t i0, float* C_part, int64_t ldc, void* ws, size_t ws_bytes,
                             void* stream);
/* Column-block form for the Redist variant of Alg. 2 (Psi = (1,1,P)): B_blk holds
 * nb (1 <= nb <= r) columns of B for rows i0 .. i0+m-1, and C_part[r x nb] = Omega[i0:i0+m, 0:r]^T B_blk
 * is the matching column block of C.  Workspace as for core_apply_block. */
sk_status_t core_apply_block_cols(sk_sketch_t h, const float* B_blk, int64_t m, int64_t nb,
                                  int64_t ldb, int64_t i0, float* C_part, int64_t ldc, void* ws,
                                  size_t ws_bytes, void* stream);

/* Host-buffer / out-of-core forms: A, B and C are HOST pointers (page-locked memory --
 * cudaHostAlloc / cudaHostRegister -- gives full PCIe bandwidth; pageable memory works but the
 * copies then serialise).  A is streamed in row blocks of `block_rows` rows through two device
 * staging buffers carved from the caller's DEVICE workspace `ws`: the H2D copy of block i+1 runs on
 * a library-internal copy stream while block i is sketched on `stream`, then B's block i is copied
 * back.  Rows of B are independent (row-block case), so any A that fits in host
 * memory can be sketched on one GPU.  nystrom_core_host additionally accumulates
 * C = sum_blocks Omega_blk^T B_blk in fixed block order (deterministic).
 * All work is enqueued on `stream` (the copy stream is joined back into it): synchronise `stream`
 * before reading B / C.  block_rows <= 0 picks a default (8192).  ws_bytes >= the size reported by
 * sketch_host_workspace_size(h, n1, block_rows).  Errors as for the device forms. */
sk_status_t sketch_host_workspace_size(sk_sketch_t h, int64_t n1, int64_t block_rows, size_t* bytes);
sk_status_t sketch_apply_host(sk_sketch_t h, const float* A_host, int64_t n1, int64_t n2, int64_t lda,
                              float* B_host, int64_t ldb, int64_t block_rows, void* ws,
                              size_t ws_bytes, void* stream);
sk_status_t nystrom_core_host(sk_sketch_t h, const float* A_host, int64_t n, int64_t lda,
                              float* B_host, int64_t ldb, float* C_host, int64_t ldc,
                              int64_t block_rows, void* ws, size_t ws_bytes, void* stream);

/* Test / debug: materialise Omega[row0 : row0+nrows, col0 : col0+ncols] (fp32, accurate transform)
 * or the raw Philox word each entry derives from (x[j&3] for tag 0, x[(j>>5)&3] for tag 1),
 * row-major into device memory `out` with leading dimension ld >= ncols.
 * Errors: SK_ERR_INVALID_VALUE if the block leaves [0, 2^62) x [0, r) or out == NULL. */
sk_status_t sketch_generate(sk_sketch_t h, int64_t row0, int64_t nrows, int64_t col0,
                            int64_t ncols, float* out, int64_t ld, void* stream);
sk_status_t sketch_generate_bits(sk_sketch_t h, int64_t row0, int64_t nrows, int64_t col0,
                                 int64_t ncols, uint32_t* out, int64_t ld, void* stream);

/* Test / debug: evaluate the device Box-Muller transform on caller-given word pairs
 * (w1[i], w2[i]) -> out_even[i] = R cos, out_odd[i] = R sin; `transform` selects the variant.
 * All pointers device, n >= 0. */
sk_status_t sketch_debug_box_muller(const uint32_t* w1, const uint32_t* w2, int64_t n,
                                    sk_omega_transform_t transform, float* out_even,
                                    float* out_odd, void* stream);

/* Phase timing, the analogue of the paper's per-phase timers (genOmegaTime, dgemm1Time, ...,
 * PAPER.md:1462-1467; Omega generation is fused into the GEMMs here, so it has no phase of its own).
 * When enabled, every kernel the handle launches is bracketed by CUDA events recorded on the
 * launch stream.  sketch_profile_read synchronises on the recorded events, writes the summed
 * device milliseconds and launch counts per phase (arrays of SK_PHASE_COUNT), and clears them. */
typedef enum {
    SK_PHASE_SKETCH_GEMM = 0, /* fused Omega-tile generation + tcgen05 A*Omega               */
    SK_PHASE_SPLITK_REDUCE = 1,
    SK_PHASE_CORE_GEMM = 2,   /* fused Omega regeneration + Omega^T*B                          */
    SK_PHASE_CORE_REDUCE = 3,
    SK_PHASE_GENERATE = 4,    /* sketch_generate / _bits (test path)                           */
    SK_PHASE_COUNT = 5
} sk_phase_t;
sk_status_t sketch_set_profiling(sk_sketch_t h, int enable);
sk_status_t sketch_profile_read(sk_sketch_t h, double* ms_per_phase, int64_t* launches_per_phase);

/* Number of kernels this library has launched in the process so far (all handles). */
uint64_t sketch_launch_count(void);

const char* sketch_status_string(sk_status_t st);
const char* sketch_last_error(void); /* thread-local detail of the last failing call */
const char* sketch_build_info(void); /* arch / version string baked in at compile time */

#ifdef __cplusplus
}
#endif
#endif /* PAPER_2603_20966_B200_SKETCH_H */
