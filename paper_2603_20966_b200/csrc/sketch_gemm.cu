// sketch_gemm.cu -- fused "generate Omega tile + tcgen05 GEMM" for B = A * Omega,
// the local product of Alg. 1 ("B-bar_ik = A_ij * Omega_jk") with Omega_jk
// regenerated in the kernel instead of communicated.
//
// One persistent CTA per SM (CG = 1) or per SM of a CTA pair (CG = 2, cluster (2,1,1),
// tcgen05 cta_group::2: the pair computes M = 256 rows per accumulator; each CTA holds its own
// 128 rows of A and HALF of the Omega tile's N columns, so each CTA generates only npad/2 Omega
// columns -- the pair shares every generated Omega element across 256 rows of A).  Warps:
//   warp 0      TMA producer: 128-row x 32-col fp32 tiles of A, SWIZZLE_128B (K-major), into an
//               a_stages-deep ring; L2 evict-first (A is streamed exactly once).  With CG = 2
//               both CTAs load their rows and the bytes are counted on the leader's barrier.
//   warp 1      MMA issuer (one elected thread of the leader CTA): tcgen05.mma kind::tf32,
//               M = 128*CG, N = npad, K = 8; NACC accumulators of 128 x npad fp32 per CTA in TMEM.
//   warp 2      TMEM allocator.
//   warps 4-19  Omega producers: Philox4x32-10 + transform, written as the K-major SWIZZLE_128B
//               B operand (row n = Omega column, 32 K-values = 128 B per row), then
//               fence.proxy.async + one mbarrier arrive per warp (remote on the leader for CG = 2).
//               Warps 4-7 also run the epilogue (tcgen05.ld 32x32b -> st.global of B or of a
//               split-K partial).
// Work unit = (m-block of 128*CG*NACC rows, K split s); units are dealt round-robin to CTA groups.
#include <map>
#include <mutex>
#include <tuple>

#include "kernels.cuh"
#include "omega_tile.cuh"
#include "philox.cuh"
#include "ptx.cuh"

namespace sk {

constexpr int kCtlWarps = 4;
#ifndef SK_CVT_WARPS_BF16
#define SK_CVT_WARPS_BF16 4
#endif
constexpr int kRngWarps = 16;  // Omega producers (the first 4 also run the epilogue)
// bf16: fewer producer warps leave more registers and issue slots per warp, and the measured optimum
// differs with the tile (same-box A/B of 8 / 10 / 12 / 14 / 16, r2af-r2ah): c2 (one column block)
// 8 warps 1.930 vs 16 warps 1.974 ms; the two-column-block c4 shape 12 warps 2.784 vs 2.844 ms.
// SK_RNG_WARPS_BF16 (compile-time) overrides both for tuning builds.
// tf32 with the fast transform: 8 warps (2.493 -> 2.437 ms at c2); with the accurate one 16 stay best
// (2.520 vs 2.691 ms with 8; r2ai).
constexpr int rng_warps(int mode, int ncol = 1, bool fast = false) {
#ifdef SK_RNG_WARPS_TF32
    if (mode == kTF32) return SK_RNG_WARPS_TF32;  // tuning builds only
#endif
    if (mode == kTF32 && fast && ncol == 1) return 8;
#ifdef SK_RNG_WARPS_BF16
    return mode == kBF16 ? SK_RNG_WARPS_BF16 : kRngWarps;
#else
    return mode == kBF16 ? (ncol == 2 ? 12 : 8) : kRngWarps;
#endif
}
// bf16 / tf32x3: warps converting each fp32 A stage (bf16 operand / A_lo)
constexpr int cvt_warps(int mode) { return (mode == kBF16 || mode == kTF32x3) ? SK_CVT_WARPS_BF16 : 0; }
constexpr int threads_for(int mode, int ncol = 1, bool fast = false) {
    return (kCtlWarps + rng_warps(mode, ncol, fast) + cvt_warps(mode)) * 32;
}

// diagnostics (sketch_set_trace, compiled in only with -DSK_TRACE: even a predicated-off check
// slows the single-thread TMA / MMA loops measurably): %globaltimer stamp of event `ev`, stage `i`
__device__ __forceinline__ void trace_stamp(const SketchGemmParams& p, int ev, uint32_t i) {
#ifdef SK_TRACE
    if (p.trace != nullptr && blockIdx.x < 160u && i < static_cast<uint32_t>(p.trace_stages)) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[(blockIdx.x * 8u + ev) * static_cast<uint32_t>(p.trace_stages) + i] = t;
    }
#else
    (void)p; (void)ev; (void)i;
#endif
}
// Work decomposition shared by every warp role (they must see the same segment sequence):
// split-K units u = group, group + ngroups, ... (m-block u / split, K slice u % split), or stream-K
// (p.sk_len > 0): the worker's contiguous range of flattened (m-block, K-iteration) indices, cut at
// m-block boundaries, so that every worker gets the same number of K iterations.
struct WorkIter {
    int64_t it, end;
    int u, group;
    __device__ __forceinline__ WorkIter(const SketchGemmParams& p, int g) : it(0), end(0), u(g), group(g) {
        if (p.sk_len > 0) {
            it = static_cast<int64_t>(g) * p.sk_len;
            end = min(it + p.sk_len, static_cast<int64_t>(p.num_mblk) * p.kiters);
        }
    }
    __device__ __forceinline__ bool next(const SketchGemmParams& p, int ngroups, int& mb, int& kb, int& ke,
                                         int& piece) {
        if (p.sk_len > 0) {
            if (it >= end) return false;
            mb = static_cast<int>(it / p.kiters);
            kb = static_cast<int>(it - static_cast<int64_t>(mb) * p.kiters);
            ke = static_cast<int>(min(static_cast<int64_t>(p.kiters), kb + (end - it)));
            piece = group - static_cast<int>((static_cast<int64_t>(mb) * p.kiters) / p.sk_len);
            it += ke - kb;
            return true;
        }
        if (u >= p.num_mblk * p.split) return false;
        mb = u / p.split;
        piece = u - mb * p.split;
        kb = piece * p.kper;
        ke = min(kb + p.kper, p.kiters);
        u += ngroups;
        return true;
    }
};

// Epilogue stores / adds of B rows (strong .gpu-scope operations, so a thread's store and later
// adds to one address stay in program order in the coherence order: a fixed fp32 summation order).
__device__ __forceinline__ void st_relaxed_v4(float* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.relaxed.gpu.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void st_relaxed(float* p, uint32_t a) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(a) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(__uint_as_float(a)),
                 "f"(__uint_as_float(b)), "f"(__uint_as_float(c)), "f"(__uint_as_float(d))
                 : "memory");
}
__device__ __forceinline__ void red_add(float* p, uint32_t a) {
    asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(__uint_as_float(a)) : "memory");
}
// ... with an L2 evict-last hint: the tf32x3 output rows are added to again 1024 K later, while the
// A stream (evict-first) passes through L2; keeping them resident avoids refetching them from DRAM
// 256-bit stores (STG.E.256): a whole 32-byte L2 sector per instruction, so a sector is never left
// partially written -- a later reduction on a partial sector makes L2 fetch it from DRAM first
__device__ __forceinline__ void st_v8(float* p, const uint32_t* v) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void st_relaxed_v8_el(float* p, const uint32_t* v, uint64_t pol) {
    asm volatile("st.relaxed.gpu.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_relaxed_v4_el(float* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t pol) {
    asm volatile("st.relaxed.gpu.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a), "r"(b),
                 "r"(c), "r"(d), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void red_add_v4_el(float* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t pol) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                 "f"(__uint_as_float(a)), "f"(__uint_as_float(b)), "f"(__uint_as_float(c)), "f"(__uint_as_float(d)),
                 "l"(pol)
                 : "memory");
}

constexpr uint32_t kATileBytes = 128 * 32 * 4;  // one 128-row x 32-fp32 TMA box
constexpr int kMaxStages = 8;

// Operand ring stage: [A_lo tile (tf32x3 only)] [Omega_hi tile] [Omega_lo tile (tf32x3, Gaussian/uniform)]
struct SmemLayout {
    uint32_t a_stage, o_stage, a_off, o_off, bar_off, total;
    uint32_t y_stage, y_off;             // bf16: ring of the second fp32 K half of each A stage
    uint32_t alo_off, ohi_off, olo_off;  // offsets inside an operand stage
};

// ks: K per pipeline step (32 for tf32 / tf32x3, 64 for bf16: a bf16 swizzle row holds 64 values).
// a_lo (tf32x3): each A stage also holds the A_lo = A - trunc_tf32(A) tiles the converter warps
// write next to the TMA'd A tiles (nacc * 16 KB more per stage).
// y_stages > 0 (bf16): an A stage's two fp32 boxes per accumulator are split over two rings: box 0
// (K 0..31) in the A ring, where the converters overwrite it with the bf16 64-K tile the MMA reads,
// and box 1 (K 32..63) in the Y ring, released as soon as it is converted -- the Y ring only has to
// cover the conversion, not the MMA, which leaves room for a deeper Omega ring.
__host__ __device__ inline SmemLayout make_layout(int nacc, int npad, int a_stages, int o_stages,
                                                  bool a_lo = false, bool olo = false, int ks = 32,
                                                  int nsubo = 1, int y_stages = 0) {
    SmemLayout L;
    L.a_stage = static_cast<uint32_t>(nacc) * kATileBytes * static_cast<uint32_t>(y_stages > 0 ? 1 : ks / 32) *
                (a_lo ? 2u : 1u);
    L.y_stage = y_stages > 0 ? static_cast<uint32_t>(nacc) * kATileBytes : 0u;
    // nsubo: 32-K sub-tiles per Omega stage (2 for tf32 with 64-wide K steps)
    const uint32_t otile = static_cast<uint32_t>(npad) * 128u * static_cast<uint32_t>(nsubo);
    L.alo_off = 0;
    L.ohi_off = 0u;
    L.olo_off = L.ohi_off + otile;
    L.o_stage = L.ohi_off + otile * (olo ? 2u : 1u);
    L.a_off = 0;
    L.y_off = L.a_off + L.a_stage * a_stages;
    L.o_off = L.y_off + L.y_stage * y_stages;
    L.bar_off = L.o_off + L.o_stage * o_stages;
    L.total = L.bar_off + (8 * kMaxStages + 4) * 8 + 16;
    return L;
}

// CL = 2 (with CG = 2): a cluster of 4 CTAs = 2 CTA pairs processing different rows of A in
// lockstep over the same K steps.  CTA (pair q, half h) needs the same Omega slice as its partner
// (pair 1-q, half h); each generates half of the slice's rows and a copier thread bulk-copies that
// half into the partner's stage (completing on the partner's full_o), so every generated Omega
// element feeds 1024 rows of A.  The partner pair's MMA commit multicasts "stage free" (pfree).
// NCOL = 2 (with CG = 2, NACC = 1): ONE 128-row A tile per CTA against TWO N = npad Omega column
// blocks (columns c0 .. c0 + 2 npad), two MMAs per K step into the two halves of TMEM -- a single
// pass over A for r <= 512 (c4); with CL = 8 (16-CTA clusters) every generated Omega element still
// feeds 2048 rows of A.
template <int CG, int NACC, int DIST, int MODE, bool FAST, int CL = 1, int NCOL = 1>
__global__ void __launch_bounds__(threads_for(MODE, NCOL, FAST), 1)
    sketch_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const SketchGemmParams p) {
    static_assert(CL == 1 || CG == 2, "Omega sharing between pairs needs CTA pairs");
    static_assert(CL >= 1 && CL <= 8, "1 to 8 CTA pairs per cluster");
    static_assert(NCOL == 1 || (NCOL == 2 && NACC == 1 && CG == 2), "two column blocks: one A tile per CTA pair half");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    constexpr bool X3 = (MODE == kTF32x3);                 // 3xTF32: A_lo and Omega_lo operands
    constexpr bool BF = (MODE == kBF16);                   // bf16 operands, K = 16 per MMA
    constexpr bool XA = X3 || BF;                          // converter warps transform A in smem
    constexpr bool ALO = X3;                               // A_lo tiles live in the A stage
    constexpr bool OLO = X3 && (DIST != kRademacher);      // +-1 is exact in tf32: no Omega_lo
    constexpr bool ARELAY = (CG == 2) && XA;               // peer A lands on its own barrier
    constexpr bool T64 = (MODE == kTF32) && (CG == 2);    // tf32 pairs: 64-wide K steps
    constexpr int KS = (BF || T64) ? 64 : 32;              // K per pipeline step
    constexpr int NBOX = KS / 32;                          // 128-B TMA boxes per accumulator
    constexpr int NSUBO = T64 ? 2 : 1;                     // 32-K Omega sub-tiles per stage
    constexpr int KMMA = T64 ? 8 : 4;                      // MMAs (per accumulator) per stage
    constexpr int kRngW = rng_warps(MODE, NCOL, FAST);     // Omega producer warps
    constexpr int kRngThreads = kRngW * 32;
    constexpr int kCvtWarps = cvt_warps(MODE);             // bf16 converter warps
    const int nh = p.npad / CG;        // Omega columns of one N block held by this CTA
    const int npad_loc = NCOL * nh;    // rows of this CTA's Omega tile (all its N blocks)
    const uint32_t osub = static_cast<uint32_t>(npad_loc) * 128u;  // bytes of one Omega sub-tile
    const SmemLayout L = make_layout(NACC, npad_loc, p.a_stages, p.o_stages, ALO, OLO, KS, NSUBO, BF ? p.y_stages : 0);
    uint8_t* sA = smem + L.a_off;
    uint8_t* sO = smem + L.o_off;
    uint8_t* sY = smem + L.y_off;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* full_a = bars;
    uint64_t* empty_a = bars + kMaxStages;
    uint64_t* full_o = bars + 2 * kMaxStages;
    uint64_t* empty_o = bars + 3 * kMaxStages;
    uint64_t* gen_done = bars + 4 * kMaxStages;  // CL = 2: this CTA's Omega half (+ A transform) written
    uint64_t* pfree = bars + 5 * kMaxStages;     // CL = 2: the partner's stage s is free
    uint64_t* conv = bars + 6 * kMaxStages;      // bf16: A stage converted (converter warps)
    uint64_t* empty_y = bars + 7 * kMaxStages;  // bf16: Y-ring slot converted (free)
    uint64_t* tmem_full = bars + 8 * kMaxStages;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 2);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const uint32_t crank_cl = (CG == 2) ? cluster_ctarank() : 0u;  // rank in the cluster
    const uint32_t crank = crank_cl & 1u;                             // rank in the CTA pair
    const uint32_t lead_rank = crank_cl & ~1u;                        // pair leader's cluster rank
    const uint32_t pairq = crank_cl >> 1;                             // pair index in the cluster
    const uint16_t pair_mask = static_cast<uint16_t>(0x3u << lead_rank);
    // every other pair of the cluster (their stages receive this CTA's Omega rows)
    const uint16_t partner_pair_mask = static_cast<uint16_t>(((1u << (2 * CL)) - 1u) & ~(0x3u << lead_rank));
    const bool leader = crank == 0;
    const int group = static_cast<int>(blockIdx.x) / (CG * CL);      // worker = pair (or cluster)
    const int ngroups = static_cast<int>(gridDim.x) / (CG * CL);
    uint32_t tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(NACC * NCOL * p.npad)) tmem_cols <<= 1;

    if (warp == 0 && lane == 0) {
        // full_a: one expect_tx arrival; with CG = 2 (tf32) the leader's barrier counts the bytes of
        // BOTH CTAs' TMA loads (the peer's loads complete_tx on it directly).  bf16 / tf32x3: each
        // CTA's A lands on its own barrier (its converter warps read it) and the MMA waits on conv.
        for (int s = 0; s < p.a_stages; ++s) {
            mbar_init(&full_a[s], 1);
            // bf16 / tf32x3: the converter warps' arrivals; the pair leader also counts the peer's converter
            // warps, which arrive on it directly (relaxed, remote)
            mbar_init(&conv[s], kCvtWarps * ((CG == 2 && leader) ? 2 : 1));  // + the peer's warps (remote)
            mbar_init(&empty_a[s], 1);
        }
        for (int s = 0; s < p.o_stages; ++s) {
            // CL = 1: own kRngW warps; CL = 2: the copier's expect_tx arrival (after gen_done),
            // plus the partner's bulk-copied half as tx bytes.  Leader: + the peer's relayed arrival.
            // CL = 1 pairs: the peer's producer warps arrive directly (relaxed, remote) on the leader
            mbar_init(&full_o[s], (CL > 1) ? (1 + (leader ? 1 : 0))
                                           : (CG == 2 ? (leader ? 2 * kRngW : kRngW) : kRngW));
            mbar_init(&empty_o[s], 1);
            mbar_init(&gen_done[s], kRngW);
            mbar_init(&pfree[s], CL > 1 ? CL - 1 : 1);  // one release per partner pair
        }
        for (int s = 0; s < (BF ? p.y_stages : 0); ++s) mbar_init(&empty_y[s], kCvtWarps);
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 4 * CG);
        fence_barrier_init();
        tma_prefetch_desc(&tmA);
    }
    if (warp == 2) {
        if constexpr (CG == 2) tmem_alloc_pair(tmem_slot, tmem_cols);
        else tmem_alloc_rt(tmem_slot, tmem_cols);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int rows_per_unit = 128 * CG * NACC * CL;   // rows of a work unit (all pairs of a cluster)
    // pair q of the cluster generates Omega slice rows [share(q), share(q+1)), as even as rows
    // allow (CL = 3: 42/43/43 of 128; the tile writers take the swizzle phase from the address)
    auto omega_share_row0 = [](int rows, uint32_t q) {
        return static_cast<int>((static_cast<uint32_t>(rows) * q) / static_cast<uint32_t>(CL));
    };
    const int pair_row0 = static_cast<int>(pairq) * 128 * CG * NACC;  // this pair's rows inside a unit
    const int kchunk = p.kchunk > 0 ? p.kchunk : 0x7fffffff;          // K iterations per accumulation

    // Epilogue of one accumulation chunk, by the warp reading TMEM lane quadrant q (lanes 32q..32q+31 =
    // rows of this CTA's 128-row tiles): tcgen05.ld -> the unit's output row (B, the split / stream-K
    // partial `s`, or a peer's receive slot) -- stored for the first chunk of the unit, added (fp32 RN,
    // same thread every time: a fixed order) for later ones -- then TMEM is handed back to the MMA.
    // In-place accumulation of the pieces of an m-block (p.inplace): flag of (m-block, piece, this CTA);
    // the 4 drain warps (128 threads, named barrier 3) wait for the piece above / publish their own.
    auto piece_flag = [&](int mb, int piece) {
        return p.flags + (static_cast<int64_t>(mb) * p.max_pieces + piece) * (CG * CL) + crank_cl;
    };
    auto wait_piece_above = [&](uint32_t q, int mb, int piece) {
        if (q == 0 && lane == 0) {
            const int32_t* f = piece_flag(mb, piece + 1);
            int32_t v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if (v != 0) break;
                __nanosleep(100);
            }
        }
        asm volatile("bar.sync 3, 128;" ::: "memory");
    };
    auto publish_piece = [&](uint32_t q, int mb, int piece) {
        asm volatile("bar.sync 3, 128;" ::: "memory");  // every drain thread's stores / adds are issued
        if (q == 0 && lane == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(piece_flag(mb, piece)), "r"(1) : "memory");
        }
    };
    auto drain = [&](uint32_t q, int mb, int s, bool first, uint32_t nd) {
        mbar_wait(tmem_full, nd & 1);
        tc_fence_after();
        const uint64_t pol_el = X3 ? l2_policy_evict_last() : 0ull;
        float* out = p.out + ((!p.inplace && (p.split > 1 || p.sk_len > 0)) ? static_cast<int64_t>(s) * p.part_stride : 0);
        const bool vec_ok = ((p.ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
        const bool vec8_ok = ((p.ldo & 7) == 0) && ((reinterpret_cast<uintptr_t>(out) & 31) == 0) &&
                             (p.npad % 8 == 0) && p.rs_ndst == 0;
#pragma unroll 1
        for (int ac = 0; ac < NACC * NCOL; ++ac) {
            const int a = ac / NCOL, h = ac % NCOL;
            const int row = mb * rows_per_unit + pair_row0 + a * 128 * CG + static_cast<int>(crank) * 128 +
                            static_cast<int>(q) * 32 + static_cast<int>(lane);
            float* orow = out + static_cast<int64_t>(row) * p.ldo + h * p.npad;
            const int rv = p.r_valid - h * p.npad;  // valid columns of this block
            if (p.rs_ndst > 0 && row < p.n1) {
                // fused reduce-scatter: the row's partial goes straight to its owner's slot
                // (NVLink store into the peer's receive buffer), no local B / split partial
                const int64_t piece = row / p.rs_piece;
                orow = p.rs_dst[piece] + (static_cast<int64_t>(p.rs_slot) * p.split + s) * p.rs_slot_elems +
                       (row - piece * p.rs_piece) * p.ldo + h * p.npad;
            }
#pragma unroll 1
            for (int cc = 0; cc < p.npad; cc += 32) {
                const uint32_t taddr = tmem_base + ((q * 32u) << 16) + static_cast<uint32_t>(ac * p.npad + cc);
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
                    if (!first) {
                        // later chunks: fire-and-forget fp32 RN adds at L2 (REDG.ADD.F32), so the drain
                        // never waits on a load; one thread owns each element and its adds are
                        // ordered by program order (same address), so the sum order is fixed
                        if (vec_ok && cc + 32 <= rv) {
#pragma unroll
                            for (int i = 0; i < 32; i += 4) {
                                if constexpr (X3) red_add_v4_el(orow + cc + i, v[i], v[i + 1], v[i + 2], v[i + 3], pol_el);
                                else red_add_v4(orow + cc + i, v[i], v[i + 1], v[i + 2], v[i + 3]);
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (cc + i < rv) red_add(orow + cc + i, v[i]);
                        }
                    } else if (vec8_ok && cc + 32 <= rv) {
#pragma unroll
                        for (int i = 0; i < 32; i += 8) {
                            if constexpr (X3)  // later chunks add to it: a strong store, ordered before them
                                st_relaxed_v8_el(orow + cc + i, v + i, pol_el);
                            else
                                st_v8(orow + cc + i, v + i);
                        }
                    } else if (vec_ok && cc + 32 <= rv) {
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            if constexpr (X3)
                                st_relaxed_v4_el(orow + cc + i, v[i], v[i + 1], v[i + 2], v[i + 3], pol_el);
                            else
                                *reinterpret_cast<float4*>(orow + cc + i) =
                                    make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                                __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            if (cc + i >= rv) continue;
                            if constexpr (X3) st_relaxed(orow + cc + i, v[i]);
                            else orow[cc + i] = __uint_as_float(v[i]);
                        }
                    }
                }
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(tmem_empty), lead_rank));
            else mbar_arrive(tmem_empty);
        }
    };

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint64_t pol = l2_policy_evict_first();
            const uint32_t a_bytes_cta = ALO ? L.a_stage / 2 : L.a_stage;  // (tf32x3: A_lo not loaded)
            uint32_t st = 0, ph = 0, ntr = 0, yst = 0, yph = 0;
            WorkIter wi(p, group);
            int mb, kb, ke, s;
            while (wi.next(p, ngroups, mb, kb, ke, s)) {
                // L2 prefetch of A, p.prefetch K steps ahead of the loads: the HBM latency under load
                // (~1.6 us) then overlaps the smem ring instead of adding to each stage's turnaround
                auto prefetch = [&](int kp) {
                    const int xp = kp * KS - p.kshift;
#pragma unroll
                    for (int a = 0; a < NACC; ++a)
#pragma unroll
                        for (int bx = 0; bx < NBOX; ++bx)
                            tma_prefetch_2d(&tmA, xp + 32 * bx,
                                            mb * rows_per_unit + pair_row0 + a * 128 * CG + static_cast<int>(crank) * 128);
                };
                if (p.prefetch > 0 && !(p.ablate & 2u))
                    for (int kp = kb; kp < min(kb + p.prefetch, ke); ++kp) prefetch(kp);
                for (int kit = kb; kit < ke; ++kit) {
                    mbar_wait(&empty_a[st], ph ^ 1);
                    if constexpr (BF) mbar_wait(&empty_y[yst], yph ^ 1);
                    trace_stamp(p, 0, ntr++);
                    if (p.prefetch > 0 && kit + p.prefetch < ke && !(p.ablate & 2u)) prefetch(kit + p.prefetch);
                    const int x = kit * KS - p.kshift;
                    if (p.ablate & 2u) {  // ablation: no A traffic, stage marked full at once
                        if (leader || ARELAY) mbar_arrive(&full_a[st]);
                        if (++st == static_cast<uint32_t>(p.a_stages)) { st = 0; ph ^= 1; }
                        if (BF && ++yst == static_cast<uint32_t>(p.y_stages)) { yst = 0; yph ^= 1; }
                        continue;
                    }
                    if constexpr (BF) {
                        // each CTA loads its own rows on its own barrier (its converters read them):
                        // K 0..31 into the A ring, K 32..63 into the Y ring
                        mbar_arrive_expect_tx(&full_a[st], 2u * a_bytes_cta);
#pragma unroll
                        for (int a = 0; a < NACC; ++a) {
                            const int row = mb * rows_per_unit + pair_row0 + a * 128 * CG + static_cast<int>(crank) * 128;
                            tma_load_2d(sA + st * L.a_stage + a * kATileBytes, &tmA, &full_a[st], x, row, pol);
                            tma_load_2d(sY + yst * L.y_stage + a * kATileBytes, &tmA, &full_a[st], x + 32, row, pol);
                        }
                        if (++yst == static_cast<uint32_t>(p.y_stages)) { yst = 0; yph ^= 1; }
                    } else if constexpr (CG == 2 && !ARELAY) {
                        // both CTAs load their own rows; bytes are counted on the leader's barrier
                        const uint32_t bar = mapa_shared(smem_u32(&full_a[st]), lead_rank);
                        if (leader) mbar_arrive_expect_tx(&full_a[st], 2 * a_bytes_cta);
#pragma unroll
                        for (int a = 0; a < NACC; ++a)
#pragma unroll
                            for (int bx = 0; bx < NBOX; ++bx)
                                tma_load_2d_pair(sA + st * L.a_stage + (a * NBOX + bx) * kATileBytes, &tmA, bar,
                                                 x + 32 * bx,
                                                 mb * rows_per_unit + pair_row0 + a * 256 + static_cast<int>(crank) * 128, pol);
                    } else {
                        mbar_arrive_expect_tx(&full_a[st], a_bytes_cta);
#pragma unroll
                        for (int a = 0; a < NACC; ++a)
#pragma unroll
                            for (int bx = 0; bx < NBOX; ++bx)
                                tma_load_2d(sA + st * L.a_stage + (a * NBOX + bx) * kATileBytes, &tmA, &full_a[st],
                                            x + 32 * bx, mb * rows_per_unit + pair_row0 + a * 128 * CG +
                                                             static_cast<int>(crank) * 128, pol);
                    }
                    if (++st == static_cast<uint32_t>(p.a_stages)) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ------------------------------------------------------------------ MMA issuer (leader)
        if (elect_one()) {
            const uint32_t idesc = make_idesc(BF ? kFmtBF16 : kFmtTF32, 128 * CG, static_cast<uint32_t>(p.npad), 0, 0);
            uint32_t sa = 0, pa = 0, so = 0, po = 0, nd = 0, ntr = 0;
            WorkIter wi(p, group);
            int mb, kb, ke, s;
            while (wi.next(p, ngroups, mb, kb, ke, s)) {
                int ci = 0;  // K iteration inside the accumulation chunk (a counter: no division here)
                for (int kit = kb; kit < ke; ++kit, ++ntr) {
                    if (ci == 0) {  // the epilogue has drained the previous chunk
                        mbar_wait(tmem_empty, (nd & 1) ^ 1);
                        tc_fence_after();
                    }
                    if constexpr (XA) mbar_wait(&conv[sa], pa);  // both CTAs' A stage converted
                    else mbar_wait(&full_a[sa], pa);
                    trace_stamp(p, 1, ntr);
                    mbar_wait(&full_o[so], po);
                    trace_stamp(p, 2, ntr);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + sa * L.a_stage);
                    const uint32_t o_base = smem_u32(sO + so * L.o_stage);
#pragma unroll
                    for (int k8 = 0; k8 < ((p.ablate & 4u) ? 0 : KMMA); ++k8) {
                        const int sub = k8 >> 2, kk = k8 & 3;  // 32-K sub-tile, 8-K step inside it
#pragma unroll
                        for (int ac = 0; ac < NACC * NCOL; ++ac) {
                            const int a = ac / NCOL, h = ac % NCOL;  // A tile, Omega column block
                            const uint64_t bdesc = sw128_desc(o_base + L.ohi_off + sub * osub + h * nh * 128 + kk * 32, 16, 1024);
                            const uint64_t adesc = sw128_desc(a_base + (a * NBOX + sub) * kATileBytes + kk * 32, 16, 1024);
                            uint32_t acc = (ci > 0 || k8 > 0) ? 1u : 0u;
                            const uint32_t d = tmem_base + ac * p.npad;
                            if constexpr (X3) {
                                // small terms first: A_lo * Omega_hi, A_hi * Omega_lo, then A_hi * Omega_hi
                                const uint64_t alo = sw128_desc(a_base + (NACC + a) * kATileBytes + k8 * 32, 16, 1024);
                                if constexpr (CG == 2) mma_tf32_pair(d, alo, bdesc, idesc, acc);
                                else mma_tf32(d, alo, bdesc, idesc, acc);
                                acc = 1u;
                                if constexpr (OLO) {
                                    const uint64_t blo = sw128_desc(o_base + L.olo_off + k8 * 32, 16, 1024);
                                    if constexpr (CG == 2) mma_tf32_pair(d, adesc, blo, idesc, acc);
                                    else mma_tf32(d, adesc, blo, idesc, acc);
                                }
                            }
                            if constexpr (BF) {
                                // bf16 A tile (converted in place by the converter warps)
                                const uint64_t abf = sw128_desc(a_base + a * kATileBytes + k8 * 32, 16, 1024);
                                if constexpr (CG == 2) mma_bf16_pair(d, abf, bdesc, idesc, acc);
                                else mma_bf16(d, abf, bdesc, idesc, acc);
                            } else {
                                if constexpr (CG == 2) mma_tf32_pair(d, adesc, bdesc, idesc, acc);
                                else mma_tf32(d, adesc, bdesc, idesc, acc);
                            }
                        }
                    }
                    if constexpr (CG == 2) {
                        mma_commit_pair(&empty_a[sa], pair_mask);
                        mma_commit_pair(&empty_o[so], pair_mask);
                        if constexpr (CL > 1) mma_commit_pair(&pfree[so], partner_pair_mask);
                    } else {
                        mma_commit(&empty_a[sa]);
                        mma_commit(&empty_o[so]);
                    }
                    if (++sa == static_cast<uint32_t>(p.a_stages)) { sa = 0; pa ^= 1; }
                    if (++so == static_cast<uint32_t>(p.o_stages)) { so = 0; po ^= 1; }
                    if (++ci == kchunk || kit + 1 == ke) {  // chunk complete: hand TMEM to the epilogue
                        if constexpr (CG == 2) mma_commit_pair(tmem_full, pair_mask);
                        else mma_commit(tmem_full);
                        ++nd;
                        ci = 0;
                    }
                }
            }
        }
    } else if (warp == 2 || warp == 3 || (warp == 1 && !leader)) {
        // ------------------------------------------------------------------ relays / copier
        // CL > 1: the peer CTA's warp 2 forwards its full_o (own share written + partners' bytes
        // landed) to the pair leader with a RELAXED cluster-scope arrive (a release.cluster arrive
        // drains in-flight TMA traffic; the relay writes nothing itself), and the copier (leader:
        // warp 3, peer: warp 1) bulk-copies this CTA's Omega share into the partner pairs' CTAs.
        const bool is_copier = (CL > 1) && ((leader && warp == 3) || (!leader && warp == 1));
        const bool is_orelay = (CG == 2) && (CL > 1) && !leader && warp == 2;
        if ((is_copier || is_orelay) && elect_one()) {
            uint64_t* bars_r = full_o;
            const uint32_t nst = static_cast<uint32_t>(p.o_stages);
            const uint32_t gen_rows = static_cast<uint32_t>(omega_share_row0(npad_loc, pairq + 1) -
                                                            omega_share_row0(npad_loc, pairq));
            const uint32_t half_bytes = gen_rows * 128u;  // this CTA's share of one sub-tile
            const uint32_t half_off = static_cast<uint32_t>(omega_share_row0(npad_loc, pairq)) * 128u;
            // the partners' shares land here: all rows of the slice but this CTA's own
            uint32_t tx = (static_cast<uint32_t>(npad_loc) - gen_rows) * 128u * (OLO ? 2u : 1u) * NSUBO;
            // ablation bit 7: copy 1/8 of each share (timing only: the result is wrong)
            const uint32_t cp_bytes = (p.ablate & 128u) ? half_bytes / 8u : half_bytes;
            if (p.ablate & 128u) tx /= 8u;
            uint32_t st = 0, ph = 0, ntr = 0;
            WorkIter wi(p, group);
            int mb, kb, ke, s;
            while (wi.next(p, ngroups, mb, kb, ke, s)) {
                for (int kit = kb; kit < ke; ++kit, ++ntr) {
                    if (is_copier) {
                        mbar_wait(&gen_done[st], ph);
                        mbar_arrive_expect_tx(&full_o[st], tx);  // local half done; partner half incoming
                        mbar_wait(&pfree[st], ph ^ 1);
                        trace_stamp(p, 5, ntr);
#pragma unroll
                        for (int pp = 1; pp < CL; ++pp) {
                            // partner CTA: same half of the pair, pair (pairq + pp) mod CL
                            const uint32_t partner = ((((pairq + pp) % CL)) << 1) | crank;
                            const uint32_t bar = mapa_shared(smem_u32(&full_o[st]), partner);
#pragma unroll
                            for (int sb = 0; sb < NSUBO; ++sb) {
                                const uint32_t src = smem_u32(sO + st * L.o_stage + L.ohi_off) + sb * osub + half_off;
                                bulk_copy_to_cta(mapa_shared(src, partner), src, cp_bytes, bar);
                            }
                            if constexpr (OLO) {
                                const uint32_t src_lo = smem_u32(sO + st * L.o_stage + L.olo_off) + half_off;
                                bulk_copy_to_cta(mapa_shared(src_lo, partner), src_lo, cp_bytes, bar);
                            }
                        }
                    } else {
                        mbar_wait(&bars_r[st], ph);
                        trace_stamp(p, 6, ntr);
                        if (p.ablate & 16u) mbar_arrive_cluster(mapa_shared(smem_u32(&bars_r[st]), lead_rank));
                        else mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&bars_r[st]), lead_rank));
                    }
                    if (++st == nst) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp >= kCtlWarps && warp < kCtlWarps + kRngW) {
        // ------------------------------------------------------------------ Omega producers + epilogue
        const int t = static_cast<int>(threadIdx.x) - kCtlWarps * 32;
        const int gen_row0 = omega_share_row0(npad_loc, pairq);                  // first generated row
        const int gen_rows = omega_share_row0(npad_loc, pairq + 1) - gen_row0;   // rows this CTA generates
        // tf32 64-K stages hold two 32-K sub-tiles: when one sub-tile has at most half as many
        // chunks as there are producers (clusters of 4 pairs), each half of the producers takes one
        // sub-tile instead of both halves idling through the sub-tiles in turn
        constexpr int kHalfThreads = kRngThreads / 2;
        const bool split_sub = (NSUBO == 2) && (gen_rows * 8 <= kHalfThreads);
        const int tt = split_sub ? (t % kHalfThreads) : t;
        const int my_sub = split_sub ? (t / kHalfThreads) : 0;
        const int nthr = split_sub ? kHalfThreads : kRngThreads;
        const int n_start = tt % gen_rows, j_start = tt / gen_rows;
        const int tq = nthr / gen_rows, tr = nthr % gen_rows;
        // this CTA's tile row n is Omega column c0 + (n / nh) npad + crank nh + n % nh; a share lies
        // inside one column block (the planner's cluster sizes divide the blocks)
        const int gen_h = gen_row0 / nh;
        const int c0_loc = p.c0 + gen_h * p.npad + static_cast<int>(crank) * nh + (gen_row0 - gen_h * nh);
        uint32_t so = 0, po = 0, nd = 0, ntr = 0;
        const uint32_t lo_off = L.olo_off - L.ohi_off;
        WorkIter wi(p, group);
        int mb, kb, ke, s;
        while (wi.next(p, ngroups, mb, kb, ke, s)) {
            for (int kit = kb; kit < ke; ++kit, ++ntr) {
                if (p.ablate & 32u) mbar_wait(&empty_o[so], po ^ 1);
                else mbar_wait_sleep(&empty_o[so], po ^ 1);
                if (t == 0) trace_stamp(p, 3, ntr);
                uint8_t* ostage = sO + so * L.o_stage;
                uint8_t* otile = ostage + L.ohi_off + gen_row0 * 128;  // this CTA's generated rows
                if (p.ablate & 1u) {
                    // ablation: stage marked full without generating Omega
                } else if constexpr (BF) {
                    if constexpr (DIST == kRademacher)
                        produce_omega_tile_bf16_r<DIST, FAST>(otile, p.k0a + static_cast<int64_t>(kit) * KS,
                                                              p.roff, gen_rows, c0_loc, p.key0, p.key1, t);
                    else
                        if (gen_rows * 8 < kRngThreads)  // small share: one-call items
                            produce_omega_tile_bf16_g<DIST, FAST, true>(otile, p.k0a + static_cast<int64_t>(kit) * KS,
                                                                  p.roff, gen_rows, c0_loc, p.key0, p.key1,
                                                                  n_start, j_start, tq, tr);
                        else
                            produce_omega_tile_bf16_g<DIST, FAST>(otile, p.k0a + static_cast<int64_t>(kit) * KS,
                                                                  p.roff, gen_rows, c0_loc, p.key0, p.key1,
                                                                  n_start, j_start, tq, tr);
                } else if constexpr (DIST == kRademacher)
                    for (int sb = 0; sb < NSUBO; ++sb)
                        produce_omega_tile_r<DIST, MODE, FAST>(otile + sb * osub,
                                                               p.k0a + static_cast<int64_t>(kit) * KS + 32 * sb,
                                                               p.roff, gen_rows, c0_loc, p.key0, p.key1, t, lo_off);
                else if (split_sub)
                    produce_omega_tile_g<DIST, MODE, FAST>(otile + my_sub * osub,
                                                           p.k0a + static_cast<int64_t>(kit) * KS + 32 * my_sub,
                                                           p.roff, gen_rows, c0_loc, p.key0, p.key1,
                                                           n_start, j_start, tq, tr, lo_off);
                else
                    for (int sb = 0; sb < NSUBO; ++sb)
                        produce_omega_tile_g<DIST, MODE, FAST>(otile + sb * osub,
                                                               p.k0a + static_cast<int64_t>(kit) * KS + 32 * sb,
                                                               p.roff, gen_rows, c0_loc, p.key0, p.key1,
                                                               n_start, j_start, tq, tr, lo_off);
                fence_proxy_async_smem();
                __syncwarp();
                if (t == 0) trace_stamp(p, 4, ntr);
                if (lane == 0) {
                    if constexpr (CL > 1) mbar_arrive(&gen_done[so]);
                    else if (CG == 2 && !leader) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&full_o[so]), lead_rank));
                    else mbar_arrive(&full_o[so]);
                }
                if (++so == static_cast<uint32_t>(p.o_stages)) { so = 0; po ^= 1; }
            }
            if (!X3 && t < 128) {
                // epilogue: warp (4+q) reads TMEM lanes 32q..32q+31 = rows of this CTA's half
                const uint32_t q = static_cast<uint32_t>(t >> 5);
                const bool top = ke == p.kiters;  // the piece holding the last K iterations stores first
                if (p.inplace && !top) wait_piece_above(q, mb, s);
                drain(q, mb, s, !p.inplace || top, nd);
                if (p.inplace) publish_piece(q, mb, s);
                ++nd;
            }
        }
    } else if constexpr (X3) {
        // ------------------------------------------------------------------ A_lo writers (tf32x3)
        // A_lo = A - trunc_tf32(A) (exact in fp32), elementwise next to the TMA'd A tiles of the same
        // stage (same SW128 layout, so the copy is layout-agnostic); the MMA reads A (as tf32, i.e.
        // truncated) and A_lo.  In their own warps this overlaps the Omega generation.
        // They also run the epilogue: after converting the last stage of each accumulation chunk
        // (kchunk K iterations) they drain TMEM into the unit's output (first chunk: store; later
        // chunks: add in fp32 round-to-nearest -- the promotion that keeps the truncating TMEM
        // accumulation to <= 1024 K), while the producers run ahead.
        const int cw = static_cast<int>(warp) - (kCtlWarps + kRngW);
        const int ct = cw * 32 + static_cast<int>(lane);
        uint32_t sa = 0, pa = 0, nd = 0;
        WorkIter wi(p, group);
        int mb, kb, ke, s;
        while (wi.next(p, ngroups, mb, kb, ke, s)) {
            int ci = 0;
            bool first = true;
            for (int kit = kb; kit < ke; ++kit) {
                if (cw == 0) mbar_wait(&full_a[sa], pa);
                asm volatile("bar.sync 2, %0;" ::"n"(kCvtWarps * 32) : "memory");
                if (!(p.ablate & 64u)) {
                    const float4* src = reinterpret_cast<const float4*>(sA + sa * L.a_stage);
                    float4* dst = reinterpret_cast<float4*>(sA + sa * L.a_stage + NACC * kATileBytes);
#pragma unroll 4
                    for (int i = ct; i < static_cast<int>(NACC * kATileBytes / 16); i += kCvtWarps * 32) {
                        float4 v = src[i];
                        v.x -= __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                        v.y -= __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                        v.z -= __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                        v.w -= __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                        dst[i] = v;
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2 && !leader) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&conv[sa]), lead_rank));
                    else mbar_arrive(&conv[sa]);
                }
                if (++sa == static_cast<uint32_t>(p.a_stages)) { sa = 0; pa ^= 1; }
                if (++ci == kchunk || kit + 1 == ke) {
                    const bool top = ke == p.kiters;
                    if (p.inplace && !top && first) wait_piece_above(static_cast<uint32_t>(cw), mb, s);
                    drain(static_cast<uint32_t>(cw), mb, s, first && (!p.inplace || top), nd);
                    if (p.inplace && kit + 1 == ke) publish_piece(static_cast<uint32_t>(cw), mb, s);
                    ++nd;
                    ci = 0;
                    first = false;
                }
            }
        }
    } else if constexpr (BF) {
        // ------------------------------------------------------------------ A converters (bf16)
        // A (two fp32 SW128 boxes of 32 K per accumulator: K 0..31 in the A ring, K 32..63 in the Y
        // ring) -> one bf16 SW128 tile of 64 K, IN PLACE over the A-ring box.  Row-local: bf16 row m
        // overwrites only fp32 row m of the A-ring box, so the 8 lanes of one warp that own row m (lane
        // j8 = 8-K chunk) order their loads before their stores with a __syncwarp.  The two loads
        // of a lane alternate even / odd chunk so that each 8-lane phase touches 8 distinct 16-B
        // bank groups; the stores are the 8 distinct chunks of one row.  In their own warps, the
        // smem-bound conversion overlaps the ALU-bound Omega generation (measured at c2 with
        // clusters of 4 pairs: the in-producer conversion took ~0.8 of the 1.3 us producer stage).
        const int cw = static_cast<int>(warp) - (kCtlWarps + kRngW);
        const uint32_t j8 = lane & 7u;
        const uint32_t hi = j8 >> 2, c0 = 2u * (j8 & 3u);
        const uint32_t ce = c0 + hi, co = c0 + 1u - hi;  // load order: even chunk first in half 0
        constexpr int kRowsPerPass = kCvtWarps * 4;        // 4 rows per warp per item
#ifndef SK_CVT_UNROLL
#define SK_CVT_UNROLL 4
#endif
        constexpr int kUnroll = SK_CVT_UNROLL;
        static_assert((NACC * 128) % (kRowsPerPass * kUnroll) == 0, "converter passes must tile the A stage");
        uint32_t sa = 0, pa = 0, ys = 0, ntr = 0;
        WorkIter wi(p, group);
        int mb, kb, ke, s;
        while (wi.next(p, ngroups, mb, kb, ke, s)) {
            for (int kit = kb; kit < ke; ++kit, ++ntr) {
                // converter warp 0 polls, a named barrier releases the other converter warps
                if (cw == 0) mbar_wait(&full_a[sa], pa);
                asm volatile("bar.sync 2, %0;" ::"n"(kCvtWarps * 32) : "memory");
                if (cw == 0 && lane == 0) trace_stamp(p, 7, ntr);
                if (!(p.ablate & 64u)) {
                    const uint32_t st0 = smem_u32(sA + sa * L.a_stage);
                    const uint32_t y0 = smem_u32(sY + ys * L.y_stage);
#pragma unroll 1
                    for (int r0 = 0; r0 < NACC * 128; r0 += kRowsPerPass * kUnroll) {
                        uint32_t rowaddr[kUnroll];
                        float4 va[kUnroll][2];
#pragma unroll
                        for (int it = 0; it < kUnroll; ++it) {
                            const int rr = r0 + it * kRowsPerPass + cw * 4 + static_cast<int>(lane >> 3);
                            const int a = rr >> 7, m = rr & 127;
                            const uint32_t sw = static_cast<uint32_t>(m & 7);
                            const uint32_t roff_b = static_cast<uint32_t>(a * kATileBytes + m * 128);
                            rowaddr[it] = st0 + roff_b;
                            const uint32_t src = (hi ? y0 : st0) + roff_b;
                            float4 x, y;
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                                         : "r"(src + ((ce ^ sw) << 4)));
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w)
                                         : "r"(src + ((co ^ sw) << 4)));
                            va[it][0] = hi ? y : x;  // K chunk c0
                            va[it][1] = hi ? x : y;  // K chunk c0 + 1
                        }
                        __syncwarp();
#pragma unroll
                        for (int it = 0; it < kUnroll; ++it) {
                            const uint32_t sw = static_cast<uint32_t>((r0 + it * kRowsPerPass + cw * 4 + (lane >> 3)) & 7);
                            st_shared_v4_u32(rowaddr[it] + ((j8 ^ sw) << 4),
                                             pack_bf16x2(va[it][0].x, va[it][0].y), pack_bf16x2(va[it][0].z, va[it][0].w),
                                             pack_bf16x2(va[it][1].x, va[it][1].y), pack_bf16x2(va[it][1].z, va[it][1].w));
                        }
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty_y[ys]);
                    if (CG == 2 && !leader) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&conv[sa]), lead_rank));
                    else mbar_arrive(&conv[sa]);
                }
                if (++sa == static_cast<uint32_t>(p.a_stages)) { sa = 0; pa ^= 1; }
                if (++ys == static_cast<uint32_t>(p.y_stages)) ys = 0;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_pair(tmem_base, tmem_cols);
        else tmem_dealloc_rt(tmem_base, tmem_cols);
    }
}

// Raises a kernel's opt-in dynamic smem limit to at least `smem` (per device and function; thread-safe,
// the attribute only ever grows).
cudaError_t raise_smem_limit(const void* fn, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> set;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    size_t& cur = set[std::make_pair(dev, fn)];
    if (smem <= cur) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) cur = smem;
    return e;
}

size_t sketch_gemm_smem_bytes(int cg, int nacc, int npad, int a_stages, int o_stages, bool xa, bool olo,
                              int ks, int nsubo, int y_stages) {
    return make_layout(nacc, npad / cg, a_stages, o_stages, xa, olo, ks, nsubo, y_stages).total + 1024;
}

int sketch_gemm_max_smem() { return 227 * 1024; }

// The kernel instantiation for a launch configuration (nullptr if not built).  Instantiated: CTA
// pairs with 2 accumulators and clusters of 2, 3 or 4 pairs (Omega sharing, Gaussian / uniform) or
// none; the column-pair variant (NCOL = 2, one accumulator) with clusters of 4 or 8 pairs; single
// CTAs and pairs without sharing for small shapes.
template <int CG, int NACC, int DIST, int CL, int NCOL>
static const void* pick_mode(int mode, bool fast) {
    if (mode == kTF32) {
        if constexpr (DIST == kGaussian)
            if (fast) return reinterpret_cast<const void*>(sketch_gemm_kernel<CG, NACC, DIST, kTF32, true, CL, NCOL>);
        return reinterpret_cast<const void*>(sketch_gemm_kernel<CG, NACC, DIST, kTF32, false, CL, NCOL>);
    }
    if (mode == kBF16) {
        if constexpr (DIST == kGaussian)
            if (fast) return reinterpret_cast<const void*>(sketch_gemm_kernel<CG, NACC, DIST, kBF16, true, CL, NCOL>);
        return reinterpret_cast<const void*>(sketch_gemm_kernel<CG, NACC, DIST, kBF16, false, CL, NCOL>);
    }
    if constexpr (NCOL == 1)
        if (mode == kTF32x3) return reinterpret_cast<const void*>(sketch_gemm_kernel<CG, NACC, DIST, kTF32x3, false, CL, NCOL>);
    return nullptr;
}

template <int CG, int NACC, int CL, int NCOL>
static const void* pick_dist(int dist, int mode, bool fast) {
    if (dist == kGaussian) return pick_mode<CG, NACC, kGaussian, CL, NCOL>(mode, fast);
    if constexpr (NCOL == 1)
        if (dist == kRademacher) return pick_mode<CG, NACC, kRademacher, CL, NCOL>(mode, fast);
    if (dist == kUniform) return pick_mode<CG, NACC, kUniform, CL, NCOL>(mode, fast);
    return nullptr;
}

static const void* pick_kernel(int cg, int nacc, int dist, int mode, bool fast, int cl, int ncol) {
    if (ncol == 2) {
        if (cg != 2 || nacc != 1 || dist == kRademacher) return nullptr;
        if (cl == 8) return pick_dist<2, 1, 8, 2>(dist, mode, fast);
        if (cl == 4) return pick_dist<2, 1, 4, 2>(dist, mode, fast);
        return nullptr;
    }
    if (ncol != 1) return nullptr;
    if (cl == 4 && cg == 2 && nacc == 2) return pick_dist<2, 2, 4, 1>(dist, mode, fast);
    if (cl == 3 && cg == 2 && nacc == 2) return pick_dist<2, 2, 3, 1>(dist, mode, fast);
    if (cl == 2 && cg == 2 && nacc == 2) return pick_dist<2, 2, 2, 1>(dist, mode, fast);
    if (cl == 2 && cg == 2 && nacc == 1) return pick_dist<2, 1, 2, 1>(dist, mode, fast);
    if (cl != 1) return nullptr;
    if (cg == 1 && nacc == 1) return pick_dist<1, 1, 1, 1>(dist, mode, fast);
    if (cg == 1 && nacc == 2) return pick_dist<1, 2, 1, 1>(dist, mode, fast);
    if (cg == 2 && nacc == 1) return pick_dist<2, 1, 1, 1>(dist, mode, fast);
    if (cg == 2 && nacc == 2) return pick_dist<2, 2, 1, 1>(dist, mode, fast);
    return nullptr;
}

// Function attributes of an instantiation, once per (device, function): the opt-in smem limit (only
// ever raised) and, for clusters of more than 8 CTAs, the non-portable cluster size.
static cudaError_t prepare_kernel(const void* fn, size_t smem, int cluster) {
    if (cudaError_t e = raise_smem_limit(fn, smem)) return e;
    if (cluster > 8) {
        static std::mutex mu;
        static std::map<std::pair<int, const void*>, bool> done;  // per (device, function), set once
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> g(mu);
        bool& d = done[std::make_pair(dev, fn)];
        if (!d) {
            if (cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) return e;
            d = true;
        }
    }
    return cudaSuccess;
}

// Clusters of cg * cl CTAs of this kernel that can be co-resident (GPC packing strands SMs for
// large clusters).  Returns 0 if the query fails or the configuration is not built.
int sketch_gemm_max_clusters(int cg, int nacc, int dist, int mode, bool fast, int cl, size_t smem, int ncol) {
    // per process, keyed by (device, kernel instantiation, smem); guarded: handles may be used from
    // several threads at once (sketch.h)
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, size_t>, int> cache;
    const void* fn = pick_kernel(cg, nacc, dist, mode, fast, cl, ncol);
    if (!fn) return 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, fn, smem);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cg * cl * 16);
    cfg.blockDim = dim3(threads_for(mode, ncol, fast && dist == kGaussian));
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cg * cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (prepare_kernel(fn, smem, cg * cl) != cudaSuccess) { cudaGetLastError(); return 0; }
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) { cudaGetLastError(); return 0; }
    std::lock_guard<std::mutex> g(mu);
    cache[key] = n;
    return n;
}

cudaError_t launch_sketch_gemm(const CUtensorMap& tmA, const SketchGemmParams& p, int cg, int nacc,
                               int dist, int mode, bool fast, int grid, size_t smem,
                               cudaStream_t s, int cl, int ncol) {
    const void* fn = pick_kernel(cg, nacc, dist, mode, fast, cl, ncol);
    if (!fn) return cudaErrorNotSupported;
    if (cudaError_t e = prepare_kernel(fn, smem, cg * cl)) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads_for(mode, ncol, fast && dist == kGaussian));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    // ablation bit 3: launch single-CTA tiles as clusters of 2 (isolates cluster placement effects)
    attr[0].val.clusterDim.x = (cg == 1 && (p.ablate & 8u)) ? 2 : cg * cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p.inplace) {
        // in-place pieces: CTAs wait for other CTAs of this grid, so the grid must be co-resident even
        // when other kernels share the GPU -- a cooperative launch is scheduled only as a whole
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
        cfg.numAttrs = 2;
    }
    void* args[] = {const_cast<CUtensorMap*>(&tmA), const_cast<SketchGemmParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace sk
