// api.cu -- the C ABI declared in include/sketch.h: handle, validation, launch planning,
// TMA tensor-map encoding, and the call sequences of sketch_apply / nystrom_core.
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sketch.h"
#include "kernels.cuh"

struct sk_timed_launch {
    int phase;
    cudaEvent_t start, end;
};

struct sk_sketch_s {
    uint64_t seed;
    int dist;
    int64_t n2;
    int64_t r;
    int mode;
    int omega_transform;
    int split_override;
    int cg_override;  // 0 auto, 1 force single-CTA tiles (ablation / tests)
    int core_simt;    // 1: force the fp32 SIMT core GEMM (tests / ablation)
    int cl_override;  // 0 auto, 1 never share Omega between CTA pairs, 2 share whenever possible
    uint32_t ablate;  // performance ablations (bench only): see SketchGemmParams::ablate
    uint64_t* trace = nullptr;  // pipeline trace buffer (diagnostics)
    int32_t trace_stages = 0;
    int profiling;
    std::mutex prof_mu;
    std::vector<sk_timed_launch> prof;
    std::vector<cudaEvent_t> event_pool;  // reused by LaunchScope (no create/destroy per launch)
    // host streaming: internal copy stream + events (created on first use, per handle)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_join = nullptr;
    std::mutex host_mu;
};

static cudaEvent_t pool_get(sk_sketch_s* h) {
    {
        std::lock_guard<std::mutex> g(h->prof_mu);
        if (!h->event_pool.empty()) {
            cudaEvent_t e = h->event_pool.back();
            h->event_pool.pop_back();
            return e;
        }
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

static std::atomic<uint64_t> g_launches{0};

// Brackets one kernel launch: counts it and, when profiling, records events on its stream.
struct LaunchScope {
    sk_sketch_s* h;
    int phase;
    cudaStream_t s;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    LaunchScope(sk_sketch_s* h_, int phase_, cudaStream_t s_) : h(h_), phase(phase_), s(s_) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (h && h->profiling) {
            e0 = pool_get(h);
            e1 = pool_get(h);
            cudaEventRecord(e0, s);
        }
    }
    ~LaunchScope() {
        if (e0) {
            cudaEventRecord(e1, s);
            std::lock_guard<std::mutex> g(h->prof_mu);
            h->prof.push_back({phase, e0, e1});
        }
    }
};

namespace {

thread_local std::string g_last_error;

sk_status_t fail(sk_status_t st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

sk_status_t cuda_fail(cudaError_t e, const char* where) {
    return fail(SK_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2D fp32 row-major tensor [rows x cols] with row stride ld (elements), box {box_cols, box_rows},
// SWIZZLE_128B, out-of-bounds elements read as zero.
sk_status_t make_map_2d(CUtensorMap* map, const float* base, int64_t rows, int64_t cols,
                        int64_t ld, uint32_t box_cols, uint32_t box_rows, bool swizzle = true) {
    auto enc = get_encode();
    if (!enc) return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string(r) + ")");
    return SK_SUCCESS;
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------- launch planning
struct SketchPlan {
    int npass;         // column passes of <= 256 columns (<= 512 with ncol = 2)
    int npad[32];      // MMA N per pass (per column block with ncol = 2)
    int ncol;          // 2: one A tile against two N = 256 Omega column blocks per pass
    int cg;            // 1: one CTA per tile; 2: CTA pair (tcgen05 cta_group::2, M = 256)
    int cl;            // 2: clusters of two CTA pairs sharing every generated Omega slice
    int nacc;
    int a_stages, o_stages, y_stages;
    int64_t sk_len;    // > 0: stream-K range length per worker (split = max pieces per m-block)
    int rows_per_unit;
    int split;
    int kiters;
    int num_mblk;
    int grid;
    size_t smem;
    size_t ws_per_split;  // bytes of one split partial (n1 x npad_max)
};

SketchPlan plan_sketch(const sk_sketch_s* h, int64_t n1, int64_t k, int kshift, size_t ws_cap,
                       int force_split = 0, bool allow_ncol = true);
SketchPlan plan_sketch_ncol1(const sk_sketch_s* h, int64_t n1, int64_t k, int kshift, size_t ws_cap, int force_split) {
    return plan_sketch(h, n1, k, kshift, ws_cap, force_split, false);
}

SketchPlan plan_sketch(const sk_sketch_s* h, int64_t n1, int64_t k, int kshift, size_t ws_cap,
                       int force_split, bool allow_ncol) {
    SketchPlan P{};
    const int64_t rpad = round_up(h->r, 16);
    const bool x3 = h->mode == sk::kTF32x3;
    P.cg = (n1 > 256 && h->cg_override != 1) ? 2 : 1;
    P.nacc = (n1 > 128 * P.cg) ? 2 : 1;
    // Wide r (256 < r <= 512, or r a multiple of 512): one pass over A per 512 columns -- each CTA
    // holds ONE 128-row A tile against two N = 256 Omega column blocks (TMEM: 2 x 256 columns), in
    // clusters of 8 CTA pairs (2048 rows share every generated Omega element) or 4; reading A once
    // instead of twice per 512 columns.  Gaussian / uniform Omega, tf32 / bf16.
    P.ncol = 1;
    {
        const char* e = getenv("SK_NCOL");  // tuning: SK_NCOL=1 forces 256-column passes
        const bool want = allow_ncol && !(e && atoi(e) == 1) && h->cl_override == 0;
        if (want && !x3 && h->dist != sk::kRademacher && P.cg == 2 && n1 > 512 && rpad > 256 &&
            (rpad <= 512 || rpad % 512 == 0)) {
            P.ncol = 2;
            P.nacc = 1;
        }
    }
    const int cols_per_pass = 256 * P.ncol;
    P.npass = static_cast<int>((rpad + cols_per_pass - 1) / cols_per_pass);
    int npad_max = 0;
    for (int i = 0; i < P.npass; ++i) {
        P.npad[i] = P.ncol == 2 ? 256 : static_cast<int>(std::min<int64_t>(256, rpad - 256 * i));
        npad_max = std::max(npad_max, P.npad[i]);
    }
    const bool bf = h->mode == sk::kBF16;
    const bool xa = x3 || bf;
    const bool t64 = (h->mode == sk::kTF32) && P.cg == 2;  // tf32 pairs run 64-wide K steps
    const int ks = (bf || t64) ? 64 : 32;
    const int nsubo = t64 ? 2 : 1;
    const bool olo = x3 && h->dist != sk::kRademacher;
    // Omega ring depth: pairs hand every stage across the pair (relay + multicast commit)
    P.o_stages = bf ? 2 : ((P.cg == 2 || x3) ? 3 : 2);
    const int budget = sk::sketch_gemm_max_smem() - 2048;
    // operand stage: Omega (+ Omega_lo); tf32x3 keeps A_lo in the A stage, bf16 converts A in place
    auto ostage_bytes = [&](int) {
        const int otile = (P.ncol * npad_max / P.cg) * 128 * nsubo;
        return otile * (olo ? 2 : 1);
    };
    int a_cap = 6;
    if (bf && P.cg == 2) { a_cap = 3; P.o_stages = 8; }  // bf16 pairs: 3 x 64 KB A, rest Omega ring
    // two column blocks (32 KB Omega stages): one more A stage for one fewer Omega stage (c4, 3 runs of
    // each: 11.26 / 11.63 / 11.53 ms vs 11.79 / 11.80 / 12.11 ms; r2bb)
    if (bf && P.ncol == 2) { a_cap = 4; P.o_stages = 3; }
    if (const char* e = getenv("SK_A_STAGES")) a_cap = std::max(1, std::min(8, atoi(e)));    // tuning
    if (const char* e = getenv("SK_O_STAGES")) P.o_stages = std::max(1, std::min(8, atoi(e)));  // tuning
    // bf16: the second fp32 K half of each A stage lives in a short ring of its own (freed once
    // converted), so the A ring holds 32 KB slots and the Omega ring gets deeper
    P.y_stages = bf ? 2 : 0;
    if (const char* e = getenv("SK_Y_STAGES")) if (bf) P.y_stages = std::max(1, std::min(8, atoi(e)));  // tuning
    for (;;) {
        const int a_slot = P.nacc * 128 * (bf ? 32 : ks) * 4 * (x3 ? 2 : 1);  // bytes of one A-ring slot
        const int y_bytes = P.y_stages * P.nacc * 128 * 32 * 4;
        P.a_stages = std::min(a_cap, (budget - y_bytes - 2 * ostage_bytes(P.nacc)) / a_slot);
        P.o_stages = std::max(2, std::min(P.o_stages, (budget - y_bytes - P.a_stages * a_slot) / ostage_bytes(P.nacc)));
        if (P.a_stages >= 2 || P.nacc == 1 || P.ncol == 2) break;
        P.nacc = 1;  // make room for >= 2 A stages
    }
    const int a_stage = P.nacc * 128 * ks * 4;  // A bytes per K step
    P.smem = sk::sketch_gemm_smem_bytes(P.cg, P.nacc, P.ncol * npad_max, P.a_stages, P.o_stages, x3, olo, ks, nsubo,
                                        P.y_stages);
    P.kiters = static_cast<int>((k + kshift + ks - 1) / ks);
    // Clusters of CTA pairs share each generated Gaussian Omega slice: every element then feeds
    // 1024 (2 pairs) or 2048 (4 pairs) rows of A instead of 512.  Omega generation is the
    // bottleneck of the fused kernel, so the automatic choice is 4 pairs (c2, max clocks: bf16
    // 2.37 -> 2.27 ms, tf32 3.17 -> 2.70 ms) except in tf32x3 mode, whose Omega_lo doubles the
    // shared bytes (6.2 -> 7.1 ms with sharing); then 2 pairs, then none if the shape does not allow
    // it.  sketch_set_cta_group(h, 2 / 4 / 8) forces none / 2 pairs / 4 pairs.
    auto cl_ok = [&](int cl) {
        // every pair generates whole 8-row swizzle atoms of each CTA's npad/2-row Omega slice
        const bool split_ok = (cl == 3) ? (npad_max % 16 == 0 && npad_max / 16 >= cl) : (npad_max % (16 * cl) == 0);
        return P.cg == 2 && P.nacc == 2 && n1 >= 512 * cl && split_ok && h->dist == sk::kGaussian;
    };
    P.cl = 1;
    const bool fast_t = h->omega_transform == SK_OMEGA_FAST;
    if (P.ncol == 2) {
        // 16-CTA clusters when the rows fill them (and the GPU packs them), else 8 CTAs
        P.cl = (n1 > 1024 && sk::sketch_gemm_max_clusters(2, 1, h->dist, h->mode, fast_t, 8, P.smem, 2) > 0) ? 8 : 4;
        if (const char* e = getenv("SK_NCOL_CL")) P.cl = atoi(e) == 8 ? 8 : 4;  // tuning
    }
    // bf16 with the fast (MUFU) transform generates Omega cheaply enough that 3 pairs per cluster
    // win: clusters of 6 CTAs pack 22 per B200 (132 SMs) against 15 of 8 CTAs (120 SMs), at 4/3
    // the generated elements per A byte (c2: 2.05 -> 1.98 ms, 25000^2: 0.571 -> 0.538 ms, 12500 x
    // 50000: 0.591 -> 0.533, 6250 x 50000: 0.359 -> 0.343; the accurate transform loses, c2 2.11 ->
    // 2.22 ms, 12500 x 50000 0.600 -> 0.631); tf32 with the fast transform likewise (c2: 2.369 -> 2.224
    // ms, round 2, r2ax).  Only for n1 >= 4 units of 1536 rows, so the ragged
    // last unit stays a small share (c4, n1 = 2048, keeps one 2048-row unit).
    const bool fast = h->omega_transform == SK_OMEGA_FAST;
    if (P.ncol == 2) {
        // (chosen above)
    } else if (h->cl_override == 0 && !x3) {
        P.cl = (fast && n1 >= 4 * 1536 && cl_ok(3)) ? 3 : cl_ok(4) ? 4 : cl_ok(2) ? 2 : 1;
    } else if (h->cl_override >= 2) {
        P.cl = cl_ok(h->cl_override) ? h->cl_override : 1;
    }
    int workers = sk::num_sms() / P.cg;
    if (P.cl > 1) {
        int mc = sk::sketch_gemm_max_clusters(P.cg, P.nacc, h->dist, h->mode, fast_t, P.cl, P.smem, P.ncol);
        if (mc <= 0 && P.ncol == 2 && P.cl == 8) {  // 16-CTA clusters do not fit: 8 CTAs
            P.cl = 4;
            mc = sk::sketch_gemm_max_clusters(P.cg, P.nacc, h->dist, h->mode, fast_t, P.cl, P.smem, P.ncol);
        }
        if (mc <= 0) {
            if (P.ncol == 2) return plan_sketch_ncol1(h, n1, k, kshift, ws_cap, force_split);
            P.cl = 1;
        } else {
            workers = std::min(mc, sk::num_sms() / (2 * P.cl));
        }
    }
    const int rows_per_unit = 128 * P.cg * P.nacc * P.cl;
    P.num_mblk = static_cast<int>((n1 + rows_per_unit - 1) / rows_per_unit);
    P.ws_per_split = static_cast<size_t>(n1) * npad_max * P.ncol * sizeof(float);
    const int nsm = workers;  // independent workers (CTAs, CTA pairs or clusters of pairs)
    // The tensor core accumulates fp32 in TMEM with a bias toward zero of ~2^-24 per K=8 MMA step
    // (measured: relF = 7e-9 x K per accumulator, tools/acc_test.py).  tf32x3 promises fp32
    // accuracy (1e-5), so it caps K per accumulator at 1024 (32 K-iterations) INSIDE the kernel: the
    // epilogue drains TMEM every kchunk iterations and adds the chunk into the unit's output in fp32
    // round-to-nearest (sketch_gemm.cu, `drain`), so any split / stream-K range keeps the cap.
    const int min_split = 1;
    int best_s = 1;
    if (force_split > 0) {
        best_s = std::min(force_split, std::max(1, P.kiters));
    } else if (h->split_override > 0) {
        best_s = std::min(h->split_override, std::max(1, P.kiters));
    } else if (min_split > 64) {
        best_s = min_split;
    }
    double best = 1e300;
    const double unit_ovh = 2.0;  // epilogue + pipeline fill, in K-iteration units
    if (force_split == 0 && h->split_override == 0 && min_split <= 64) {
        for (int s = min_split; s <= std::max(min_split, std::min(64, std::max(1, P.kiters / 4))); ++s) {
            const int64_t units = static_cast<int64_t>(P.num_mblk) * s;
            const int64_t waves = (units + nsm - 1) / nsm;
            const int kper = (P.kiters + s - 1) / s;
            double t = static_cast<double>(waves) * (kper + unit_ovh);
            if (s > 1)
                t += static_cast<double>(s + 1) * n1 * npad_max * P.ncol * 4.0 /
                     (static_cast<double>(nsm) * a_stage * P.cg);
            if (t < best * 0.995) { best = t; best_s = s; }
        }
    }
    if (best_s > 1 && force_split == 0 && ws_cap < static_cast<size_t>(best_s) * P.ws_per_split)
        best_s = std::max<int>(1, static_cast<int>(ws_cap / P.ws_per_split));
    // each split must own >= 1 K iteration
    const int kper = (P.kiters + best_s - 1) / best_s;
    P.split = (P.kiters + kper - 1) / kper;
    const int64_t units = static_cast<int64_t>(P.num_mblk) * P.split;
    P.grid = static_cast<int>(std::min<int64_t>(units, nsm)) * P.cg * P.cl;
    P.rows_per_unit = rows_per_unit;
    P.sk_len = 0;
    // Stream-K: every worker gets the same number of K iterations of the flattened (m-block, K)
    // space, cut at m-block boundaries, when wave quantisation of the split-K units would leave
    // workers idle (e.g. 13 m-blocks on 15 clusters).  Not for an explicit split (fused
    // reduce-scatter slots, tests).
    if (force_split == 0 && h->split_override == 0 && getenv("SK_NO_STREAMK") == nullptr && best < 1e299 &&
        P.num_mblk > 0 && P.kiters > 0) {
        const int64_t total = static_cast<int64_t>(P.num_mblk) * P.kiters;
        const int64_t L = (total + nsm - 1) / nsm;
        const int pieces = static_cast<int>((P.kiters + L - 1) / L) + 1;
        const double t_sk = static_cast<double>(L) + unit_ovh * (1.0 + static_cast<double>(L) / P.kiters) +
                            static_cast<double>(pieces + 1) * n1 * npad_max * P.ncol * 4.0 /
                                (static_cast<double>(nsm) * a_stage * P.cg);
        if (t_sk < best * 0.97 && ws_cap >= static_cast<size_t>(pieces) * P.ws_per_split) {
            P.sk_len = L;
            P.split = pieces;
            P.grid = static_cast<int>((total + L - 1) / L) * P.cg * P.cl;
        }
    }
    if ((h->ablate & 8u) && (P.grid & 1)) P.grid += 1;  // cluster-of-2 ablation needs an even grid
    if (getenv("SK_DEBUG_PLAN"))  // tuning diagnostics
        fprintf(stderr, "[sketch plan] n1=%lld k=%lld cg=%d cl=%d nacc=%d ncol=%d a=%d y=%d o=%d split=%d sk_len=%lld kiters=%d mblk=%d grid=%d smem=%zu\n",
                static_cast<long long>(n1), static_cast<long long>(k), P.cg, P.cl, P.nacc, P.ncol, P.a_stages, P.y_stages,
                P.o_stages, P.split, static_cast<long long>(P.sk_len), P.kiters, P.num_mblk, P.grid, P.smem);
    return P;
}

size_t sketch_ws_bytes(const sk_sketch_s* h, int64_t n1, int64_t k) {
    const SketchPlan P = plan_sketch(h, n1, k, 127, ~size_t(0));
    return P.split > 1 ? P.split * P.ws_per_split : 0;
}

struct CorePlan {
    bool tc;             // tcgen05 path (r <= 256) vs fp32 SIMT
    int chunks;
    int chunk_rows;      // SIMT: rows of B per chunk
    int64_t base, step;  // tcgen05: 128-aligned chunk grid in global Omega rows
    int npad, nacc;
};

CorePlan plan_core_simt(const sk_sketch_s* h, int64_t m) {
    CorePlan C{};
    C.tc = false;
    const int64_t tiles = ((h->r + 63) / 64) * ((h->r + 63) / 64);
    const int64_t want = std::max<int64_t>(1, (2 * sk::num_sms() + tiles - 1) / tiles);
    const int64_t maxc = std::max<int64_t>(1, (m + 31) / 32);
    const int64_t chunks = std::min(want, maxc);
    C.chunk_rows = static_cast<int>(round_up((m + chunks - 1) / chunks, 32));
    C.chunks = static_cast<int>((m + C.chunk_rows - 1) / C.chunk_rows);
    return C;
}

// tcgen05 core: one CTA per (128-aligned chunk of B rows, block of C); SIMT only on request.
// tf32 / bf16: blocks of up to 256 x 256, about one wave of CTAs.  tf32x3 (3xTF32): 128 x 128 blocks
// (the hi + lo operands double the ring) and chunks of <= 1024 rows -- the TMEM accumulation
// truncates (~7e-9 relative per accumulated K), so K per accumulator is capped as in
// the sketch GEMM and the partials are summed in fp32 round-to-nearest by core_reduce.
CorePlan plan_core(const sk_sketch_s* h, int64_t m, int64_t i0 = 0, int64_t nb = -1) {
    if (h->core_simt) return plan_core_simt(h, m);
    if (nb < 0) nb = h->r;
    const bool x3 = h->mode == sk::kTF32x3;
    CorePlan C{};
    C.tc = true;
    C.npad = static_cast<int>(std::min<int64_t>(x3 ? 128 : 256, round_up(nb, 16)));
    C.nacc = (!x3 && h->r > 128) ? 2 : 1;
    C.base = i0 & ~static_cast<int64_t>(127);
    const int64_t span = std::max<int64_t>(1, i0 + m - C.base);
    const int64_t sms = sk::num_sms();
    const char* core_nacc_env = getenv("SK_CORE_NACC");  // tuning: force 256 / 128-row C blocks
    if (!x3 && h->r > 128 && h->r <= 256 && nb <= 256) {
        // 256-row blocks of C (nacc 2) or 128-row blocks (nacc 1: twice the CTAs, each generating half
        // the Omega columns -- the same total) and the rows per chunk: the pair minimising waves x the
        // per-CTA time measured for r = 256 (profiles/r2_core_plan_sweep.txt: one wave takes ~19 us +
        // 0.0625 us per row with nacc 2, ~13.5 us + 0.054 us per row with nacc 1).  6250 rows: nacc 1,
        // 128-row chunks (27.0 -> 20.8 us); 25000: nacc 1, 384 rows (37.3 -> 35.1); 12500 / 50000 stay
        // nacc 2 with 128 / 384 rows.
        double best = 1e30;
        for (int na = 2; na >= 1; --na) {
            const int64_t blk = (h->r + 128 * na - 1) / (128 * na);
            for (int64_t st = 128; st <= 4096; st += 128) {
                // (depends on span only through round_up(span, 128): see core_ws_bytes)
                const int64_t ctas = ((span + st - 1) / st) * blk;
                const double t = static_cast<double>((ctas + sms - 1) / sms) *
                                 (na == 2 ? 19.0 + 0.0625 * st : 13.5 + 0.054 * st);
                if (t < best) { best = t; C.nacc = na; C.step = st; }
                if (ctas <= sms) break;  // one wave: longer chunks only cost more
            }
        }
        if (core_nacc_env) C.nacc = atoi(core_nacc_env) == 1 ? 1 : 2;  // tuning
    }
    const int64_t blocks = ((h->r + 128 * C.nacc - 1) / (128 * C.nacc)) * ((nb + C.npad - 1) / C.npad);
    const int64_t want = std::max<int64_t>(1, sms / blocks);
    if (x3 || !(h->r > 128 && h->r <= 256 && nb <= 256) || core_nacc_env)
        C.step = round_up((span + want - 1) / want, 128);
    if (x3) {
        // <= 1024 rows per chunk; when that leaves more CTAs than SMs (one CTA per SM), take the chunk
        // length minimising waves x (rows + ~128 rows of fixed per-CTA cost): 50000 rows, r = 256:
        // 1024-row chunks = 196 CTAs in 2 waves -> 768-row chunks = 264 CTAs in 2 shorter waves
        C.step = std::min<int64_t>(C.step, 1024);
        int64_t best = -1;
        for (int64_t st = 128; st <= 1024; st += 128) {
            const int64_t ctas = ((span + st - 1) / st) * blocks;
            const int64_t cost = ((ctas + sk::num_sms() - 1) / sk::num_sms()) * (st + 128);
            if (best < 0 || cost <= best) { best = cost; C.step = st; }
            if (ctas <= sk::num_sms()) break;  // one wave: longer chunks only cost more
        }
    }
    const char* core_step_env = getenv("SK_CORE_STEP");  // tuning: rows per chunk (x 128)
    if (core_step_env) C.step = std::max<int64_t>(128, round_up(atoi(core_step_env), 128));
    C.chunks = static_cast<int>((span + C.step - 1) / C.step);
    return C;
}

size_t core_ws_bytes(const sk_sketch_s* h, int64_t m) {
    // largest chunk count of either plan over every block offset: i0 % 128 widens the span to m .. m + 127
    // rows.  Chunk lengths are multiples of 128, so a tcgen05 plan's chunk count depends on the span only
    // through round_up(span, 128) -- one of the two values the offsets 0 and 127 give (+ 1 for the
    // round-up of the one-wave chunk length)
    const int64_t chunks = std::max<int64_t>(
        std::max(plan_core(h, m, 0).chunks, plan_core(h, m, 127).chunks) + 1, plan_core_simt(h, m).chunks);
    // (plan_core with nb = r: narrower column blocks -- core_apply_block_cols -- have as many chunks or fewer)
    return static_cast<size_t>(chunks) * h->r * h->r * sizeof(float);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

sk_status_t check_handle(const sk_sketch_s* h) {
    if (!h) return fail(SK_ERR_INVALID_VALUE, "NULL handle");
    return SK_SUCCESS;
}

sk_status_t check_mode(const sk_sketch_s* h) {
    if (h->omega_transform == SK_OMEGA_FAST && h->mode == sk::kTF32x3)
        return fail(SK_ERR_UNSUPPORTED, "SK_OMEGA_FAST is not allowed with SK_MODE_TF32X3");
    return SK_SUCCESS;
}

// B_part[m x r] = A[m x k] * Omega[k0 : k0+k, :r]
// Fused reduce-scatter target (f1): output rows go to peer receive buffers, see sketch.h
struct RsTarget {
    float* dst[8];
    int32_t ndst;
    int32_t slot;
    int64_t piece;
    int64_t slot_elems;
    int32_t split;
};

sk_status_t apply_impl(sk_sketch_s* h, const float* A, int64_t m, int64_t k, int64_t lda,
                       int64_t k0, float* B, int64_t ldb, void* ws, size_t ws_bytes,
                       cudaStream_t stream, const RsTarget* rs = nullptr) {
    if (m == 0) return SK_SUCCESS;
    // Omega tile rows start at a 128-aligned global row (+ roff = k0 % 4); the matching A columns
    // start kshift (a multiple of 4) columns left of column 0 and are zero-filled by TMA.
    const int kshift = static_cast<int>(k0 & 124);
    const int roff = static_cast<int>(k0 & 3);
    const SketchPlan P = plan_sketch(h, m, k, kshift, rs ? ~size_t(0) : ws_bytes, rs ? rs->split : 0);
    if (rs && (P.npass != 1 || P.split != rs->split || P.ncol != 1))
        return fail(SK_ERR_UNSUPPORTED, "fused reduce-scatter needs r <= 256 and split <= K iterations");
    CUtensorMap map;
    sk_status_t st = make_map_2d(&map, A, m, k, lda, 32, 128);
    if (st != SK_SUCCESS) return st;
    // In-place accumulation of split / stream-K pieces (no partials, no reduce kernel) whenever no
    // piece can wait on a unit its own worker runs later: stream-K (a lower piece is the LAST unit of
    // its worker, the piece above the FIRST unit of the next worker), or split-K whose pieces of one
    // m-block fall in the same wave (one wave, or a wave width that is a multiple of the split); and
    // only for <= 4 pieces per m-block: pieces that finish together publish one after another, so a
    // long chain costs more than the reduce it saves (c4: 7 pieces, 2.75 -> 2.80 ms; 106 rows with 132
    // stream-K pieces: 0.67 ms; c2: 1.951 -> 1.933 ms and 25000 x 25000: 0.525 -> 0.505 ms; r2w, r2y).
    const int ngroups = P.grid / (P.cg * P.cl);
    const int64_t units = static_cast<int64_t>(P.num_mblk) * P.split;
    const bool pieces = P.split > 1 || P.sk_len > 0;
    const char* ip_env = getenv("SK_INPLACE");  // tuning: SK_INPLACE=0 keeps partials + reduce
    const char* ipm_env = getenv("SK_INPLACE_MAX");  // tuning: most pieces per m-block accumulated in place
    const int inplace_max = ipm_env ? atoi(ipm_env) : 4;
    // Under Nsight Compute a cooperative cluster launch fails ("LaunchFailed", and ncu ends the process;
    // r2ct): profiled runs take the partials + reduce path.  ncu exports NV_COMPUTE_PROFILER_PERFWORKS_DIR
    // to the target (r2cv); CUDA_INJECTION64_PATH covers the other injection-based tools.
    static const bool profiled =
        getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr || getenv("CUDA_INJECTION64_PATH") != nullptr;
    const bool inplace = !rs && pieces && !profiled && !(ip_env && atoi(ip_env) == 0) &&
                         P.split <= inplace_max && (P.sk_len > 0 || units <= ngroups || ngroups % P.split == 0);
    const size_t inplace_flag_bytes =
        static_cast<size_t>(std::max(P.num_mblk, 1)) * P.split * P.cg * P.cl * sizeof(int32_t);
    if (inplace && (!ws || ws_bytes < inplace_flag_bytes))
        return fail(SK_ERR_WORKSPACE, "workspace too small for the piece flags");
    for (int pass = 0; pass < P.npass; ++pass) {
        sk::SketchGemmParams p{};
        const int c0 = 256 * P.ncol * pass;
        const int pass_cols = P.ncol * P.npad[pass];  // output columns of this pass (and partial row length)
        p.r_valid = static_cast<int32_t>(std::min<int64_t>(h->r - c0, pass_cols));
        p.npad = P.npad[pass];
        p.c0 = c0;
        p.k0a = k0 - kshift;
        p.kshift = kshift;
        p.roff = roff;
        p.n1 = static_cast<int32_t>(m);
        p.kiters = P.kiters;
        p.num_mblk = P.num_mblk;
        p.split = P.split;
        p.kper = (P.kiters + P.split - 1) / P.split;
        p.a_stages = P.a_stages;
        p.o_stages = P.o_stages;
        p.y_stages = P.y_stages;
        p.prefetch = 0;
        p.kchunk = (h->mode == sk::kTF32x3) ? 1024 / 32 : 0;  // tf32x3: <= 1024 K per TMEM accumulation
        p.sk_len = P.sk_len;
        if (const char* e = getenv("SK_PREFETCH")) p.prefetch = std::max(0, std::min(16, atoi(e)));  // tuning
        p.key0 = static_cast<uint32_t>(h->seed);
        p.key1 = static_cast<uint32_t>(h->seed >> 32);
        p.ablate = h->ablate;
        p.trace = h->trace;
        p.trace_stages = h->trace_stages;
        if (rs) {
            for (int j = 0; j < 8; ++j) p.rs_dst[j] = j < rs->ndst ? rs->dst[j] : nullptr;
            p.rs_ndst = rs->ndst;
            p.rs_slot = rs->slot;
            p.rs_piece = rs->piece;
            p.rs_slot_elems = rs->slot_elems;
            p.out = rs->dst[0];
            p.ldo = p.npad;
            p.part_stride = 0;
        } else if (inplace) {
            // pieces accumulate into B in descending piece order (flags at the head of the workspace)
            p.out = B + c0;
            p.ldo = ldb;
            p.part_stride = 0;
            p.inplace = 1;
            p.max_pieces = P.split;
            p.flags = static_cast<int32_t*>(ws);
        } else if (P.split > 1 || P.sk_len > 0) {
            p.out = static_cast<float*>(ws);
            p.ldo = pass_cols;
            p.part_stride = m * static_cast<int64_t>(pass_cols);
        } else {
            p.out = B + c0;
            p.ldo = ldb;
            p.part_stride = 0;
        }
        cudaError_t e;
        if (inplace) {  // zero the piece flags (a few KB) ahead of the kernel on the same stream
            e = cudaMemsetAsync(ws, 0, inplace_flag_bytes, stream);
            if (e != cudaSuccess) return cuda_fail(e, "flag memset");
        }
        {
            LaunchScope ls(h, SK_PHASE_SKETCH_GEMM, stream);
            e = sk::launch_sketch_gemm(map, p, P.cg, P.nacc, h->dist, h->mode,
                                       h->omega_transform == SK_OMEGA_FAST, P.grid, P.smem, stream, P.cl, P.ncol);
        }
        if (e != cudaSuccess) return cuda_fail(e, "sketch_gemm launch");
        if (inplace) {
            // nothing to reduce: B is complete when the kernel ends
        } else if (P.sk_len > 0 && !rs) {
            LaunchScope ls(h, SK_PHASE_SPLITK_REDUCE, stream);
            e = sk::launch_streamk_reduce(static_cast<const float*>(ws), p.part_stride, p.n1, p.r_valid, pass_cols,
                                          B + c0, ldb, P.rows_per_unit, P.kiters, P.sk_len, stream);
            if (e != cudaSuccess) return cuda_fail(e, "streamk_reduce launch");
        } else if (P.split > 1 && !rs) {
            LaunchScope ls(h, SK_PHASE_SPLITK_REDUCE, stream);
            e = sk::launch_splitk_reduce(static_cast<const float*>(ws), p.part_stride, P.split,
                                         p.n1, p.r_valid, pass_cols, B + c0, ldb, stream);
            if (e != cudaSuccess) return cuda_fail(e, "splitk_reduce launch");
        }
    }
    return SK_SUCCESS;
}

// C[r x r] (ldc) = Omega[i0 : i0+m, :r]^T * B[m x r]
sk_status_t core_impl(sk_sketch_s* h, const float* B, int64_t m, int64_t ldb, int64_t i0,
                      float* C, int64_t ldc, void* ws, cudaStream_t stream, int64_t nb = -1,
                      float* C_mc = nullptr) {
    if (nb < 0) nb = h->r;
    CorePlan CP = plan_core(h, m, i0, nb);
    if (CP.tc && (!aligned16(B) || (ldb & 3))) CP = plan_core_simt(h, m);  // TMA needs 16-B rows
    // the callers validated the workspace against core_ws_bytes(h, m): the partials of this plan must fit
    if (static_cast<size_t>(CP.chunks) * h->r * nb * sizeof(float) > core_ws_bytes(h, std::max<int64_t>(m, 1)))
        return fail(SK_ERR_WORKSPACE, "internal: core plan exceeds the workspace bound");
    if (C_mc && !CP.tc) return fail(SK_ERR_UNSUPPORTED, "multicast core needs the tcgen05 core (16-B aligned B rows)");
    if (C_mc && m == 0) return SK_SUCCESS;  // nothing to add
    if (CP.tc && m > 0) {
        CUtensorMap map;
        if (sk_status_t st = make_map_2d(&map, B, m, nb, ldb, 32, 32, false)) return st;
        sk::CoreTcParams q{};
        q.part = static_cast<float*>(ws);
        q.ldp = nb;
        q.i0 = i0;
        q.base = CP.base;
        q.step = CP.step;
        q.m = static_cast<int32_t>(m);
        q.r = static_cast<int32_t>(h->r);
        q.nb = static_cast<int32_t>(nb);
        q.npad = CP.npad;
        q.nchunks = CP.chunks;
        q.key0 = static_cast<uint32_t>(h->seed);
        q.key1 = static_cast<uint32_t>(h->seed >> 32);
        // partials [nchunks * r, r] stored by TMA in 32x32 tiles when r is a multiple of 32
        CUtensorMap omap;
        q.tma_store = (!C_mc && h->r % 32 == 0 && nb % 4 == 0 && aligned16(ws)) ? 1 : 0;
        q.mc_out = C_mc;
        q.ldc_mc = ldc;
        if (q.tma_store) {
            if (sk_status_t st = make_map_2d(&omap, q.part, static_cast<int64_t>(q.nchunks) * h->r, nb, nb, 32, 32))
                return st;
        } else {
            omap = map;  // unused
        }
        cudaError_t e;
        {
            LaunchScope ls(h, SK_PHASE_CORE_GEMM, stream);
            e = sk::launch_core_gemm_tc(map, omap, q, CP.nacc, h->dist, h->omega_transform == SK_OMEGA_FAST,
                                        h->mode == sk::kTF32x3, stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "core_gemm_tc launch");
        if (C_mc) return SK_SUCCESS;  // the epilogue added every partial into C on every rank
        {
            LaunchScope ls(h, SK_PHASE_CORE_REDUCE, stream);
            e = sk::launch_core_reduce(q.part, q.nchunks, q.r, q.nb, C, ldc, stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "core_reduce launch");
        return SK_SUCCESS;
    }
    sk::CoreGemmParams p{};
    p.B = B;
    p.ldb = ldb;
    p.part = static_cast<float*>(ws);
    p.ldp = nb;
    p.i0 = i0;
    p.m = static_cast<int32_t>(m);
    p.r = static_cast<int32_t>(h->r);
    p.nb = static_cast<int32_t>(nb);
    p.chunk_rows = CP.chunk_rows;
    p.chunks = CP.chunks;
    p.key0 = static_cast<uint32_t>(h->seed);
    p.key1 = static_cast<uint32_t>(h->seed >> 32);
    if (m == 0) {
        cudaError_t e = cudaMemset2DAsync(C, ldc * sizeof(float), 0, nb * sizeof(float), h->r, stream);
        return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "memset C");
    }
    cudaError_t e;
    {
        LaunchScope ls(h, SK_PHASE_CORE_GEMM, stream);
        e = sk::launch_core_gemm(p, h->dist, h->omega_transform == SK_OMEGA_FAST, stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "core_gemm launch");
    {
        LaunchScope ls(h, SK_PHASE_CORE_REDUCE, stream);
        e = sk::launch_core_reduce(p.part, p.chunks, p.r, p.nb, C, ldc, stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "core_reduce launch");
    return SK_SUCCESS;
}

}  // namespace

namespace sk {
int num_sms() {
    static const int n = [] {  // thread-safe one-time initialisation
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        return v;
    }();
    return n;
}
}  // namespace sk

extern "C" {

sk_status_t sketch_create(uint64_t seed, sk_dist_t dist, int64_t n2, int64_t r, sk_sketch_t* out) {
    if (!out) return fail(SK_ERR_INVALID_VALUE, "out == NULL");
    if (n2 < 1) return fail(SK_ERR_INVALID_VALUE, "n2 must be >= 1");
    if (r < 1 || r > 4096) return fail(SK_ERR_INVALID_VALUE, "r must be in [1, 4096]");
    if (dist != SK_DIST_GAUSSIAN && dist != SK_DIST_RADEMACHER && dist != SK_DIST_UNIFORM)
        return fail(SK_ERR_INVALID_VALUE, "unknown distribution");
    auto* h = new (std::nothrow) sk_sketch_s;
    if (!h) return fail(SK_ERR_INVALID_VALUE, "out of host memory");
    h->seed = seed;
    h->dist = static_cast<int>(dist);
    h->n2 = n2;
    h->r = r;
    h->mode = sk::kTF32x3;
    h->omega_transform = SK_OMEGA_ACCURATE;
    h->split_override = 0;
    h->cg_override = 0;
    h->core_simt = 0;
    h->cl_override = 0;
    h->ablate = 0;
    h->profiling = 0;
    *out = h;
    return SK_SUCCESS;
}

sk_status_t sketch_destroy(sk_sketch_t h) {
    if (h) {
        for (auto& t : h->prof) { cudaEventDestroy(t.start); cudaEventDestroy(t.end); }
        for (auto e : h->event_pool) cudaEventDestroy(e);
        if (h->copy_stream) {
            for (int i = 0; i < 2; ++i) { cudaEventDestroy(h->ev_h2d[i]); cudaEventDestroy(h->ev_done[i]); }
            cudaEventDestroy(h->ev_join);
            cudaStreamDestroy(h->copy_stream);
        }
        delete h;
    }
    return SK_SUCCESS;
}

sk_status_t sketch_set_profiling(sk_sketch_t h, int enable) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    h->profiling = enable ? 1 : 0;
    return SK_SUCCESS;
}

sk_status_t sketch_profile_read(sk_sketch_t h, double* ms, int64_t* launches) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (!ms || !launches) return fail(SK_ERR_INVALID_VALUE, "NULL output arrays");
    for (int i = 0; i < SK_PHASE_COUNT; ++i) { ms[i] = 0.0; launches[i] = 0; }
    std::vector<sk_timed_launch> v;
    {
        std::lock_guard<std::mutex> g(h->prof_mu);
        v.swap(h->prof);
    }
    sk_status_t st = SK_SUCCESS;
    for (auto& t : v) {
        float e = 0.f;
        cudaError_t err = cudaEventSynchronize(t.end);
        if (err == cudaSuccess) err = cudaEventElapsedTime(&e, t.start, t.end);
        if (err != cudaSuccess && st == SK_SUCCESS) st = cuda_fail(err, "profile event");
        ms[t.phase] += e;
        launches[t.phase] += 1;
    }
    {
        std::lock_guard<std::mutex> g(h->prof_mu);
        for (auto& t : v) {
            h->event_pool.push_back(t.start);
            h->event_pool.push_back(t.end);
        }
    }
    return st;
}

uint64_t sketch_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

sk_status_t sketch_set_mode(sk_sketch_t h, sk_mode_t mode) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (mode != SK_MODE_TF32X3 && mode != SK_MODE_TF32 && mode != SK_MODE_BF16)
        return fail(SK_ERR_INVALID_VALUE, "unknown mode");
    h->mode = static_cast<int>(mode);
    return SK_SUCCESS;
}

sk_status_t sketch_set_omega_transform(sk_sketch_t h, sk_omega_transform_t t) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (t != SK_OMEGA_ACCURATE && t != SK_OMEGA_FAST)
        return fail(SK_ERR_INVALID_VALUE, "unknown omega transform");
    h->omega_transform = static_cast<int>(t);
    return SK_SUCCESS;
}

sk_status_t sketch_set_split_k(sk_sketch_t h, int32_t split_k) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (split_k < 0 || split_k > 64) return fail(SK_ERR_INVALID_VALUE, "split_k must be in [0, 64]");
    h->split_override = split_k;
    return SK_SUCCESS;
}

sk_status_t sketch_set_cta_group(sk_sketch_t h, int32_t cg) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (!(cg == 0 || cg == 1 || cg == 2 || cg == 4 || cg == 6 || cg == 8))
        return fail(SK_ERR_INVALID_VALUE, "cta group must be 0 (auto), 1, 2, 4, 6 or 8");
    h->cg_override = (cg >= 4) ? 0 : cg;                // 4 / 6 / 8: pairs + sharing
    h->cl_override = (cg == 2) ? 1 : (cg >= 4) ? cg / 2 : 0;  // 2: pairs, no sharing
    return SK_SUCCESS;
}

sk_status_t sketch_set_core_impl(sk_sketch_t h, int32_t simt) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    h->core_simt = simt ? 1 : 0;
    return SK_SUCCESS;
}

sk_status_t sketch_set_ablation(sk_sketch_t h, uint32_t flags) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    h->ablate = flags & 255u;
    return SK_SUCCESS;
}

sk_status_t sketch_set_trace(sk_sketch_t h, uint64_t* dev_buf, int32_t stages) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (dev_buf && stages <= 0) return fail(SK_ERR_INVALID_VALUE, "trace needs stages > 0");
#ifndef SK_TRACE
    if (dev_buf) return fail(SK_ERR_UNSUPPORTED, "library built without SK_TRACE (SK_BUILD_TRACE=1)");
#endif
    h->trace = dev_buf;
    h->trace_stages = dev_buf ? stages : 0;
    return SK_SUCCESS;
}

sk_status_t sketch_workspace_size(sk_sketch_t h, int64_t n1, size_t* bytes) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (!bytes || n1 < 0) return fail(SK_ERR_INVALID_VALUE, "bad workspace query");
    *bytes = std::max(sketch_ws_bytes(h, std::max<int64_t>(n1, 1), h->n2), core_ws_bytes(h, std::max<int64_t>(n1, 1)));
    return SK_SUCCESS;
}

static sk_status_t validate_apply(sk_sketch_t h, const float* A, int64_t m, int64_t k, int64_t lda,
                                  int64_t k0, const float* B, int64_t ldb, void* ws,
                                  size_t ws_bytes, bool check_ws = true) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (sk_status_t st = check_mode(h)) return st;
    if (m < 0 || k < 1) return fail(SK_ERR_INVALID_VALUE, "need m >= 0 and k >= 1");
    if (m > (1ll << 31) - 256) return fail(SK_ERR_UNSUPPORTED, "m >= 2^31 rows");
    if (k0 < 0 || k0 + k > h->n2)
        return fail(SK_ERR_SHAPE_MISMATCH, "Omega rows [k0, k0+k) exceed the handle's n2");
    if (m > 0 && (!A || !B)) return fail(SK_ERR_INVALID_VALUE, "NULL matrix pointer");
    if (lda < k) return fail(SK_ERR_SHAPE_MISMATCH, "lda < number of columns of A");
    if (ldb < h->r) return fail(SK_ERR_SHAPE_MISMATCH, "ldb < r");
    if (!aligned16(A) || (lda & 3)) return fail(SK_ERR_ALIGNMENT, "A must be 16-byte aligned with lda % 4 == 0");
    if (!check_ws) return SK_SUCCESS;
    size_t need = 0;
    sketch_workspace_size(h, m, &need);
    if (ws_bytes < need || (need > 0 && !ws))
        return fail(SK_ERR_WORKSPACE, "workspace smaller than sketch_workspace_size (" +
                                          std::to_string(need) + " bytes)");
    if (ws && !aligned16(ws)) return fail(SK_ERR_ALIGNMENT, "workspace must be 16-byte aligned");
    return SK_SUCCESS;
}

sk_status_t sketch_apply(sk_sketch_t h, const float* A, int64_t n1, int64_t n2, int64_t lda,
                         float* B, int64_t ldb, void* ws, size_t ws_bytes, void* stream) {
    if (h && n2 != h->n2) return fail(SK_ERR_SHAPE_MISMATCH, "n2 != handle n2");
    if (sk_status_t st = validate_apply(h, A, n1, n2, lda, 0, B, ldb, ws, ws_bytes)) return st;
    return apply_impl(h, A, n1, n2, lda, 0, B, ldb, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

sk_status_t sketch_apply_block(sk_sketch_t h, const float* A_blk, int64_t m, int64_t k,
                               int64_t lda, int64_t k0, float* B_part, int64_t ldb, void* ws,
                               size_t ws_bytes, void* stream) {
    if (sk_status_t st = validate_apply(h, A_blk, m, k, lda, k0, B_part, ldb, ws, ws_bytes)) return st;
    return apply_impl(h, A_blk, m, k, lda, k0, B_part, ldb, ws, ws_bytes,
                      static_cast<cudaStream_t>(stream));
}

sk_status_t sketch_plan_info(sk_sketch_t h, int64_t m, int64_t k, int32_t* rows_per_unit, int32_t* split,
                             int32_t* cluster_pairs, int32_t* grid) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (m < 1 || k < 1) return fail(SK_ERR_INVALID_VALUE, "bad plan query");
    const SketchPlan P = plan_sketch(h, m, k, 0, ~size_t(0));
    if (rows_per_unit) *rows_per_unit = P.rows_per_unit;
    if (split) *split = P.split;
    if (cluster_pairs) *cluster_pairs = P.cl;
    if (grid) *grid = P.grid;
    return SK_SUCCESS;
}

sk_status_t sketch_rs_split(sk_sketch_t h, int64_t m, int64_t k, int32_t* split) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (!split || m < 1 || k < 1) return fail(SK_ERR_INVALID_VALUE, "bad reduce-scatter split query");
    *split = plan_sketch(h, m, k, 127, ~size_t(0)).split;
    return SK_SUCCESS;
}

sk_status_t sketch_apply_block_rs(sk_sketch_t h, const float* A_blk, int64_t m, int64_t k, int64_t lda,
                                  int64_t k0, float* const* dst, int32_t ndst, int64_t piece_rows,
                                  int32_t slot, int64_t slot_elems, int32_t split, void* stream) {
    if (sk_status_t st = validate_apply(h, A_blk, m, k, lda, k0, A_blk, h ? h->r : 0, nullptr, 0, false))
        return st;
    if (h->r > 256) return fail(SK_ERR_UNSUPPORTED, "fused reduce-scatter supports r <= 256 (one column pass)");
    if (!dst || ndst < 1 || ndst > 8) return fail(SK_ERR_INVALID_VALUE, "need 1 <= ndst <= 8 destinations");
    if (piece_rows < 1 || (m + piece_rows - 1) / piece_rows > ndst)
        return fail(SK_ERR_INVALID_VALUE, "row pieces exceed the destinations");
    if (slot < 0 || split < 1) return fail(SK_ERR_INVALID_VALUE, "need slot >= 0 and split >= 1");
    const int64_t npad = round_up(h->r, 16);
    if ((slot_elems & 3) || slot_elems < piece_rows * npad)
        return fail(SK_ERR_SHAPE_MISMATCH, "slot_elems must be a multiple of 4 and >= piece_rows * round_up(r, 16)");
    RsTarget rs{};
    for (int j = 0; j < ndst; ++j) {
        if (!dst[j] || !aligned16(dst[j])) return fail(SK_ERR_ALIGNMENT, "destinations must be 16-byte aligned");
        rs.dst[j] = dst[j];
    }
    rs.ndst = ndst;
    rs.slot = slot;
    rs.piece = piece_rows;
    rs.slot_elems = slot_elems;
    rs.split = split;
    return apply_impl(h, A_blk, m, k, lda, k0, nullptr, 0, nullptr, 0, static_cast<cudaStream_t>(stream), &rs);
}

sk_status_t sketch_reduce_slots(sk_sketch_t h, const float* slots, int32_t nslots, int64_t slot_elems,
                                int64_t rows, float* B, int64_t ldb, void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    const int64_t npad = round_up(h->r, 16);
    if (rows < 0 || nslots < 1 || !slots || (rows > 0 && !B)) return fail(SK_ERR_INVALID_VALUE, "bad slot reduce");
    if (ldb < h->r || slot_elems < rows * npad) return fail(SK_ERR_SHAPE_MISMATCH, "slot / B extents");
    if (rows == 0) return SK_SUCCESS;
    LaunchScope ls(h, SK_PHASE_SPLITK_REDUCE, static_cast<cudaStream_t>(stream));
    cudaError_t e = sk::launch_splitk_reduce(slots, slot_elems, nslots, static_cast<int32_t>(rows),
                                             static_cast<int32_t>(h->r), static_cast<int32_t>(npad), B, ldb,
                                             static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "slot reduce launch");
}

sk_status_t sketch_sum_peers(const float* const* src, int32_t n, int64_t elems, float* out, void* stream) {
    if (!src || !out || n < 1 || n > 8 || elems < 0) return fail(SK_ERR_INVALID_VALUE, "bad peer sum");
    if (elems & 3) return fail(SK_ERR_SHAPE_MISMATCH, "elems must be a multiple of 4");
    for (int j = 0; j < n; ++j)
        if (!src[j] || !aligned16(src[j])) return fail(SK_ERR_ALIGNMENT, "sources must be 16-byte aligned");
    if (!aligned16(out)) return fail(SK_ERR_ALIGNMENT, "out must be 16-byte aligned");
    if (elems == 0) return SK_SUCCESS;
    cudaError_t e;
    {
        LaunchScope ls(nullptr, 0, static_cast<cudaStream_t>(stream));
        e = sk::launch_sum_peers(src, n, elems, out, static_cast<cudaStream_t>(stream));
    }
    return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "peer sum launch");
}

sk_status_t sketch_multimem_sum(const float* mc_src, int64_t elems, float* out, float* mc_out, void* stream) {
    if (!mc_src || elems < 0 || (!out && !mc_out)) return fail(SK_ERR_INVALID_VALUE, "bad multicast reduction arguments");
    if (elems % 4 != 0) return fail(SK_ERR_SHAPE_MISMATCH, "elems must be a multiple of 4");
    if (!aligned16(mc_src) || (out && !aligned16(out)) || (mc_out && !aligned16(mc_out)))
        return fail(SK_ERR_ALIGNMENT, "multicast reduction needs 16-byte aligned buffers");
    cudaError_t e;
    {
        LaunchScope ls(nullptr, 0, static_cast<cudaStream_t>(stream));
        e = sk::launch_multimem_sum(mc_src, elems, out, mc_out, static_cast<cudaStream_t>(stream));
    }
    return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "multimem sum launch");
}

sk_status_t sketch_pack_cols(const float* B, int64_t rows, int64_t ldb, const int64_t* cb, int32_t nblk,
                             float* out, void* stream) {
    if (!cb || nblk < 1 || nblk > 64 || rows < 0) return fail(SK_ERR_INVALID_VALUE, "bad column-pack arguments");
    if (cb[0] != 0) return fail(SK_ERR_INVALID_VALUE, "cb[0] must be 0");
    for (int j = 0; j < nblk; ++j)
        if (cb[j + 1] < cb[j]) return fail(SK_ERR_INVALID_VALUE, "column bounds must be non-decreasing");
    if (cb[nblk] > ldb) return fail(SK_ERR_SHAPE_MISMATCH, "cb[nblk] > ldb");
    if (rows == 0 || cb[nblk] == 0) return SK_SUCCESS;
    if (!B || !out) return fail(SK_ERR_INVALID_VALUE, "NULL matrix pointer");
    cudaError_t e;
    {
        LaunchScope ls(nullptr, 0, static_cast<cudaStream_t>(stream));
        e = sk::launch_pack_cols(B, rows, ldb, cb, nblk, out, static_cast<cudaStream_t>(stream));
    }
    return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "pack_cols launch");
}

sk_status_t core_apply_block(sk_sketch_t h, const float* B_blk, int64_t m, int64_t ldb,
                             int64_t i0, float* C_part, int64_t ldc, void* ws, size_t ws_bytes,
                             void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (sk_status_t st = check_mode(h)) return st;
    if (m < 0 || i0 < 0 || i0 + m > h->n2)
        return fail(SK_ERR_SHAPE_MISMATCH, "Omega rows [i0, i0+m) exceed the handle's n2");
    if ((m > 0 && !B_blk) || !C_part) return fail(SK_ERR_INVALID_VALUE, "NULL matrix pointer");
    if (ldb < h->r || ldc < h->r) return fail(SK_ERR_SHAPE_MISMATCH, "ldb / ldc < r");
    const size_t need = core_ws_bytes(h, std::max<int64_t>(m, 1));
    if (ws_bytes < need || !ws)
        return fail(SK_ERR_WORKSPACE, "workspace smaller than sketch_workspace_size");
    return core_impl(h, B_blk, m, ldb, i0, C_part, ldc, ws, static_cast<cudaStream_t>(stream));
}

sk_status_t core_apply_block_mc(sk_sketch_t h, const float* B_blk, int64_t m, int64_t ldb, int64_t i0,
                                float* C_mc, int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (sk_status_t st = check_mode(h)) return st;
    if (m < 0 || i0 < 0 || i0 + m > h->n2)
        return fail(SK_ERR_SHAPE_MISMATCH, "Omega rows [i0, i0+m) exceed the handle's n2");
    if ((m > 0 && !B_blk) || !C_mc) return fail(SK_ERR_INVALID_VALUE, "NULL matrix pointer");
    if (ldb < h->r || ldc < h->r) return fail(SK_ERR_SHAPE_MISMATCH, "ldb / ldc < r");
    if (!aligned16(C_mc) || (ldc & 3)) return fail(SK_ERR_ALIGNMENT, "C_mc and ldc must be 16-byte aligned");
    const size_t need = core_ws_bytes(h, std::max<int64_t>(m, 1));
    if (ws_bytes < need || !ws)
        return fail(SK_ERR_WORKSPACE, "workspace smaller than sketch_workspace_size");
    return core_impl(h, B_blk, m, ldb, i0, nullptr, ldc, ws, static_cast<cudaStream_t>(stream), -1, C_mc);
}

sk_status_t core_apply_block_cols(sk_sketch_t h, const float* B_blk, int64_t m, int64_t nb, int64_t ldb,
                                  int64_t i0, float* C_part, int64_t ldc, void* ws, size_t ws_bytes,
                                  void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (sk_status_t st = check_mode(h)) return st;
    if (m < 0 || i0 < 0 || i0 + m > h->n2)
        return fail(SK_ERR_SHAPE_MISMATCH, "Omega rows [i0, i0+m) exceed the handle's n2");
    if (nb < 1 || nb > h->r) return fail(SK_ERR_INVALID_VALUE, "nb must be in [1, r]");
    if ((m > 0 && !B_blk) || !C_part) return fail(SK_ERR_INVALID_VALUE, "NULL matrix pointer");
    if (ldb < nb || ldc < nb) return fail(SK_ERR_SHAPE_MISMATCH, "ldb / ldc < nb");
    const size_t need = core_ws_bytes(h, std::max<int64_t>(m, 1));
    if (ws_bytes < need || !ws)
        return fail(SK_ERR_WORKSPACE, "workspace smaller than sketch_workspace_size");
    return core_impl(h, B_blk, m, ldb, i0, C_part, ldc, ws, static_cast<cudaStream_t>(stream), nb);
}

sk_status_t nystrom_core(sk_sketch_t h, const float* A, int64_t n, int64_t lda, float* B,
                         int64_t ldb, float* C, int64_t ldc, void* ws, size_t ws_bytes,
                         void* stream) {
    if (h && n != h->n2) return fail(SK_ERR_SHAPE_MISMATCH, "n != handle n2 (A must be n2 x n2)");
    if (sk_status_t st = validate_apply(h, A, n, n, lda, 0, B, ldb, ws, ws_bytes)) return st;
    if (!C) return fail(SK_ERR_INVALID_VALUE, "NULL C");
    if (ldc < h->r) return fail(SK_ERR_SHAPE_MISMATCH, "ldc < r");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (sk_status_t st = apply_impl(h, A, n, n, lda, 0, B, ldb, ws, ws_bytes, s)) return st;
    return core_impl(h, B, n, ldb, 0, C, ldc, ws, s);
}

sk_status_t sketch_generate(sk_sketch_t h, int64_t row0, int64_t nrows, int64_t col0,
                            int64_t ncols, float* out, int64_t ld, void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (!out || row0 < 0 || nrows < 0 || col0 < 0 || ncols < 0 || col0 + ncols > h->r ||
        row0 + nrows > (1ll << 62) || ld < ncols)
        return fail(SK_ERR_INVALID_VALUE, "block outside [0, 2^62) x [0, r) or bad ld");
    LaunchScope ls(h, SK_PHASE_GENERATE, static_cast<cudaStream_t>(stream));
    cudaError_t e = sk::launch_generate(h->seed, h->dist, row0, nrows, col0, ncols, out, ld, false,
                                        static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "generate launch");
}

sk_status_t sketch_generate_bits(sk_sketch_t h, int64_t row0, int64_t nrows, int64_t col0,
                                 int64_t ncols, uint32_t* out, int64_t ld, void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (!out || row0 < 0 || nrows < 0 || col0 < 0 || ncols < 0 || col0 + ncols > h->r ||
        row0 + nrows > (1ll << 62) || ld < ncols)
        return fail(SK_ERR_INVALID_VALUE, "block outside [0, 2^62) x [0, r) or bad ld");
    LaunchScope ls(h, SK_PHASE_GENERATE, static_cast<cudaStream_t>(stream));
    cudaError_t e = sk::launch_generate(h->seed, h->dist, row0, nrows, col0, ncols, out, ld, true,
                                        static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "generate_bits launch");
}

sk_status_t sketch_debug_box_muller(const uint32_t* w1, const uint32_t* w2, int64_t n,
                                    sk_omega_transform_t transform, float* out_even,
                                    float* out_odd, void* stream) {
    if (n < 0 || (n > 0 && (!w1 || !w2 || !out_even || !out_odd)))
        return fail(SK_ERR_INVALID_VALUE, "bad debug_box_muller arguments");
    LaunchScope ls(nullptr, SK_PHASE_GENERATE, static_cast<cudaStream_t>(stream));
    cudaError_t e = sk::launch_debug_box_muller(w1, w2, n, transform == SK_OMEGA_FAST, out_even,
                                                out_odd, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SK_SUCCESS : cuda_fail(e, "debug_box_muller launch");
}

// ------------------------------------------------------------------------------- host streaming
static int64_t host_block_rows(int64_t n1, int64_t block_rows) {
    int64_t b = block_rows > 0 ? block_rows : 8192;
    b = std::min<int64_t>(b, std::max<int64_t>(n1, 1));
    return round_up(b, 4);
}

struct HostWs {
    size_t a_off[2], b_off[2], cacc_off, cpart_off, inner_off, total, a_elems, ld_dev;
};

static HostWs host_ws_layout(sk_sketch_s* h, int64_t n1, int64_t n2, int64_t block_rows) {
    HostWs W{};
    const int64_t br = host_block_rows(n1, block_rows);
    W.ld_dev = static_cast<size_t>(round_up(n2, 4));
    W.a_elems = static_cast<size_t>(br) * W.ld_dev;
    size_t inner = 0;
    sketch_workspace_size(h, br, &inner);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = round_up(static_cast<int64_t>(off + bytes), 256); return o; };
    for (int i = 0; i < 2; ++i) W.a_off[i] = take(W.a_elems * sizeof(float));
    for (int i = 0; i < 2; ++i) W.b_off[i] = take(static_cast<size_t>(br) * h->r * sizeof(float));
    W.cacc_off = take(static_cast<size_t>(h->r) * h->r * sizeof(float));
    W.cpart_off = take(static_cast<size_t>(h->r) * h->r * sizeof(float));
    W.inner_off = take(inner);
    W.total = off;
    return W;
}

static sk_status_t host_stream_impl(sk_sketch_s* h, const float* A, int64_t n1, int64_t n2, int64_t lda,
                                    float* B, int64_t ldb, float* C, int64_t ldc, int64_t block_rows,
                                    void* ws, size_t ws_bytes, cudaStream_t s) {
    const HostWs W = host_ws_layout(h, n1, n2, block_rows);
    if (ws_bytes < W.total || !ws) return fail(SK_ERR_WORKSPACE, "workspace smaller than sketch_host_workspace_size");
    if (!aligned16(ws)) return fail(SK_ERR_ALIGNMENT, "workspace must be 16-byte aligned");
    std::lock_guard<std::mutex> g(h->host_mu);
    if (!h->copy_stream) {
        if (cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "copy stream");
        for (int i = 0; i < 2; ++i) {
            cudaEventCreateWithFlags(&h->ev_h2d[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&h->ev_done[i], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
    }
    uint8_t* base = static_cast<uint8_t*>(ws);
    const int64_t br = host_block_rows(n1, block_rows);
    const size_t inner_bytes = W.total - W.inner_off;
    float* Cacc = reinterpret_cast<float*>(base + W.cacc_off);
    float* Cpart = reinterpret_cast<float*>(base + W.cpart_off);
    cudaError_t e;
    // the copy stream starts after everything already enqueued on `s`
    if ((e = cudaEventRecord(h->ev_join, s)) != cudaSuccess) return cuda_fail(e, "event");
    if ((e = cudaStreamWaitEvent(h->copy_stream, h->ev_join, 0)) != cudaSuccess) return cuda_fail(e, "event");
    const int64_t nblk = (n1 + br - 1) / br;
    for (int64_t bi = 0; bi < nblk; ++bi) {
        const int slot = static_cast<int>(bi & 1);
        const int64_t r0 = bi * br, rows = std::min(br, n1 - r0);
        float* Ad = reinterpret_cast<float*>(base + W.a_off[slot]);
        float* Bd = reinterpret_cast<float*>(base + W.b_off[slot]);
        // H2D of block bi on the copy stream, once the compute that used this slot is done
        if (bi >= 2 && (e = cudaStreamWaitEvent(h->copy_stream, h->ev_done[slot], 0)) != cudaSuccess)
            return cuda_fail(e, "event");
        e = cudaMemcpy2DAsync(Ad, W.ld_dev * sizeof(float), A + r0 * lda, lda * sizeof(float),
                              n2 * sizeof(float), rows, cudaMemcpyHostToDevice, h->copy_stream);
        if (e != cudaSuccess) return cuda_fail(e, "H2D of an A block");
        if ((e = cudaEventRecord(h->ev_h2d[slot], h->copy_stream)) != cudaSuccess) return cuda_fail(e, "event");
        // sketch (and core) of block bi on the caller's stream
        if ((e = cudaStreamWaitEvent(s, h->ev_h2d[slot], 0)) != cudaSuccess) return cuda_fail(e, "event");
        if (sk_status_t st = apply_impl(h, Ad, rows, n2, static_cast<int64_t>(W.ld_dev), 0, Bd, h->r,
                                        base + W.inner_off, inner_bytes, s))
            return st;
        if (C) {
            if (sk_status_t st = core_impl(h, Bd, rows, h->r, r0, Cpart, h->r, base + W.inner_off, s)) return st;
            LaunchScope ls(h, SK_PHASE_CORE_REDUCE, s);
            if ((e = sk::launch_accumulate(Cacc, Cpart, h->r * h->r, bi == 0, s)) != cudaSuccess)
                return cuda_fail(e, "accumulate C");
        }
        e = cudaMemcpy2DAsync(B + r0 * ldb, ldb * sizeof(float), Bd, h->r * sizeof(float), h->r * sizeof(float),
                              rows, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e, "D2H of a B block");
        if ((e = cudaEventRecord(h->ev_done[slot], s)) != cudaSuccess) return cuda_fail(e, "event");
    }
    if (C) {
        e = cudaMemcpy2DAsync(C, ldc * sizeof(float), Cacc, h->r * sizeof(float), h->r * sizeof(float), h->r,
                              cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e, "D2H of C");
    }
    // join: `s` also waits for the copy stream's last operation
    if ((e = cudaEventRecord(h->ev_join, h->copy_stream)) != cudaSuccess) return cuda_fail(e, "event");
    if ((e = cudaStreamWaitEvent(s, h->ev_join, 0)) != cudaSuccess) return cuda_fail(e, "event");
    return SK_SUCCESS;
}

sk_status_t sketch_host_workspace_size(sk_sketch_t h, int64_t n1, int64_t block_rows, size_t* bytes) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (!bytes || n1 < 0) return fail(SK_ERR_INVALID_VALUE, "bad workspace query");
    *bytes = host_ws_layout(h, std::max<int64_t>(n1, 1), h->n2, block_rows).total;
    return SK_SUCCESS;
}

sk_status_t sketch_apply_host(sk_sketch_t h, const float* A_host, int64_t n1, int64_t n2, int64_t lda,
                              float* B_host, int64_t ldb, int64_t block_rows, void* ws,
                              size_t ws_bytes, void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (sk_status_t st = check_mode(h)) return st;
    if (n2 != h->n2) return fail(SK_ERR_SHAPE_MISMATCH, "n2 != handle n2");
    if (n1 < 0) return fail(SK_ERR_INVALID_VALUE, "n1 < 0");
    if (n1 > 0 && (!A_host || !B_host)) return fail(SK_ERR_INVALID_VALUE, "NULL matrix pointer");
    if (lda < n2 || ldb < h->r) return fail(SK_ERR_SHAPE_MISMATCH, "lda < n2 or ldb < r");
    if (n1 == 0) return SK_SUCCESS;
    return host_stream_impl(h, A_host, n1, n2, lda, B_host, ldb, nullptr, 0, block_rows, ws, ws_bytes,
                            static_cast<cudaStream_t>(stream));
}

sk_status_t nystrom_core_host(sk_sketch_t h, const float* A_host, int64_t n, int64_t lda,
                              float* B_host, int64_t ldb, float* C_host, int64_t ldc,
                              int64_t block_rows, void* ws, size_t ws_bytes, void* stream) {
    if (check_handle(h)) return SK_ERR_INVALID_VALUE;
    if (sk_status_t st = check_mode(h)) return st;
    if (n != h->n2) return fail(SK_ERR_SHAPE_MISMATCH, "n != handle n2 (A must be n2 x n2)");
    if (!A_host || !B_host || !C_host) return fail(SK_ERR_INVALID_VALUE, "NULL matrix pointer");
    if (lda < n || ldb < h->r || ldc < h->r) return fail(SK_ERR_SHAPE_MISMATCH, "lda / ldb / ldc too small");
    return host_stream_impl(h, A_host, n, n, lda, B_host, ldb, C_host, ldc, block_rows, ws, ws_bytes,
                            static_cast<cudaStream_t>(stream));
}

const char* sketch_status_string(sk_status_t st) {
    switch (st) {
        case SK_SUCCESS: return "SK_SUCCESS";
        case SK_ERR_INVALID_VALUE: return "SK_ERR_INVALID_VALUE";
        case SK_ERR_SHAPE_MISMATCH: return "SK_ERR_SHAPE_MISMATCH";
        case SK_ERR_ALIGNMENT: return "SK_ERR_ALIGNMENT";
        case SK_ERR_UNSUPPORTED: return "SK_ERR_UNSUPPORTED";
        case SK_ERR_WORKSPACE: return "SK_ERR_WORKSPACE";
        case SK_ERR_CUDA: return "SK_ERR_CUDA";
        case SK_ERR_NCCL: return "SK_ERR_NCCL";
    }
    return "SK_ERR_UNKNOWN";
}

const char* sketch_last_error(void) { return g_last_error.c_str(); }

const char* sketch_build_info(void) {
    return "libsketch sm_100a (tcgen05 sketch GEMM: tf32 / bf16 / 3xTF32, fused Philox4x32-10 Omega tiles; "
           "tcgen05 core GEMM with regenerated Omega; fixed-order reductions)";
}

}  // extern "C"
