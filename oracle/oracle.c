/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference for the hot path of
 * arXiv 2603.20966 ("Communication Lower Bounds and Algorithms for Sketching
 * with Random Dense Matrices"):
 *
 *     B = A * Omega          (sec. 1: "mapped ... by multiplying
 *                             it with a random matrix Omega in R^{n2 x r}")
 *     C = Omega^T * B        (sec. 1: "first computing B = A Omega
 *                             and then computing C = Omega^T B")
 *
 * with Omega regenerated from a counter-based Philox generator with a shared
 * seed (sec. 6.3: "generate the entire Omega with a shared
 * seed on each process ... counter-based pseudorandom number generation
 * algorithm Philox [salmon2011parallel]").  The paper fixes neither the counter
 * layout nor the Gaussian transform; this file follows the reading O1 recorded
 * in DESIGN.md ("Readings of the paper", R1-R4), step by step:
 *
 *   Philox4x32-10 (Salmon et al. 2011, the reference the paper cites at
 *   PAPER.md:1190), key = (seed & 0xffffffff, seed >> 32).
 *   Gaussian / uniform stream (tag 0): element (j, k) of Omega (global row j,
 *     global column k) uses counter (q & 0xffffffff, q >> 32, k, 0), q = j >> 2;
 *     x = Philox(ctr, key).  Raw word U[j,k] = x[j & 3].
 *     uniform:  (U >> 8) * 2^-24.
 *     Gaussian (Box-Muller, "Gaussian random matrices"): p = j & 2,
 *       u1 = ((x[p] >> 8) + 1) * 2^-24 in (0,1],  u2 = (x[p+1] >> 8) * 2^-24 in [0,1),
 *       R = sqrt(-2 ln u1);  z = R cos(2 pi u2) for even j, R sin(2 pi u2) for odd j.
 *       Evaluated in fp64 with the angle reduced exactly in quarter turns, then
 *       rounded ONCE to fp32: Omega[j,k] is that fp32 value.
 *   Rademacher stream (tag 1): counter (g & 0xffffffff, g >> 32, k, 1), g = j >> 7;
 *     bit = (x[(j >> 5) & 3] >> (j & 31)) & 1;  Omega[j,k] = bit ? -1 : +1.
 *
 *   B[i,k] = sum_{j < n2} (double)A[i,j] * (double)Omega[j,k], j increasing.
 *   C[a,b] = sum_{i < n}  (double)Omega[i,a] * B[i,b],         i increasing.
 *
 * Nothing here is shared with the CUDA path (paper_2603_20966_b200/csrc): no
 * headers, no tables, no helpers.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------------------
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random numbers:
 * as easy as 1, 2, 3"; cited by the paper at PAPER.md:1190).
 * One round:  (c0,c1,c2,c3) <- (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0));
 * the key is bumped by the Weyl constants (W0, W1) between rounds.
 * ------------------------------------------------------------------------- */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Distribution codes (same numbering as the public header, restated here). */
enum { ORACLE_GAUSSIAN = 0, ORACLE_RADEMACHER = 1, ORACLE_UNIFORM = 2 };

static void philox_for(uint64_t seed, uint64_t blk, uint32_t col, uint32_t tag, uint32_t x[4])
{
    uint32_t ctr[4] = { (uint32_t)(blk & 0xffffffffu), (uint32_t)(blk >> 32), col, tag };
    uint32_t key[2] = { (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32) };
    oracle_philox4x32_10(ctr, key, x);
}

/* Raw Philox word from which element (j,k) is derived (reading O1). */
uint32_t oracle_omega_word(uint64_t seed, int dist, uint64_t j, uint64_t k)
{
    uint32_t x[4];
    if (dist == ORACLE_RADEMACHER) {
        philox_for(seed, j >> 7, (uint32_t)k, 1u, x);
        return x[(j >> 5) & 3u];
    }
    philox_for(seed, j >> 2, (uint32_t)k, 0u, x);
    return x[j & 3u];
}

/* Box-Muller in fp64, angle reduced exactly in quarter turns.
 * w1, w2: the two raw words of the pair.  Writes z_even = R cos(2 pi u2),
 * z_odd = R sin(2 pi u2), each in fp64 (not yet rounded). */
void oracle_box_muller(uint32_t w1, uint32_t w2, double *z_even, double *z_odd)
{
    double u1 = ((double)(w1 >> 8) + 1.0) * 0x1p-24;   /* (0, 1]  */
    double u2 = (double)(w2 >> 8) * 0x1p-24;           /* [0, 1)  */
    double R = sqrt(-2.0 * log(u1));
    /* 2 pi u2 = (pi/2) * v with v = 4 u2 in [0,4) quarter turns (exact).
     * v = q + f, q = nearest integer (mod 4), f in [-1/2, 1/2] (exact). */
    double v = 4.0 * u2;
    double qd = floor(v + 0.5);
    double f = v - qd;
    int q = ((int)qd) & 3;
    double phi = f * (M_PI / 2.0);
    double s = sin(phi), c = cos(phi);
    double cv, sv;   /* cos(2 pi u2), sin(2 pi u2) */
    switch (q) {
        case 0:  cv =  c; sv =  s; break;
        case 1:  cv = -s; sv =  c; break;
        case 2:  cv = -c; sv = -s; break;
        default: cv =  s; sv = -c; break;
    }
    *z_even = R * cv;
    *z_odd = R * sv;
}

/* Omega[j,k] in fp32 (rounded once from the fp64 value). */
float oracle_omega_value(uint64_t seed, int dist, uint64_t j, uint64_t k)
{
    if (dist == ORACLE_RADEMACHER) {
        uint32_t w = oracle_omega_word(seed, dist, j, k);
        return ((w >> (j & 31u)) & 1u) ? -1.0f : 1.0f;
    }
    uint32_t x[4];
    philox_for(seed, j >> 2, (uint32_t)k, 0u, x);
    if (dist == ORACLE_UNIFORM)
        return (float)((double)(x[j & 3u] >> 8) * 0x1p-24);
    unsigned p = (unsigned)(j & 2u);
    double ze, zo;
    oracle_box_muller(x[p], x[p + 1], &ze, &zo);
    return (float)((j & 1u) ? zo : ze);
}

/* Materialise rows [row0,row0+nrows) x cols [col0,col0+ncols) of Omega,
 * row-major with leading dimension ld (elements). */
void oracle_omega(uint64_t seed, int dist, int64_t row0, int64_t nrows,
                  int64_t col0, int64_t ncols, float *out, int64_t ld)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t c = 0; c < ncols; ++c)
            out[i * ld + c] = oracle_omega_value(seed, dist, (uint64_t)(row0 + i), (uint64_t)(col0 + c));
}

void oracle_omega_words(uint64_t seed, int dist, int64_t row0, int64_t nrows,
                        int64_t col0, int64_t ncols, uint32_t *out, int64_t ld)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t c = 0; c < ncols; ++c)
            out[i * ld + c] = oracle_omega_word(seed, dist, (uint64_t)(row0 + i), (uint64_t)(col0 + c));
}

/* B[i,k] = sum_j A[i,j] * Omega[k0 + j, k] for i < n1, k < r, fp64, j increasing.
 * A: fp32 row-major (lda); Omega rows start at global row k0 (block form,
 * PAPER.md:411 "GenRandom(n2/p2, r/p3)" for block column j of the grid).
 * Omega is materialised first (plain definition), then the triple loop runs. */
void oracle_sketch(uint64_t seed, int dist, const float *A, int64_t n1, int64_t n2,
                   int64_t lda, int64_t k0, int64_t r, double *B, int64_t ldb)
{
    float *Om = (float *)malloc((size_t)n2 * (size_t)r * sizeof(float));
    oracle_omega(seed, dist, k0, n2, 0, r, Om, r);
    #pragma omp parallel
    {
        double *acc = (double *)malloc((size_t)r * sizeof(double));
        #pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < n1; ++i) {
            for (int64_t k = 0; k < r; ++k) acc[k] = 0.0;
            const float *a = A + i * lda;
            for (int64_t j = 0; j < n2; ++j) {
                double aij = (double)a[j];
                const float *om = Om + j * r;
                for (int64_t k = 0; k < r; ++k) acc[k] += aij * (double)om[k];
            }
            for (int64_t k = 0; k < r; ++k) B[i * ldb + k] = acc[k];
        }
        free(acc);
    }
    free(Om);
}

/* C[a,b] = sum_i Omega[i0 + i, a] * B[i, b], fp64, i increasing (PAPER.md:611,
 * Alg. 2 line "C-bar = Omega^T B").  B: fp64 row-major n x r (ldb). */
void oracle_core(uint64_t seed, int dist, const double *B, int64_t n, int64_t ldb,
                 int64_t i0, int64_t r, double *C, int64_t ldc)
{
    float *Om = (float *)malloc((size_t)n * (size_t)r * sizeof(float));
    oracle_omega(seed, dist, i0, n, 0, r, Om, r);
    #pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < r; ++a) {
        for (int64_t b = 0; b < r; ++b) {
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) s += (double)Om[i * r + a] * B[i * ldb + b];
            C[a * ldc + b] = s;
        }
    }
    free(Om);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Vectorised oracle_box_muller for exhaustive transform checks: fp64 results rounded once
 * to fp32 (RN), i.e. the correctly rounded reference Gaussians. */
void oracle_box_muller_many(const uint32_t *w1, const uint32_t *w2, int64_t n,
                            float *z_even, float *z_odd)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double ze, zo;
        oracle_box_muller(w1[i], w2[i], &ze, &zo);
        z_even[i] = (float)ze;
        z_odd[i] = (float)zo;
    }
}
