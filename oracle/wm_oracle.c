/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Only tests/, the smoke() check in
 * __graft_entry__.py and bench.py's cpu_baseline leg may load this library, and
 * only as the checker; the product (paper_0707_2347_b200) never links it.
 *
 * A plain-C restatement of the reference's ring layer
 * (/root/reference/proj/include/winomem/ring.hpp):
 *   wmo_splitmix_fill   <- SplitMix64 + Matrix::fill_random   ring.hpp:93-105,202-205
 *   wmo_fnv1a64         <- fnv1a64 / Matrix::hash             ring.hpp:107-114,208
 *   wmo_block_addsub    <- block_addsub                       ring.hpp:241-278
 *   wmo_classical_modp  <- classical_mul (lazy u64 path, p<2^16, and the
 *                          per-step-reduce path otherwise)    ring.hpp:315-384
 *   wmo_classical_f64   <- the same contraction over the reals (config 5 has no
 *                          reference float path: SPEC.md:94 -- parity for it is
 *                          pinned only by this restatement)
 *   wmo_real_fill       <- builder-defined float generator
 *                          x = 2*((next()>>11)*2^-53) - 1
 * Row striping over POSIX threads is an oracle-side speed-up only (the
 * reference is single-threaded); every output element is computed exactly as
 * the reference computes it, so results are bit-identical at any thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* state after i+1 calls is seed + (i+1)*gamma, so the stream is index-addressable */
void wmo_splitmix_fill(uint32_t* out, uint64_t count, uint64_t seed, uint32_t p) {
    const uint64_t gamma = 0x9e3779b97f4a7c15ull;
    for (uint64_t i = 0; i < count; ++i) out[i] = (uint32_t)(sm64_mix(seed + (i + 1) * gamma) % p);
}

void wmo_splitmix_raw(uint64_t* out, uint64_t count, uint64_t seed) {
    const uint64_t gamma = 0x9e3779b97f4a7c15ull;
    for (uint64_t i = 0; i < count; ++i) out[i] = sm64_mix(seed + (i + 1) * gamma);
}

void wmo_real_fill(double* out, uint64_t count, uint64_t seed) {
    const uint64_t gamma = 0x9e3779b97f4a7c15ull;
    for (uint64_t i = 0; i < count; ++i) {
        double u = (double)(sm64_mix(seed + (i + 1) * gamma) >> 11) * 0x1.0p-53;
        out[i] = 2.0 * u - 1.0;
    }
}

uint64_t wmo_fnv1a64(const uint32_t* data, uint64_t count) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < count; ++i) {
        h ^= data[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* dst <- sa*a + sb*b mod p over an r x c window (row strides lda/ldb/ldd) */
void wmo_block_addsub(uint64_t r, uint64_t c, uint32_t p, uint32_t* dst, uint64_t ldd,
                      const uint32_t* a, uint64_t lda, const uint32_t* b, uint64_t ldb,
                      uint32_t sa, uint32_t sb) {
    for (uint64_t i = 0; i < r; ++i)
        for (uint64_t j = 0; j < c; ++j) {
            uint64_t v = (uint64_t)sa * a[i * lda + j] + (uint64_t)sb * b[i * ldb + j];
            dst[i * ldd + j] = (uint32_t)(v % p);
        }
}

typedef struct {
    uint64_t m, k, n, lda, ldb, ldc, row0, row1;
    const uint32_t *A, *B;
    uint32_t* C;
    uint32_t alpha, beta, p;
} modp_job;

static void* modp_worker(void* arg) {
    const modp_job* j = (const modp_job*)arg;
    enum { TILE = 64 };
    uint64_t acc[TILE];
    const uint32_t p = j->p;
    for (uint64_t i = j->row0; i < j->row1; ++i) {
        for (uint64_t j0 = 0; j0 < j->n; j0 += TILE) {
            const uint64_t w = (j->n - j0) < TILE ? (j->n - j0) : TILE;
            for (uint64_t t = 0; t < w; ++t) acc[t] = 0;
            if (p < (1u << 16)) {
                for (uint64_t l = 0; l < j->k; ++l) {
                    const uint64_t av = j->A[i * j->lda + l];
                    const uint32_t* brow = j->B + l * j->ldb + j0;
                    for (uint64_t t = 0; t < w; ++t) acc[t] += av * brow[t];
                }
                for (uint64_t t = 0; t < w; ++t) acc[t] %= p;
            } else {
                for (uint64_t l = 0; l < j->k; ++l) {
                    const uint64_t av = j->A[i * j->lda + l];
                    const uint32_t* brow = j->B + l * j->ldb + j0;
                    for (uint64_t t = 0; t < w; ++t) acc[t] = (acc[t] + av * brow[t]) % p;
                }
            }
            for (uint64_t t = 0; t < w; ++t) {
                uint64_t dot = (acc[t] * j->alpha) % p;
                uint32_t* c = j->C + i * j->ldc + j0 + t;
                *c = (uint32_t)((j->beta == 0) ? dot : (dot + (uint64_t)j->beta * *c) % p);
            }
        }
    }
    return NULL;
}

/* C <- alpha*A*B + beta*C mod p, exact, C disjoint from A and B. */
void wmo_classical_modp(uint64_t m, uint64_t k, uint64_t n, const uint32_t* A, uint64_t lda,
                        const uint32_t* B, uint64_t ldb, uint32_t* C, uint64_t ldc,
                        uint32_t alpha, uint32_t beta, uint32_t p, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > m) nthreads = (int)m;
    modp_job* jobs = (modp_job*)calloc((size_t)nthreads, sizeof(modp_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        modp_job* j = &jobs[t];
        j->m = m; j->k = k; j->n = n; j->lda = lda; j->ldb = ldb; j->ldc = ldc;
        j->row0 = m * (uint64_t)t / (uint64_t)nthreads;
        j->row1 = m * (uint64_t)(t + 1) / (uint64_t)nthreads;
        j->A = A; j->B = B; j->C = C; j->alpha = alpha % p; j->beta = beta % p; j->p = p;
        if (nthreads > 1) pthread_create(&th[t], NULL, modp_worker, j);
        else modp_worker(j);
    }
    if (nthreads > 1)
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

typedef struct {
    uint64_t m, k, n, lda, ldb, ldc, row0, row1;
    const double *A, *B;
    double* C;
    double alpha, beta;
} f64_job;

static void* f64_worker(void* arg) {
    const f64_job* j = (const f64_job*)arg;
    enum { TILE = 128 };
    double acc[TILE];
    for (uint64_t i = j->row0; i < j->row1; ++i) {
        for (uint64_t j0 = 0; j0 < j->n; j0 += TILE) {
            const uint64_t w = (j->n - j0) < TILE ? (j->n - j0) : TILE;
            for (uint64_t t = 0; t < w; ++t) acc[t] = 0.0;
            for (uint64_t l = 0; l < j->k; ++l) {
                const double av = j->A[i * j->lda + l];
                const double* brow = j->B + l * j->ldb + j0;
                for (uint64_t t = 0; t < w; ++t) acc[t] += av * brow[t];
            }
            for (uint64_t t = 0; t < w; ++t) {
                double* c = j->C + i * j->ldc + j0 + t;
                *c = j->alpha * acc[t] + (j->beta == 0.0 ? 0.0 : j->beta * *c);
            }
        }
    }
    return NULL;
}

/* classical C <- alpha*A*B + beta*C over the reals (the config-5 reference) */
void wmo_classical_f64(uint64_t m, uint64_t k, uint64_t n, const double* A, uint64_t lda,
                       const double* B, uint64_t ldb, double* C, uint64_t ldc, double alpha,
                       double beta, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > m) nthreads = (int)m;
    f64_job* jobs = (f64_job*)calloc((size_t)nthreads, sizeof(f64_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        f64_job* j = &jobs[t];
        j->m = m; j->k = k; j->n = n; j->lda = lda; j->ldb = ldb; j->ldc = ldc;
        j->row0 = m * (uint64_t)t / (uint64_t)nthreads;
        j->row1 = m * (uint64_t)(t + 1) / (uint64_t)nthreads;
        j->A = A; j->B = B; j->C = C; j->alpha = alpha; j->beta = beta;
        if (nthreads > 1) pthread_create(&th[t], NULL, f64_worker, j);
        else f64_worker(j);
    }
    if (nthreads > 1)
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

/* Winograd (std2 formulas, Table 1) over the reals, recursion to `cutoff`,
 * with fresh temporaries per level -- the config-5 CPU restatement used for
 * the float64 cpu_baseline (there is no reference float path). */
static void f64_add(uint64_t r, uint64_t c, double* d, uint64_t ldd, const double* a,
                    uint64_t lda, const double* b, uint64_t ldb, double sb) {
    for (uint64_t i = 0; i < r; ++i)
        for (uint64_t j = 0; j < c; ++j) d[i * ldd + j] = a[i * lda + j] + sb * b[i * ldb + j];
}

void wmo_winograd_f64(uint64_t n, const double* A, uint64_t lda, const double* B,
                      uint64_t ldb, double* C, uint64_t ldc, uint64_t cutoff) {
    if (n <= cutoff || (n & 1)) {
        wmo_classical_f64(n, n, n, A, lda, B, ldb, C, ldc, 1.0, 0.0, 1);
        return;
    }
    const uint64_t h = n / 2;
    const double *A11 = A, *A12 = A + h, *A21 = A + h * lda, *A22 = A + h * lda + h;
    const double *B11 = B, *B12 = B + h, *B21 = B + h * ldb, *B22 = B + h * ldb + h;
    double *C11 = C, *C12 = C + h, *C21 = C + h * ldc, *C22 = C + h * ldc + h;
    double* X = (double*)malloc(h * h * sizeof(double));
    double* Y = (double*)malloc(h * h * sizeof(double));
    f64_add(h, h, X, h, A11, lda, A21, lda, -1.0);            /* S3 */
    f64_add(h, h, Y, h, B22, ldb, B12, ldb, -1.0);            /* T3 */
    wmo_winograd_f64(h, X, h, Y, h, C21, ldc, cutoff);        /* P7 */
    f64_add(h, h, X, h, A21, lda, A22, lda, 1.0);             /* S1 */
    f64_add(h, h, Y, h, B12, ldb, B11, ldb, -1.0);            /* T1 */
    wmo_winograd_f64(h, X, h, Y, h, C22, ldc, cutoff);        /* P5 */
    f64_add(h, h, X, h, X, h, A11, lda, -1.0);                /* S2 */
    f64_add(h, h, Y, h, B22, ldb, Y, h, -1.0);                /* T2 */
    wmo_winograd_f64(h, X, h, Y, h, C12, ldc, cutoff);        /* P6 */
    f64_add(h, h, X, h, A12, lda, X, h, -1.0);                /* S4 */
    wmo_winograd_f64(h, X, h, B22, ldb, C11, ldc, cutoff);    /* P3 */
    wmo_winograd_f64(h, A11, lda, B11, ldb, X, h, cutoff);    /* P1 */
    f64_add(h, h, C12, ldc, X, h, C12, ldc, 1.0);             /* U2 */
    f64_add(h, h, C21, ldc, C12, ldc, C21, ldc, 1.0);         /* U3 */
    f64_add(h, h, C12, ldc, C12, ldc, C22, ldc, 1.0);         /* U4 */
    f64_add(h, h, C22, ldc, C21, ldc, C22, ldc, 1.0);         /* U7 */
    f64_add(h, h, C12, ldc, C12, ldc, C11, ldc, 1.0);         /* U5 */
    f64_add(h, h, Y, h, Y, h, B21, ldb, -1.0);                /* T4 */
    wmo_winograd_f64(h, A22, lda, Y, h, C11, ldc, cutoff);    /* P4 */
    f64_add(h, h, C21, ldc, C21, ldc, C11, ldc, -1.0);        /* U6 */
    wmo_winograd_f64(h, A12, lda, B21, ldb, C11, ldc, cutoff);/* P2 */
    f64_add(h, h, C11, ldc, X, h, C11, ldc, 1.0);             /* U1 */
    free(X);
    free(Y);
}
