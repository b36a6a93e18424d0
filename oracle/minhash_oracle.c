/*
 * minhash_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).
 *
 * CPU restatement of the reference's compiled hot loops, applied to every row of a
 * CSR batch.  Nothing in the product path links or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs do.
 *
 * oracle_sign_iterative_csr  restates kernels.sign_iterative
 *     /root/reference/pkg/src/minhashlab/kernels.py:44-73
 *     (feature-outer / hash-inner; h starts at (a*x) % p and advances by
 *      dh = (x+b) % p with a conditional subtract; strict '<' keeps the first
 *      (smallest, for ascending ids) feature on ties; first feature seeds best/arg)
 * oracle_sign_random_csr     restates kernels.sign_random
 *     /root/reference/pkg/src/minhashlab/kernels.py:21-41
 *     (hash-outer / feature-inner; (a_i*x + b_i) % p per visit; strict '<')
 *
 * Arithmetic is int64 exactly as numba runs it (kernels.py:18; exact for
 * p <= MAX_VECTOR_PRIME, modmath.py:19).  Beyond MAX_VECTOR_PRIME the reference
 * switches to _signature_by_rows (minhash.py:102-127: exact Python-int eval_all per
 * feature, ascending ids, strict '<'); here the same loops run with 128-bit
 * products, which is that exact fallback.  Rows are independent, so rows are spread
 * over OpenMP threads (the reference allows concurrency across documents,
 * SPEC.md:224); each row's loop order is the reference's.
 */
#include <stdint.h>
#include <stdlib.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define MAX_VECTOR_PRIME 3037000499LL /* modmath.py:19 */

/* (w * x + c) mod p, exact for any w, c < p < 2^63 and x < 2^32 */
static inline int64_t mulmod_exact(int64_t w, int64_t x, int64_t c, int64_t p) {
    return (int64_t)(((unsigned __int128)(uint64_t)w * (uint64_t)x + (uint64_t)c) % (uint64_t)p);
}

/* p > MAX_VECTOR_PRIME: _signature_by_rows, minhash.py:113-127 (eval_all per feature,
 * families.py:153-168: h_i(x) = (a x + i ((x + b) mod p)) mod p; strict '<') */
static void sign_iterative_row_exact(const uint32_t* ids, int64_t m, int64_t a, int64_t b, int64_t p, int32_t n,
                                     int64_t* best, int64_t* arg) {
    for (int64_t j = 0; j < m; ++j) {
        const int64_t x = (int64_t)ids[j];
        const int64_t ax = mulmod_exact(a, x, 0, p);
        const int64_t dh = (int64_t)(((uint64_t)x + (uint64_t)b) % (uint64_t)p);
        int64_t h = ax;
        for (int32_t i = 0; i < n; ++i) {
            if (j == 0 || h < best[i]) {
                best[i] = h;
                arg[i] = x;
            }
            h = (int64_t)(((uint64_t)h + (uint64_t)dh) % (uint64_t)p);
        }
    }
}

static void sign_random_row_exact(const uint32_t* ids, int64_t m, const int64_t* a, const int64_t* b, int64_t p,
                                  int32_t n, int64_t* out) {
    for (int32_t i = 0; i < n; ++i) {
        int64_t best = 0, arg = 0;
        for (int64_t j = 0; j < m; ++j) {
            const int64_t hv = mulmod_exact(a[i], (int64_t)ids[j], b[i], p);
            if (j == 0 || hv < best) {
                best = hv;
                arg = (int64_t)ids[j];
            }
        }
        out[i] = arg;
    }
}

static void sign_iterative_row(const uint32_t* ids, int64_t m, int64_t a, int64_t b, int64_t p, int32_t n,
                               int64_t* best, int64_t* arg) {
    if (p > MAX_VECTOR_PRIME) {
        sign_iterative_row_exact(ids, m, a, b, p, n, best, arg);
        return;
    }
    /* kernels.py:53-61: the first feature seeds every (best, arg) */
    int64_t x = (int64_t)ids[0];
    int64_t dh = (x + b) % p;
    int64_t h = (a * x) % p;
    for (int32_t i = 0; i < n; ++i) {
        best[i] = h;
        arg[i] = x;
        h += dh;
        if (h >= p) h -= p;
    }
    /* kernels.py:62-72: remaining features, add/compare only */
    for (int64_t j = 1; j < m; ++j) {
        x = (int64_t)ids[j];
        dh = (x + b) % p;
        h = (a * x) % p;
        for (int32_t i = 0; i < n; ++i) {
            if (h < best[i]) {
                best[i] = h;
                arg[i] = x;
            }
            h += dh;
            if (h >= p) h -= p;
        }
    }
}

static void sign_random_row(const uint32_t* ids, int64_t m, const int64_t* a, const int64_t* b, int64_t p,
                            int32_t n, int64_t* out) {
    if (p > MAX_VECTOR_PRIME) {
        sign_random_row_exact(ids, m, a, b, p, n, out);
        return;
    }
    /* kernels.py:28-41 */
    for (int32_t i = 0; i < n; ++i) {
        const int64_t ai = a[i], bi = b[i];
        int64_t best = (ai * (int64_t)ids[0] + bi) % p;
        int64_t arg = (int64_t)ids[0];
        for (int64_t j = 1; j < m; ++j) {
            const int64_t hv = (ai * (int64_t)ids[j] + bi) % p;
            if (hv < best) {
                best = hv;
                arg = (int64_t)ids[j];
            }
        }
        out[i] = arg;
    }
}

/* out: int64[n_sets * n]; rows with no features are left untouched (the reference
 * raises before calling its kernel, minhash.py:97-98).  threads <= 0: OpenMP default. */
void oracle_sign_iterative_csr(const int64_t* indptr, const uint32_t* ids, int64_t n_sets, int64_t a,
                               int64_t b, int64_t p, int32_t n, int64_t* out, int32_t threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        int64_t* best = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
        for (int64_t s = 0; s < n_sets; ++s) {
            const int64_t lo = indptr[s], m = indptr[s + 1] - indptr[s];
            if (m <= 0) continue;
            sign_iterative_row(ids + lo, m, a, b, p, n, best, out + s * (int64_t)n);
        }
        free(best);
    }
}

void oracle_sign_random_csr(const int64_t* indptr, const uint32_t* ids, int64_t n_sets, const int64_t* a,
                            const int64_t* b, int64_t p, int32_t n, int64_t* out, int32_t threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int64_t s = 0; s < n_sets; ++s) {
        const int64_t lo = indptr[s], m = indptr[s + 1] - indptr[s];
        if (m <= 0) continue;
        sign_random_row(ids + lo, m, a, b, p, n, out + s * (int64_t)n);
    }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
