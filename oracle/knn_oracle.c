/*
 * knn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's brute-force kNN hot path, used as
 * the parity checker for the CUDA engine.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library.  The product path
 * (paper_0804_1448_b200/) never links or calls it.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libknnref.so, compiled from
 * /root/reference/proj/src by oracle/Makefile) and against the golden fixtures
 * in tests/golden/ that were generated from that build (oracle/gen_golden.py).
 *
 * Reference anchors (paths relative to /root/reference/proj):
 *   - seeds / RNG ............ include/knn/rng.hpp:9-38, src/bench.cpp:39-46
 *   - per-pair keys .......... include/knn/metric.hpp:22-44 (sequential, no FMA:
 *                              CMakeLists.txt:16 -ffp-contract=off)
 *   - Mahalanobis ............ src/metric.cpp:20-82 (Cholesky M = L L^T, y = L^T x)
 *   - top-k tie rule ......... src/topk.cpp:11-33 ((key, index) lexicographic)
 *   - bf_knn ................. src/bruteforce.cpp:42-100 (validate, keys, select,
 *                              sqrt for the squared kinds)
 *
 * Compile with -ffp-contract=off so the double accumulations round exactly as
 * the reference's do.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { KO_EUCLIDEAN = 0, KO_MANHATTAN = 1, KO_CHEBYSHEV = 2, KO_MAHALANOBIS = 3 };
enum { KO_OK = 0, KO_EINVAL = 1, KO_ENOMEM = 2 };

/* ---------------------------------------------------------------- RNG ---- */

/* splitmix64 step (rng.hpp:9-14). */
static uint64_t ko_splitmix_step(uint64_t *state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* derive_seed(master, a, b, c) (rng.hpp:17-28). */
uint64_t ko_derive_seed(uint64_t master, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t st = master;
    uint64_t acc = ko_splitmix_step(&st);
    st ^= a * 0x9e3779b97f4a7c15ULL;
    acc ^= ko_splitmix_step(&st);
    st ^= b * 0xbf58476d1ce4e5b9ULL;
    acc ^= ko_splitmix_step(&st);
    st ^= c * 0x94d049bb133111ebULL;
    acc ^= ko_splitmix_step(&st);
    return acc;
}

/* MT19937-64 (the engine std::mt19937_64 pins down; rng.hpp:30-38 relies on it). */
typedef struct {
    uint64_t s[312];
    int pos;
} ko_mt64;

static void ko_mt64_seed(ko_mt64 *g, uint64_t seed) {
    g->s[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->s[i] = 6364136223846793005ULL * (g->s[i - 1] ^ (g->s[i - 1] >> 62)) + (uint64_t)i;
    g->pos = 312;
}

static void ko_mt64_twist(ko_mt64 *g) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
        uint64_t y = (g->s[i] & upper) | (g->s[(i + 1) % 312] & lower);
        uint64_t v = g->s[(i + 156) % 312] ^ (y >> 1);
        if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
        g->s[i] = v;
    }
    g->pos = 0;
}

static uint64_t ko_mt64_next(ko_mt64 *g) {
    if (g->pos >= 312) ko_mt64_twist(g);
    uint64_t x = g->s[g->pos++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* Raw mt19937_64 draws (for pinning the engine against the reference). */
void ko_mt64_draws(uint64_t seed, uint64_t *out, size_t count) {
    ko_mt64 g;
    ko_mt64_seed(&g, seed);
    for (size_t i = 0; i < count; ++i) out[i] = ko_mt64_next(&g);
}

/* generate_uniform (bench.cpp:39-46): doubles (bits >> 11) * 2^-53. */
void ko_fill_uniform_f64(double *out, size_t count, uint64_t seed) {
    ko_mt64 g;
    ko_mt64_seed(&g, seed);
    for (size_t i = 0; i < count; ++i) out[i] = (double)(ko_mt64_next(&g) >> 11) * 0x1.0p-53;
}

/* FP32 variant used by the GPU benchmark: (bits >> 40) * 2^-24 is exactly
 * representable in float and never rounds up to 1.0f. */
void ko_fill_uniform_f32(float *out, size_t count, uint64_t seed) {
    ko_mt64 g;
    ko_mt64_seed(&g, seed);
    for (size_t i = 0; i < count; ++i) out[i] = (float)(ko_mt64_next(&g) >> 40) * 0x1.0p-24f;
}

/* Counter-based FP32 uniform for very large sets (config E): element i of a
 * stream is splitmix64(seed + i) >> 40 scaled by 2^-24.  Reproducible at any
 * offset, so a host can regenerate any subsample of a device-generated set. */
void ko_fill_counter_f32(float *out, size_t begin, size_t count, uint64_t seed) {
    for (size_t i = 0; i < count; ++i) {
        uint64_t st = seed + (uint64_t)(begin + i);
        out[i] = (float)(ko_splitmix_step(&st) >> 40) * 0x1.0p-24f;
    }
}

/* ---------------------------------------------------------- metrics ---- */

/* metric.hpp:22-29: squared L2, coordinates accumulated in order. */
static double ko_key_l2(const double *a, const double *b, size_t d) {
    double acc = 0.0;
    for (size_t c = 0; c < d; ++c) {
        double t = a[c] - b[c];
        acc += t * t;
    }
    return acc;
}

/* metric.hpp:31-35 */
static double ko_key_l1(const double *a, const double *b, size_t d) {
    double acc = 0.0;
    for (size_t c = 0; c < d; ++c) acc += fabs(a[c] - b[c]);
    return acc;
}

/* metric.hpp:37-44 */
static double ko_key_linf(const double *a, const double *b, size_t d) {
    double acc = 0.0;
    for (size_t c = 0; c < d; ++c) {
        double t = fabs(a[c] - b[c]);
        if (t > acc) acc = t;
    }
    return acc;
}

double ko_key(const double *a, const double *b, size_t d, int metric) {
    switch (metric) {
        case KO_MANHATTAN: return ko_key_l1(a, b, d);
        case KO_CHEBYSHEV: return ko_key_linf(a, b, d);
        default: return ko_key_l2(a, b, d);
    }
}

/* Cholesky factor of a symmetric positive-definite d x d matrix
 * (metric.cpp:20-61): returns KO_EINVAL for asymmetry beyond 1e-12 relative or
 * a non-positive pivot; L is lower-triangular row-major. */
int ko_cholesky(const double *M, size_t d, double *L) {
    for (size_t i = 0; i < d; ++i)
        for (size_t j = i + 1; j < d; ++j) {
            double x = M[i * d + j], y = M[j * d + i];
            double scale = fabs(x) > fabs(y) ? fabs(x) : fabs(y);
            if (fabs(x - y) > 1e-12 * scale) return KO_EINVAL;
        }
    memset(L, 0, d * d * sizeof(double));
    for (size_t i = 0; i < d; ++i) {
        for (size_t j = 0; j <= i; ++j) {
            double s = M[i * d + j];
            for (size_t c = 0; c < j; ++c) s -= L[i * d + c] * L[j * d + c];
            if (i == j) {
                if (!(s > 0.0)) return KO_EINVAL;
                L[i * d + i] = sqrt(s);
            } else {
                L[i * d + j] = s / L[j * d + j];
            }
        }
    }
    return KO_OK;
}

/* y = L^T x per row (metric.cpp:63-82). */
void ko_whiten(const double *L, size_t d, const double *in, size_t n, double *out) {
    for (size_t p = 0; p < n; ++p) {
        const double *x = in + p * d;
        double *y = out + p * d;
        for (size_t r = 0; r < d; ++r) {
            double acc = 0.0;
            for (size_t c = r; c < d; ++c) acc += L[c * d + r] * x[c];
            y[r] = acc;
        }
    }
}

/* --------------------------------------------------------- selection ---- */

typedef struct {
    double key;
    int64_t idx;
} ko_pair;

/* (key, index) lexicographic order, topk.cpp:11-13. */
static int ko_less(const ko_pair *a, const ko_pair *b) {
    return a->key < b->key || (a->key == b->key && a->idx < b->idx);
}

/* Bounded max-heap of the k best pairs: the root is the worst kept pair. */
static void ko_sift_down(ko_pair *h, size_t len, size_t at) {
    for (;;) {
        size_t l = 2 * at + 1, r = l + 1, big = at;
        if (l < len && ko_less(&h[big], &h[l])) big = l;
        if (r < len && ko_less(&h[big], &h[r])) big = r;
        if (big == at) return;
        ko_pair t = h[at];
        h[at] = h[big];
        h[big] = t;
        at = big;
    }
}

static void ko_sift_up(ko_pair *h, size_t at) {
    while (at > 0) {
        size_t p = (at - 1) / 2;
        if (!ko_less(&h[p], &h[at])) return;
        ko_pair t = h[p];
        h[p] = h[at];
        h[at] = t;
        at = p;
    }
}

/* The k smallest of keys[0..m) under the (key, index) order, ascending.
 * Same result as nth_element + sort in topk.cpp:17-33. */
void ko_select_k(const double *keys, size_t m, size_t k, ko_pair *out) {
    size_t len = 0;
    for (size_t j = 0; j < m; ++j) {
        ko_pair c = {keys[j], (int64_t)j};
        if (len < k) {
            out[len] = c;
            ko_sift_up(out, len);
            ++len;
        } else if (ko_less(&c, &out[0])) {
            out[0] = c;
            ko_sift_down(out, len, 0);
        }
    }
    /* heap-sort in place: repeatedly move the max to the end */
    for (size_t end = len; end > 1; --end) {
        ko_pair t = out[0];
        out[0] = out[end - 1];
        out[end - 1] = t;
        ko_sift_down(out, end - 1, 0);
    }
}

/* ------------------------------------------------------------ search ---- */

/* bf_knn (bruteforce.cpp:42-100) for row-major double inputs.  `mahal` is the
 * d x d inverse covariance when metric == KO_MAHALANOBIS, else ignored.
 * Outputs are n x k row-major: index and finalized distance (sqrt for the
 * squared kinds, bruteforce.cpp:67-69,89-93).  threads <= 0 uses all cores. */
int ko_knn(const double *Q, size_t n, const double *R, size_t m, size_t d, size_t k,
           int metric, const double *mahal, int threads, int64_t *out_idx, double *out_dist) {
    if (n == 0 || m == 0 || d == 0) return KO_EINVAL;
    if (k == 0 || k > m) return KO_EINVAL;
    const double *q = Q, *r = R;
    double *wq = NULL, *wr = NULL, *L = NULL;
    if (metric == KO_MAHALANOBIS) {
        L = (double *)malloc(d * d * sizeof(double));
        wq = (double *)malloc(n * d * sizeof(double));
        wr = (double *)malloc(m * d * sizeof(double));
        if (!L || !wq || !wr) { free(L); free(wq); free(wr); return KO_ENOMEM; }
        if (ko_cholesky(mahal, d, L) != KO_OK) { free(L); free(wq); free(wr); return KO_EINVAL; }
        ko_whiten(L, d, Q, n, wq);
        ko_whiten(L, d, R, m, wr);
        q = wq;
        r = wr;
    }
    const int kind = metric == KO_MAHALANOBIS ? KO_EUCLIDEAN : metric;
    const int root = kind == KO_EUCLIDEAN;
    int status = KO_OK;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        double *row = (double *)malloc(m * sizeof(double));
        ko_pair *best = (ko_pair *)malloc(k * sizeof(ko_pair));
        if (!row || !best) {
            status = KO_ENOMEM;
        } else {
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
            for (int64_t i = 0; i < (int64_t)n; ++i) {
                const double *qi = q + (size_t)i * d;
                for (size_t j = 0; j < m; ++j) row[j] = ko_key(qi, r + j * d, d, kind);
                ko_select_k(row, m, k, best);
                for (size_t t = 0; t < k; ++t) {
                    out_idx[(size_t)i * k + t] = best[t].idx;
                    out_dist[(size_t)i * k + t] = root ? sqrt(best[t].key) : best[t].key;
                }
            }
        }
        free(row);
        free(best);
    }
    free(L);
    free(wq);
    free(wr);
    return status;
}

/* Convenience for FP32 inputs: widen exactly to double, then ko_knn. */
int ko_knn_f32(const float *Q, size_t n, const float *R, size_t m, size_t d, size_t k,
               int metric, const double *mahal, int threads, int64_t *out_idx, double *out_dist) {
    double *q = (double *)malloc(n * d * sizeof(double));
    double *r = (double *)malloc(m * d * sizeof(double));
    if (!q || !r) { free(q); free(r); return KO_ENOMEM; }
    for (size_t i = 0; i < n * d; ++i) q[i] = (double)Q[i];
    for (size_t i = 0; i < m * d; ++i) r[i] = (double)R[i];
    int s = ko_knn(q, n, r, m, d, k, metric, mahal, threads, out_idx, out_dist);
    free(q);
    free(r);
    return s;
}

/* Exact double key of one (query, reference) pair, finalized like bf_knn
 * reports it: used by the tolerance comparator to recompute the distance of
 * a returned index. */
double ko_pair_distance_f32(const float *a, const float *b, size_t d, int metric) {
    double x[4096], y[4096];
    double *xa = d <= 4096 ? x : (double *)malloc(d * sizeof(double));
    double *ya = d <= 4096 ? y : (double *)malloc(d * sizeof(double));
    for (size_t c = 0; c < d; ++c) { xa[c] = a[c]; ya[c] = b[c]; }
    double key = ko_key(xa, ya, d, metric);
    if (xa != x) free(xa);
    if (ya != y) free(ya);
    return metric == KO_EUCLIDEAN ? sqrt(key) : key;
}

int ko_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
