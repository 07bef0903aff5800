/*
 * pmf_oracle.c -- CPU restatement of the parmf reference (TEST INFRASTRUCTURE, see pmf_oracle.h).
 * Built by oracle/Makefile into oracle/build/liborc.so with -O2 -ffp-contract=off.
 */
#define _POSIX_C_SOURCE 199309L
#include "pmf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---- std::mt19937 (C++ [rand.eng.mers] parameters), restated for the C oracle ------------- */
typedef struct {
    uint32_t mt[624];
    int idx;
} mt19937;

static void mt_seed(mt19937* g, uint32_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 624; ++i)
        g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
    g->idx = 624;
}

static uint32_t mt_next(mt19937* g) {
    if (g->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            const uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
            g->mt[i] = g->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        g->idx = 0;
    }
    uint32_t y = g->mt[g->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* model.hpp:77-79 unit_open_closed == tests/testutil.hpp:49-51 unit: (gen()+1) / 2^32 in (0,1] */
static double unit_open_closed(mt19937* g) {
    return ((double)mt_next(g) + 1.0) * (1.0 / 4294967296.0);
}

uint32_t orc_mt19937_first(uint32_t seed, int skip) {
    mt19937 g;
    mt_seed(&g, seed);
    for (int i = 0; i < skip; ++i) mt_next(&g);
    return mt_next(&g);
}

#define REAL float
#define SUF _f32
#define SQRT sqrtf
#include "pmf_oracle_impl.inc"
#undef REAL
#undef SUF
#undef SQRT

#define REAL double
#define SUF _f64
#define SQRT sqrt
#include "pmf_oracle_impl.inc"
#undef REAL
#undef SUF
#undef SQRT

/* ---- tests/testutil.hpp generators ---------------------------------------------------------- */

/* open-addressing set of int64 keys (stands in for std::unordered_set in testutil.hpp:113-131;
 * only membership matters, so the draw sequence is identical) */
typedef struct {
    int64_t* keys;
    uint64_t cap;
} keyset;

static void ks_init(keyset* s, uint64_t expected) {
    uint64_t cap = 16;
    while (cap < expected * 2 + 16) cap <<= 1;
    s->cap = cap;
    s->keys = (int64_t*)malloc(sizeof(int64_t) * cap);
    for (uint64_t i = 0; i < cap; ++i) s->keys[i] = -1;
}

/* returns 1 if inserted, 0 if already present */
static int ks_insert(keyset* s, int64_t key) {
    uint64_t h = (uint64_t)key * 0x9E3779B97F4A7C15ull;
    uint64_t i = (h >> 17) & (s->cap - 1);
    for (;;) {
        if (s->keys[i] == key) return 0;
        if (s->keys[i] < 0) {
            s->keys[i] = key;
            return 1;
        }
        i = (i + 1) & (s->cap - 1);
    }
}

static double tu_uniform(mt19937* g, double lo, double hi) {  /* testutil.hpp:53-55 */
    return lo + (hi - lo) * unit_open_closed(g);
}

static double tu_gaussian(mt19937* g) {  /* testutil.hpp:57-60 Box-Muller */
    const double u1 = unit_open_closed(g), u2 = unit_open_closed(g);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static uint32_t tu_bounded(mt19937* g, uint32_t n) { return mt_next(g) % n; }  /* :62-64 */

/* testutil.hpp:68-85 random_triplets */
int64_t orc_random_triplets(int32_t m, int32_t n, int32_t target, uint32_t seed, double lo,
                            double hi, orc_triplet_f64* out) {
    mt19937 g;
    mt_seed(&g, seed);
    keyset s;
    ks_init(&s, (uint64_t)target);
    int64_t count = 0;
    const int64_t cells = (int64_t)m * n;
    while (count < target && count < cells) {
        const int32_t i = (int32_t)tu_bounded(&g, (uint32_t)m);
        const int32_t j = (int32_t)tu_bounded(&g, (uint32_t)n);
        const int64_t key = (int64_t)i * n + j;
        if (!ks_insert(&s, key)) continue;
        out[count].user = i;
        out[count].item = j;
        out[count].rating = tu_uniform(&g, lo, hi);
        ++count;
    }
    free(s.keys);
    return count;
}

/* testutil.hpp:89-106 planted_full */
int64_t orc_planted_full(int32_t m, int32_t n, int k, double scale, uint32_t seed,
                         orc_triplet_f64* out) {
    mt19937 g;
    mt_seed(&g, seed);
    double* w = (double*)malloc(sizeof(double) * (size_t)m * k);
    double* h = (double*)malloc(sizeof(double) * (size_t)n * k);
    for (int64_t x = 0; x < (int64_t)m * k; ++x) w[x] = unit_open_closed(&g) * scale;
    for (int64_t x = 0; x < (int64_t)n * k; ++x) h[x] = unit_open_closed(&g) * scale;
    int64_t c = 0;
    for (int32_t i = 0; i < m; ++i)
        for (int32_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int t = 0; t < k; ++t) s += w[(size_t)i * k + t] * h[(size_t)j * k + t];
            out[c].user = i;
            out[c].item = j;
            out[c].rating = s;
            ++c;
        }
    free(w);
    free(h);
    return c;
}

/* testutil.hpp:111-132 synth_ratings: planted rank + biases + noise, quantised to 1..5,
 * uniform users, Zipf(0.8) items via CDF lower_bound, deduplicated (user,item). */
int64_t orc_synth_ratings(int32_t m, int32_t n, int true_rank, int64_t target_nnz, uint32_t seed,
                          orc_triplet_f64* out) {
    mt19937 g;
    mt_seed(&g, seed);
    const double fscale = 0.45 / sqrt((double)true_rank);
    double* w = (double*)malloc(sizeof(double) * (size_t)m * true_rank);
    double* h = (double*)malloc(sizeof(double) * (size_t)n * true_rank);
    double* bu = (double*)malloc(sizeof(double) * (size_t)m);
    double* bi = (double*)malloc(sizeof(double) * (size_t)n);
    double* cdf = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t x = 0; x < (int64_t)m * true_rank; ++x) w[x] = tu_gaussian(&g) * fscale;
    for (int64_t x = 0; x < (int64_t)n * true_rank; ++x) h[x] = tu_gaussian(&g) * fscale;
    for (int32_t x = 0; x < m; ++x) bu[x] = tu_gaussian(&g) * 0.35;
    for (int32_t x = 0; x < n; ++x) bi[x] = tu_gaussian(&g) * 0.35;
    double acc = 0.0;
    for (int32_t j = 0; j < n; ++j) {
        acc += 1.0 / pow((double)j + 1.0, 0.8);
        cdf[j] = acc;
    }
    for (int32_t j = 0; j < n; ++j) cdf[j] /= acc;
    keyset s;
    ks_init(&s, (uint64_t)target_nnz);
    int64_t count = 0;
    while (count < target_nnz) {
        const int32_t i = (int32_t)tu_bounded(&g, (uint32_t)m);
        const double r = unit_open_closed(&g);
        /* std::lower_bound: first cdf[j] >= r (== n if none) */
        int32_t lo = 0, hi = n;
        while (lo < hi) {
            const int32_t mid = lo + (hi - lo) / 2;
            if (cdf[mid] < r) lo = mid + 1;
            else hi = mid;
        }
        const int32_t j = lo;
        const int64_t key = (int64_t)i * n + j;
        if (!ks_insert(&s, key)) continue;
        double score = 3.6 + bu[i] + bi[j] + tu_gaussian(&g) * 0.35;
        for (int t = 0; t < true_rank; ++t)
            score += w[(size_t)i * true_rank + t] * h[(size_t)j * true_rank + t] /
                     (fscale * fscale) * 0.12;
        score = fmin(5.0, fmax(1.0, round(score)));
        out[count].user = i;
        out[count].item = j;
        out[count].rating = score;
        ++count;
    }
    free(s.keys);
    free(w);
    free(h);
    free(bu);
    free(bi);
    free(cdf);
    return count;
}

/* testutil.hpp:136-144 carve_probe: Fisher-Yates with bounded(), probe = last probe_count
 * entries (caller splits the array: train = [0, count-probe_count), probe = the tail). */
void orc_carve_probe(orc_triplet_f64* train, int64_t count, int64_t probe_count, uint32_t seed) {
    (void)probe_count;
    mt19937 g;
    mt_seed(&g, seed);
    for (uint32_t i = (uint32_t)count; i > 1; --i) {
        const uint32_t r = tu_bounded(&g, i);
        orc_triplet_f64 tmp = train[i - 1];
        train[i - 1] = train[r];
        train[r] = tmp;
    }
}

/* runtime.hpp:91-136 partition_balanced: binary search on the bottleneck, then a greedy sweep.
 * bounds has p+1 entries. */
int orc_partition_balanced(const int64_t* costs, int32_t count, int p, int32_t* bounds) {
    if (p < 1) return ORC_INVALID_ARGUMENT;
    int64_t lo = 0, total = 0;
    for (int32_t i = 0; i < count; ++i) {
        if (costs[i] < 0) return ORC_INVALID_ARGUMENT;
        if (costs[i] > lo) lo = costs[i];
        total += costs[i];
    }
    int64_t hi = total;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        int blocks = 1;
        int64_t cur = 0;
        for (int32_t i = 0; i < count; ++i) {
            if (cur + costs[i] > mid) {
                ++blocks;
                cur = costs[i];
            } else {
                cur += costs[i];
            }
        }
        if (blocks <= p) hi = mid;
        else lo = mid + 1;
    }
    int nb = 0;
    bounds[nb++] = 0;
    int64_t cur = 0;
    for (int32_t i = 0; i < count; ++i) {
        if (cur + costs[i] > lo && nb <= p - 1) {
            bounds[nb++] = i;
            cur = costs[i];
        } else {
            cur += costs[i];
        }
    }
    while (nb < p + 1) bounds[nb++] = count;
    return ORC_OK;
}
