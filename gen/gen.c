/*
 * gen.c -- seeded synthetic input generators shared by the oracle and the CUDA path.
 *
 * This module holds NONE of the method's arithmetic (no partitioning, no
 * aggregation, no correction).  It only turns a root seed into graphs,
 * features, labels, train masks and initial weights, following the canonical
 * definitions written down in DESIGN.md §3 ("input recipe"):
 *
 *   mix(x)        splitmix64 finalizer (with the golden-gamma pre-add)
 *   h(a,b,...)    mix(a ^ mix(b ^ ...)), innermost argument hashed first
 *   scramble      4-round balanced Feistel bijection on [0,N) with cycle walking
 *   RMAT sample i level l:  r = h(h(seed_graph, i, attempt), l) >> 11, quadrant by
 *                 comparing r against a, a+b, a+b+c scaled by 2^53; reject ids >= N
 *   SBM pair u<v: edge iff h(seed_graph, u, v) < p * 2^64
 *
 * Graph construction: drop self loops, symmetrise, deduplicate, scramble ids,
 * sort every adjacency list ascending -> CSR (rowptr int64[N+1], col int32[nnz]).
 * Every result is independent of the OpenMP thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t h2(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b)); }
static inline uint64_t h3(uint64_t a, uint64_t b, uint64_t c) { return mix64(a ^ mix64(b ^ mix64(c))); }

uint64_t gen_mix(uint64_t x) { return mix64(x); }
uint64_t gen_h2(uint64_t a, uint64_t b) { return h2(a, b); }
uint64_t gen_h3(uint64_t a, uint64_t b, uint64_t c) { return h3(a, b, c); }

/* ---------------- Feistel bijection (id scrambling only) ---------------- */
typedef struct { uint64_t seed; int half; uint64_t mask; int64_t n; } feistel_t;

static feistel_t feistel_make(int64_t n, uint64_t seed) {
    int lg = 0;
    while (((int64_t)1 << lg) < n) lg++;
    int bits = 2 * ((lg + 1) / 2);
    if (bits < 2) bits = 2;
    feistel_t f; f.seed = seed; f.half = bits / 2; f.mask = (1ULL << f.half) - 1; f.n = n;
    return f;
}
static inline uint64_t feistel_once(const feistel_t* f, uint64_t x) {
    uint64_t L = x >> f->half, R = x & f->mask;
    for (uint64_t r = 0; r < 4; r++) {
        uint64_t nl = R;
        uint64_t nr = L ^ (h3(f->seed, r, R) & f->mask);
        L = nl; R = nr;
    }
    return (L << f->half) | R;
}
static inline int64_t feistel_apply(const feistel_t* f, int64_t v) {
    uint64_t y = feistel_once(f, (uint64_t)v);
    while (y >= (uint64_t)f->n) y = feistel_once(f, y);
    return (int64_t)y;
}

void gen_scramble(int64_t n, uint64_t seed, const int64_t* in, int64_t* out, int64_t count) {
    feistel_t f = feistel_make(n, seed);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; i++) out[i] = feistel_apply(&f, in[i]);
}

/* ---------------- edge list -> CSR ---------------- */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}
static void sort_i32(int32_t* a, int64_t n) {
    if (n < 24) {
        for (int64_t i = 1; i < n; i++) {
            int32_t v = a[i]; int64_t j = i - 1;
            while (j >= 0 && a[j] > v) { a[j + 1] = a[j]; j--; }
            a[j + 1] = v;
        }
    } else {
        qsort(a, (size_t)n, sizeof(int32_t), cmp_i32);
    }
}

/* Build a symmetric, deduplicated, self-loop-free CSR from undirected pairs (src[i], dst[i]).
 * Pairs with src<0 are ignored.  Returns nnz; rowptr must hold n+1 entries; *col_out is
 * malloc'ed and owned by the caller (free with gen_free). */
static int64_t build_csr(int64_t n, const int32_t* src, const int32_t* dst, int64_t m,
                         int64_t* rowptr, int32_t** col_out) {
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        int32_t u = src[i], v = dst[i];
        if (u < 0 || u == v) continue;
        #pragma omp atomic
        cnt[u]++;
        #pragma omp atomic
        cnt[v]++;
    }
    int64_t* off = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
    off[0] = 0;
    for (int64_t v = 0; v < n; v++) off[v + 1] = off[v] + cnt[v];
    int64_t tot = off[n];
    int32_t* tmp = (int32_t*)malloc((size_t)(tot > 0 ? tot : 1) * sizeof(int32_t));
    int64_t* pos = cnt;  /* reuse as fill cursor */
    memcpy(pos, off, (size_t)n * sizeof(int64_t));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        int32_t u = src[i], v = dst[i];
        if (u < 0 || u == v) continue;
        int64_t p, q;
        #pragma omp atomic capture
        p = pos[u]++;
        #pragma omp atomic capture
        q = pos[v]++;
        tmp[p] = v; tmp[q] = u;
    }
    /* sort + dedup each row in place; record unique length */
    int64_t* ulen = pos;
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; v++) {
        int32_t* a = tmp + off[v];
        int64_t len = off[v + 1] - off[v];
        sort_i32(a, len);
        int64_t k = 0;
        for (int64_t j = 0; j < len; j++)
            if (k == 0 || a[j] != a[k - 1]) a[k++] = a[j];
        ulen[v] = k;
    }
    rowptr[0] = 0;
    for (int64_t v = 0; v < n; v++) rowptr[v + 1] = rowptr[v] + ulen[v];
    int64_t nnz = rowptr[n];
    int32_t* col = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
    #pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; v++)
        memcpy(col + rowptr[v], tmp + off[v], (size_t)ulen[v] * sizeof(int32_t));
    free(tmp); free(off); free(cnt);
    *col_out = col;
    return nnz;
}

void gen_free(void* p) { free(p); }

/* ---------------- RMAT ---------------- */
/* Graph500-style RMAT: `num_samples` undirected samples on 2^scale ids, ids >= n rejected
 * (the attempt counter advances), then ids scrambled by the Feistel bijection seeded with
 * seed_perm.  Returns nnz (directed CSR entries); *col_out malloc'ed. */
int64_t gen_rmat(int scale, int64_t n, int64_t num_samples, double a, double b, double c,
                 uint64_t seed_graph, uint64_t seed_perm, int64_t* rowptr, int32_t** col_out) {
    const uint64_t t1 = (uint64_t)(a * 9007199254740992.0);
    const uint64_t t2 = (uint64_t)((a + b) * 9007199254740992.0);
    const uint64_t t3 = (uint64_t)((a + b + c) * 9007199254740992.0);
    uint64_t lvl[64];
    for (int l = 0; l < 64; l++) lvl[l] = mix64((uint64_t)l);
    int32_t* src = (int32_t*)malloc((size_t)num_samples * sizeof(int32_t));
    int32_t* dst = (int32_t*)malloc((size_t)num_samples * sizeof(int32_t));
    feistel_t f = feistel_make(n, seed_perm);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < num_samples; i++) {
        for (uint64_t att = 0;; att++) {
            uint64_t key = h3(seed_graph, (uint64_t)i, att);
            uint64_t u = 0, v = 0;
            for (int l = 0; l < scale; l++) {
                uint64_t r = mix64(key ^ lvl[l]) >> 11;
                uint64_t bu = (r >= t2);                 /* quadrants c,d: row bit 1 */
                uint64_t bv = (r >= t1 && r < t2) || (r >= t3); /* quadrants b,d: col bit 1 */
                u = (u << 1) | bu; v = (v << 1) | bv;
            }
            if (u < (uint64_t)n && v < (uint64_t)n) {
                src[i] = (int32_t)feistel_apply(&f, (int64_t)u);
                dst[i] = (int32_t)feistel_apply(&f, (int64_t)v);
                break;
            }
        }
    }
    int64_t nnz = build_csr(n, src, dst, num_samples, rowptr, col_out);
    free(src); free(dst);
    return nnz;
}

/* ---------------- SBM ---------------- */
/* Stochastic block model: community(v) given; pair u<v is an edge iff
 * h(seed_graph,u,v) < p*2^64, p = p_in for same community else p_out. */
int64_t gen_sbm(int64_t n, const int32_t* community, double p_in, double p_out,
                uint64_t seed_graph, int64_t* rowptr, int32_t** col_out) {
    const uint64_t tin = (p_in >= 1.0) ? UINT64_MAX : (uint64_t)(p_in * 18446744073709551616.0);
    const uint64_t tout = (p_out >= 1.0) ? UINT64_MAX : (uint64_t)(p_out * 18446744073709551616.0);
    /* count per u, then fill (two passes keep it deterministic) */
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t u = 0; u < n; u++) {
        int64_t k = 0;
        for (int64_t v = u + 1; v < n; v++) {
            uint64_t t = community[u] == community[v] ? tin : tout;
            uint64_t x = h3(seed_graph, (uint64_t)u, (uint64_t)v);
            if (x < t || t == UINT64_MAX) k++;
        }
        cnt[u] = k;
    }
    int64_t* off = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
    off[0] = 0;
    for (int64_t u = 0; u < n; u++) off[u + 1] = off[u] + cnt[u];
    int64_t m = off[n];
    int32_t* src = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    int32_t* dst = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t u = 0; u < n; u++) {
        int64_t k = off[u];
        for (int64_t v = u + 1; v < n; v++) {
            uint64_t t = community[u] == community[v] ? tin : tout;
            uint64_t x = h3(seed_graph, (uint64_t)u, (uint64_t)v);
            if (x < t || t == UINT64_MAX) { src[k] = (int32_t)u; dst[k] = (int32_t)v; k++; }
        }
    }
    int64_t nnz = build_csr(n, src, dst, m, rowptr, col_out);
    free(src); free(dst); free(cnt); free(off);
    return nnz;
}

/* ---------------- node data ---------------- */
/* x[v][f] = ((int32)(h(seed,v,f) >> 40) - 2^23) * 2^-23 for f < F, 0 for F <= f < F_pad.
 * Exact in fp32.  Optional signal: +signal on dim (community[v] mod F). */
void gen_features(int64_t n, int32_t F, int32_t F_pad, uint64_t seed, const int32_t* community,
                  float signal, float* x) {
    #pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; v++) {
        float* row = x + v * (int64_t)F_pad;
        for (int32_t f = 0; f < F; f++) {
            int32_t q = (int32_t)(h3(seed, (uint64_t)v, (uint64_t)f) >> 40) - (1 << 23);
            row[f] = (float)q * (1.0f / 8388608.0f);
        }
        for (int32_t f = F; f < F_pad; f++) row[f] = 0.0f;
        if (community) row[community[v] % F] += signal;
    }
}

/* label(v) = h(seed, v) mod K */
void gen_labels(int64_t n, int32_t K, uint64_t seed, int32_t* y) {
    #pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; v++) y[v] = (int32_t)(h2(seed, (uint64_t)v) % (uint64_t)K);
}

/* train(v) <=> h(seed, v) < threshold (threshold = frac * 2^64, computed by the caller) */
void gen_train_mask(int64_t n, uint64_t seed, uint64_t threshold, uint8_t* mask) {
    #pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; v++) mask[v] = h2(seed, (uint64_t)v) < threshold ? 1 : 0;
}

/* Glorot-uniform [fan_in x fan_out] logical block written into a [rows_pad x cols_pad]
 * row-major fp32 buffer (padding = 0).  w = (2u-1)*sqrt(6/(fan_in+fan_out)),
 * u = (h(h(seed, layer, mat), i*fan_out+j) >> 11) * 2^-53, computed in f64, rounded once. */
void gen_glorot(int32_t fan_in, int32_t fan_out, int32_t rows_pad, int32_t cols_pad,
                uint64_t seed, uint64_t layer, uint64_t mat, float* w) {
    double lim = sqrt(6.0 / (double)(fan_in + fan_out));
    uint64_t key = h3(seed, layer, mat);
    for (int32_t i = 0; i < rows_pad; i++)
        for (int32_t j = 0; j < cols_pad; j++) {
            float val = 0.0f;
            if (i < fan_in && j < fan_out) {
                uint64_t r = h2(key, (uint64_t)i * (uint64_t)fan_out + (uint64_t)j) >> 11;
                double u = (double)r * (1.0 / 9007199254740992.0);
                val = (float)((2.0 * u - 1.0) * lim);
            }
            w[(int64_t)i * cols_pad + j] = val;
        }
}

int gen_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
