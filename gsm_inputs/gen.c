/*
 * gsm_inputs/gen.c — seeded, deterministic synthetic INPUT generators.
 *
 * This module is shared by both sides of the parity check (the CPU oracle under
 * oracle/ and the CUDA path under paper_2003_01527_b200/).  It holds NONE of the
 * matching method's arithmetic: it only draws graphs and labels.
 *
 * Every random number is a pure function of (seed, stream, index) through a
 * splitmix64 cascade, and every probability is compared as a 32-bit integer
 * threshold, so the output is bit-identical regardless of thread count,
 * machine, or caller.
 *
 * Workloads (BASELINE.json configs):
 *   - R-MAT (Graph500 a,b,c,d = .57,.19,.19,.05) with a random vertex permutation;
 *   - Erdos-Renyi G(n, m), m edges uniformly without replacement;
 *   - road-like W x H lattice: 4-neighbour edges plus, per cell, no diagonal,
 *     one random-orientation diagonal, or both;
 *   - uniform node labels in [0, L).
 * All edge lists go through gen_csr_build: symmetrise, drop self-loops,
 * dedup, sort each neighbour list ascending (SPEC CsrGraph invariants).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define STREAM_RMAT 0x524d4154ULL  /* "RMAT" */
#define STREAM_PERM 0x5045524dULL  /* "PERM" */
#define STREAM_GRID 0x47524944ULL  /* "GRID" */
#define STREAM_ER 0x45524552ULL    /* "ERER" */
#define STREAM_LABEL 0x4c41424cULL /* "LABL" */

static inline uint64_t sm64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

/* counter-based draw: a pure function of (seed, stream, index) */
uint64_t gen_draw(uint64_t seed, uint64_t stream, uint64_t idx) {
    return sm64(sm64(sm64(seed) ^ stream) ^ idx);
}

int gen_num_threads(void) { return omp_get_max_threads(); }

/* ---------------------------------------------------------------- R-MAT */
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return (x > y) - (x < y);
}

/* Samples num_samples directed R-MAT edges on 2^scale vertices.  Quadrant
 * thresholds are 32-bit integers: t_a = a*2^32, t_ab = (a+b)*2^32,
 * t_abc = (a+b+c)*2^32.  After sampling, vertex ids are relabelled by a random
 * permutation (rank of draw(seed, PERM, v), ties by v).  Returns 0 on success. */
int gen_rmat_edges(int scale, int64_t num_samples, uint64_t seed, uint32_t t_a, uint32_t t_ab,
                   uint32_t t_abc, int32_t* src, int32_t* dst) {
    if (scale < 1 || scale > 30) return 1;
    const int64_t n = (int64_t)1 << scale;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < num_samples; ++e) {
        uint32_t u = 0, v = 0;
        for (int l = 0; l < scale; ++l) {
            uint32_t x = (uint32_t)(gen_draw(seed, STREAM_RMAT, (uint64_t)e * 64u + (uint64_t)l) >> 32);
            uint32_t bu, bv;
            if (x < t_a) { bu = 0; bv = 0; }
            else if (x < t_ab) { bu = 0; bv = 1; }
            else if (x < t_abc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        src[e] = (int32_t)u;
        dst[e] = (int32_t)v;
    }
    /* random permutation: key = high bits of draw | v  (unique keys) */
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
    int32_t* newid = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    if (!keys || !newid) { free(keys); free(newid); return 2; }
    const uint64_t lowmask = (uint64_t)n - 1;
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v)
        keys[v] = (gen_draw(seed, STREAM_PERM, (uint64_t)v) & ~lowmask) | (uint64_t)v;
    qsort(keys, (size_t)n, sizeof(uint64_t), cmp_u64);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) newid[keys[p] & lowmask] = (int32_t)p;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < num_samples; ++e) {
        src[e] = newid[src[e]];
        dst[e] = newid[dst[e]];
    }
    free(keys);
    free(newid);
    return 0;
}

/* ---------------------------------------------------------------- grid */
/* Road-like lattice.  Vertex id = y*W + x.  Writes at most
 * 2*W*H + 2*(W-1)*(H-1) edges; returns the number written (or -1).
 * Per cell (x,y), x<W-1, y<H-1: r = draw(seed, GRID, cell) >> 32;
 *   r <  t_none          -> no diagonal
 *   r <  t_none_one      -> one diagonal, orientation by bit 0 of the full draw
 *   otherwise            -> both diagonals.
 * If d1_out/d2_out are non-NULL they receive #cells with one / both diagonals. */
int64_t gen_grid_edges(int64_t W, int64_t H, uint64_t seed, uint32_t t_none, uint32_t t_none_one,
                       int32_t* src, int32_t* dst, int64_t* d1_out, int64_t* d2_out) {
    if (W < 1 || H < 1 || W * H > 0x7fffffffLL) return -1;
    int64_t m = 0, d1 = 0, d2 = 0;
    for (int64_t y = 0; y < H; ++y)
        for (int64_t x = 0; x < W; ++x) {
            int64_t id = y * W + x;
            if (x + 1 < W) { src[m] = (int32_t)id; dst[m] = (int32_t)(id + 1); ++m; }
            if (y + 1 < H) { src[m] = (int32_t)id; dst[m] = (int32_t)(id + W); ++m; }
            if (x + 1 < W && y + 1 < H) {
                uint64_t full = gen_draw(seed, STREAM_GRID, (uint64_t)id);
                uint32_t r = (uint32_t)(full >> 32);
                int main_d = 0, anti_d = 0;
                if (r < t_none) {
                } else if (r < t_none_one) {
                    if (full & 1) main_d = 1; else anti_d = 1;
                    ++d1;
                } else {
                    main_d = anti_d = 1;
                    ++d2;
                }
                if (main_d) { src[m] = (int32_t)id; dst[m] = (int32_t)(id + W + 1); ++m; }
                if (anti_d) { src[m] = (int32_t)(id + 1); dst[m] = (int32_t)(id + W); ++m; }
            }
        }
    if (d1_out) *d1_out = d1;
    if (d2_out) *d2_out = d2;
    return m;
}

/* ---------------------------------------------------------------- Erdos-Renyi */
/* G(n, m): draws t = 0,1,2,... give (u,v) = (hi32*n>>32, lo32*n>>32); loops and
 * repeats are skipped until m distinct undirected edges exist.  Open-addressing
 * hash set, sequential (m is small in every config).  Returns m or -1. */
int64_t gen_er_edges(int64_t n, int64_t m, uint64_t seed, int32_t* src, int32_t* dst) {
    if (n < 2 || m < 0 || m > n * (n - 1) / 2) return -1;
    int64_t cap = 16;
    while (cap < 4 * m + 16) cap <<= 1;
    uint64_t* table = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)cap);
    if (!table) return -1;
    for (int64_t i = 0; i < cap; ++i) table[i] = ~0ULL;
    int64_t got = 0;
    for (uint64_t t = 0; got < m; ++t) {
        uint64_t r = gen_draw(seed, STREAM_ER, t);
        uint64_t u = ((r >> 32) * (uint64_t)n) >> 32;
        uint64_t v = ((r & 0xffffffffULL) * (uint64_t)n) >> 32;
        if (u == v) continue;
        if (u > v) { uint64_t s = u; u = v; v = s; }
        uint64_t key = (u << 32) | v;
        uint64_t h = sm64(key) & (uint64_t)(cap - 1);
        int dup = 0;
        while (table[h] != ~0ULL) {
            if (table[h] == key) { dup = 1; break; }
            h = (h + 1) & (uint64_t)(cap - 1);
        }
        if (dup) continue;
        table[h] = key;
        src[got] = (int32_t)u;
        dst[got] = (int32_t)v;
        ++got;
    }
    free(table);
    return m;
}

/* ---------------------------------------------------------------- labels */
void gen_uniform_labels(int64_t n, uint32_t num_labels, uint64_t seed, uint32_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v)
        out[v] = (uint32_t)(((gen_draw(seed, STREAM_LABEL, (uint64_t)v) >> 32) * (uint64_t)num_labels) >> 32);
}

/* ---------------------------------------------------------------- CSR build */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

static void sort_i32(int32_t* a, int64_t len) {
    if (len < 2) return;
    if (len <= 24) { /* insertion sort for short lists */
        for (int64_t i = 1; i < len; ++i) {
            int32_t x = a[i];
            int64_t j = i - 1;
            while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
            a[j + 1] = x;
        }
        return;
    }
    qsort(a, (size_t)len, sizeof(int32_t), cmp_i32);
}

/* Canonical undirected CSR from a directed edge list: both directions stored,
 * self-loops dropped, duplicates merged, each list sorted ascending.
 * offsets: caller buffer of n+1; cols: caller buffer of capacity >= 2*m.
 * Returns nnz (= offsets[n]) or -1 (id out of range / alloc failure). */
int64_t gen_csr_build(int64_t n, int64_t m, const int32_t* src, const int32_t* dst, int64_t* offsets,
                      int32_t* cols) {
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!cnt) return -1;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t e = 0; e < m; ++e) {
        int32_t u = src[e], v = dst[e];
        if (u < 0 || v < 0 || u >= n || v >= n) { bad = 1; continue; }
        if (u == v) continue;
        __atomic_fetch_add(&cnt[u], 1, __ATOMIC_RELAXED);
        __atomic_fetch_add(&cnt[v], 1, __ATOMIC_RELAXED);
    }
    if (bad) { free(cnt); return -1; }
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m + 1));
    if (!start || !tmp) { free(cnt); free(start); free(tmp); return -1; }
    start[0] = 0;
    for (int64_t v = 0; v < n; ++v) start[v + 1] = start[v] + cnt[v];
    memcpy(cnt, start, sizeof(int64_t) * (size_t)n); /* cnt becomes a write cursor */
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        int32_t u = src[e], v = dst[e];
        if (u == v) continue;
        tmp[__atomic_fetch_add(&cnt[u], 1, __ATOMIC_RELAXED)] = v;
        tmp[__atomic_fetch_add(&cnt[v], 1, __ATOMIC_RELAXED)] = u;
    }
    /* sort + dedup each list in place; cnt[v] := deduplicated length */
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t v = 0; v < n; ++v) {
        int32_t* a = tmp + start[v];
        int64_t len = start[v + 1] - start[v];
        sort_i32(a, len);
        int64_t w = 0;
        for (int64_t i = 0; i < len; ++i)
            if (w == 0 || a[i] != a[w - 1]) a[w++] = a[i];
        cnt[v] = w;
    }
    offsets[0] = 0;
    for (int64_t v = 0; v < n; ++v) offsets[v + 1] = offsets[v] + cnt[v];
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v)
        memcpy(cols + offsets[v], tmp + start[v], sizeof(int32_t) * (size_t)cnt[v]);
    int64_t nnz = offsets[n];
    free(cnt);
    free(start);
    free(tmp);
    return nnz;
}
