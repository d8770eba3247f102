/*
 * oracle/oracle.c — CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2003_01527_b200/) never links, imports or calls it, and this file
 * shares no code, header, helper or constant with the CUDA path.
 *
 * What it computes:
 *   the set of all maps f : V_Q -> V_G that are injective, edge-preserving
 *   ((u,w) in E_Q  =>  (f(u),f(w)) in E_G; non-induced, P:136 checks only query
 *   edges) and label-respecting (label_G(f(u)) = label_Q(u)).
 *
 * How: plain Ullmann/VF2-style depth-first backtracking — the CPU method the
 * paper contrasts GSM with ("depth-first search with backtracking to formulate
 * solutions incrementally", §2.1), written in the order SURVEY §8(c)
 * "Oracle algorithm" states:
 *   1. order the query vertices by BFS from query vertex 0 (the oracle's own
 *      order, never the product's plan); parent = earliest-ordered neighbour;
 *   2. position 0: every data vertex with a matching label (or every vertex of
 *      an optional root subset);
 *   3. position i: for v in N(f(parent)): skip on label mismatch, skip if v is
 *      already used, skip unless v is adjacent to f(j) for every other earlier
 *      query neighbour j (binary search in the sorted CSR), else recurse;
 *   4. a full map is a row, stored as a tuple indexed by query-vertex id.
 * No degree filter, no symmetry breaking, no pruning beyond the definition.
 * Rows are returned unsorted; oracle/__init__.py sorts them lexicographically.
 *
 * Parallelism: position-0 candidates are split over OpenMP threads; each
 * thread's DFS is sequential.  Counts are exact uint64.
 *
 * Also here: two independent exact counters used as full-scale pins
 * (SURVEY §8(c) "Triangle" / configs [4]):
 *   oracle_count_triangles — Schank-Wagner forward counting over the
 *     (degree, id) orientation, merge intersection;
 *   oracle_count_k4 — the same orientation, K4 = sum over oriented triangles
 *     (u,v,w) of |N+(u) & N+(v) & N+(w)|.
 * Both count each unlabeled clique exactly once; all-embedding counts are
 * 6*T and 24*K4 (|Aut(K3)| = 6, |Aut(K4)| = 24).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define OR_MAXK 32

typedef struct {
    uint64_t count;
    int64_t nrows;
    int32_t k;
    int32_t* rows; /* nrows * k, row-major, column j = f(query vertex j); malloc'd */
    int32_t status; /* 0 ok, 1 bad argument, 2 allocation failure */
} oracle_result;

typedef struct {
    /* graph */
    const int64_t* off;
    const int32_t* cols;
    const uint32_t* labels;
    /* query, in the oracle's BFS order */
    int k;
    int order[OR_MAXK];           /* order[i] = query vertex at position i */
    int parent[OR_MAXK];          /* parent[i] = earlier position (i >= 1)   */
    int nother[OR_MAXK];          /* other earlier neighbours (non-parent)   */
    int other[OR_MAXK][OR_MAXK];
    int use_labels;
    uint32_t qlabel[OR_MAXK];     /* by position */
    int want_rows;
} or_ctx;

typedef struct {
    int32_t f[OR_MAXK];   /* f by position */
    uint64_t count;
    int32_t* rows;
    int64_t nrows, cap;
    int failed;
} or_thread;

static int adjacent(const or_ctx* c, int32_t a, int32_t b) {
    /* is b in N(a)?  binary search in the sorted list */
    int64_t lo = c->off[a], hi = c->off[a + 1];
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        int32_t x = c->cols[mid];
        if (x == b) return 1;
        if (x < b) lo = mid + 1; else hi = mid;
    }
    return 0;
}

static void emit(const or_ctx* c, or_thread* t) {
    t->count++;
    if (!c->want_rows) return;
    if (t->nrows == t->cap) {
        int64_t ncap = t->cap ? 2 * t->cap : 1024;
        int32_t* nr = (int32_t*)realloc(t->rows, sizeof(int32_t) * (size_t)(ncap * c->k));
        if (!nr) { t->failed = 1; return; }
        t->rows = nr;
        t->cap = ncap;
    }
    int32_t* row = t->rows + t->nrows * c->k;
    for (int i = 0; i < c->k; ++i) row[c->order[i]] = t->f[i];  /* index by query-vertex id */
    t->nrows++;
}

static void dfs(const or_ctx* c, or_thread* t, int i) {
    if (i == c->k) { emit(c, t); return; }
    int32_t a = t->f[c->parent[i]];
    for (int64_t e = c->off[a]; e < c->off[a + 1]; ++e) {
        int32_t v = c->cols[e];
        if (c->use_labels && c->labels[v] != c->qlabel[i]) continue;
        int used = 0;
        for (int j = 0; j < i; ++j)
            if (t->f[j] == v) { used = 1; break; }
        if (used) continue;
        int ok = 1;
        for (int q = 0; q < c->nother[i]; ++q)
            if (!adjacent(c, t->f[c->other[i][q]], v)) { ok = 0; break; }
        if (!ok) continue;
        t->f[i] = v;
        dfs(c, t, i + 1);
    }
}

/* qedges: 2*nqe ints.  qlabels NULL => labels ignored.  labels NULL with
 * qlabels non-NULL => status 1.  roots NULL => position 0 ranges over all
 * vertices; else only over roots[0..nroots).  Query must be connected. */
int oracle_match(int64_t n, const int64_t* off, const int32_t* cols, const uint32_t* labels, int k,
                 int nqe, const int32_t* qedges, const uint32_t* qlabels, const int32_t* roots,
                 int64_t nroots, int nthreads, int want_rows, oracle_result* out) {
    memset(out, 0, sizeof(*out));
    out->k = k;
    if (k < 1 || k > OR_MAXK || n < 1 || (qlabels && !labels)) { out->status = 1; return 1; }
    int adj[OR_MAXK][OR_MAXK];
    memset(adj, 0, sizeof(adj));
    for (int e = 0; e < nqe; ++e) {
        int a = qedges[2 * e], b = qedges[2 * e + 1];
        if (a < 0 || b < 0 || a >= k || b >= k || a == b) { out->status = 1; return 1; }
        adj[a][b] = adj[b][a] = 1;
    }
    or_ctx c;
    memset(&c, 0, sizeof(c));
    c.off = off; c.cols = cols; c.labels = labels; c.k = k;
    c.use_labels = qlabels != NULL;
    c.want_rows = want_rows;
    /* 1. BFS order from query vertex 0 */
    int pos[OR_MAXK];
    for (int u = 0; u < k; ++u) pos[u] = -1;
    int head = 0, tail = 0;
    c.order[tail++] = 0;
    pos[0] = 0;
    while (head < tail) {
        int x = c.order[head++];
        for (int y = 0; y < k; ++y)
            if (adj[x][y] && pos[y] < 0) { pos[y] = tail; c.order[tail++] = y; }
    }
    if (tail != k) { out->status = 1; return 1; } /* disconnected query */
    for (int i = 0; i < k; ++i) {
        int u = c.order[i];
        c.qlabel[i] = qlabels ? qlabels[u] : 0;
        c.parent[i] = -1;
        c.nother[i] = 0;
        for (int j = 0; j < i; ++j) {  /* earlier positions adjacent to u */
            if (!adj[u][c.order[j]]) continue;
            if (c.parent[i] < 0) c.parent[i] = j;  /* earliest-ordered neighbour */
            else c.other[i][c.nother[i]++] = j;
        }
    }
    int64_t ncand = roots ? nroots : n;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    or_thread* th = (or_thread*)calloc((size_t)nthreads, sizeof(or_thread));
    if (!th) { out->status = 2; return 2; }
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 16)
    for (int64_t r = 0; r < ncand; ++r) {
        or_thread* t = &th[omp_get_thread_num()];
        int32_t v = roots ? roots[r] : (int32_t)r;
        if (v < 0 || v >= n) continue;
        if (c.use_labels && labels[v] != c.qlabel[0]) continue;
        t->f[0] = v;
        dfs(&c, t, 1);
    }
    uint64_t total = 0;
    int64_t nrows = 0;
    int failed = 0;
    for (int i = 0; i < nthreads; ++i) {
        total += th[i].count;
        nrows += th[i].nrows;
        failed |= th[i].failed;
    }
    out->count = total;
    if (want_rows && !failed) {
        out->rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nrows * k + 1));
        if (!out->rows) failed = 1;
        else {
            int64_t w = 0;
            for (int i = 0; i < nthreads; ++i) {
                memcpy(out->rows + w * k, th[i].rows, sizeof(int32_t) * (size_t)(th[i].nrows * k));
                w += th[i].nrows;
            }
            out->nrows = nrows;
        }
    }
    for (int i = 0; i < nthreads; ++i) free(th[i].rows);
    free(th);
    if (failed) { out->status = 2; return 2; }
    return 0;
}

void oracle_result_free(oracle_result* r) {
    if (r && r->rows) { free(r->rows); r->rows = NULL; }
}

/* ------------------------------------------------------------ exact clique counters */
/* Degree-ordered orientation: u -> v iff (deg u, u) < (deg v, v).  Out-lists
 * keep ascending id order (filtered from the sorted CSR). */
typedef struct { int64_t* off; int32_t* col; } or_oriented;

static int orient(int64_t n, const int64_t* off, const int32_t* cols, or_oriented* o) {
    o->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    o->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(off[n] / 2 + 1));
    if (!o->off || !o->col) return 1;
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!cnt) return 1;
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < n; ++u) {
        int64_t du = off[u + 1] - off[u], c0 = 0;
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
            int32_t v = cols[e];
            int64_t dv = off[v + 1] - off[v];
            if (du < dv || (du == dv && u < v)) c0++;
        }
        cnt[u] = c0;
    }
    o->off[0] = 0;
    for (int64_t u = 0; u < n; ++u) o->off[u + 1] = o->off[u] + cnt[u];
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t u = 0; u < n; ++u) {
        int64_t du = off[u + 1] - off[u], w = o->off[u];
        for (int64_t e = off[u]; e < off[u + 1]; ++e) {
            int32_t v = cols[e];
            int64_t dv = off[v + 1] - off[v];
            if (du < dv || (du == dv && u < v)) o->col[w++] = v;
        }
    }
    free(cnt);
    return 0;
}

static int64_t merge_count(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {
    int64_t i = 0, j = 0, c = 0;
    while (i < na && j < nb) {
        if (a[i] < b[j]) ++i;
        else if (a[i] > b[j]) ++j;
        else { ++c; ++i; ++j; }
    }
    return c;
}

/* roots == NULL: every vertex u; else only the cliques whose LOWEST vertex in the
 * (degree, id) orientation is one of roots[0..nroots) — the vertex the forward
 * algorithm counts each clique at (SURVEY §8(c) configs[4] pin (ii), root-restricted
 * for shard parity: a clique belongs to the root shard of its lowest-ranked vertex). */
uint64_t oracle_count_triangles_roots(int64_t n, const int64_t* off, const int32_t* cols, const int32_t* roots,
                                      int64_t nroots, uint64_t* per_root, int nthreads) {
    or_oriented o;
    if (orient(n, off, cols, &o)) return ~0ULL;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    const int64_t nu = roots ? nroots : n;
    uint64_t t = 0;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 256) reduction(+ : t)
    for (int64_t r = 0; r < nu; ++r) {
        const int64_t u = roots ? (int64_t)roots[r] : r;
        uint64_t tu = 0;
        for (int64_t e = o.off[u]; e < o.off[u + 1]; ++e) {
            int32_t v = o.col[e];
            tu += (uint64_t)merge_count(o.col + o.off[u], o.off[u + 1] - o.off[u], o.col + o.off[v],
                                        o.off[v + 1] - o.off[v]);
        }
        if (per_root) per_root[r] = tu;
        t += tu;
    }
    free(o.off);
    free(o.col);
    return t;
}

uint64_t oracle_count_triangles(int64_t n, const int64_t* off, const int32_t* cols, int nthreads) {
    return oracle_count_triangles_roots(n, off, cols, NULL, 0, NULL, nthreads);
}

uint64_t oracle_count_k4_roots(int64_t n, const int64_t* off, const int32_t* cols, const int32_t* roots,
                               int64_t nroots, uint64_t* per_root, int nthreads) {
    or_oriented o;
    if (orient(n, off, cols, &o)) return ~0ULL;
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    int64_t maxout = 0;
    for (int64_t u = 0; u < n; ++u)
        if (o.off[u + 1] - o.off[u] > maxout) maxout = o.off[u + 1] - o.off[u];
    uint64_t total = 0;
#pragma omp parallel num_threads(nthreads) reduction(+ : total)
    {
        int32_t* s = (int32_t*)malloc(sizeof(int32_t) * (size_t)(maxout + 1));
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < (roots ? nroots : n); ++r) {
            const int64_t u = roots ? (int64_t)roots[r] : r;
            uint64_t tu = 0;
            for (int64_t e = o.off[u]; e < o.off[u + 1]; ++e) {
                int32_t v = o.col[e];
                /* s = N+(u) & N+(v) */
                const int32_t *a = o.col + o.off[u], *b = o.col + o.off[v];
                int64_t na = o.off[u + 1] - o.off[u], nb = o.off[v + 1] - o.off[v], i = 0, j = 0, ns = 0;
                while (i < na && j < nb) {
                    if (a[i] < b[j]) ++i;
                    else if (a[i] > b[j]) ++j;
                    else { s[ns++] = a[i]; ++i; ++j; }
                }
                for (int64_t x = 0; x < ns; ++x) {
                    int32_t w = s[x];
                    tu += (uint64_t)merge_count(s, ns, o.col + o.off[w], o.off[w + 1] - o.off[w]);
                }
            }
            if (per_root) per_root[r] = tu;
            total += tu;
        }
        free(s);
    }
    free(o.off);
    free(o.col);
    return total;
}

uint64_t oracle_count_k4(int64_t n, const int64_t* off, const int32_t* cols, int nthreads) {
    return oracle_count_k4_roots(n, off, cols, NULL, 0, NULL, nthreads);
}

/* ------------------------------------------------------------ labeled house counter */
/* Exact count of the labeled house query (square 0-1-2-3 + roof 4 on edge 0-1;
 * SURVEY §8(d) configs[3]) with f(0) restricted to roots (NULL = every vertex),
 * per root.  Independent of the DFS: it counts instead of enumerating.
 *
 * For f(0) = a and f(1) = b (an edge, labels l0, l1) the remaining vertices
 * split into the roof x = f(4) in N(a) & N(b) with label l4, and the path
 * a - y - z - b with y = f(3) in N(a) (label l3), z = f(2) in N(b) (label l2),
 * y ~ z.  Under the caller-checked label conditions l4 not in {l0..l3},
 * l1 != l3, l0 != l2 every pair of query vertices is either adjacent or has
 * different labels, so injectivity holds automatically and the two parts are
 * independent given (a, b):
 *     count(a) = sum_{b in N(a), L(b)=l1}  c(a,b) * p(a,b),
 *     c(a,b)  = |{x in N(a) & N(b) : L(x) = l4}|,
 *     p(a,b)  = sum_{z in N(b), L(z)=l2} w_a(z),   w_a(z) = |{y in N(a) & N(z) : L(y) = l3}|.
 * w_a is accumulated once per root in a dense per-thread array (touched entries reset). */
static int64_t merge_count_label(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, const uint32_t* lab,
                                 uint32_t want) {
    int64_t i = 0, j = 0, c = 0;
    while (i < na && j < nb) {
        if (a[i] < b[j]) ++i;
        else if (a[i] > b[j]) ++j;
        else { c += lab[a[i]] == want; ++i; ++j; }
    }
    return c;
}

uint64_t oracle_count_house_roots(int64_t n, const int64_t* off, const int32_t* cols, const uint32_t* lab,
                                  const uint32_t* ql /* 5 labels */, const int32_t* roots, int64_t nroots,
                                  uint64_t* per_root, int nthreads) {
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    const int64_t nu = roots ? nroots : n;
    uint64_t total = 0;
    int fail = 0;
#pragma omp parallel num_threads(nthreads) reduction(+ : total)
    {
        int64_t* w = (int64_t*)calloc((size_t)n, sizeof(int64_t));
        int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
        if (!w || !touched) {
#pragma omp atomic write
            fail = 1;
        }
#pragma omp for schedule(dynamic, 16)
        for (int64_t r = 0; r < nu; ++r) {
            if (!w || !touched) continue;
            const int64_t a = roots ? (int64_t)roots[r] : r;
            uint64_t ta = 0;
            if (lab[a] == ql[0]) {
                int64_t nt = 0;
                for (int64_t e = off[a]; e < off[a + 1]; ++e) {  /* y = f(3) */
                    const int32_t y = cols[e];
                    if (lab[y] != ql[3]) continue;
                    for (int64_t f = off[y]; f < off[y + 1]; ++f) {  /* z = f(2) candidates */
                        const int32_t z = cols[f];
                        if (lab[z] != ql[2]) continue;
                        if (w[z]++ == 0) touched[nt++] = z;
                    }
                }
                for (int64_t e = off[a]; e < off[a + 1]; ++e) {  /* b = f(1) */
                    const int32_t b = cols[e];
                    if (lab[b] != ql[1]) continue;
                    int64_t p = 0;
                    for (int64_t f = off[b]; f < off[b + 1]; ++f) {
                        const int32_t z = cols[f];
                        if (lab[z] == ql[2]) p += w[z];
                    }
                    if (!p) continue;
                    const int64_t c = merge_count_label(cols + off[a], off[a + 1] - off[a], cols + off[b],
                                                        off[b + 1] - off[b], lab, ql[4]);
                    ta += (uint64_t)c * (uint64_t)p;
                }
                for (int64_t t = 0; t < nt; ++t) w[touched[t]] = 0;
            }
            if (per_root) per_root[r] = ta;
            total += ta;
        }
        free(w);
        free(touched);
    }
    return fail ? ~0ULL : total;
}

int oracle_num_threads(void) { return omp_get_max_threads(); }
