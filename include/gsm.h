/*
 * gsm.h — C ABI of the B200-native GSM hot path (Gunrock Subgraph Matching,
 * Wang & Owens, arXiv 2003.01527).  Library: paper_2003_01527_b200/libgsm.so.
 *
 * What the library computes (§3.2 "two outputs: the subgraph
 * counting and subgraph enumeration"; §1 "enumeration of all subgraph
 * isomorphisms"; Alg. 1):  given an undirected data graph G in CSR
 * form and a small connected query Q (k <= 32 vertices), the set of all maps
 * f : V_Q -> V_G that are
 *     injective,
 *     edge-preserving   ((u,w) in E_Q  =>  (f(u), f(w)) in E_G; non-induced,
 *                        the paper's verify step checks only query edges),
 *     label-respecting  (label_G(f(u)) = label_Q(u); node labels only).
 * The count is exact (uint64).  Enumeration rows are int32, row-major,
 * column j = f(query vertex j), sorted lexicographically as unsigned tuples.
 *
 * The method (Alg. 1): a host pass orders the query vertices by d_M, P_f, deg
 * and derives symmetry-breaking "constraints on node ID values"
 * (P:71); a filter kernel builds candidate sets by label and degree (Alg. 1
 * line 8); then |Q|-1 breadth-first verify iterations (Alg. 1
 * lines 9-15) each expand every partial result through the
 * CSR list of one already-matched data vertex ("Advance"), verify the other
 * query edges, injectivity and the ID constraints ("Compute"), and compact the
 * survivors into the next frontier ("Write_to_Partial").  Frontiers are
 * processed in chunks so device memory stays bounded ("memory
 * linear to matched subgraphs").
 *
 * Conventions for every function:
 *   - returns gsm_status; never throws across the ABI;
 *   - on error a thread-local message is available from gsm_last_error();
 *   - on error every output struct is zeroed and every output handle is NULL;
 *   - struct arguments carry struct_size = sizeof(struct) for versioning.
 *
 * Threading: a gsm_graph is bound to one CUDA device and is not thread-safe;
 * use one handle per device per process.  gsm_match is synchronous with
 * respect to the host (it returns when its results are final).
 *
 * Memory: gsm_match keeps its grow-only device work buffers (frontier chunks,
 * per-row plans, counters — at most mem_budget_bytes plus O(n)) inside the
 * graph handle and reuses them on the next call; gsm_free releases them.
 */
#ifndef GSM_H_
#define GSM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSM_MAX_QUERY_NODES 32

#if defined(__GNUC__)
#define GSM_API __attribute__((visibility("default")))
#else
#define GSM_API
#endif

typedef enum {
    GSM_OK = 0,
    GSM_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, bad struct_size, query labels on an unlabeled graph */
    GSM_ERR_INVALID_GRAPH = 2,    /* n <= 0, non-monotone offsets, unsorted/duplicate neighbour,
                                     self-loop, asymmetric edge, id out of range */
    GSM_ERR_INVALID_QUERY = 3,    /* k == 0 or k > 32, self-loop or duplicate edge, vertex out of
                                     range, disconnected query */
    GSM_ERR_OUT_OF_MEMORY = 4,    /* device allocation failed even at the minimum chunk size, or the
                                     enumeration output does not fit (SPEC S:238 resource limit) */
    GSM_ERR_CUDA = 5,             /* any other CUDA runtime error (message has the CUDA string) */
    GSM_ERR_NO_DEVICE = 6         /* no CUDA device / driver: there is NO CPU fallback */
} gsm_status;

/* Opaque device-resident data graph (a relabelled CSR replica; see gsm_load_graph). */
typedef struct gsm_graph gsm_graph;

typedef struct {
    uint32_t struct_size; /* = sizeof(gsm_load_opts) */
    int32_t device;       /* CUDA device ordinal the graph lives on */
    int32_t validate;     /* 1: check the CSR invariants on the device, O(n + m log d) */
    int32_t reserved;
    void* stream;         /* cudaStream_t used for loading; NULL = a library-owned stream */
} gsm_load_opts;

/*
 * gsm_load_graph — build the device replica of an undirected CSR data graph.
 *
 *   num_nodes           n >= 1.
 *   row_offsets         int64[n+1], row_offsets[0] = 0, non-decreasing.
 *   col_indices         int32[row_offsets[n]]; list of v = col_indices[row_offsets[v] ..
 *                       row_offsets[v+1]), strictly ascending, no self-loops, each undirected
 *                       edge stored in both directions (SPEC CsrGraph S:22-29; PAPER P:148
 *                       "compressed sparse row").
 *   labels              uint32[n] node labels, or NULL = unlabeled.
 *   pointers_on_device  0: the three arrays are host memory; 1: device memory on opts->device.
 *                       Either way they are only BORROWED for the duration of the call — the
 *                       library keeps its own copy.
 *   opts                may be NULL (device 0, no validation, library stream).
 *   out                 receives the handle; release with gsm_free.
 *
 * Load-time work (reported separately from match time, like the paper excludes
 * GSI's preprocessing but not its own processing): copy, optional
 * validation, and a relabelling of the vertices by ascending (degree, id) with
 * each list re-sorted, which makes the symmetry-breaking order "≺" a plain
 * integer compare and each list's "higher-ranked neighbours" a contiguous
 * suffix.  Results are always reported in the caller's original vertex ids.
 */
GSM_API gsm_status gsm_load_graph(int64_t num_nodes, const int64_t* row_offsets, const int32_t* col_indices,
                          const uint32_t* labels, int32_t pointers_on_device, const gsm_load_opts* opts,
                          gsm_graph** out);

/* Releases a graph (idempotent on NULL). */
GSM_API gsm_status gsm_free(gsm_graph* g);

/* Basic facts about a loaded graph (host-readable). */
GSM_API gsm_status gsm_graph_info(const gsm_graph* g, int64_t* num_nodes, int64_t* num_directed_edges,
                          int32_t* labeled, int32_t* device);

/* Query graph Q: k = num_nodes vertices 0..k-1 ("small query graph"). */
typedef struct {
    int32_t num_nodes;      /* k, 1 <= k <= 32 */
    int32_t num_edges;      /* undirected edges */
    const int32_t* edges;   /* HOST int32[2*num_edges]: (a0,b0,a1,b1,...) */
    const uint32_t* labels; /* HOST uint32[k], or NULL = label-agnostic */
} gsm_query;

typedef enum { GSM_MODE_COUNT = 0, GSM_MODE_ENUMERATE = 1 } gsm_mode;

enum {
    /* report one embedding per Aut(Q) orbit instead of all embeddings (SURVEY §8(c) amb. 1) */
    GSM_FLAG_UNIQUE = 1u,
    /* test-only: search all embeddings directly, without ID constraints */
    GSM_FLAG_NO_SYMMETRY = 2u,
    /* record per-kernel CUDA-event times and algorithmic-byte counters in gsm_result.prof */
    GSM_FLAG_PROFILE = 4u,
    /* gsm_plan_query only: plan as a COUNT-mode match does — the two last positions an
       independent pair of non-adjacent query vertices when Q allows it */
    GSM_FLAG_PLAN_COUNT = 8u,
    /* store intermediate partial results as level-wise (parent row, vertex) pairs — 8 bytes per
       partial result at any width instead of 4 x width (PAPER P:136/"store the value
       to partial results ... to further save memory usage"; bijective, so listings are exact) */
    GSM_FLAG_COMPRESSED_PARTIALS = 16u,
    /* multi-GPU skew (SURVEY §8(e) mitigation): with num_shards = P > 1, shard by the LEVEL-1
       partial result instead of the root: every rank expands all roots one level and keeps the
       pairs (f(π[0]), f(π[1])) whose hash mod P == shard_index, so one hub root's subtree is
       spread over all ranks.  Each embedding still belongs to exactly one shard.  Applies where
       level 1 is a breadth-first expand (k >= 3, not the clique bitmap path, not a pair/fused
       tail at level 1); elsewhere the call shards by root as without the flag. */
    GSM_FLAG_SHARD_LEVEL1 = 32u
};

typedef struct {
    uint32_t struct_size;     /* = sizeof(gsm_match_opts) */
    gsm_mode mode;
    uint32_t flags;           /* GSM_FLAG_* */
    int32_t shard_index;      /* root-candidate shard (multi-GPU); 0 */
    int32_t num_shards;       /* 0 or 1 = all roots; P = keep the root candidates v whose rank in the
                                 ascending (degree, original id) order satisfies rank % P == shard_index
                                 (each embedding belongs to exactly one shard: the one of its root
                                 f(π[0]); P may be as large as n, e.g. to isolate one root) */
    int32_t refine_rounds;    /* neighbourhood-encoding filter (Alg. 1 lines 7-8): 0 = label +
                                 degree only; R >= 1 = R rounds of NE(v) >= NE_Q(u), effective
                                 degree, and the 1-step look-ahead condition (every query neighbour
                                 of u has a candidate among v's neighbours), each
                                 recomputed over the surviving vertices.  Sound: never changes the
                                 result, only the candidate sets. */
    int32_t lookahead;        /* k-look-ahead in the verification step (§3.3, Table 2;
                                 SPEC S:225-233): 0 = off; 1 = a new partial result whose image v of
                                 π[i] has, for some unmapped query neighbour u' of π[i], no neighbour
                                 left that can host u' (|N(v) ∩ C(u')| minus the mapped ones known to
                                 be there) is dropped; 2 = additionally such a neighbour must itself
                                 have a candidate neighbour for each later query neighbour of u'.
                                 Necessary conditions only: never changes the result, only the
                                 intermediate rows (level_rows) — DESIGN.md reading R17. */
    const int32_t* root_subset; /* HOST, optional (test/parity sampling): only embeddings with
                                   f(query vertex 0) in the subset (original ids).  Forces the
                                   query order to start at vertex 0 and implies NO_SYMMETRY. */
    int64_t root_subset_len;
    uint64_t mem_budget_bytes; /* device bytes for intermediate frontiers; 0 = 1/4 of free HBM.
                                  Frontiers are cut into chunks that fit (exact upper bound). */
    void* stream;             /* cudaStream_t; NULL = the graph's stream */
} gsm_match_opts;

/* Per-kernel profile (filled when GSM_FLAG_PROFILE is set).  Times are sums of
 * CUDA-event durations of the individual launches on the match stream;
 * alg_bytes are the ALGORITHMIC bytes those launches had to move
 * (DESIGN.md §4 "algorithmic bytes"). */
typedef struct {
    uint64_t launches;
    double ms;
    double alg_bytes;
} gsm_kernel_prof;

enum {
    GSM_K_FILTER = 0,   /* K1 candidate filter (cmask + |C(u)|)          */
    GSM_K_ROOTS = 1,    /* root compaction / sharding                    */
    GSM_K_PLAN = 2,     /* per-row pivot choice + range (pre-expand)     */
    GSM_K_SCAN = 3,     /* work scan (CUB) + merge-path partition        */
    GSM_K_EXPAND = 4,   /* K2/K3/K4 expand + verify + compact            */
    GSM_K_FINALIZE = 5, /* id map, Aut expansion, radix sort             */
    GSM_K_TAIL = 6,     /* fused last two positions (COUNT mode, clique-like tails) */
    GSM_K_CLIQUE = 7,   /* clique queries K3/K4 (COUNT mode): per-root local bitmaps */
    GSM_K_COUNT_ = 8
};

typedef struct {
    uint64_t count;          /* embeddings (all, or unique with GSM_FLAG_UNIQUE) */
    uint64_t count_unique;   /* orbit representatives found by the symmetric search
                                (= count when NO_SYMMETRY or UNIQUE) */
    uint64_t automorphisms;  /* |Aut(Q)| (labels respected) */
    int32_t width;           /* k */
    int32_t num_levels;      /* k */
    uint64_t num_rows;       /* ENUMERATE: rows in `rows` (= count) */
    int32_t* rows;           /* ENUMERATE: DEVICE int32[num_rows * k], library-owned,
                                release with gsm_result_free; NULL in COUNT mode */
    float ms_total, ms_plan, ms_filter, ms_expand, ms_finalize; /* host wall times */
    int32_t order[GSM_MAX_QUERY_NODES];        /* query order π (position -> query vertex) */
    uint64_t candidates[GSM_MAX_QUERY_NODES];  /* |C(u)| per query vertex u after the filter */
    uint64_t level_rows[GSM_MAX_QUERY_NODES];  /* partial results produced at each position */
    uint64_t level_work[GSM_MAX_QUERY_NODES];  /* candidates examined at each position */
    uint64_t num_chunks;     /* expand launches (chunks over all levels) */
    uint64_t kernel_launches;/* all kernels this call launched */
    gsm_kernel_prof prof[GSM_K_COUNT_];
    int32_t device;
    int32_t symmetric;       /* 1 if ID constraints were used */
    uint64_t level_frontier_bytes[GSM_MAX_QUERY_NODES]; /* bytes of the stored partial results of each
                                width w = i+1 (summed over chunks; plain 4w, compressed 8 per row) */
    int32_t compressed;      /* 1 if intermediate partial results used the compressed layout */
    int32_t level1_sharded;  /* 1 if GSM_FLAG_SHARD_LEVEL1 sharded this call by level-1 pairs */
} gsm_result;

/*
 * gsm_match — count or enumerate the embeddings of q in g (Alg. 1).
 *   opts may be NULL (COUNT, all embeddings, all roots, default budget).
 *   On success *out holds the result; ENUMERATE rows must be released with
 *   gsm_result_free.  An empty candidate set, or k > n, is GSM_OK with count 0
 *   (SPEC S:220/S:224).  The library never falls back to the CPU.
 */
GSM_API gsm_status gsm_match(const gsm_graph* g, const gsm_query* q, const gsm_match_opts* opts, gsm_result* out);

/* Frees result rows (idempotent); zeroes rows/num_rows. */
GSM_API gsm_status gsm_result_free(gsm_result* r);

/* Copies ENUMERATE rows to dst (host memory if dst_on_device == 0, else device
 * memory on the graph's device); dst must hold num_rows * width int32. */
GSM_API gsm_status gsm_result_copy_rows(const gsm_result* r, int32_t* dst, int32_t dst_on_device);

/*
 * gsm_plan_query — HOST-ONLY (no device needed): the query-side plan the match
 * would use for candidate-set sizes cand[k] (NULL = all equal): order π by
 * d_M, then |C(u)| (the exact-count form of P_f), then degree, then id
 * (SPEC S:135), spanning-tree parents and non-tree edges
 * (Alg. 1 lines 3-4), and the symmetry-breaking ID constraints
 * built by the Grochow-Kellis stabiliser chain (reading R9).
 */
typedef struct {
    int32_t k;
    int32_t order[GSM_MAX_QUERY_NODES];   /* position -> query vertex */
    int32_t parent[GSM_MAX_QUERY_NODES];  /* position -> earlier position (-1 at 0) */
    uint32_t backward[GSM_MAX_QUERY_NODES]; /* position -> bitmask of earlier adjacent positions */
    int32_t num_conditions;
    int32_t cond_lo[GSM_MAX_QUERY_NODES * GSM_MAX_QUERY_NODES / 2]; /* query vertex a ... */
    int32_t cond_hi[GSM_MAX_QUERY_NODES * GSM_MAX_QUERY_NODES / 2]; /* ... with f(a) ≺ f(b), b here */
    uint64_t automorphisms;               /* |Aut(Q)| */
} gsm_plan_info;

GSM_API gsm_status gsm_plan_query(const gsm_query* q, const uint64_t* cand, uint32_t flags, gsm_plan_info* out);

/*
 * gsm_sort_rows — lexicographic (unsigned tuple) in-place sort of num_rows x width int32 rows
 * in DEVICE memory on `device`, values in [0, max_id].  Used to merge the enumerated row
 * shards of several GPUs; the same LSD radix sort gsm_match uses to order its
 * output.  Synchronous on `stream` (NULL = legacy default stream).
 */
GSM_API gsm_status gsm_sort_rows(int32_t* rows, uint64_t num_rows, int32_t width, int64_t max_id, int32_t device,
                                 void* stream);

/*
 * gsm_merge_rows — merge two lexicographically sorted (unsigned tuple) row blocks
 * a (na x width) and b (nb x width) into out ((na + nb) x width), all int32 in DEVICE memory
 * on `device`; out must not overlap a or b.  The P-way merge of the locally sorted ENUMERATE
 * shards of P GPUs ("a P-way merge of the locally pre-sorted
 * shards") is a tree of these.  Equal rows keep a's first.  Merge-path partition: each thread
 * binary-searches its output diagonal, then merges 8 rows.  Synchronous on `stream` (NULL =
 * legacy default stream).  Errors: GSM_ERR_INVALID_ARGUMENT (null pointer with a non-zero
 * count, width outside 1..32), GSM_ERR_CUDA.
 */
GSM_API gsm_status gsm_merge_rows(const int32_t* a, uint64_t na, const int32_t* b, uint64_t nb, int32_t width,
                                  int32_t* out, int32_t device, void* stream);

/*
 * gsm_filter_candidates — the candidate filter alone (Alg. 1 lines 6-9, PAPER P:108-110,
 * P:129): out[v] for every data vertex v (ORIGINAL id order) = bitmask of the query
 * vertices u with v in C(u): label(v) = label_Q(u) and deg(v) >= deg_Q(u), then
 * refine_rounds rounds of the NE / effective-degree refinement exactly as gsm_match uses them.
 *   out            uint32[n]: host memory (out_on_device = 0) or device memory on g's device.
 * Errors as gsm_match (invalid query, labels on an unlabeled graph, no device).
 */
GSM_API gsm_status gsm_filter_candidates(const gsm_graph* g, const gsm_query* q, int32_t refine_rounds,
                                         uint32_t* out, int32_t out_on_device);

/* Thread-local message for the last non-OK status ("" if none). */
GSM_API const char* gsm_last_error(void);

/* Library version string. */
GSM_API const char* gsm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GSM_H_ */
