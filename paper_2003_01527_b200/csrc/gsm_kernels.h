// gsm_kernels.h — launchers for the hot-path kernels (gsm_kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gsm_common.h"

namespace gsm {

struct FilterQuery {
    int32_t k;
    int32_t use_labels;
    uint32_t qlabel[kMaxK];
    int32_t qdeg[kMaxK];
    uint32_t qadj[kMaxK];  // query adjacency bitmasks (refinement: 1-step look-ahead)
};

// mask width: 1, 2 or 4 bytes per vertex (k <= 8, 16, 32)
inline int mask_bytes_for(int k) { return k <= 8 ? 1 : (k <= 16 ? 2 : 4); }

// ----------------------------------------------------------------------------
// A frontier of partial results (Alg. 1's M[i]) of width W, in one of two layouts:
//  * plain: int32 rows, row-major (4 W bytes per row);
//  * compressed ("store the value to partial
//    results ... to further save memory usage", P:163 optimisation 4): level-wise
//    (parent index, vertex) pairs — row r of width w is row pv[w][r].x of width w-1
//    extended by vertex pv[w][r].y — 8 bytes per row at any width; the chain ends in a
//    plain frontier `base` of width bw (the roots, or rows handed over in plain form).
// Depth-first chunk processing keeps every ancestor chunk resident while its children
// are expanded, so a chain is always valid.  Bijective (the tuple is recovered exactly,
// unlike a lossy hash, so listings stay possible — DESIGN.md reading R6).
// ----------------------------------------------------------------------------
struct Frontier {
    int32_t W = 0;
    const int32_t* rows = nullptr;     // plain rows (width W), or nullptr when compressed
    const int32_t* base = nullptr;     // compressed: plain rows of width bw the chains end in
    int32_t bw = 0;
    const int2* pv[kMaxK + 1] = {};    // compressed: pv[w] for w = bw+1 .. W
};

// the row as a pointer: into the plain rows, or reconstructed into buf (W <= kMaxK)
__device__ __forceinline__ const int32_t* frontier_row(const Frontier& F, int64_t r, int32_t* buf) {
    if (F.rows) return F.rows + r * F.W;
    for (int w = F.W; w > F.bw; --w) {
        const int2 e = F.pv[w][r];
        buf[w - 1] = e.y;
        r = e.x;
    }
    for (int c = 0; c < F.bw; ++c) buf[c] = F.base[r * F.bw + c];
    return buf;
}

// K1 (Alg. 1 line 8): cmask[v] bit u = [label(v) = label_Q(u)] and [deg(v) >= deg_Q(u)];
// counts[u] += |C(u)|  (counts must be zeroed by the caller).
void launch_filter(const DevGraph& g, const FilterQuery& q, void* cmask, unsigned long long* counts,
                   cudaStream_t s);

// K5 NE refinement (Alg. 1 lines 7-8): `rounds` passes of NE / effective-degree pruning of
// cmask (qne: device int64[k] query NE), then counts[u] = |C(u)| recomputed.  tmp: n mask words.
// out[new2old[v]] = (uint32) cmask[v]
void launch_mask_to_original(const DevGraph& g, const void* cmask, int mask_bytes, uint32_t* out, cudaStream_t s);

void launch_refine(const DevGraph& g, const FilterQuery& q, const int64_t* qne, int rounds, void* cmask, void* tmp,
                   unsigned long long* counts, cudaStream_t s);

// Roots: stable compaction of {v : bit `bit` of cmask[v]} in ascending new id, keeping global
// rank r with r % nshards == shard (written at r / nshards).  Returns the number written.
int64_t launch_roots(const DevGraph& g, const void* cmask, int mask_bytes, int bit, int shard, int nshards,
                     int32_t* roots, cudaStream_t s);

// Root subset (original ids, device array): new ids with the cmask bit set (order preserved).
int64_t launch_root_subset(const DevGraph& g, const void* cmask, int mask_bytes, int bit, const int32_t* subset_old,
                           int64_t len, int32_t* roots, cudaStream_t s);

// Per-row pivot choice and candidate range (the "Advance" source list).
// Also writes, per row and per backward position q, the exact admissible segment of that
// neighbour's list (cbeg/clen, R x nb): the pivot's is the candidate list, the others are
// the membership lists the verify step binary-searches.
void launch_plan_rows(const DevGraph& g, const Frontier& F, int64_t R, const LevelPlan& L, int64_t* rbeg,
                      int64_t* rlen, uint8_t* rpiv, int64_t* cbeg, int32_t* clen, cudaStream_t s);

// Inclusive scan of rlen into P[1..R] (P[0] = 0); returns nothing (caller reads P[R]).
size_t scan_temp_bytes(int64_t R);
void launch_scan(const int64_t* rlen, int64_t R, int64_t* P, void* tmp, size_t tmp_bytes, cudaStream_t s);

// Merge-path partition of diagonals [D0, D1) into tiles of TD: tile_ra[t] for t = 0..ntiles.
void launch_partition(const int64_t* P, int64_t R, int64_t S, int64_t D0, int64_t D1, int64_t TD, int64_t ntiles,
                      int64_t* tile_ra, cudaStream_t s);

struct ExpandArgs {
    Frontier F;            // input rows (R x width)
    int64_t R;
    const int64_t* P;      // R+1 work offsets
    const int64_t* rbeg;   // R pivot-range starts (index into cols)
    const uint8_t* rpiv;   // R pivot index into L.bpos
    const int64_t* cbeg;   // R x nb admissible segment starts (index into cols)
    const int32_t* clen;   // R x nb admissible segment lengths
    const int64_t* tile_ra;
    int64_t D0, D1, TD, ntiles;
    const int64_t* off;
    const int32_t* cols;
    const void* cmask;
    int32_t* out;          // survivors (width+1 ints each), unless count_only or out_pv
    int2* out_pv;          // compressed output: (input row index, new vertex) per survivor
    unsigned long long* out_count;  // survivors (atomic)
    unsigned long long* stats;      // [items, mask_checked, probes, survivors, lists]
    // look-ahead tables (L.nla > 0): c1[v*k + u] = min(255, |N(v) ∩ C(u)|); ok1 = per-vertex
    // mask of u whose later query neighbours all have a candidate neighbour; c2[v*k + u] =
    // min(255, |{w ∈ N(v) : ok1[w] bit u}|)
    const uint8_t* la_c1;
    const uint8_t* la_c2;
    const void* la_ok1;
    int32_t la_k;
};

// look-ahead precomputation (one edge pass each): out[v*k + u] = min(255, |{w in N(v): mask[w] bit u}|)
void launch_la_counts(const DevGraph& g, int k, int mask_bytes, const void* mask, uint8_t* out, cudaStream_t s);
// ok1[w] = bits u with cmask[w] bit u and c1[w*k + u''] >= 1 for every u'' in dmask[u]
void launch_la_ok1(const DevGraph& g, int k, int mask_bytes, const void* cmask, const uint8_t* c1,
                   const uint32_t* dmask_host, void* ok1, cudaStream_t s);

// Tile size (merge steps per CTA) for a given input width / for a level plan (the COUNT-mode
// last level uses the walking kernel with its own, larger tile).
int64_t expand_tile(int width);
int64_t expand_tile_for(const LevelPlan& L);

// K2+K3+K4 fused: expand + verify + compact (Alg. 1 lines 11-13).
void launch_expand(const ExpandArgs& a, const LevelPlan& L, int mask_bytes, cudaStream_t s);

// Fused tail (COUNT mode): positions k-2 and k-1 in one kernel (candidate-set inheritance).
struct TailArgs {
    Frontier F;             // rows of width k-2
    int64_t R;
    const int64_t* rbeg;    // plan of position k-2 (k_plan_rows)
    const int64_t* rlen;
    const uint8_t* rpiv;
    const int64_t* cbeg;
    const int32_t* clen;
    const int64_t* off;
    const int32_t* up;      // plain lists: N+(v) starts at off[v] + up[v]
    const int32_t* cols;    // plain or keyed lists (same as position k-2's)
    const void* cmask;
    int32_t rel;            // +1: f(π[k-1]) ≻ f(π[k-2]); -1: ≺; 0: unconstrained
    int32_t cap;            // per-warp candidate buffer (int32 entries)
    int32_t bratio;         // phase-2 strategy threshold in percent (see tail_bratio)
    int32_t nxlo, nxhi;     // extra ID bounds of π[k-1] not implied by π[k-2]'s interval
    int32_t xlo[kMaxK], xhi[kMaxK];
    unsigned long long* count;
    const int64_t* rows_idx;  // k_tail_block: indices of the rows to process (NULL = 0..R-1)
    int64_t* overflow;      // rows left to the next stage
    unsigned long long* noverflow;
    unsigned long long* next;  // dynamic row scheduler (zeroed before each launch)
    unsigned long long* cyc;   // optional (GSM_TRACE=2): warp cycles [phase1, small-RC pairs, big-RC c loop, #small, #big]
    unsigned long long* stats;
};
// Reorders row indices by descending pivot length (largest rows first: better makespan).
void sort_rows_by_len_desc(const int64_t* rlen, int64_t* idx, int64_t n, cudaStream_t s);
int tail_cap();
int tail_bratio();
int tail_block_cap();
void launch_tail_block(const TailArgs& a, const LevelPlan& Lc, const LevelPlan& Ld, int mask_bytes, cudaStream_t s);
void launch_tail(const TailArgs& a, const LevelPlan& Lc, const LevelPlan& Ld, int mask_bytes, cudaStream_t s);
void launch_gather_rows(const Frontier& F, const int64_t* idx, int64_t n, int32_t* out, cudaStream_t s);

// Pair tail (COUNT mode): positions p = k-2 and q = k-1 not adjacent in Q and without an ID
// condition between them: count(r) = |Cp(r)| |Cq(r)| - |Cp(r) ∩ Cq(r)| per row r of width k-2.
// exact adjacency test v ∈ N(f) for v already inside the admissible range of f's segment:
// hub bitmap when both are hubs, else binary search in the shorter of seg and N(v)
struct MemberCtx {
    const int64_t* off = nullptr;
    const uint32_t* hub_bits = nullptr;
    int32_t hub_base = 0, hub_words = 0;
    int32_t swap_min = 0;   // segments longer than this may search f in N(v) instead (0 = never)
};

struct PairArgs {
    Frontier F;
    MemberCtx mem;
    int64_t R;
    const int64_t *pbeg, *plen, *pcbeg;  // k_plan_rows of position p
    const uint8_t* ppiv;
    const int32_t* pclen;
    const int64_t *qbeg, *qlen, *qcbeg;  // k_plan_rows of position q (same input rows)
    const uint8_t* qpiv;
    const int32_t* qclen;
    const int32_t* colsp;   // plain or keyed lists of p's / q's label
    const int32_t* colsq;
    const void* cmask;
    int32_t need_both;      // 0 when Cp and Cq are disjoint (different labels)
    unsigned long long* count;
    unsigned long long* next;   // dynamic row scheduler (zeroed)
    unsigned long long* stats;  // [items, -, probes, -, -]
    const int64_t* rows_idx;    // warp pass: the rows to process (NULL = 0..R-1)
    int64_t* overflow;          // thread pass: rows whose two segments exceed `thread_max`
    unsigned long long* noverflow;
    int32_t thread_max;
};
// Thread pass: one thread per row for rows with short segments (labeled queries: most);
// longer rows are appended to a.overflow for the warp pass (launch_pair).
void launch_pair_thread(const PairArgs& a, const LevelPlan& Lp, const LevelPlan& Lq, int mask_bytes, cudaStream_t s);
void launch_pair(const PairArgs& a, const LevelPlan& Lp, const LevelPlan& Lq, int mask_bytes, cudaStream_t s);

// Clique queries K3/K4 in COUNT mode (gsm_clique.cu): per-root local bitmaps over
// N+(u).  Adds the number of cliques (orbit representatives) to *count.
struct CliqueRun {
    int k;                  // 3 or 4
    const int32_t* roots;   // level-0 frontier (new ids)
    int64_t R;
    const int64_t* off;
    const int32_t* cols;
    const int32_t* up;
    unsigned long long* count;
    unsigned long long* stats;  // 5: [list entries read, global probes, bitmap words, cliques, sum |N+(u)|]
    int32_t* over_roots;    // out (capacity R): roots with |N+(u)| beyond the per-CTA tables,
    int64_t n_over;         // left to the breadth-first path (set by run_clique)
    struct Workspace* ws;   // per-graph grow-only buffers (gsm_workspace.h)
    const uint32_t* hub_bits = nullptr;  // DevGraph hub bitmap (nullptr = none)
    int32_t hub_base = 0, hub_words = 0;
    const int4* nplus = nullptr;      // DevGraph packed N+(v) descriptors
    const int32_t* nh_off = nullptr;  // DevGraph hashed N+(v) tables (nullptr = none)
    const int32_t* nh_tab = nullptr;
};
int64_t run_clique(CliqueRun& r, cudaStream_t s);  // returns kernel launches
int clique_dsmem(int K);

// Finalize ("Return ... subgraph enumeration M").
void launch_to_query_order(const int32_t* in, int64_t N, int k, const int32_t* order, const int32_t* new2old,
                           int32_t* out, cudaStream_t s);
void launch_aut_expand(const int32_t* in, int64_t N, int k, const int8_t* sigmas, int64_t num_aut, int32_t* out,
                       cudaStream_t s);
// Lexicographic sort of N rows x k int32 columns (values in [0, n)).  Uses `out` as destination.
void sort_rows(const int32_t* rows, int64_t N, int k, int64_t n, int32_t* out, cudaStream_t s);

}  // namespace gsm
