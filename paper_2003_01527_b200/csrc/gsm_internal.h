// gsm_internal.h — shared between the host plan, the driver and the kernels of
// libgsm (product side).  Nothing here is visible across the C ABI.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "gsm.h"

namespace gsm {

constexpr int kMaxK = GSM_MAX_QUERY_NODES;

// ----------------------------------------------------------------------------
// Host plan (PreCompute_on_CPUs, Alg. 1 lines 1-5)
// ----------------------------------------------------------------------------
struct QueryPlan {
    int k = 0;
    uint32_t adj[kMaxK] = {};     // adjacency bitmask per query vertex
    uint32_t qlabel[kMaxK] = {};  // labels (if use_labels)
    bool use_labels = false;
    int qdeg[kMaxK] = {};

    // symmetry breaking: "constraints on node ID values", Grochow-Kellis
    bool symmetric = false;
    std::vector<std::pair<int, int>> conds;  // (a, b): f(a) ≺ f(b)
    uint64_t aut_size = 1;
    std::vector<std::vector<int8_t>> aut_list;  // all automorphisms (sigma[u]) if listed
    bool aut_list_complete = false;

    // order (Compute_query_node_sequence_info)
    int order[kMaxK] = {};    // position -> query vertex
    int pos[kMaxK] = {};      // query vertex -> position
    int parent[kMaxK] = {};   // position -> earlier position (spanning tree)
    uint32_t backward[kMaxK] = {};  // position -> mask of earlier adjacent positions (nn + ne)
};

// Validates and loads a gsm_query (connected; no loops/dups).
// Returns GSM_OK or GSM_ERR_INVALID_QUERY / GSM_ERR_INVALID_ARGUMENT with msg.
gsm_status load_query(const gsm_query* q, QueryPlan* plan, std::string* msg);

// Aut(Q) order, GK conditions, optional automorphism list (<= list_cap).
void compute_symmetry(QueryPlan* plan, bool with_conditions, size_t list_cap);

// Greedy order: max d_M, min |C(u)|, max deg, min id (cand may be NULL).
// forced_first >= 0 pins position 0 (root-subset sampling).
void compute_order(QueryPlan* plan, const uint64_t* cand, int forced_first);

// COUNT mode: if Q has two non-adjacent vertices a, b with no symmetry condition between
// them and Q - {a, b} connected, order Q - {a, b} greedily and put a, b last (the "pair
// tail": their candidate sets are independent given the rest).  Returns false otherwise.
// forced_first >= 0 keeps that query vertex at position 0 (root-subset sampling).
bool compute_order_pair_tail(QueryPlan* plan, const uint64_t* cand, int forced_first = -1);

// ----------------------------------------------------------------------------
// Per-level device plan (Verify_Constraints at position i, Alg. 1 lines 10-14)
// ----------------------------------------------------------------------------
struct LevelPlan {
    int32_t width;       // i: columns of an input row (positions 0..i-1)
    int32_t qv;          // query vertex π[i]: cmask bit to test
    int32_t check_mask;  // 0 when the cmask bit is implied (no labels, deg_Q <= |B(i)|)
    int32_t nb;          // |B(i)|: earlier positions adjacent to π[i]
    int32_t bpos[kMaxK];
    int32_t nlo;         // positions j with f(π[j]) ≺ f(π[i])  (candidate must be larger)
    int32_t lo[kMaxK];
    int32_t nhi;         // positions j with f(π[i]) ≺ f(π[j])  (candidate must be smaller)
    int32_t hi[kMaxK];
    int32_t ninj;        // positions needing an explicit injectivity compare
    int32_t inj[kMaxK];
    int32_t count_only;  // last level in COUNT mode: count survivors, write nothing
    // label-grouped lists (set by the driver when the graph has them and Q is labeled):
    // candidates are keys key_base | id in the (label, id)-sorted lists; idmask decodes
    int32_t keyed;
    int32_t key_base;
    int32_t idmask;
    // keyed lists: key of each backward neighbour's image in OTHER lists = its query label <<
    // idbits (-1: unknown / not keyed -> plain ids); lets a membership test search the shorter list
    int32_t bkey[kMaxK];
    // k-look-ahead (DESIGN R17): the unmapped query neighbours of π[i]
    int32_t la_depth;    // 0 (off), 1 or 2
    int32_t nla;
    int32_t la_u[kMaxK];
    // level-1 sharding (GSM_FLAG_SHARD_LEVEL1, position 1 only): keep the survivors v of row r
    // with pair_shard(f_r(0), v, shard_p) == shard_s; shard_p <= 1 = off
    int32_t shard_p;
    int32_t shard_s;
};

#ifdef __CUDACC__
#define GSM_HD __host__ __device__ __forceinline__
#else
#define GSM_HD inline
#endif
GSM_HD int32_t pair_shard(int32_t a, int32_t b, int32_t P) {
    uint32_t h = (uint32_t)a * 0x9E3779B1u ^ ((uint32_t)b + 0x7F4A7C15u) * 0x85EBCA6Bu;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    return (int32_t)(h % (uint32_t)P);
}

LevelPlan make_level_plan(const QueryPlan& p, int i, bool count_only);

}  // namespace gsm
