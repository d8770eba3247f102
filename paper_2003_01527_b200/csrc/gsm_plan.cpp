// gsm_plan.cpp — host query plan (Alg. 1 "PreCompute_on_CPUs").
//
//  * compute_order: "the query order is determined in the following priority
//    order: d_M, P_f, and deg ... If all three are equal, the order is chosen
//    arbitrarily".  P_f(u) (VF3's probability that a data vertex is
//    compatible: same label, degree >= deg(u)) is replaced by the exact
//    integer |C(u)| = n * P_f(u) measured by the filter kernel, so no float ties
//    (reading R7).  d_M(u) = edges from u into already-ordered vertices
//    (P:130), updated after every pick; ties -> lowest query id.  The first pick
//    has d_M = 0 everywhere and is decided by (|C(u)|, -deg, id).
//  * Spanning-tree parent = earliest-ordered neighbour ("nn", Alg. 1 line 3,
//    P:131); all other backward edges are the non-tree edges ("ne", line 4).
//  * compute_symmetry: "a set of constraints on node ID values of the query
//    graph in order to avoid generating partial results, which eventually
//    become duplicated combinations".  The paper gives no construction;
//    we use the Grochow-Kellis stabiliser chain (reading R9):
//      A := Aut(Q); while |A| > 1: u := smallest id with |orbit_A(u)| > 1;
//      add f(u) ≺ f(w) for every other w in orbit_A(u); A := Stab_A(u).
//    |Aut(Q)| = product of the orbit sizes (orbit-stabiliser theorem).
#include <algorithm>
#include <cstring>
#include <string>

#include "gsm_internal.h"

namespace gsm {

static inline bool qadj(const QueryPlan& p, int a, int b) { return (p.adj[a] >> b) & 1u; }

gsm_status load_query(const gsm_query* q, QueryPlan* plan, std::string* msg) {
    *plan = QueryPlan();
    if (!q) { *msg = "query is NULL"; return GSM_ERR_INVALID_ARGUMENT; }
    const int k = q->num_nodes;
    if (k < 1 || k > kMaxK) { *msg = "query must have 1..32 vertices"; return GSM_ERR_INVALID_QUERY; }
    if (q->num_edges < 0 || (q->num_edges > 0 && !q->edges)) { *msg = "bad query edge list"; return GSM_ERR_INVALID_QUERY; }
    plan->k = k;
    for (int e = 0; e < q->num_edges; ++e) {
        int a = q->edges[2 * e], b = q->edges[2 * e + 1];
        if (a < 0 || b < 0 || a >= k || b >= k) { *msg = "query edge endpoint out of range"; return GSM_ERR_INVALID_QUERY; }
        if (a == b) { *msg = "query self-loop"; return GSM_ERR_INVALID_QUERY; }
        if (qadj(*plan, a, b)) { *msg = "duplicate query edge"; return GSM_ERR_INVALID_QUERY; }
        plan->adj[a] |= 1u << b;
        plan->adj[b] |= 1u << a;
    }
    for (int u = 0; u < k; ++u) plan->qdeg[u] = __builtin_popcount(plan->adj[u]);
    // connectivity (frontier expansion presumes a connected query)
    uint32_t seen = 1u, frontier = 1u;
    while (frontier) {
        uint32_t next = 0;
        for (int u = 0; u < k; ++u)
            if ((frontier >> u) & 1u) next |= plan->adj[u];
        frontier = next & ~seen;
        seen |= next;
    }
    const uint32_t all = (k == 32) ? 0xffffffffu : ((1u << k) - 1u);
    if ((seen & all) != all) { *msg = "query graph is disconnected"; return GSM_ERR_INVALID_QUERY; }
    if (q->labels) {
        plan->use_labels = true;
        for (int u = 0; u < k; ++u) plan->qlabel[u] = q->labels[u];
    }
    return GSM_OK;
}

// ---------------------------------------------------------------- automorphisms
namespace {

struct AutSearch {
    const QueryPlan& p;
    int8_t sigma[kMaxK];
    int8_t prescribed[kMaxK];  // -1 = free
    uint32_t used = 0;
    // listing mode
    std::vector<std::vector<int8_t>>* out = nullptr;
    size_t cap = 0;
    bool overflow = false;

    explicit AutSearch(const QueryPlan& plan) : p(plan) {
        for (int u = 0; u < kMaxK; ++u) prescribed[u] = -1;
    }

    bool compatible(int u, int w) const {
        if (p.qdeg[u] != p.qdeg[w]) return false;
        if (p.use_labels && p.qlabel[u] != p.qlabel[w]) return false;
        for (int x = 0; x < u; ++x)
            if (qadj(p, u, x) != qadj(p, w, sigma[x])) return false;
        return true;
    }

    // returns true when a complete automorphism was found (existence mode)
    bool run(int u) {
        if (u == p.k) {
            if (!out) return true;
            if (out->size() >= cap) { overflow = true; return true; }
            out->emplace_back(sigma, sigma + p.k);
            return false;  // keep enumerating
        }
        int lo = 0, hi = p.k;
        if (prescribed[u] >= 0) { lo = prescribed[u]; hi = lo + 1; }
        for (int w = lo; w < hi; ++w) {
            if ((used >> w) & 1u) continue;
            if (!compatible(u, w)) continue;
            sigma[u] = (int8_t)w;
            used |= 1u << w;
            bool done = run(u + 1);
            used &= ~(1u << w);
            if (done) return true;
        }
        return false;
    }
};

// Is there an automorphism fixing every vertex in `fixed` and mapping u -> w?
bool exists_aut(const QueryPlan& p, uint32_t fixed, int u, int w) {
    AutSearch s(p);
    for (int x = 0; x < p.k; ++x)
        if ((fixed >> x) & 1u) s.prescribed[x] = (int8_t)x;
    if (((fixed >> u) & 1u) && u != w) return false;
    s.prescribed[u] = (int8_t)w;
    return s.run(0);
}

}  // namespace

void compute_symmetry(QueryPlan* plan, bool with_conditions, size_t list_cap) {
    QueryPlan& p = *plan;
    p.conds.clear();
    p.aut_size = 1;
    uint32_t fixed = 0;
    // stabiliser chain
    for (;;) {
        int chosen = -1;
        std::vector<int> orbit;
        for (int u = 0; u < p.k && chosen < 0; ++u) {
            if ((fixed >> u) & 1u) continue;
            std::vector<int> orb;
            for (int w = 0; w < p.k; ++w)
                if (w == u || exists_aut(p, fixed, u, w)) orb.push_back(w);
            if (orb.size() > 1) { chosen = u; orbit = orb; }
        }
        if (chosen < 0) break;
        p.aut_size *= (uint64_t)orbit.size();
        for (int w : orbit)
            if (w != chosen) p.conds.emplace_back(chosen, w);
        fixed |= 1u << chosen;
    }
    p.symmetric = with_conditions && !p.conds.empty();
    if (!with_conditions) p.conds.clear();
    // explicit automorphism list (for Aut-expansion of enumerated representatives)
    p.aut_list.clear();
    p.aut_list_complete = false;
    if (list_cap > 0 && p.aut_size <= list_cap) {
        AutSearch s(p);
        s.out = &p.aut_list;
        s.cap = list_cap;
        s.run(0);
        p.aut_list_complete = !s.overflow && p.aut_list.size() == p.aut_size;
    }
}

// ---------------------------------------------------------------- order
// Greedy order of the query vertices not in `excluded`, then `tail` (in order).
static void order_greedy(QueryPlan& p, const uint64_t* cand, int forced_first, uint32_t excluded,
                         const int* tail, int ntail) {
    uint32_t placed = 0;
    const int nfree = p.k - ntail;
    for (int i = 0; i < nfree; ++i) {
        int best = -1;
        int best_dm = -1;
        for (int u = 0; u < p.k; ++u) {
            if (((placed | excluded) >> u) & 1u) continue;
            int dm = __builtin_popcount(p.adj[u] & placed);
            if (i > 0 && dm == 0) continue;  // keep the prefix connected
            if (best < 0) { best = u; best_dm = dm; continue; }
            uint64_t cu = cand ? cand[u] : 0, cb = cand ? cand[best] : 0;
            bool better;
            if (dm != best_dm) better = dm > best_dm;                  // max d_M
            else if (cu != cb) better = cu < cb;                       // min P_f (= |C(u)|/n)
            else if (p.qdeg[u] != p.qdeg[best]) better = p.qdeg[u] > p.qdeg[best];  // max deg
            else better = false;                                        // min id (scan order)
            if (better) { best = u; best_dm = dm; }
        }
        if (i == 0 && forced_first >= 0) best = forced_first;
        p.order[i] = best;
        p.pos[best] = i;
        placed |= 1u << best;
    }
    for (int t = 0; t < ntail; ++t) {
        p.order[nfree + t] = tail[t];
        p.pos[tail[t]] = nfree + t;
    }
    for (int i = 0; i < p.k; ++i) {
        int u = p.order[i];
        p.backward[i] = 0;
        p.parent[i] = -1;
        for (int j = 0; j < i; ++j)
            if (qadj(p, u, p.order[j])) {
                p.backward[i] |= 1u << j;
                if (p.parent[i] < 0) p.parent[i] = j;  // earliest-ordered neighbour
            }
    }
}

void compute_order(QueryPlan* plan, const uint64_t* cand, int forced_first) {
    order_greedy(*plan, cand, forced_first, 0u, nullptr, 0);
}

// vertices of `mask` connected in Q (restricted to mask)
static bool connected_within(const QueryPlan& p, uint32_t mask) {
    if (!mask) return false;
    uint32_t seen = mask & (~mask + 1u), frontier = seen;
    while (frontier) {
        uint32_t next = 0;
        for (int u = 0; u < p.k; ++u)
            if ((frontier >> u) & 1u) next |= p.adj[u] & mask;
        frontier = next & ~seen;
        seen |= next;
    }
    return seen == mask;
}

bool compute_order_pair_tail(QueryPlan* plan, const uint64_t* cand, int forced_first) {
    QueryPlan& p = *plan;
    if (p.k < 3) return false;
    const uint32_t all = p.k == 32 ? 0xffffffffu : ((1u << p.k) - 1u);
    int ba = -1, bb = -1;
    double bestv = -1;
    for (int a = 0; a < p.k; ++a)
        for (int b = a + 1; b < p.k; ++b) {
            if (qadj(p, a, b)) continue;
            if (a == forced_first || b == forced_first) continue;  // π[0] is pinned (root_subset)
            bool cond = false;
            for (auto& c : p.conds)
                if ((c.first == a && c.second == b) || (c.first == b && c.second == a)) cond = true;
            if (cond) continue;
            if (!connected_within(p, all & ~((1u << a) | (1u << b)))) continue;
            const double v = cand ? (double)cand[a] * (double)cand[b] : 1.0;
            if (v > bestv) { bestv = v; ba = a; bb = b; }
        }
    if (ba < 0) return false;
    const int tail[2] = {ba, bb};
    order_greedy(p, cand, forced_first, (1u << ba) | (1u << bb), tail, 2);
    return true;
}

LevelPlan make_level_plan(const QueryPlan& p, int i, bool count_only) {
    LevelPlan L;
    std::memset(&L, 0, sizeof(L));
    L.width = i;
    L.qv = p.order[i];
    L.count_only = count_only ? 1 : 0;
    uint32_t covered = 0;
    for (int j = 0; j < i; ++j)
        if ((p.backward[i] >> j) & 1u) { L.bpos[L.nb++] = j; covered |= 1u << j; }
    if (p.symmetric)
        for (auto& c : p.conds) {
            int pa = p.pos[c.first], pb = p.pos[c.second];
            if (pb == i && pa < i) { L.lo[L.nlo++] = pa; covered |= 1u << pa; }  // f(a) ≺ v
            if (pa == i && pb < i) { L.hi[L.nhi++] = pb; covered |= 1u << pb; }  // v ≺ f(b)
        }
    // adjacency (no self-loops) and strict ID bounds already imply v != f(j)
    for (int j = 0; j < i; ++j)
        if (!((covered >> j) & 1u)) L.inj[L.ninj++] = j;
    L.check_mask = (p.use_labels || p.qdeg[L.qv] > L.nb) ? 1 : 0;
    L.keyed = 0;
    L.key_base = 0;
    L.idmask = -1;
    for (int q = 0; q < kMaxK; ++q) L.bkey[q] = 0;  // plain lists: a vertex's key is its id
    return L;
}

}  // namespace gsm
