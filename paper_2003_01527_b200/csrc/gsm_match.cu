// gsm_match.cu — gsm_match: the GSM driver (Alg. 1).
//
//   PreCompute_on_CPUs (lines 1-5)   -> gsm_plan.cpp (order, nn, ne, ID constraints)
//   Filter_candidate_set (lines 6-9) -> K1 filter kernel + root compaction
//   while |M[i]| < |Q| (lines 10-15) -> per position i: plan_rows, scan,
//                                       merge-path partition, fused expand kernel
//   return |M|/|Q| and M (line 16)   -> count reduction / finalize (id map,
//                                       Aut-expansion, lexicographic sort)
//
// Chunked frontier ("memory linear to
// matched subgraphs"): a position's work space (rows + candidate items, i.e.
// its merge-path diagonals) is cut into chunks no larger than the next level's
// row capacity.  Survivors <= candidate items, so a chunk can never overflow;
// each chunk's output is consumed depth-first before the next chunk runs.
#include <chrono>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

#include "gsm_common.h"
#include "gsm_kernels.h"
#include "gsm_workspace.h"

namespace gsm {

const DevGraph& graph_of(const gsm_graph* h);
int device_of(const gsm_graph* h);
cudaStream_t stream_of(const gsm_graph* h);
bool labeled_of(const gsm_graph* h);
Workspace& workspace_of(const gsm_graph* h);

namespace {

using Clock = std::chrono::steady_clock;
inline double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// Per-kernel CUDA-event bracketing (GSM_FLAG_PROFILE) + launch accounting.
struct Recorder {
    bool prof = false;
    cudaStream_t s = 0;
    gsm_result* res = nullptr;
    struct Mark { int kind; cudaEvent_t a, b; };
    std::vector<Mark> marks;
    ~Recorder() {
        for (auto& m : marks) {
            cudaEventDestroy(m.a);
            cudaEventDestroy(m.b);
        }
    }
    template <class F>
    void run(int kind, int launches, F&& f) {
        res->kernel_launches += launches;
        res->prof[kind].launches += launches;
        if (!prof) { f(); return; }
        Mark m{kind, nullptr, nullptr};
        GSM_CUDA(cudaEventCreate(&m.a));
        GSM_CUDA(cudaEventCreate(&m.b));
        marks.push_back(m);
        GSM_CUDA(cudaEventRecord(m.a, s));
        f();
        GSM_CUDA(cudaEventRecord(m.b, s));
    }
    void finish() {
        if (!prof) return;
        GSM_CUDA(cudaStreamSynchronize(s));
        for (auto& m : marks) {
            float ms = 0;
            GSM_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
            res->prof[m.kind].ms += ms;
        }
    }
};

template <typename T>
T read_scalar(const T* dptr, cudaStream_t s) {
    T h{};
    const auto t0 = Clock::now();
    GSM_CUDA(cudaMemcpyAsync(&h, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    GSM_CUDA(cudaStreamSynchronize(s));
    g_trace.sync_ms += ms_since(t0);
    g_trace.syncs++;
    return h;
}

class Matcher {
   public:
    Matcher(const gsm_graph* gh, QueryPlan& plan, const gsm_match_opts& o, gsm_result* res, cudaStream_t s)
        : g_(graph_of(gh)), plan_(plan), opts_(o), res_(res), s_(s), ws_(workspace_of(gh)), lv_(ws_.lv),
          cmask_(ws_.cmask), final_count_(ws_.final_count), stats_(ws_.stats), ovf_idx_(ws_.ovf_idx),
          ovf_rows_(ws_.ovf_rows), ovf_n_(ws_.ovf_n) {
        rec_.prof = (o.flags & GSM_FLAG_PROFILE) != 0;
        rec_.s = s;
        rec_.res = res;
    }

    void run();

   private:
    void process(int w, const Frontier& F, int64_t R);
    void ensure_caps();
    void process_generic(int w, const Frontier& F, int64_t R);
    void process_tail(int w, const Frontier& F, int64_t R);
    void process_pair(int w, const Frontier& F, int64_t R);
    static Frontier plain(const int32_t* rows, int w) {
        Frontier f;
        f.W = w;
        f.rows = rows;
        return f;
    }
    bool tail_eligible(TailArgs* ta) const;
    bool clique_eligible() const;
    void append_output(const int32_t* rows, int64_t R);
    void finalize();

    const DevGraph& g_;
    QueryPlan& plan_;
    const gsm_match_opts& opts_;
    gsm_result* res_;
    cudaStream_t s_;
    Recorder rec_;

    Workspace& ws_;                                 // per-graph buffers, reused across matches
    std::vector<std::unique_ptr<LevelBufs>>& lv_;   // index = width 1..k
    DevBuf<uint8_t>& cmask_;
    DevBuf<unsigned long long>& final_count_;       // COUNT mode: survivors at the last level
    DevBuf<unsigned long long>& stats_;             // 5 per width (+ tail slot)
    DevBuf<int64_t>& ovf_idx_;
    DevBuf<int32_t>& ovf_rows_;
    DevBuf<unsigned long long>& ovf_n_;
    int k_ = 0;
    int mask_bytes_ = 1;
    bool count_mode_ = true;
    std::vector<LevelPlan> lplan_;
    DevBuf<int32_t> arena_;                       // ENUMERATE: rows in position order, new ids
    int64_t arena_rows_ = 0;
    int64_t budget_ = 0;
    double t_expand_ms_ = 0;
    bool tail_ = false;        // fuse the last two positions (COUNT mode)
    TailArgs tail_args_;
    double tail_rows_ = 0;     // rows handled by the fused tail
    bool clique_ = false;      // K3/K4 COUNT: per-root local bitmaps (gsm_clique.cu)
    bool pair_ = false;        // COUNT: last two positions independent (k_pair)
    LevelPlan lq_;             // plan of position k-1 over rows of width k-2 (pair tail)
    double pair_rows_ = 0;
    bool compress_ = false;    // intermediate frontiers as (parent, vertex) pairs
    bool deferred_counts_ = false;
    bool caps_ready_ = false;  // |C(u)| read back with the result (unlabeled queries)
};

void Matcher::run() {
    const auto t_all = Clock::now();
    k_ = plan_.k;
    count_mode_ = opts_.mode == GSM_MODE_COUNT;
    mask_bytes_ = mask_bytes_for(k_);

    // ---- Filter_candidate_set (Alg. 1 lines 6-9): K1 over every data vertex
    auto t0 = Clock::now();
    FilterQuery fq;
    std::memset(&fq, 0, sizeof(fq));
    fq.k = k_;
    fq.use_labels = plan_.use_labels ? 1 : 0;
    for (int u = 0; u < k_; ++u) {
        fq.qlabel[u] = plan_.qlabel[u];
        fq.qdeg[u] = plan_.qdeg[u];
        fq.qadj[u] = plan_.adj[u];
    }
    cmask_.ensure((size_t)g_.n * mask_bytes_, s_);
    DevBuf<unsigned long long>& counts = ws_.counts;
    counts.ensure(kMaxK, s_);
    GSM_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * kMaxK, s_));
    rec_.run(GSM_K_FILTER, 1, [&] { launch_filter(g_, fq, cmask_.p, counts.p, s_); });
    res_->prof[GSM_K_FILTER].alg_bytes +=
        (double)g_.n * (8.0 + (plan_.use_labels ? 4.0 : 0.0) + mask_bytes_);
    if (opts_.refine_rounds > 0) {  // Alg. 1 lines 7-8: NE filter + refinement rounds
        int64_t hqne[kMaxK] = {};
        for (int u = 0; u < k_; ++u)
            for (int w = 0; w < k_; ++w)
                if ((plan_.adj[u] >> w) & 1u) hqne[u] += plan_.use_labels ? (int64_t)plan_.qlabel[w] + 1 : 1;
        DevBuf<int64_t> dqne;
        DevBuf<uint8_t> tmp;
        dqne.ensure(kMaxK, s_);
        tmp.ensure((size_t)g_.n * mask_bytes_, s_);
        GSM_CUDA(cudaMemcpyAsync(dqne.p, hqne, sizeof(hqne), cudaMemcpyHostToDevice, s_));
        rec_.run(GSM_K_FILTER, 2 * opts_.refine_rounds + 1,
                 [&] { launch_refine(g_, fq, dqne.p, opts_.refine_rounds, cmask_.p, tmp.p, counts.p, s_); });
        res_->prof[GSM_K_FILTER].alg_bytes +=
            opts_.refine_rounds * ((double)g_.nnz * (4.0 + mask_bytes_ + (plan_.use_labels ? 4.0 : 0.0)) +
                                   (double)g_.n * (16.0 + 3.0 * mask_bytes_)) + (double)g_.n * mask_bytes_;
    }
    uint64_t cand[kMaxK];
    bool empty = false;
    // Unlabeled query without refinement: |C(u)| = #{v : deg(v) >= deg_Q(u)} is non-increasing
    // in deg_Q(u), so the order (max d_M, min |C(u)|, max deg, min id) is the order by (max d_M,
    // max deg, min id) and C(u) is empty iff deg_Q(u) > max degree: the counts are not needed
    // before the search, and are read back with the result (one host sync fewer per match).
    deferred_counts_ = !plan_.use_labels && opts_.refine_rounds == 0;
    if (deferred_counts_) {
        for (int u = 0; u < k_; ++u) {
            cand[u] = (uint64_t)(kMaxK + 1 - plan_.qdeg[u]);  // order-equivalent proxy
            if (plan_.qdeg[u] > g_.max_degree) empty = true;
        }
    } else {
        unsigned long long hc[kMaxK];
        GSM_CUDA(cudaMemcpyAsync(hc, counts.p, sizeof(hc), cudaMemcpyDeviceToHost, s_));
        GSM_CUDA(cudaStreamSynchronize(s_));
        for (int u = 0; u < k_; ++u) {
            cand[u] = hc[u];
            res_->candidates[u] = hc[u];
            if (hc[u] == 0) empty = true;
        }
    }
    // ---- query order with the exact |C(u)|
    compute_order(&plan_, cand, opts_.root_subset ? 0 : -1);
    {   // COUNT mode: order the two last positions as an independent pair when Q allows it
        // (under root_subset the pair keeps π[0] = query vertex 0 in front)
        if (count_mode_ && k_ >= 3 && knobs().pair_tail)
            pair_ = compute_order_pair_tail(&plan_, cand, opts_.root_subset ? 0 : -1);
    }
    for (int i = 0; i < k_; ++i) res_->order[i] = plan_.order[i];
    res_->num_levels = k_;
    res_->width = k_;
    for (int w = 0; w <= k_; ++w) {  // reuse the graph's grow-only buffers; reset per-match state
        lv_[w]->cap_rows = 0;
        lv_[w]->stats = nullptr;
        lv_[w]->rows_in = 0;
    }
    lplan_.resize(k_);
    for (int i = 1; i < k_; ++i) {
        LevelPlan& L = lplan_[i];
        L = make_level_plan(plan_, i, count_mode_ && i == k_ - 1);
        if (opts_.refine_rounds > 0) L.check_mask = 1;  // NE-refined cmask is stronger than the degree test
        if (plan_.use_labels && g_.lkeys && plan_.qlabel[L.qv] <= g_.max_label) {
            L.keyed = 1;
            L.key_base = (int32_t)(plan_.qlabel[L.qv] << g_.idbits);
            L.idmask = (int32_t)((1u << g_.idbits) - 1u);
            // the label is implied by the key range; the degree by |B(i)| unless NE-refined
            L.check_mask = (opts_.refine_rounds > 0 || plan_.qdeg[L.qv] > L.nb) ? 1 : 0;
            for (int q = 0; q < L.nb; ++q) {
                const uint32_t lb = plan_.qlabel[plan_.order[L.bpos[q]]];
                L.bkey[q] = lb <= g_.max_label ? (int32_t)(lb << g_.idbits) : -1;
            }
        } else if (plan_.use_labels && g_.lkeys) {
            for (int q = 0; q < L.nb; ++q) L.bkey[q] = -1;  // plain list of an unkeyed label: no swap
        }
    }

    // ---- k-look-ahead: per position, the unmapped query neighbours of π[i]
    {
        const int la = knobs().lookahead >= 0 ? knobs().lookahead : opts_.lookahead;
        bool any = false;
        for (int i = 1; i < k_; ++i) {
            LevelPlan& L = lplan_[i];
            L.nla = 0;
            L.la_depth = la;
            if (la <= 0) continue;
            for (int p = i + 1; p < k_; ++p) {
                const int u = plan_.order[p];
                if ((plan_.adj[plan_.order[i]] >> u) & 1u) L.la_u[L.nla++] = u;
            }
            any |= L.nla > 0;
        }
        if (any && !empty) {
            ws_.la_c1.ensure((size_t)g_.n * k_, s_);
            rec_.run(GSM_K_FILTER, 1, [&] { launch_la_counts(g_, k_, mask_bytes_, cmask_.p, ws_.la_c1.p, s_); });
            res_->prof[GSM_K_FILTER].alg_bytes += (double)g_.nnz * (4.0 + mask_bytes_) + (double)g_.n * (16.0 + k_);
            if (la >= 2) {
                // D(u) = query neighbours of u placed after u; ok1[w] bit u = w hosts u and has a
                // candidate neighbour for every vertex of D(u)
                uint32_t dmask[kMaxK] = {};
                for (int u = 0; u < k_; ++u)
                    for (int w = 0; w < k_; ++w)
                        if (((plan_.adj[u] >> w) & 1u) && plan_.pos[w] > plan_.pos[u]) dmask[u] |= 1u << w;
                ws_.la_ok1.ensure((size_t)g_.n * mask_bytes_, s_);
                ws_.la_c2.ensure((size_t)g_.n * k_, s_);
                rec_.run(GSM_K_FILTER, 2, [&] {
                    launch_la_ok1(g_, k_, mask_bytes_, cmask_.p, ws_.la_c1.p, dmask, ws_.la_ok1.p, s_);
                    launch_la_counts(g_, k_, mask_bytes_, ws_.la_ok1.p, ws_.la_c2.p, s_);
                });
                res_->prof[GSM_K_FILTER].alg_bytes += (double)g_.n * (2.0 * mask_bytes_ + k_) +
                                                      (double)g_.nnz * (4.0 + mask_bytes_) + (double)g_.n * (16.0 + k_);
            }
        } else {
            for (int i = 1; i < k_; ++i) lplan_[i].nla = 0;
        }
    }

    tail_ = tail_eligible(&tail_args_);
    clique_ = clique_eligible();
    if (pair_) {
        tail_ = false;
        lq_ = lplan_[k_ - 1];
        lq_.width = k_ - 2;  // rows of the first k-2 positions; q never refers to p = k-2
        int n = 0;
        for (int t = 0; t < lq_.ninj; ++t)
            if (lq_.inj[t] != k_ - 2) lq_.inj[n++] = lq_.inj[t];
        lq_.ninj = n;
    }

    // ---- level-1 sharding (GSM_FLAG_SHARD_LEVEL1): every rank takes all roots and keeps its
    //      share of the (f(π[0]), f(π[1])) pairs, where level 1 is a breadth-first expand
    const bool level1 = (opts_.flags & GSM_FLAG_SHARD_LEVEL1) && opts_.num_shards > 1 && !opts_.root_subset &&
                        !clique_ && k_ >= 3 && !((pair_ || tail_) && k_ - 2 == 1);
    if (level1) {
        lplan_[1].shard_p = opts_.num_shards;
        lplan_[1].shard_s = opts_.shard_index;
    }
    res_->level1_sharded = level1 ? 1 : 0;

    // ---- roots = C(π[0]) (level-0 frontier)
    int64_t R0 = 0;
    if (!empty && (int64_t)k_ <= g_.n) {
        const int bit = plan_.order[0];
        if (opts_.root_subset) {
            DevBuf<int32_t> sub;
            sub.ensure(opts_.root_subset_len, s_);
            GSM_CUDA(cudaMemcpyAsync(sub.p, opts_.root_subset, sizeof(int32_t) * opts_.root_subset_len,
                                     cudaMemcpyHostToDevice, s_));
            lv_[1]->rows.ensure(opts_.root_subset_len, s_);
            rec_.run(GSM_K_ROOTS, 1, [&] {
                R0 = launch_root_subset(g_, cmask_.p, mask_bytes_, bit, sub.p, opts_.root_subset_len,
                                        lv_[1]->rows.p, s_);
            });
        } else {
            const int nsh = (opts_.num_shards > 1 && !level1) ? opts_.num_shards : 1;
            const int sh = nsh > 1 ? opts_.shard_index : 0;
            lv_[1]->rows.ensure(g_.n, s_);
            rec_.run(GSM_K_ROOTS, 3, [&] {
                R0 = launch_roots(g_, cmask_.p, mask_bytes_, bit, sh, nsh, lv_[1]->rows.p, s_);
            });
        }
        res_->prof[GSM_K_ROOTS].alg_bytes += 2.0 * (double)g_.n * mask_bytes_ + 4.0 * (double)R0;
    }
    res_->level_rows[0] = (uint64_t)R0;
    res_->level_frontier_bytes[0] = 4 * (uint64_t)R0;
    res_->ms_filter = (float)ms_since(t0);

    // ---- verify iterations (Alg. 1 lines 10-15)
    t0 = Clock::now();
    final_count_.ensure(1, s_);
    GSM_CUDA(cudaMemsetAsync(final_count_.p, 0, sizeof(unsigned long long), s_));
    stats_.ensure(5 * (kMaxK + 1), s_);
    GSM_CUDA(cudaMemsetAsync(stats_.p, 0, sizeof(unsigned long long) * 5 * (kMaxK + 1), s_));
    for (int w = 1; w < k_; ++w) lv_[w]->stats = stats_.p + 5 * w;

    uint64_t found = 0;
    if (k_ == 1) {
        found = (uint64_t)R0;
        if (!count_mode_ && R0 > 0) append_output(lv_[1]->rows.p, R0);
    } else if (R0 > 0 && clique_) {
        CliqueRun cr;
        cr.k = k_;
        cr.roots = lv_[1]->rows.p;
        cr.R = R0;
        cr.off = g_.off;
        cr.cols = g_.cols;
        cr.up = g_.up;
        cr.count = final_count_.p;
        cr.stats = stats_.p;  // slot 0 (the frontier levels use slots 1..k-1, the tail slot kMaxK)
        DevBuf<int32_t>& over = ws_.ck_over;
        over.ensure(R0, s_);
        cr.over_roots = over.p;
        cr.ws = &ws_;
        cr.hub_bits = g_.hub_bits;
        cr.hub_base = g_.hub_base;
        cr.hub_words = g_.hub_words;
        cr.nh_off = g_.nh_off;
        cr.nplus = g_.nplus;
        cr.nh_tab = g_.nh_tab;
        int64_t launches = 0;
        rec_.run(GSM_K_CLIQUE, 1, [&] { launches = run_clique(cr, s_); });
        res_->kernel_launches += launches > 0 ? launches - 1 : 0;
        res_->num_chunks++;
        // roots whose N+(u) exceeds the per-CTA tables: the breadth-first path (same counter)
        if (cr.n_over > 0) process(1, plain(over.p, 1), cr.n_over);
    } else if (R0 > 0) {
        process(1, plain(lv_[1]->rows.p, 1), R0);
    }
    // one host sync for the result: final count, per-level stats, deferred |C(u)|
    // (pinned staging, so the copies are truly asynchronous and share the one sync)
    std::vector<unsigned long long> hv(Workspace::kPin, 0);
    unsigned long long* hp = ws_.pinned();
    if (!hp) hp = hv.data();  // pageable fallback: each copy then blocks by itself
    unsigned long long *hfound = hp, *hcand = hp + 1, *hstat = hp + 1 + kMaxK;
    const size_t nstat = 5 * (kMaxK + 1);
    *hfound = 0;
    if (k_ > 1 && count_mode_ && R0 > 0)
        GSM_CUDA(cudaMemcpyAsync(hfound, final_count_.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s_));
    if (k_ > 1)
        GSM_CUDA(cudaMemcpyAsync(hstat, stats_.p, sizeof(unsigned long long) * nstat, cudaMemcpyDeviceToHost, s_));
    if (deferred_counts_)
        GSM_CUDA(cudaMemcpyAsync(hcand, counts.p, sizeof(unsigned long long) * kMaxK, cudaMemcpyDeviceToHost, s_));
    {
        const auto ts = Clock::now();
        GSM_CUDA(cudaStreamSynchronize(s_));
        g_trace.sync_ms += ms_since(ts);
        g_trace.syncs++;
    }
    if (deferred_counts_)
        for (int u = 0; u < k_; ++u) res_->candidates[u] = hcand[u];
    if (k_ > 1 && R0 > 0) found = count_mode_ ? (uint64_t)*hfound : (uint64_t)arena_rows_;
    std::vector<unsigned long long> hs(hstat, hstat + nstat);
    // per-level stats -> result + algorithmic bytes of the expand kernel
    if (k_ > 1) {
        double eb = 0;
        for (int w = 1; w < k_; ++w) {
            const unsigned long long* st = hs.data() + 5 * w;
            const LevelPlan& L = lplan_[w];
            // staged rows (entries, work offsets, pivot start + index, membership segments),
            // list entries read, cmask bytes, binary-search probes, survivor rows written
            eb += lv_[w]->rows_in * (4.0 * w + 8 + 8 + 1 + 12.0 * L.nb) + 4.0 * st[0] +
                  (double)mask_bytes_ * st[1] + 4.0 * st[2] + (L.count_only ? 0.0 : 4.0 * (w + 1) * st[3]);
            res_->level_work[w] = st[0];
            res_->level_rows[w] = st[3];  // partial results with w+1 matched positions
        }
        res_->prof[GSM_K_EXPAND].alg_bytes += eb;
        if (clique_) {
            // per root: id + packed N+ descriptor (4 + 16 B); per S(u) entry: the entry and its
            // descriptor (4 + 16 B); row items — list entries streamed, hub-bitmap words, keys
            // looked up — 4 B each; a hashed-N+ bucket probe (or binary-search probe) 32 B (the
            // bucket is one sector and the test must read all of it)
            const unsigned long long* st = hs.data();
            res_->prof[GSM_K_CLIQUE].alg_bytes +=
                20.0 * (double)R0 + 20.0 * (double)st[4] + 4.0 * (double)st[0] + 32.0 * (double)st[1];
            res_->level_work[k_ - 1] += st[0];
        }
        if (pair_) {  // staged row + both plans' segments; candidates and probes
            const unsigned long long* st = hs.data() + 5 * kMaxK;
            const int w = k_ - 2;
            res_->prof[GSM_K_TAIL].alg_bytes += pair_rows_ * (4.0 * w + 2 * 17.0 + 12.0 * (lplan_[w].nb + lq_.nb)) +
                                                4.0 * st[0] + 4.0 * st[2];
            res_->level_work[k_ - 1] += st[0];
        }
        if (tail_) {
            const unsigned long long* st = hs.data() + 5 * kMaxK;
            const int w = k_ - 2;
            const LevelPlan& L = lplan_[w];
            res_->prof[GSM_K_TAIL].alg_bytes +=
                tail_rows_ * (4.0 * w + 8 + 8 + 1 + 12.0 * L.nb) + 4.0 * st[0] + 4.0 * st[2];
            res_->level_work[k_ - 1] += st[0];
        }
    }
    if (k_ > 1 && count_mode_) res_->level_rows[k_ - 1] = found;
    res_->count_unique = found;
    const bool expand_orbits = plan_.symmetric && !(opts_.flags & GSM_FLAG_UNIQUE);
    res_->count = expand_orbits ? found * plan_.aut_size : found;
    res_->symmetric = plan_.symmetric ? 1 : 0;
    res_->ms_expand = (float)ms_since(t0);

    t0 = Clock::now();
    if (!count_mode_) finalize();
    res_->ms_finalize = (float)ms_since(t0);
    rec_.finish();
    res_->ms_total = (float)ms_since(t_all);
}

void Matcher::ensure_caps() {
    // frontier capacities (A7 chunking), computed on first use: matches that never expand a
    // breadth-first level (clique path, k = 1) skip the memory queries
    if (caps_ready_) return;
    caps_ready_ = true;
    size_t free_b = 0, total_b = 0;
    GSM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    {   // allocatable = free + what the stream-ordered pool holds but nobody uses + this graph's
        // cached frontier buffers (they are released and re-grown to the new chunk sizes);
        // default budget = min(total/4, 0.9 x allocatable), stable across calls
        int dev = 0;
        GSM_CUDA(cudaGetDevice(&dev));
        cudaMemPool_t pool;
        GSM_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t reserved = 0, used = 0;
        GSM_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
        GSM_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
        double cached = 0;
        for (int w = 2; w <= k_; ++w) cached += sizeof(int32_t) * (double)lv_[w]->rows.n;
        const double avail = 0.9 * ((double)free_b + (double)(reserved > used ? reserved - used : 0) + cached);
        budget_ = opts_.mem_budget_bytes ? (int64_t)opts_.mem_budget_bytes
                                         : (int64_t)std::min((double)total_b / 4.0, avail);
    }
    compress_ = ((opts_.flags & GSM_FLAG_COMPRESSED_PARTIALS) || knobs().compress > 0) && knobs().compress != 0;
    res_->compressed = compress_ ? 1 : 0;
    // per-width share of the budget for frontiers of width 2..k (k only when enumerating)
    const int nfront = count_mode_ ? std::max(0, k_ - 2) : k_ - 1;
    for (int w = 2; w <= k_; ++w) {
        const int64_t share = nfront > 0 ? budget_ / nfront : budget_;
        // stored partial result + its row plan (rbeg/rlen/P, piv, per-backward segments)
        const int64_t per_row = (compress_ && w < k_ ? 8 : 4 * w) + 8 * 3 + 1 + 1 + 12 * (w - 1);
        lv_[w]->cap_rows = std::max<int64_t>(share / per_row, 1);
    }

}

void Matcher::process(int w, const Frontier& F, int64_t R) {
    if (R <= 0) return;
    if (pair_ && w == k_ - 2) process_pair(w, F, R);
    else if (tail_ && w == k_ - 2) process_tail(w, F, R);
    else process_generic(w, F, R);
}

// Eligibility of the clique path: COUNT mode, K3 or K4, unlabeled, every position adjacent
// to all earlier ones, and the symmetry conditions chain f(π[0]) ≺ ... ≺ f(π[k-1]).
bool Matcher::clique_eligible() const {
    if (!knobs().clique) return false;
    if (!count_mode_ || (k_ != 3 && k_ != 4) || plan_.use_labels) return false;
    for (int i = 1; i < k_; ++i) {
        const LevelPlan& L = lplan_[i];
        if (plan_.backward[i] != (1u << i) - 1u) return false;
        if (L.keyed || L.nhi != 0 || L.nlo != i) return false;
    }
    return true;
}

// Eligibility of the fused tail: COUNT mode; B(k-1) = B(k-2) ∪ {k-2}; π[k-1] has the
// label of π[k-2] (or Q is unlabeled); π[k-1]'s ID bounds from earlier positions
// include π[k-2]'s (so RC(r) holds every admissible image of π[k-1]).
bool Matcher::tail_eligible(TailArgs* ta) const {
    if (!knobs().fused_tail) return false;
    if (!count_mode_ || k_ < 3) return false;
    const int c = k_ - 2, d = k_ - 1;
    if (plan_.backward[d] != (plan_.backward[c] | (1u << c))) return false;
    if (plan_.use_labels && plan_.qlabel[plan_.order[c]] != plan_.qlabel[plan_.order[d]]) return false;
    const LevelPlan &Lc = lplan_[c], &Ld = lplan_[d];
    if (Lc.keyed != Ld.keyed) return false;
    auto has = [](const int32_t* a, int n, int x) {
        for (int i = 0; i < n; ++i)
            if (a[i] == x) return true;
        return false;
    };
    for (int i = 0; i < Lc.nlo; ++i)
        if (!has(Ld.lo, Ld.nlo, Lc.lo[i])) return false;
    for (int i = 0; i < Lc.nhi; ++i)
        if (!has(Ld.hi, Ld.nhi, Lc.hi[i])) return false;
    std::memset(ta, 0, sizeof(*ta));
    ta->rel = has(Ld.lo, Ld.nlo, c) ? 1 : (has(Ld.hi, Ld.nhi, c) ? -1 : 0);
    for (int i = 0; i < Ld.nlo; ++i)
        if (Ld.lo[i] != c && !has(Lc.lo, Lc.nlo, Ld.lo[i])) ta->xlo[ta->nxlo++] = Ld.lo[i];
    for (int i = 0; i < Ld.nhi; ++i)
        if (Ld.hi[i] != c && !has(Lc.hi, Lc.nhi, Ld.hi[i])) ta->xhi[ta->nxhi++] = Ld.hi[i];
    return true;
}

void Matcher::process_tail(int w, const Frontier& F, int64_t R) {
    LevelBufs& B = *lv_[w];
    const LevelPlan& L = lplan_[w];
    B.rbeg.ensure(R, s_);
    B.rlen.ensure(R, s_);
    B.rpiv.ensure(R, s_);
    B.cbeg.ensure((size_t)R * L.nb, s_);
    B.clen.ensure((size_t)R * L.nb, s_);
    rec_.run(GSM_K_PLAN, 1, [&] { launch_plan_rows(g_, F, R, L, B.rbeg.p, B.rlen.p, B.rpiv.p, B.cbeg.p, B.clen.p, s_); });
    res_->prof[GSM_K_PLAN].alg_bytes += (double)R * (4.0 * w + 16.0 * L.nb + 12.0 * L.nb + 8 + 8 + 1);
    ovf_idx_.ensure(R, s_);
    ovf_n_.ensure(1, s_);
    GSM_CUDA(cudaMemsetAsync(ovf_n_.p, 0, sizeof(unsigned long long), s_));
    TailArgs a = tail_args_;
    a.F = F;
    a.R = R;
    a.rbeg = B.rbeg.p;
    a.rlen = B.rlen.p;
    a.rpiv = B.rpiv.p;
    a.cbeg = B.cbeg.p;
    a.clen = B.clen.p;
    a.off = g_.off;
    a.up = g_.up;
    a.cols = L.keyed ? g_.lkeys : g_.cols;
    a.cmask = cmask_.p;
    a.cap = tail_cap();
    a.bratio = tail_bratio();
    a.count = final_count_.p;
    a.overflow = ovf_idx_.p;
    a.noverflow = ovf_n_.p;
    ws_.sched.ensure(1, s_);
    GSM_CUDA(cudaMemsetAsync(ws_.sched.p, 0, sizeof(unsigned long long), s_));
    a.next = ws_.sched.p;
    DevBuf<unsigned long long> cyc;
    if (knobs().trace == 2) {
        cyc.ensure(8, s_);
        GSM_CUDA(cudaMemsetAsync(cyc.p, 0, sizeof(unsigned long long) * 8, s_));
        a.cyc = cyc.p;
    }
    a.stats = stats_.p + 5 * (kMaxK + 0);  // tail counters: slot kMaxK
    rec_.run(GSM_K_TAIL, 1, [&] { launch_tail(a, L, lplan_[w + 1], mask_bytes_, s_); });
    res_->num_chunks++;
    tail_rows_ += (double)R;
    int64_t nov = (int64_t)read_scalar(ovf_n_.p, s_);
    if (a.cyc) {
        unsigned long long hc[8];
        GSM_CUDA(cudaMemcpyAsync(hc, cyc.p, sizeof(hc), cudaMemcpyDeviceToHost, s_));
        GSM_CUDA(cudaStreamSynchronize(s_));
        std::fprintf(stderr, "[gsm tail] rows %lld: warp-cycles phase1 %.3g, small-RC pairs %.3g (%llu rows), "
                     "big-RC %.3g (%llu rows), overflow rows %lld\n", (long long)R, (double)hc[0], (double)hc[1],
                     hc[3], (double)hc[2], hc[4], (long long)nov);
    }
    if (nov > 0) {  // rows whose list did not fit a warp's buffer: one CTA per row
        DevBuf<int64_t> idx;
        idx.ensure(nov, s_);
        GSM_CUDA(cudaMemcpyAsync(idx.p, ovf_idx_.p, sizeof(int64_t) * nov, cudaMemcpyDeviceToDevice, s_));
        GSM_CUDA(cudaMemsetAsync(ovf_n_.p, 0, sizeof(unsigned long long), s_));
        sort_rows_by_len_desc(B.rlen.p, idx.p, nov, s_);  // largest rows first
        res_->kernel_launches += 5;
        GSM_CUDA(cudaMemsetAsync(ws_.sched.p, 0, sizeof(unsigned long long), s_));
        TailArgs b = a;
        b.R = nov;
        b.rows_idx = idx.p;
        b.cap = tail_block_cap();
        rec_.run(GSM_K_TAIL, 1, [&] { launch_tail_block(b, L, lplan_[w + 1], mask_bytes_, s_); });
        res_->num_chunks++;
        nov = (int64_t)read_scalar(ovf_n_.p, s_);
    }
    if (nov > 0) {  // still too big for a CTA: generic breadth-first path
        ovf_rows_.ensure((size_t)nov * w, s_);
        launch_gather_rows(F, ovf_idx_.p, nov, ovf_rows_.p, s_);
        res_->kernel_launches++;
        DevBuf<int32_t> rows;
        rows.ensure((size_t)nov * w, s_);
        GSM_CUDA(cudaMemcpyAsync(rows.p, ovf_rows_.p, sizeof(int32_t) * nov * w, cudaMemcpyDeviceToDevice, s_));
        process_generic(w, plain(rows.p, w), nov);
    }
}

// Pair tail (COUNT): per row of width k-2, |Cp| |Cq| - |Cp ∩ Cq| (k_pair)
void Matcher::process_pair(int w, const Frontier& F, int64_t R) {
    LevelBufs& B = *lv_[w];
    const LevelPlan& Lp = lplan_[w];
    B.rbeg.ensure(R, s_);
    B.rlen.ensure(R, s_);
    B.rpiv.ensure(R, s_);
    B.cbeg.ensure((size_t)R * Lp.nb, s_);
    B.clen.ensure((size_t)R * Lp.nb, s_);
    // q's plan goes to the width-(k-1) level buffers: with the pair tail that level is never
    // expanded, and the per-graph workspace keeps them across calls (no pool round trip)
    LevelBufs& Q = *lv_[k_ - 1];
    DevBuf<int64_t>& qbeg = Q.rbeg;
    DevBuf<int64_t>& qlen = Q.rlen;
    DevBuf<uint8_t>& qpiv = Q.rpiv;
    DevBuf<int64_t>& qcbeg = Q.cbeg;
    DevBuf<int32_t>& qclen = Q.clen;
    qbeg.ensure(R, s_);
    qlen.ensure(R, s_);
    qpiv.ensure(R, s_);
    qcbeg.ensure((size_t)R * lq_.nb, s_);
    qclen.ensure((size_t)R * lq_.nb, s_);
    rec_.run(GSM_K_PLAN, 2, [&] {
        launch_plan_rows(g_, F, R, Lp, B.rbeg.p, B.rlen.p, B.rpiv.p, B.cbeg.p, B.clen.p, s_);
        launch_plan_rows(g_, F, R, lq_, qbeg.p, qlen.p, qpiv.p, qcbeg.p, qclen.p, s_);
    });
    res_->prof[GSM_K_PLAN].alg_bytes += (double)R * (2 * 4.0 * w + 28.0 * (Lp.nb + lq_.nb) + 2 * 17.0);
    PairArgs a;
    std::memset(&a, 0, sizeof(a));
    a.F = F;
    a.R = R;
    a.pbeg = B.rbeg.p;
    a.plen = B.rlen.p;
    a.ppiv = B.rpiv.p;
    a.pcbeg = B.cbeg.p;
    a.pclen = B.clen.p;
    a.qbeg = qbeg.p;
    a.qlen = qlen.p;
    a.qpiv = qpiv.p;
    a.qcbeg = qcbeg.p;
    a.qclen = qclen.p;
    a.colsp = Lp.keyed ? g_.lkeys : g_.cols;
    a.colsq = lq_.keyed ? g_.lkeys : g_.cols;
    a.cmask = cmask_.p;
    a.need_both = !(plan_.use_labels && plan_.qlabel[Lp.qv] != plan_.qlabel[lq_.qv]);
    a.mem.off = g_.off;
    a.mem.hub_bits = knobs().member_hub ? g_.hub_bits : nullptr;
    a.mem.hub_base = g_.hub_base;
    a.mem.hub_words = g_.hub_words;
    a.mem.swap_min = knobs().member_swap;
    a.count = final_count_.p;
    ws_.sched.ensure(1, s_);
    GSM_CUDA(cudaMemsetAsync(ws_.sched.p, 0, sizeof(unsigned long long), s_));
    a.next = ws_.sched.p;
    a.stats = stats_.p + 5 * kMaxK;
    // thread per row for short segments, the rest (appended to an overflow list) warp per row
    const int thread_max = knobs().pair_thread_max;  // measured: 16 ~ 64 > 0 > 256
    ovf_idx_.ensure(R, s_);
    ovf_n_.ensure(1, s_);
    GSM_CUDA(cudaMemsetAsync(ovf_n_.p, 0, sizeof(unsigned long long), s_));
    a.overflow = ovf_idx_.p;
    a.noverflow = ovf_n_.p;
    a.thread_max = thread_max;
    rec_.run(GSM_K_TAIL, 1, [&] { launch_pair_thread(a, Lp, lq_, mask_bytes_, s_); });
    const int64_t nov = (int64_t)read_scalar(ovf_n_.p, s_);
    if (nov > 0) {
        PairArgs b = a;
        b.R = nov;
        b.rows_idx = ovf_idx_.p;
        rec_.run(GSM_K_TAIL, 1, [&] { launch_pair(b, Lp, lq_, mask_bytes_, s_); });
    }
    res_->num_chunks++;
    pair_rows_ += (double)R;
}

void Matcher::process_generic(int w, const Frontier& F, int64_t R) {
    if (R <= 0) return;
    ensure_caps();
    LevelBufs& B = *lv_[w];
    const LevelPlan& L = lplan_[w];
    // per-row pivot choice and admissible segment
    B.rbeg.ensure(R, s_);
    B.rlen.ensure(R, s_);
    B.rpiv.ensure(R, s_);
    B.cbeg.ensure((size_t)R * L.nb, s_);
    B.clen.ensure((size_t)R * L.nb, s_);
    B.P.ensure(R + 1, s_);
    const size_t tb = scan_temp_bytes(R);
    B.scan_tmp.ensure(tb, s_);
    rec_.run(GSM_K_PLAN, 1, [&] { launch_plan_rows(g_, F, R, L, B.rbeg.p, B.rlen.p, B.rpiv.p, B.cbeg.p, B.clen.p, s_); });
    res_->prof[GSM_K_PLAN].alg_bytes += (double)R * (4.0 * w + 16.0 * L.nb + 12.0 * L.nb + 8 + 8 + 1);
    rec_.run(GSM_K_SCAN, 1, [&] { launch_scan(B.rlen.p, R, B.P.p, B.scan_tmp.p, tb, s_); });
    res_->prof[GSM_K_SCAN].alg_bytes += (double)R * 16.0;
    const int64_t S = read_scalar(B.P.p + R, s_);
    if (S <= 0) return;

    const int64_t total = R + S;
    const int64_t TD = expand_tile_for(L);
    const bool last = (w == k_ - 1);
    int64_t chunk;
    // intermediate output (not the last level) in the compressed layout when enabled
    const bool cout = compress_ && !last;
    if (last && count_mode_) {
        chunk = TD * ((int64_t)1 << 22);  // only bounds the tile array
    } else {
        chunk = std::min<int64_t>(total, lv_[w + 1]->cap_rows);
        if (chunk < TD) chunk = std::min<int64_t>(total, TD);
        for (;;) {  // the budget is an estimate: on OOM halve this level's chunk (down to one tile)
            try {
                if (cout) lv_[w + 1]->pv.ensure((size_t)chunk, s_);
                else lv_[w + 1]->rows.ensure((size_t)chunk * (w + 1), s_);
                break;
            } catch (const Failure& f) {
                if (f.status != GSM_ERR_OUT_OF_MEMORY || chunk <= TD) throw;
                chunk = std::max<int64_t>(TD, chunk / 2);
                lv_[w + 1]->cap_rows = chunk;
            }
        }
        lv_[w + 1]->out_count.ensure(1, s_);
    }
    chunk = std::min(chunk, total);
    B.tile_ra.ensure((size_t)((chunk + TD - 1) / TD + 1), s_);

    ExpandArgs a;
    std::memset(&a, 0, sizeof(a));
    a.F = F;
    a.R = R;
    a.P = B.P.p;
    a.rbeg = B.rbeg.p;
    a.rpiv = B.rpiv.p;
    a.cbeg = B.cbeg.p;
    a.clen = B.clen.p;
    a.tile_ra = B.tile_ra.p;
    a.TD = TD;
    a.off = g_.off;
    a.cols = L.keyed ? g_.lkeys : g_.cols;
    a.cmask = cmask_.p;
    a.stats = B.stats;
    a.la_c1 = ws_.la_c1.p;
    a.la_c2 = ws_.la_c2.p;
    a.la_ok1 = ws_.la_ok1.p;
    a.la_k = k_;
    B.rows_in += (double)R;
    for (int64_t D0 = 0; D0 < total; D0 += chunk) {
        const int64_t D1 = std::min(D0 + chunk, total);
        const int64_t ntiles = (D1 - D0 + TD - 1) / TD;
        rec_.run(GSM_K_SCAN, 1, [&] { launch_partition(B.P.p, R, S, D0, D1, TD, ntiles, B.tile_ra.p, s_); });
        res_->prof[GSM_K_SCAN].alg_bytes += (double)(ntiles + 1) * 8.0 * 2;
        a.D0 = D0;
        a.D1 = D1;
        a.ntiles = ntiles;
        res_->num_chunks++;
        if (last && count_mode_) {
            a.out = nullptr;
            a.out_count = final_count_.p;
            rec_.run(GSM_K_EXPAND, 1, [&] { launch_expand(a, L, mask_bytes_, s_); });
            continue;
        }
        LevelBufs& N = *lv_[w + 1];
        GSM_CUDA(cudaMemsetAsync(N.out_count.p, 0, sizeof(unsigned long long), s_));
        a.out = cout ? nullptr : N.rows.p;
        a.out_pv = cout ? N.pv.p : nullptr;
        a.out_count = N.out_count.p;
        rec_.run(GSM_K_EXPAND, 1, [&] { launch_expand(a, L, mask_bytes_, s_); });
        const int64_t R2 = (int64_t)read_scalar(N.out_count.p, s_);
        if (R2 == 0) continue;
        res_->level_frontier_bytes[w] += (uint64_t)R2 * (cout ? 8u : 4u * (w + 1));
        if (last) {
            append_output(N.rows.p, R2);
        } else if (cout) {  // the new level extends F's chains by (row of F, vertex) pairs
            Frontier F2 = F;
            if (F.rows) {
                F2.rows = nullptr;
                F2.base = F.rows;
                F2.bw = F.W;
            }
            F2.W = w + 1;
            F2.pv[w + 1] = N.pv.p;
            process(w + 1, F2, R2);
        } else {
            process(w + 1, plain(N.rows.p, w + 1), R2);
        }
    }
}

void Matcher::append_output(const int32_t* rows, int64_t R) {
    const int64_t need = arena_rows_ + R;
    if ((size_t)(need * k_) > arena_.n) {
        size_t cap = std::max<size_t>((size_t)need * k_, arena_.n + arena_.n / 2);
        int32_t* np = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * cap, s_));
        if (arena_rows_) GSM_CUDA(cudaMemcpyAsync(np, arena_.p, sizeof(int32_t) * arena_rows_ * k_,
                                                  cudaMemcpyDeviceToDevice, s_));
        arena_.release();
        arena_.p = np;
        arena_.n = cap;
        arena_.s = s_;
    }
    GSM_CUDA(cudaMemcpyAsync(arena_.p + arena_rows_ * k_, rows, sizeof(int32_t) * R * k_,
                             cudaMemcpyDeviceToDevice, s_));
    arena_rows_ = need;
}

void Matcher::finalize() {
    const int64_t N = arena_rows_;
    const bool expand = plan_.symmetric && !(opts_.flags & GSM_FLAG_UNIQUE);
    const int64_t naut = expand ? (int64_t)plan_.aut_list.size() : 1;
    const int64_t total = N * naut;
    res_->num_rows = (uint64_t)total;
    if (total == 0) return;
    // 1. position order -> query-vertex order, new ids -> original ids
    DevBuf<int32_t> dorder, q;
    dorder.ensure(k_, s_);
    GSM_CUDA(cudaMemcpyAsync(dorder.p, plan_.order, sizeof(int32_t) * k_, cudaMemcpyHostToDevice, s_));
    q.ensure((size_t)N * k_, s_);
    rec_.run(GSM_K_FINALIZE, 1, [&] { launch_to_query_order(arena_.p, N, k_, dorder.p, g_.new2old, q.p, s_); });
    arena_.release();
    // 2. all embeddings = {f∘σ : σ in Aut(Q)} of every representative
    DevBuf<int32_t> all;
    const int32_t* src = q.p;
    if (expand && naut > 1) {
        std::vector<int8_t> sig((size_t)naut * k_);
        for (int64_t a = 0; a < naut; ++a)
            for (int u = 0; u < k_; ++u) sig[a * k_ + u] = plan_.aut_list[a][u];
        DevBuf<int8_t> dsig;
        dsig.ensure(sig.size(), s_);
        GSM_CUDA(cudaMemcpyAsync(dsig.p, sig.data(), sig.size(), cudaMemcpyHostToDevice, s_));
        all.ensure((size_t)total * k_, s_);
        rec_.run(GSM_K_FINALIZE, 1, [&] { launch_aut_expand(q.p, N, k_, dsig.p, naut, all.p, s_); });
        GSM_CUDA(cudaStreamSynchronize(s_));
        src = all.p;
    }
    // 3. lexicographic sort into the library-owned result buffer
    // library-owned result rows: from the same stream-ordered pool as every other buffer
    int32_t* out = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * (size_t)total * k_, s_));
    try {
        rec_.run(GSM_K_FINALIZE, 4, [&] { sort_rows(src, total, k_, g_.n, out, s_); });
        GSM_CUDA(cudaStreamSynchronize(s_));
    } catch (...) {
        cudaFreeAsync(out, s_);
        cudaStreamSynchronize(s_);
        throw;
    }
    res_->rows = out;
}

void match_impl(const gsm_graph* gh, const gsm_query* q, const gsm_match_opts* user_opts, gsm_result* out) {
    if (!gh) fail(GSM_ERR_INVALID_ARGUMENT, "graph is NULL");
    gsm_match_opts opts;
    std::memset(&opts, 0, sizeof(opts));
    if (user_opts) {
        if (user_opts->struct_size != sizeof(gsm_match_opts)) fail(GSM_ERR_INVALID_ARGUMENT, "gsm_match_opts.struct_size mismatch");
        opts = *user_opts;
    } else {
        opts.struct_size = sizeof(opts);
        opts.mode = GSM_MODE_COUNT;
    }
    if (opts.mode != GSM_MODE_COUNT && opts.mode != GSM_MODE_ENUMERATE) fail(GSM_ERR_INVALID_ARGUMENT, "bad mode");
    if (opts.num_shards > 1 && (opts.shard_index < 0 || opts.shard_index >= opts.num_shards))
        fail(GSM_ERR_INVALID_ARGUMENT, "shard_index out of range");
    if (opts.refine_rounds < 0 || opts.refine_rounds > 64) fail(GSM_ERR_INVALID_ARGUMENT, "refine_rounds out of range");
    if (opts.lookahead < 0 || opts.lookahead > 2) fail(GSM_ERR_INVALID_ARGUMENT, "lookahead must be 0, 1 or 2");
    if (opts.root_subset_len < 0 || (opts.root_subset_len > 0 && !opts.root_subset))
        fail(GSM_ERR_INVALID_ARGUMENT, "bad root_subset");
    if (!opts.root_subset) opts.root_subset_len = 0;

    const auto t0 = Clock::now();
    load_knobs();
    g_trace = HostTrace();
    QueryPlan plan;
    std::string msg;
    gsm_status st = load_query(q, &plan, &msg);
    if (st != GSM_OK) fail(st, msg);
    if (plan.use_labels && !labeled_of(gh)) fail(GSM_ERR_INVALID_ARGUMENT, "query has labels but the data graph is unlabeled");

    const bool want_sym = !(opts.flags & GSM_FLAG_NO_SYMMETRY) && !opts.root_subset;
    const bool need_list = opts.mode == GSM_MODE_ENUMERATE && !(opts.flags & GSM_FLAG_UNIQUE);
    compute_symmetry(&plan, want_sym, need_list ? (size_t)1 << 16 : 0);
    if (need_list && plan.symmetric && !plan.aut_list_complete) compute_symmetry(&plan, false, 0);
    if ((opts.flags & GSM_FLAG_UNIQUE) && !plan.symmetric && plan.aut_size > 1)
        fail(GSM_ERR_INVALID_ARGUMENT, "GSM_FLAG_UNIQUE cannot be combined with NO_SYMMETRY or root_subset");
    out->automorphisms = plan.aut_size;

    const int dev = device_of(gh);
    int prev = 0;
    GSM_CUDA(cudaGetDevice(&prev));
    GSM_CUDA(cudaSetDevice(dev));
    out->device = dev;
    cudaStream_t s = opts.stream ? (cudaStream_t)opts.stream : stream_of(gh);
    const float plan_ms = (float)ms_since(t0);
    try {
        Matcher m(gh, plan, opts, out, s);
        m.run();
#ifdef GSM_DEVICE_CHECKS
        GSM_CUDA(cudaStreamSynchronize(s));
        if (const unsigned f = dcheck_collect()) {
            char buf[96];
            std::snprintf(buf, sizeof(buf), "device check failed: flags 0x%x (gsm_common.h DCHK_*)", f);
            fail(GSM_ERR_CUDA, buf);
        }
#endif
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaSetDevice(prev);
        throw;
    }
    out->ms_plan = plan_ms;
    out->ms_total += plan_ms;
    {
        if (knobs().trace == 1)
            std::fprintf(stderr,
                         "[gsm] k=%d count=%llu total %.1f ms (filter %.1f expand %.1f finalize %.1f) | allocs %ld "
                         "(%.2f GB, %.1f ms) syncs %ld (%.1f ms, includes kernel waits) chunks %llu\n",
                         plan.k, (unsigned long long)out->count, out->ms_total, out->ms_filter, out->ms_expand,
                         out->ms_finalize, g_trace.allocs, g_trace.alloc_bytes / 1e9, g_trace.alloc_ms,
                         g_trace.syncs, g_trace.sync_ms, (unsigned long long)out->num_chunks);
    }
    g_trace = HostTrace();
    cudaSetDevice(prev);
}

}  // namespace
}  // namespace gsm

extern "C" {

gsm_status gsm_match(const gsm_graph* g, const gsm_query* q, const gsm_match_opts* opts, gsm_result* out) {
    if (!out) {
        gsm::set_error("out is NULL");
        return GSM_ERR_INVALID_ARGUMENT;
    }
    std::memset(out, 0, sizeof(*out));
    try {
        gsm::clear_error();
        gsm::match_impl(g, q, opts, out);
        return GSM_OK;
    } catch (const gsm::Failure& f) {
        if (out->rows) cudaFree(out->rows);
        std::memset(out, 0, sizeof(*out));
        gsm::set_error(f.msg);
        return f.status;
    } catch (const std::bad_alloc&) {
        std::memset(out, 0, sizeof(*out));
        gsm::set_error("host allocation failed");
        return GSM_ERR_OUT_OF_MEMORY;
    } catch (...) {
        std::memset(out, 0, sizeof(*out));
        gsm::set_error("unexpected exception in gsm_match");
        return GSM_ERR_CUDA;
    }
}

gsm_status gsm_result_free(gsm_result* r) {
    if (!r) return GSM_OK;
    if (r->rows) {  // pool allocation (cudaMallocAsync); cudaFree synchronises and releases it
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(r->device);
        cudaFree(r->rows);
        cudaSetDevice(prev);
    }
    r->rows = nullptr;
    r->num_rows = 0;
    return GSM_OK;
}

gsm_status gsm_result_copy_rows(const gsm_result* r, int32_t* dst, int32_t dst_on_device) {
    if (!r || (!dst && r->num_rows)) {
        gsm::set_error("bad arguments to gsm_result_copy_rows");
        return GSM_ERR_INVALID_ARGUMENT;
    }
    if (!r->num_rows) return GSM_OK;
    if (!r->rows) {
        gsm::set_error("result has no rows (COUNT mode or already freed)");
        return GSM_ERR_INVALID_ARGUMENT;
    }
    cudaError_t e = cudaMemcpy(dst, r->rows, sizeof(int32_t) * r->num_rows * (size_t)r->width,
                               dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        gsm::set_error(std::string("cudaMemcpy: ") + cudaGetErrorString(e));
        return GSM_ERR_CUDA;
    }
    return GSM_OK;
}

gsm_status gsm_sort_rows(int32_t* rows, uint64_t num_rows, int32_t width, int64_t max_id, int32_t device,
                         void* stream) {
    if (num_rows == 0) return GSM_OK;
    if (!rows || width < 1 || max_id < 0) {
        gsm::set_error("bad arguments to gsm_sort_rows");
        return GSM_ERR_INVALID_ARGUMENT;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    try {
        gsm::clear_error();
        GSM_CUDA(cudaSetDevice(device));
        cudaStream_t s = (cudaStream_t)stream;
        gsm::DevBuf<int32_t> tmp;
        tmp.ensure((size_t)num_rows * width, s);
        gsm::sort_rows(rows, (int64_t)num_rows, width, max_id + 1, tmp.p, s);
        GSM_CUDA(cudaMemcpyAsync(rows, tmp.p, sizeof(int32_t) * num_rows * width, cudaMemcpyDeviceToDevice, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        cudaSetDevice(prev);
        return GSM_OK;
    } catch (const gsm::Failure& f) {
        cudaSetDevice(prev);
        gsm::set_error(f.msg);
        return f.status;
    } catch (...) {
        cudaSetDevice(prev);
        gsm::set_error("unexpected exception in gsm_sort_rows");
        return GSM_ERR_CUDA;
    }
}

gsm_status gsm_filter_candidates(const gsm_graph* g, const gsm_query* q, int32_t refine_rounds, uint32_t* out,
                                 int32_t out_on_device) {
    int prev = 0;
    cudaGetDevice(&prev);
    try {
        gsm::clear_error();
        gsm::load_knobs();
        if (!g || !out) gsm::fail(GSM_ERR_INVALID_ARGUMENT, "graph or out is NULL");
        if (refine_rounds < 0 || refine_rounds > 64) gsm::fail(GSM_ERR_INVALID_ARGUMENT, "refine_rounds out of range");
        gsm::QueryPlan plan;
        std::string msg;
        gsm_status st = gsm::load_query(q, &plan, &msg);
        if (st != GSM_OK) gsm::fail(st, msg);
        if (plan.use_labels && !gsm::labeled_of(g))
            gsm::fail(GSM_ERR_INVALID_ARGUMENT, "query has labels but the data graph is unlabeled");
        GSM_CUDA(cudaSetDevice(gsm::device_of(g)));
        const gsm::DevGraph& G = gsm::graph_of(g);
        cudaStream_t s = gsm::stream_of(g);
        const int k = plan.k, mb = gsm::mask_bytes_for(k);
        gsm::FilterQuery fq;
        std::memset(&fq, 0, sizeof(fq));
        fq.k = k;
        fq.use_labels = plan.use_labels ? 1 : 0;
        for (int u = 0; u < k; ++u) {
            fq.qlabel[u] = plan.qlabel[u];
            fq.qdeg[u] = plan.qdeg[u];
            fq.qadj[u] = plan.adj[u];
        }
        gsm::Workspace& ws = gsm::workspace_of(g);
        ws.cmask.ensure((size_t)G.n * mb, s);
        ws.counts.ensure(gsm::kMaxK, s);
        GSM_CUDA(cudaMemsetAsync(ws.counts.p, 0, sizeof(unsigned long long) * gsm::kMaxK, s));
        gsm::launch_filter(G, fq, ws.cmask.p, ws.counts.p, s);
        if (refine_rounds > 0) {
            int64_t hqne[gsm::kMaxK] = {};
            for (int u = 0; u < k; ++u)
                for (int w = 0; w < k; ++w)
                    if ((plan.adj[u] >> w) & 1u) hqne[u] += plan.use_labels ? (int64_t)plan.qlabel[w] + 1 : 1;
            gsm::DevBuf<int64_t> dqne;
            gsm::DevBuf<uint8_t> tmp;
            dqne.ensure(gsm::kMaxK, s);
            tmp.ensure((size_t)G.n * mb, s);
            GSM_CUDA(cudaMemcpyAsync(dqne.p, hqne, sizeof(hqne), cudaMemcpyHostToDevice, s));
            gsm::launch_refine(G, fq, dqne.p, refine_rounds, ws.cmask.p, tmp.p, ws.counts.p, s);
        }
        gsm::DevBuf<uint32_t> dout;
        uint32_t* dst = out;
        if (!out_on_device) {
            dout.ensure((size_t)G.n, s);
            dst = dout.p;
        }
        gsm::launch_mask_to_original(G, ws.cmask.p, mb, dst, s);
        if (!out_on_device)
            GSM_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(uint32_t) * G.n, cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        cudaSetDevice(prev);
        return GSM_OK;
    } catch (const gsm::Failure& f) {
        cudaSetDevice(prev);
        gsm::set_error(f.msg);
        return f.status;
    } catch (...) {
        cudaSetDevice(prev);
        gsm::set_error("unexpected exception in gsm_filter_candidates");
        return GSM_ERR_CUDA;
    }
}

gsm_status gsm_plan_query(const gsm_query* q, const uint64_t* cand, uint32_t flags, gsm_plan_info* out) {
    if (!out) {
        gsm::set_error("out is NULL");
        return GSM_ERR_INVALID_ARGUMENT;
    }
    std::memset(out, 0, sizeof(*out));
    try {
        gsm::clear_error();
        gsm::QueryPlan plan;
        std::string msg;
        gsm_status st = gsm::load_query(q, &plan, &msg);
        if (st != GSM_OK) {
            gsm::set_error(msg);
            return st;
        }
        gsm::compute_symmetry(&plan, !(flags & GSM_FLAG_NO_SYMMETRY), 0);
        gsm::compute_order(&plan, cand, -1);
        if (flags & GSM_FLAG_PLAN_COUNT) gsm::compute_order_pair_tail(&plan, cand);
        out->k = plan.k;
        for (int i = 0; i < plan.k; ++i) {
            out->order[i] = plan.order[i];
            out->parent[i] = plan.parent[i];
            out->backward[i] = plan.backward[i];
        }
        out->num_conditions = (int32_t)plan.conds.size();
        for (size_t c = 0; c < plan.conds.size(); ++c) {
            out->cond_lo[c] = plan.conds[c].first;
            out->cond_hi[c] = plan.conds[c].second;
        }
        out->automorphisms = plan.aut_size;
        return GSM_OK;
    } catch (...) {
        gsm::set_error("unexpected exception in gsm_plan_query");
        return GSM_ERR_INVALID_QUERY;
    }
}

}  // extern "C"
