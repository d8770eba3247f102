// gsm_graph.cu — gsm_load_graph / gsm_free: the device replica of the data graph.
//
// PAPER P:148 (§3.3): "We store graphs in a space-efficient fashion on the GPU
// by using compressed sparse row (CSR)".  P:47: the method inputs CSR and does
// no index building on G.  We add one O(m log m) relabelling at load time
// (reported as load time, never inside gsm_match): vertices are
// renumbered by ascending (degree, original id) and every list is re-sorted.
// After it, the symmetry-breaking total order ≺ on data vertices (P:71
// constraints) is plain integer '<' on new ids, and
// N+(v) = {w in N(v) : v ≺ w} is the contiguous suffix of v's sorted list
// starting at up[v].  Every id crossing the ABI is an original id.
#include <vector>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>

#include "gsm_common.h"
#include "gsm_workspace.h"

struct gsm_graph {
    gsm::DevGraph g;
    std::unique_ptr<gsm::Workspace> ws{new gsm::Workspace()};
    int device = 0;
    cudaStream_t stream = 0;
    bool own_stream = false;
    bool labeled = false;
};

namespace gsm {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }

HostTrace g_trace;

static thread_local Knobs g_knobs;
const Knobs& knobs() { return g_knobs; }

static int env_or(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}

void load_knobs() {
    Knobs k;
    k.clique = env_or("GSM_CLIQUE", k.clique);
    k.clique_warp = env_or("GSM_CLIQUE_WARP", k.clique_warp) ? 32 : 0;
    k.clique_dsmem = env_or("GSM_CLIQUE_DSMEM", 0);
    k.clique_dmax = env_or("GSM_CLIQUE_DMAX", 0);
    k.clique_stream = env_or("GSM_CLIQUE_STREAM", k.clique_stream);
    k.clique_hash = env_or("GSM_CLIQUE_HASH", k.clique_hash);
    k.clique_occ = env_or("GSM_CLIQUE_OCC", k.clique_occ);
    k.pair_tail = env_or("GSM_PAIR_TAIL", k.pair_tail);
    k.pair_thread_max = env_or("GSM_PAIR_THREAD_MAX", k.pair_thread_max);
    k.fused_tail = env_or("GSM_FUSED_TAIL", k.fused_tail);
    k.tail_cap = std::min(6144, std::max(64, env_or("GSM_TAIL_CAP", k.tail_cap))) & ~1;
    k.tail_block_cap = std::min(48 * 1024, std::max(256, env_or("GSM_TAIL_BLOCK_CAP", k.tail_block_cap)));
    k.tail_bratio = env_or("GSM_TAIL_BRATIO_PCT", k.tail_bratio);
    k.count_walk = env_or("GSM_COUNT_WALK", k.count_walk);
    k.expand_td = std::min(2048, std::max(128, env_or("GSM_EXPAND_TD", k.expand_td)));
    const int u = env_or("GSM_EXPAND_ILP", 1);
    k.expand_ilp = (u == 2 || u == 4) ? u : 1;
    k.trace = env_or("GSM_TRACE", 0);
    k.lookahead = env_or("GSM_LOOKAHEAD", -1);
    k.compress = env_or("GSM_COMPRESS", -1);
    k.plan_groups = env_or("GSM_PLAN_GROUPS", k.plan_groups);
    k.member_hub = env_or("GSM_MEMBER_HUB", k.member_hub);
    k.member_swap = env_or("GSM_MEMBER_SWAP", k.member_swap);
    k.hub_bits = std::max(0, env_or("GSM_HUB_BITS", k.hub_bits)) & ~31;
    k.clique_hub = env_or("GSM_CLIQUE_HUB", k.clique_hub);
    k.clique_hub_ratio = env_or("GSM_CLIQUE_HUB_RATIO", k.clique_hub_ratio);
    k.order = env_or("GSM_ORDER", k.order);
    k.nhash_min = std::max(0, env_or("GSM_NHASH_MIN", k.nhash_min));
    k.lidx_min = std::max(0, env_or("GSM_LIDX_MIN", k.lidx_min));
    k.clique_ranges = env_or("GSM_CLIQUE_RANGES", k.clique_ranges);
    k.clique_ntsel = env_or("GSM_CLIQUE_NTSEL", k.clique_ntsel);
    k.clique_lazy_ck = env_or("GSM_CLIQUE_LAZYCK", k.clique_lazy_ck);
    k.filter_bps = std::max(1, std::min(512, env_or("GSM_FILTER_BPS", k.filter_bps)));
    k.bigsort = env_or("GSM_BIGSORT", k.bigsort);
    k.bigsort_min = std::max(2, env_or("GSM_BIGSORT_MIN", k.bigsort_min));
    {
        const int fu = env_or("GSM_FILTER_U", k.filter_u);
        k.filter_u = (fu == 1 || fu == 2 || fu == 4) ? fu : 1;
    }
    k.clique_nh_stream = env_or("GSM_CLIQUE_NH_STREAM", k.clique_nh_stream);
    g_knobs = k;
}

#ifdef GSM_DEVICE_CHECKS
static std::vector<unsigned (*)()>& dcheck_readers() {
    static std::vector<unsigned (*)()> v;
    return v;
}
void dcheck_register(unsigned (*fn)()) { dcheck_readers().push_back(fn); }
unsigned dcheck_collect() {
    unsigned f = 0;
    for (auto fn : dcheck_readers()) f |= fn();
    return f;
}
#endif

void* dev_alloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    g_trace.alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    g_trace.allocs++;
    g_trace.alloc_bytes += (double)bytes;
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        char buf[160];
        std::snprintf(buf, sizeof(buf), "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
        fail(e == cudaErrorMemoryAllocation ? GSM_ERR_OUT_OF_MEMORY : GSM_ERR_CUDA, buf);
    }
    return p;
}

void dev_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// ---------------------------------------------------------------- validation kernels
__global__ void k_validate_offsets(const int64_t* __restrict__ off, int64_t n, int64_t nnz, int* err) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        if (off[v] > off[v + 1]) atomicOr(err, 1);
        if (v == 0 && off[0] != 0) atomicOr(err, 1);
        if (v == n - 1 && off[n] != nnz) atomicOr(err, 1);
    }
}

// warp per vertex: ids in range, no self-loop, strictly ascending, symmetric
__global__ void k_validate_lists(const int64_t* __restrict__ off, const int32_t* __restrict__ cols, int64_t n,
                                 int* err) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = warp; u < n; u += nwarps) {
        const int64_t b = off[u], e = off[u + 1];
        for (int64_t i = b + lane; i < e; i += 32) {
            const int32_t c = cols[i];
            if (c < 0 || c >= n) { atomicOr(err, 2); continue; }
            if (c == u) atomicOr(err, 4);
            if (i > b && cols[i - 1] >= c) atomicOr(err, 8);
            // symmetric: u in N(c)
            int64_t lo = off[c], hi = off[c + 1];
            bool found = false;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                int32_t x = cols[mid];
                if (x == u) { found = true; break; }
                if (x < u) lo = mid + 1; else hi = mid;
            }
            if (!found) atomicOr(err, 16);
        }
    }
}

// ---------------------------------------------------------------- relabel kernels
__global__ void k_degree_keys(const int64_t* __restrict__ off, int64_t n, uint64_t* keys, int* maxdeg) {
    int local = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int64_t d = off[v + 1] - off[v];
        keys[v] = ((uint64_t)d << 32) | (uint64_t)v;
        local = max(local, (int)d);
    }
    for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxdeg, local);
}

__global__ void k_permutation(const uint64_t* __restrict__ sorted, const int64_t* __restrict__ off, int64_t n,
                              int32_t* new2old, int32_t* old2new, int64_t* newdeg) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = sorted[p];
        int32_t old = (int32_t)(k & 0xffffffffu);
        new2old[p] = old;
        old2new[old] = (int32_t)p;
        newdeg[p] = off[old + 1] - off[old];
    }
}

// ---------------------------------------------------------------- approximate degeneracy order
// (GSM_ORDER=1; any strict total order ≺ is valid, SURVEY §8(c) amb. 9).  Peeling in rounds:
// every remaining vertex whose remaining degree is <= (1 + eps) x the remaining average is
// removed in round r (O(log n / eps) rounds); rank = (round, degree, id).  Orienting by it
// bounds |N+(u)| by the remaining degree at removal, <= 2(1 + eps) x the degeneracy.
__global__ void k_adg_init(const int64_t* __restrict__ off, int64_t n, int32_t* __restrict__ dr,
                           uint8_t* __restrict__ lvl) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        dr[v] = (int32_t)(off[v + 1] - off[v]);
        lvl[v] = 0xff;
    }
}

// sum of remaining degrees and remaining count ([0], [1])
__global__ void k_adg_stats(const int32_t* __restrict__ dr, const uint8_t* __restrict__ lvl, int64_t n,
                            unsigned long long* __restrict__ acc) {
    unsigned long long sd = 0, c = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (lvl[v] == 0xff) {
            sd += (unsigned long long)max(dr[v], 0);
            ++c;
        }
    for (int o = 16; o; o >>= 1) {
        sd += __shfl_xor_sync(0xffffffffu, sd, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0 && c) {
        atomicAdd(acc, sd);
        atomicAdd(acc + 1, c);
    }
}

// round r: remove the remaining vertices with dr <= thr (queued)
__global__ void k_adg_mark(const int32_t* __restrict__ dr, uint8_t* __restrict__ lvl, int64_t n, int64_t thr, int r,
                           int32_t* __restrict__ q, unsigned long long* __restrict__ qn) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (lvl[v] == 0xff && (int64_t)dr[v] <= thr) {
            lvl[v] = (uint8_t)r;
            q[atomicAdd(qn, 1ull)] = (int32_t)v;
        }
}

// warp per removed vertex: its still-remaining neighbours lose one remaining degree
__global__ void k_adg_peel(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                           const int32_t* __restrict__ q, int64_t qn, const uint8_t* __restrict__ lvl,
                           int32_t* __restrict__ dr) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < qn; t += nw) {
        const int32_t v = q[t];
        for (int64_t x = off[v] + lane; x < off[v + 1]; x += 32) {
            const int32_t w = cols[x];
            if (lvl[w] == 0xff) atomicSub(&dr[w], 1);
        }
    }
}

__global__ void k_adg_keys(const int64_t* __restrict__ off, const uint8_t* __restrict__ lvl, int64_t n,
                           uint64_t* __restrict__ keys) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t dd = off[v + 1] - off[v];
        const uint64_t d = (uint64_t)(dd < (1 << 24) - 1 ? dd : (1 << 24) - 1);
        keys[v] = ((uint64_t)lvl[v] << 56) | (d << 32) | (uint64_t)v;
    }
}

// warp per new vertex p: emit (p, old2new[w]) keys for its old list
__global__ void k_edge_keys(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                            const int64_t* __restrict__ noff, const int32_t* __restrict__ new2old,
                            const int32_t* __restrict__ old2new, int64_t n, uint64_t* ekeys) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = warp; p < n; p += nwarps) {
        const int32_t old = new2old[p];
        const int64_t b = off[old], e = off[old + 1], dst = noff[p];
        for (int64_t i = b + lane; i < e; i += 32)
            ekeys[dst + (i - b)] = ((uint64_t)p << 32) | (uint32_t)old2new[cols[i]];
    }
}

// warp per new vertex p: its old list mapped to new ids (unsorted), at the new offset
__global__ void k_edge_cols(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                            const int64_t* __restrict__ noff, const int32_t* __restrict__ new2old,
                            const int32_t* __restrict__ old2new, int64_t n, int32_t* out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = warp; p < n; p += nwarps) {
        const int32_t old = new2old[p];
        const int64_t b = off[old], e = off[old + 1], dst = noff[p];
        for (int64_t i = b + lane; i < e; i += 32) out[dst + (i - b)] = old2new[cols[i]];
    }
}

__global__ void k_extract_cols(const uint64_t* __restrict__ ekeys, int64_t nnz, int32_t* cols) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
        cols[i] = (int32_t)(ekeys[i] & 0xffffffffu);
}

__global__ void k_up(const int64_t* __restrict__ off, const int32_t* __restrict__ cols, int64_t n, int32_t* up) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = off[v], hi = off[v + 1];
        const int64_t b = lo;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (cols[mid] < v) lo = mid + 1; else hi = mid;
        }
        up[v] = (int32_t)(lo - b);
    }
}

__global__ void k_max_label(const uint32_t* __restrict__ labels, int64_t n, unsigned* out) {
    unsigned m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        m = max(m, labels[v]);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// warp per vertex p of the relabelled CSR: key (p, label(w) << idbits | w)
__global__ void k_label_edge_keys(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                                  const uint32_t* __restrict__ labels, int64_t n, int idbits, uint64_t* ekeys) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = warp; p < n; p += nwarps)
        for (int64_t i = off[p] + lane; i < off[p + 1]; i += 32) {
            const int32_t w = cols[i];
            ekeys[i] = ((uint64_t)p << 32) | (((uint64_t)labels[w] << idbits) | (uint32_t)w);
        }
}

__global__ void k_permute_labels(const uint32_t* __restrict__ labels, const int32_t* __restrict__ new2old, int64_t n,
                                 uint32_t* out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        out[p] = labels[new2old[p]];
}

// hub bitmap: warp per hub a, one bit per entry of N+(a) (all inside the hub range)
__global__ void k_hub_bits(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                           const int32_t* __restrict__ up, int32_t base, int32_t H, int hw, uint32_t* bits) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < H;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t a = base + (int32_t)r;
        uint32_t* row = const_cast<uint32_t*>(hub_row(bits, hw, (int)r));
        for (int64_t e = off[a] + up[a] + lane; e < off[a + 1]; e += 32) {
            const int c = cols[e] - base;
            atomicOr(row + (c >> 5), 1u << (c & 31));
        }
    }
}

static int grid_for(int64_t items, int threads = 256) {
    int64_t b = (items + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 64) b = 148 * 64;
    return (int)b;
}

// ---------------------------------------------------------------- hashed N+(v) tables
// buckets per vertex (0 when |N+(v)| < nh_min)
__global__ void k_nh_sizes(const int64_t* __restrict__ off, const int32_t* __restrict__ up, int64_t n, int nh_min,
                           int64_t* __restrict__ nb) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t L = off[v + 1] - off[v] - up[v];
        nb[v] = L >= nh_min ? (int64_t)nh_buckets(L) : 0;
    }
}

__global__ void k_nh_offsets(const int64_t* __restrict__ nb, const int64_t* __restrict__ excl, int64_t n,
                             int32_t* __restrict__ nh_off) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        nh_off[v] = nb[v] ? (int32_t)excl[v] : -1;
}

// warp per vertex: insert every entry of N+(v) into v's table (first free slot of its bucket,
// else the next bucket); the entries of one list are distinct, so no duplicate checks
__global__ void k_nh_insert(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                            const int32_t* __restrict__ up, const int32_t* __restrict__ nh_off, int64_t n,
                            int32_t* __restrict__ tab) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
        const int32_t tb = nh_off[v];
        if (tb < 0) continue;
        const int64_t b0 = off[v] + up[v], e = off[v + 1];
        const unsigned B = nh_buckets(e - b0);
        for (int64_t x = b0 + lane; x < e; x += 32) {
            const int32_t key = cols[x];
            unsigned b = nh_hash(key, B);
            for (bool done = false; !done; b = (b + 1) & (B - 1)) {
                int32_t* slot = tab + 8 * ((int64_t)tb + b);
                for (int q = 0; q < 8; ++q)
                    if (atomicCAS(slot + q, -1, key) == -1) {
                        done = true;
                        break;
                    }
            }
        }
    }
}

// label index: per indexed vertex, nl + 1 relative offsets (segment starts of labels 0..nl-1, then
// the list length); warp per vertex, lanes over labels, each a binary search in the keyed list
__global__ void k_lidx_sizes(const int64_t* __restrict__ off, int64_t n, int lmin, int nl, int64_t* __restrict__ sz) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        sz[v] = off[v + 1] - off[v] >= lmin ? nl + 1 : 0;
}

__global__ void k_lidx_build(const int64_t* __restrict__ off, const int32_t* __restrict__ lkeys,
                             const int64_t* __restrict__ sz, const int64_t* __restrict__ excl, int64_t n, int nl,
                             int idbits, int32_t* __restrict__ lidx_off, int32_t* __restrict__ lidx) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n; v += nw) {
        if (sz[v] == 0) {
            if (lane == 0) lidx_off[v] = -1;
            continue;
        }
        const int64_t b = off[v], e = off[v + 1];
        if (lane == 0) lidx_off[v] = (int32_t)excl[v];
        for (int l = lane; l <= nl; l += 32) {
            int64_t lo = b, hi = e;
            const int64_t key = (int64_t)l << idbits;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)lkeys[mid] < key) lo = mid + 1; else hi = mid;
            }
            lidx[excl[v] + l] = (int32_t)(lo - b);
        }
    }
}

// number of trailing vertices (new order) with degree >= big, and where their lists start;
// degrees are non-decreasing in the (degree, id) order, so they form a suffix
__global__ void k_big_suffix(const int64_t* __restrict__ off, int64_t n, int64_t big, int64_t* out) {
    // the first vertex with degree >= big: a binary search by one thread (log2 n steps)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (off[mid + 1] - off[mid] < big) lo = mid + 1; else hi = mid;
        }
        out[0] = n - lo;
        out[1] = off[lo];
    }
}

// warp per long list: (list index << 32 | id) keys of its entries
__global__ void k_big_keys(const int64_t* __restrict__ off, const int32_t* __restrict__ ecols, int64_t first,
                           int64_t nbig, int64_t base, uint64_t* __restrict__ keys) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < nbig; b += nw) {
        const int64_t v = first + b;
        for (int64_t x = off[v] + lane; x < off[v + 1]; x += 32)
            keys[x - base] = ((uint64_t)b << 32) | (uint32_t)ecols[x];
    }
}

__global__ void k_nplus(const int64_t* __restrict__ off, const int32_t* __restrict__ up,
                        const int32_t* __restrict__ nh_off, int64_t n, int4* __restrict__ np) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = off[v] + up[v];
        np[v] = make_int4((int32_t)(uint32_t)(b & 0xffffffffLL), (int32_t)(b >> 32), (int32_t)(off[v + 1] - b),
                          nh_off ? nh_off[v] : -1);
    }
}

// keys = (peeling round, degree, id) of the approximate degeneracy order (k_adg_*)
static void adg_keys(const int64_t* off, const int32_t* cols, int64_t n, int64_t nnz, uint64_t* keys, cudaStream_t s) {
    (void)nnz;
    DevBuf<int32_t> dr, q;
    DevBuf<uint8_t> lvl;
    DevBuf<unsigned long long> acc;
    dr.ensure(n, s);
    q.ensure(n, s);
    lvl.ensure(n, s);
    acc.ensure(3, s);
    const unsigned gb = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    k_adg_init<<<gb, 256, 0, s>>>(off, n, dr.p, lvl.p);
    GSM_LAUNCH("k_adg_init");
    const double eps = 0.25;
    for (int r = 0; r < 254; ++r) {
        GSM_CUDA(cudaMemsetAsync(acc.p, 0, 3 * sizeof(unsigned long long), s));
        k_adg_stats<<<gb, 256, 0, s>>>(dr.p, lvl.p, n, acc.p);
        GSM_LAUNCH("k_adg_stats");
        unsigned long long h[2];
        GSM_CUDA(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        if (h[1] == 0) break;
        // the last admissible round takes everything left
        const int64_t thr = r == 253 ? INT64_MAX : (int64_t)((1.0 + eps) * (double)h[0] / (double)h[1]);
        k_adg_mark<<<gb, 256, 0, s>>>(dr.p, lvl.p, n, thr, r, q.p, acc.p + 2);
        GSM_LAUNCH("k_adg_mark");
        unsigned long long qn = 0;
        GSM_CUDA(cudaMemcpyAsync(&qn, acc.p + 2, sizeof(qn), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        if (qn == h[1]) break;  // nothing remains to update
        k_adg_peel<<<(unsigned)std::min<int64_t>((qn + 7) / 8, 148 * 64), 256, 0, s>>>(off, cols, q.p, (int64_t)qn,
                                                                                     lvl.p, dr.p);
        GSM_LAUNCH("k_adg_peel");
    }
    k_adg_keys<<<gb, 256, 0, s>>>(off, lvl.p, n, keys);
    GSM_LAUNCH("k_adg_keys");
}

static int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && (x >> b)) ++b;
    return b;
}

static void free_graph(gsm_graph* h) {
    if (!h) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(h->device);
    DevGraph& g = h->g;
    cudaStreamSynchronize(h->stream);
    h->ws.reset();  // frees the cached match workspace (stream-ordered)
    // graph arrays come from the device's stream-ordered pool (kept cached by its release
    // threshold, so a load/free/load cycle does not re-map memory)
    for (void* p : {(void*)g.off, (void*)g.cols, (void*)g.up, (void*)g.labels, (void*)g.lkeys, (void*)g.new2old,
                    (void*)g.old2new, (void*)g.hub_bits, (void*)g.nh_off, (void*)g.nh_tab, (void*)g.nplus,
                    (void*)g.lidx_off, (void*)g.lidx})
        if (p) cudaFreeAsync(p, h->stream);
    cudaStreamSynchronize(h->stream);
    if (h->own_stream) cudaStreamDestroy(h->stream);
    cudaSetDevice(cur);
    delete h;
}

static void load_graph_impl(int64_t n, const int64_t* row_offsets, const int32_t* col_indices, const uint32_t* labels,
                            int32_t on_device, const gsm_load_opts* opts, gsm_graph** out) {
    if (!out) fail(GSM_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    load_knobs();
    // GSM_TRACE=1: per-phase load times (a stream sync after each phase; tracing only)
    auto tph = std::chrono::steady_clock::now();
    cudaStream_t stream_for_trace = nullptr;
    cudaStream_t* out_stream = &stream_for_trace;
    auto phase = [&](const char* name) {
        if (knobs().trace != 1 || !*out_stream) return;
        cudaStreamSynchronize(*out_stream);
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[gsm load] %-26s %8.2f ms\n", name, std::chrono::duration<double, std::milli>(t - tph).count());
        tph = t;
    };
    if (opts && opts->struct_size != sizeof(gsm_load_opts)) fail(GSM_ERR_INVALID_ARGUMENT, "gsm_load_opts.struct_size mismatch");
    if (n <= 0) fail(GSM_ERR_INVALID_GRAPH, "graph has no vertices");
    if (n >= (int64_t)0x7fffffff) fail(GSM_ERR_INVALID_GRAPH, "more than 2^31-1 vertices");
    if (!row_offsets || !col_indices) fail(GSM_ERR_INVALID_ARGUMENT, "CSR pointer is NULL");
    int ndev = 0;
    cudaError_t de = cudaGetDeviceCount(&ndev);
    if (de != cudaSuccess || ndev == 0) {
        (void)cudaGetLastError();
        fail(GSM_ERR_NO_DEVICE, std::string("no CUDA device: ") + cudaGetErrorString(de));
    }
    const int device = opts ? opts->device : 0;
    if (device < 0 || device >= ndev) fail(GSM_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    GSM_CUDA(cudaSetDevice(device));

    std::unique_ptr<gsm_graph, void (*)(gsm_graph*)> h(new gsm_graph(), free_graph);
    h->device = device;
    if (opts && opts->stream) {
        h->stream = (cudaStream_t)opts->stream;
    } else {
        GSM_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    cudaStream_t s = h->stream;
    stream_for_trace = s;
    // keep freed pool memory cached between matches
    cudaMemPool_t pool;
    GSM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    GSM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));

    int64_t nnz = 0;
    if (on_device) GSM_CUDA(cudaMemcpyAsync(&nnz, row_offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    else nnz = row_offsets[n];
    GSM_CUDA(cudaStreamSynchronize(s));
    if (nnz < 0) fail(GSM_ERR_INVALID_GRAPH, "row_offsets[n] < 0");

    // input replica on the device (borrowed zero-copy when already there)
    DevBuf<int64_t> in_off;
    DevBuf<int32_t> in_cols;
    DevBuf<uint32_t> in_lab;
    const int64_t* d_off = row_offsets;
    const int32_t* d_cols = col_indices;
    const uint32_t* d_lab = labels;
    if (!on_device) {
        in_off.ensure(n + 1, s);
        in_cols.ensure(nnz, s);
        GSM_CUDA(cudaMemcpyAsync(in_off.p, row_offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
        if (nnz) GSM_CUDA(cudaMemcpyAsync(in_cols.p, col_indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
        d_off = in_off.p;
        d_cols = in_cols.p;
        if (labels) {
            in_lab.ensure(n, s);
            GSM_CUDA(cudaMemcpyAsync(in_lab.p, labels, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s));
            d_lab = in_lab.p;
        }
    }
    if (opts && opts->validate) {
        DevBuf<int> err;
        err.ensure(1, s);
        GSM_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), s));
        k_validate_offsets<<<grid_for(n), 256, 0, s>>>(d_off, n, nnz, err.p);
        GSM_LAUNCH("k_validate_offsets");
        int herr = 0;
        GSM_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        if (herr) fail(GSM_ERR_INVALID_GRAPH, "row_offsets are not a valid CSR offset array");
        k_validate_lists<<<grid_for(n * 32), 256, 0, s>>>(d_off, d_cols, n, err.p);
        GSM_LAUNCH("k_validate_lists");
        GSM_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        if (herr & 2) fail(GSM_ERR_INVALID_GRAPH, "neighbour id out of range");
        if (herr & 4) fail(GSM_ERR_INVALID_GRAPH, "self-loop");
        if (herr & 8) fail(GSM_ERR_INVALID_GRAPH, "neighbour list not strictly ascending (unsorted or duplicate)");
        if (herr & 16) fail(GSM_ERR_INVALID_GRAPH, "asymmetric edge (graph must be undirected)");
    }

    DevGraph& g = h->g;
    g.n = n;
    g.nnz = nnz;
    g.off = static_cast<int64_t*>(dev_alloc(sizeof(int64_t) * (n + 1), s));
    g.cols = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * (nnz ? nnz : 1), s));
    g.up = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * n, s));
    g.new2old = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * n, s));
    g.old2new = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * n, s));

    phase("upload + validate");
    // 1. rank by (degree, id) (GSM_ORDER=1: by (peeling round, degree, id), k_adg_*)
    {
        DevBuf<uint64_t> keys, sorted;
        DevBuf<int> maxdeg;
        keys.ensure(n, s);
        sorted.ensure(n, s);
        maxdeg.ensure(1, s);
        GSM_CUDA(cudaMemsetAsync(maxdeg.p, 0, sizeof(int), s));
        k_degree_keys<<<grid_for(n), 256, 0, s>>>(d_off, n, keys.p, maxdeg.p);
        GSM_LAUNCH("k_degree_keys");
        int hmax = 0;
        GSM_CUDA(cudaMemcpyAsync(&hmax, maxdeg.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        g.max_degree = hmax;
        int end_bit = 32 + bits_for((uint64_t)hmax);
        if (knobs().order == 1 && n > 1) {
            end_bit = 64;
            adg_keys(d_off, d_cols, n, nnz, keys.p, s);
        }
        size_t tmp_bytes = 0;
        GSM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.p, sorted.p, n, 0, end_bit, s));
        DevBuf<uint8_t> tmp;
        tmp.ensure(tmp_bytes, s);
        GSM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.p, sorted.p, n, 0, end_bit, s));
        DevBuf<int64_t> newdeg;
        newdeg.ensure(n, s);
        k_permutation<<<grid_for(n), 256, 0, s>>>(sorted.p, d_off, n, g.new2old, g.old2new, newdeg.p);
        GSM_LAUNCH("k_permutation");
        GSM_CUDA(cudaMemsetAsync(g.off, 0, sizeof(int64_t), s));
        size_t sb = 0;
        GSM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, sb, newdeg.p, g.off + 1, n, s));
        DevBuf<uint8_t> stmp;
        stmp.ensure(sb, s);
        GSM_CUDA(cub::DeviceScan::InclusiveSum(stmp.p, sb, newdeg.p, g.off + 1, n, s));
    }
    phase("rank + offsets");
    // 2. relabelled lists, each re-sorted (segmented sort of 32-bit ids: the rows are
    //    already in their new order, only the ids inside a list move)
    if (nnz > 0 && nnz > (int64_t)INT32_MAX) {  // beyond 32-bit segmented-sort sizes: (row, id) keys
        DevBuf<uint64_t> ekeys, esorted;
        ekeys.ensure(nnz, s);
        esorted.ensure(nnz, s);
        k_edge_keys<<<grid_for(n * 32), 256, 0, s>>>(d_off, d_cols, g.off, g.new2old, g.old2new, n, ekeys.p);
        GSM_LAUNCH("k_edge_keys");
        const int end_bit = 32 + bits_for((uint64_t)n);
        size_t tmp_bytes = 0;
        GSM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, ekeys.p, esorted.p, nnz, 0, end_bit, s));
        DevBuf<uint8_t> tmp;
        tmp.ensure(tmp_bytes, s);
        GSM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, ekeys.p, esorted.p, nnz, 0, end_bit, s));
        k_extract_cols<<<grid_for(nnz), 256, 0, s>>>(esorted.p, nnz, g.cols);
        GSM_LAUNCH("k_extract_cols");
    } else if (nnz > 0) {
        DevBuf<int32_t> ecols;
        ecols.ensure(nnz, s);
        k_edge_cols<<<grid_for(n * 32), 256, 0, s>>>(d_off, d_cols, g.off, g.new2old, g.old2new, n, ecols.p);
        GSM_LAUNCH("k_edge_cols");
        // Under the (degree, id) order the long lists are the last ranks.  CUB's segmented sort
        // runs few, long segments at low occupancy (ncu: 43 ms, 12.5 % warps active on
        // R-MAT-24), so the lists of degree >= kBig are sorted together by one radix sort of
        // (list index, id) keys and only the prefix of short lists goes through the
        // segmented sort.
        const int64_t kBig = knobs().bigsort_min;
        int64_t nbig = 0, split = nnz;
        if (knobs().bigsort && knobs().order == 0 && g.max_degree >= kBig) {
            DevBuf<int64_t> hv;
            hv.ensure(2, s);
            k_big_suffix<<<grid_for(n), 256, 0, s>>>(g.off, n, kBig, hv.p);
            GSM_LAUNCH("k_big_suffix");
            int64_t h[2];
            GSM_CUDA(cudaMemcpyAsync(h, hv.p, sizeof(h), cudaMemcpyDeviceToHost, s));
            GSM_CUDA(cudaStreamSynchronize(s));
            nbig = h[0];
            split = h[1];
        }
        const int64_t nsmall = n - nbig;
        if (split > 0) {
            size_t tmp_bytes = 0;
            GSM_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, ecols.p, g.cols, split, nsmall, g.off,
                                                        g.off + 1, s));
            DevBuf<uint8_t> tmp;
            tmp.ensure(tmp_bytes, s);
            GSM_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.p, tmp_bytes, ecols.p, g.cols, split, nsmall, g.off,
                                                        g.off + 1, s));
        }
        if (nbig > 0) {
            const int64_t E = nnz - split;
            DevBuf<uint64_t> bk, bs;
            bk.ensure(E, s);
            bs.ensure(E, s);
            k_big_keys<<<grid_for(nbig * 32), 256, 0, s>>>(g.off, ecols.p, nsmall, nbig, split, bk.p);
            GSM_LAUNCH("k_big_keys");
            const int end_bit = 32 + bits_for((uint64_t)nbig);
            size_t tb = 0;
            GSM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, bk.p, bs.p, E, 0, end_bit, s));
            DevBuf<uint8_t> tmp;
            tmp.ensure(tb, s);
            GSM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, bk.p, bs.p, E, 0, end_bit, s));
            k_extract_cols<<<grid_for(E), 256, 0, s>>>(bs.p, E, g.cols + split);
            GSM_LAUNCH("k_extract_cols(big)");
        }
    }
    k_up<<<grid_for(n), 256, 0, s>>>(g.off, g.cols, n, g.up);
    GSM_LAUNCH("k_up");
    phase("relabelled lists");
    // 3. hub adjacency bitmap of the H highest-ranked vertices (load-time derived data)
    if (knobs().hub_bits > 0) {
        const int32_t H = (int32_t)std::min<int64_t>(n, knobs().hub_bits) & ~31;
        if (H >= 64) {
            g.hub_base = (int32_t)(n - H);
            g.hub_words = H / 32;
            g.hub_bytes = 4 * hub_total_words(g.hub_words);
            g.hub_bits = static_cast<uint32_t*>(dev_alloc((size_t)g.hub_bytes, s));
            GSM_CUDA(cudaMemsetAsync(g.hub_bits, 0, (size_t)g.hub_bytes, s));
            k_hub_bits<<<grid_for((int64_t)H * 32), 256, 0, s>>>(g.off, g.cols, g.up, g.hub_base, H, g.hub_words,
                                                                 g.hub_bits);
            GSM_LAUNCH("k_hub_bits");
        }
    }
    phase("hub bitmap");
    // 4. hashed N+(v) tables of the vertices with |N+(v)| >= nh_min (load-time derived data)
    if (knobs().nhash_min > 0 && nnz > 0) {
        DevBuf<int64_t> nb, excl;
        nb.ensure(n, s);
        excl.ensure(n + 1, s);
        k_nh_sizes<<<grid_for(n), 256, 0, s>>>(g.off, g.up, n, knobs().nhash_min, nb.p);
        GSM_LAUNCH("k_nh_sizes");
        GSM_CUDA(cudaMemsetAsync(excl.p, 0, sizeof(int64_t), s));
        size_t sb = 0;
        GSM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, sb, nb.p, excl.p + 1, n, s));
        DevBuf<uint8_t> stmp;
        stmp.ensure(sb, s);
        GSM_CUDA(cub::DeviceScan::InclusiveSum(stmp.p, sb, nb.p, excl.p + 1, n, s));
        int64_t total = 0;
        GSM_CUDA(cudaMemcpyAsync(&total, excl.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        if (total > 0 && total < (int64_t)INT32_MAX) {
            g.nh_min = knobs().nhash_min;
            g.nh_buckets_total = total;
            g.nh_off = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * n, s));
            g.nh_tab = static_cast<int32_t*>(dev_alloc(32 * (size_t)total, s));
            GSM_CUDA(cudaMemsetAsync(g.nh_tab, 0xff, 32 * (size_t)total, s));
            k_nh_offsets<<<grid_for(n), 256, 0, s>>>(nb.p, excl.p, n, g.nh_off);
            GSM_LAUNCH("k_nh_offsets");
            k_nh_insert<<<grid_for(n * 32), 256, 0, s>>>(g.off, g.cols, g.up, g.nh_off, n, g.nh_tab);
            GSM_LAUNCH("k_nh_insert");
        }
    }
    phase("hashed N+ tables");
    g.nplus = static_cast<int4*>(dev_alloc(sizeof(int4) * n, s));
    k_nplus<<<grid_for(n), 256, 0, s>>>(g.off, g.up, g.nh_off, n, g.nplus);
    GSM_LAUNCH("k_nplus");
    phase("N+ descriptors");
    if (labels) {
        g.labels = static_cast<uint32_t*>(dev_alloc(sizeof(uint32_t) * n, s));
        k_permute_labels<<<grid_for(n), 256, 0, s>>>(d_lab, g.new2old, n, g.labels);
        GSM_LAUNCH("k_permute_labels");
        h->labeled = true;
        // label-grouped lists: each list re-sorted by (label, id) as packed 31-bit keys,
        // so a labeled query's admissible candidates form one contiguous segment
        DevBuf<unsigned> maxl;
        maxl.ensure(1, s);
        GSM_CUDA(cudaMemsetAsync(maxl.p, 0, sizeof(unsigned), s));
        k_max_label<<<grid_for(n), 256, 0, s>>>(g.labels, n, maxl.p);
        GSM_LAUNCH("k_max_label");
        unsigned hmax = 0;
        GSM_CUDA(cudaMemcpyAsync(&hmax, maxl.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        const int idbits = bits_for((uint64_t)(n > 1 ? n - 1 : 1));
        const int lbits = hmax ? bits_for((uint64_t)hmax) : 0;
        g.max_label = hmax;
        if (nnz > 0 && idbits + lbits <= 31) {
            g.idbits = idbits;
            g.lkeys = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * nnz, s));
            DevBuf<uint64_t> ekeys, esorted;
            ekeys.ensure(nnz, s);
            esorted.ensure(nnz, s);
            k_label_edge_keys<<<grid_for(n * 32), 256, 0, s>>>(g.off, g.cols, g.labels, n, idbits, ekeys.p);
            GSM_LAUNCH("k_label_edge_keys");
            const int end_bit = 32 + bits_for((uint64_t)n);
            size_t tmp_bytes = 0;
            GSM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, ekeys.p, esorted.p, nnz, 0, end_bit, s));
            DevBuf<uint8_t> tmp;
            tmp.ensure(tmp_bytes, s);
            GSM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, ekeys.p, esorted.p, nnz, 0, end_bit, s));
            k_extract_cols<<<grid_for(nnz), 256, 0, s>>>(esorted.p, nnz, g.lkeys);
            GSM_LAUNCH("k_extract_cols(lkeys)");
            const int nl = (int)hmax + 1;
            if (knobs().lidx_min > 0 && nl <= 64) {
                DevBuf<int64_t> sz, excl;
                sz.ensure(n, s);
                excl.ensure(n + 1, s);
                k_lidx_sizes<<<grid_for(n), 256, 0, s>>>(g.off, n, knobs().lidx_min, nl, sz.p);
                GSM_LAUNCH("k_lidx_sizes");
                GSM_CUDA(cudaMemsetAsync(excl.p, 0, sizeof(int64_t), s));
                size_t sb = 0;
                GSM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, sb, sz.p, excl.p + 1, n, s));
                DevBuf<uint8_t> stmp;
                stmp.ensure(sb, s);
                GSM_CUDA(cub::DeviceScan::InclusiveSum(stmp.p, sb, sz.p, excl.p + 1, n, s));
                int64_t total = 0;
                GSM_CUDA(cudaMemcpyAsync(&total, excl.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                GSM_CUDA(cudaStreamSynchronize(s));
                if (total > 0 && total < (int64_t)INT32_MAX) {
                    g.lidx_off = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * n, s));
                    g.lidx = static_cast<int32_t*>(dev_alloc(sizeof(int32_t) * total, s));
                    k_lidx_build<<<grid_for(n * 32), 256, 0, s>>>(g.off, g.lkeys, sz.p, excl.p, n, nl, idbits,
                                                                  g.lidx_off, g.lidx);
                    GSM_LAUNCH("k_lidx_build");
                }
            }
        }
    }
    phase("labels + keyed lists");
    GSM_CUDA(cudaStreamSynchronize(s));
    *out = h.release();
}

}  // namespace gsm

extern "C" {

gsm_status gsm_load_graph(int64_t num_nodes, const int64_t* row_offsets, const int32_t* col_indices,
                          const uint32_t* labels, int32_t pointers_on_device, const gsm_load_opts* opts,
                          gsm_graph** out) {
    try {
        gsm::clear_error();
        gsm::load_graph_impl(num_nodes, row_offsets, col_indices, labels, pointers_on_device, opts, out);
        return GSM_OK;
    } catch (const gsm::Failure& f) {
        gsm::set_error(f.msg);
        if (out) *out = nullptr;
        return f.status;
    } catch (const std::bad_alloc&) {
        gsm::set_error("host allocation failed");
        if (out) *out = nullptr;
        return GSM_ERR_OUT_OF_MEMORY;
    } catch (...) {
        gsm::set_error("unexpected exception in gsm_load_graph");
        if (out) *out = nullptr;
        return GSM_ERR_CUDA;
    }
}

gsm_status gsm_free(gsm_graph* g) {
    gsm::free_graph(g);
    return GSM_OK;
}

gsm_status gsm_graph_info(const gsm_graph* g, int64_t* num_nodes, int64_t* num_directed_edges, int32_t* labeled,
                          int32_t* device) {
    if (!g) {
        gsm::set_error("graph is NULL");
        return GSM_ERR_INVALID_ARGUMENT;
    }
    if (num_nodes) *num_nodes = g->g.n;
    if (num_directed_edges) *num_directed_edges = g->g.nnz;
    if (labeled) *labeled = g->labeled ? 1 : 0;
    if (device) *device = g->device;
    return GSM_OK;
}

const char* gsm_last_error(void) { return gsm::g_last_error.c_str(); }

const char* gsm_version(void) { return "gsm-b200 0.1 (sm_100a)"; }

}  // extern "C"

// accessors used by gsm_match.cu
namespace gsm {
const DevGraph& graph_of(const gsm_graph* h) { return h->g; }
int device_of(const gsm_graph* h) { return h->device; }
cudaStream_t stream_of(const gsm_graph* h) { return h->stream; }
bool labeled_of(const gsm_graph* h) { return h->labeled; }
Workspace& workspace_of(const gsm_graph* h) { return *h->ws; }
}  // namespace gsm
