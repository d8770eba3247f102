// gsm_common.h — device-side types and error plumbing shared by the .cu files
// of libgsm (product side).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "gsm.h"
#include "gsm_internal.h"

namespace gsm {

// ---------------------------------------------------------------- device checks
// Build with -DGSM_DEVICE_CHECKS (libgsm_checked.so, _build.build(checked=True)): kernels test
// their shared-memory / staging / table indices against the sizes they were launched with and
// OR a bit into a per-translation-unit device flag instead of touching memory out of bounds
// unchecked; gsm_match collects the flags after every call and fails with GSM_ERR_CUDA
// ("device check failed") if any is set.  The stand-in for compute-sanitizer, which this
// GPU pool does not allow.  Release builds compile the checks away.
#ifdef GSM_DEVICE_CHECKS
void dcheck_register(unsigned (*read_and_clear)());
unsigned dcheck_collect();
#ifdef __CUDACC__
static __device__ unsigned int g_dcheck_tu;
static unsigned dcheck_read_tu() {
    unsigned h = 0, z = 0;
    cudaMemcpyFromSymbol(&h, g_dcheck_tu, sizeof(h));
    cudaMemcpyToSymbol(g_dcheck_tu, &z, sizeof(z));
    return h;
}
static const bool g_dcheck_registered = (dcheck_register(&dcheck_read_tu), true);
#define GSM_DCHECK(cond, bit)                                            \
    do {                                                                 \
        if (!(cond)) atomicOr(&::gsm::g_dcheck_tu, (unsigned)(bit));     \
    } while (0)
#endif
#else
#define GSM_DCHECK(cond, bit) \
    do {                      \
    } while (0)
#endif
enum : unsigned {
    DCHK_WARP_D = 1u,        // k_clique_warp root with |N+(u)| > 32
    DCHK_CTA_D = 2u,         // k_clique_cta root beyond the launch's dmax
    DCHK_CUCKOO = 4u,        // cuckoo slot outside the 2P table
    DCHK_PAIRQ = 8u,         // level-3 pair queue index >= 32
    DCHK_AROW = 16u,         // bit-row word outside the triangular row block
    DCHK_SLAB = 32u,         // global-slab CTA beyond the slabs allocated
    DCHK_STAGE = 64u,        // k_expand staging slot / row index beyond the tile capacity
    DCHK_NH = 128u,          // hashed N+(v) probe walked more buckets than the table has
    DCHK_MERGE = 256u,       // merge-path output index beyond na + nb
};


// Relabelled device CSR (new ids = rank by ascending (degree, original id)).
struct DevGraph {
    int64_t n = 0;
    int64_t nnz = 0;
    int64_t* off = nullptr;       // n+1
    int32_t* cols = nullptr;      // nnz, ascending per list (new ids)
    int32_t* up = nullptr;        // n: neighbours with smaller new id; N+(v) = cols[off[v]+up[v], off[v+1])
    uint32_t* labels = nullptr;   // n (new ids) or nullptr
    // label-grouped lists (labeled graphs whose label and id bits fit 31 bits): list of v
    // re-sorted by (label(w), w), stored as keys label(w) << idbits | w, same offsets
    int32_t* lkeys = nullptr;
    int32_t idbits = 0;
    // label index of the keyed lists (vertices with degree >= lidx_min, labels <= 63): lidx_off[v]
    // = first entry of v's (max_label + 2) int32 offsets (relative to off[v]) where each label's
    // segment starts, or -1 — a plan row's label segment is two loads instead of two binary
    // searches over the whole list
    int32_t* lidx_off = nullptr;
    int32_t* lidx = nullptr;
    uint32_t max_label = 0;
    int32_t* new2old = nullptr;   // n
    int32_t* old2new = nullptr;   // n
    int32_t max_degree = 0;
    // Hub adjacency bitmap ("dense core"): the H highest-ranked vertices
    // [hub_base, n) — the highest degrees — with, per hub a, the bits of N+(a) (which lies
    // entirely inside the hub range, N+(a) ⊂ (a, n)).  Upper-triangular by 32-row blocks:
    // row r = a - hub_base keeps words [r/32, hub_words); hub_row() gives a pointer that is
    // indexed by the column's full word index c >> 5.  An adjacency test of two hubs is one
    // L2-resident load instead of a binary search.  nullptr = disabled (GSM_HUB_BITS=0).
    uint32_t* hub_bits = nullptr;
    int32_t hub_base = 0;
    int32_t hub_words = 0;        // H / 32
    int64_t hub_bytes = 0;
    // Hashed N+(v) ("membership tables"): for every v with |N+(v)| >= nh_min, an
    // open-addressing table of N+(v) in 32-byte buckets of 8 int32 slots (one DRAM sector;
    // nh_buckets(|N+(v)|) buckets, load <= 1/2, -1 = empty, slots filled from slot 0, overflow
    // to the next bucket).  nh_off[v] = first bucket of v's table, or -1.  A membership test
    // x ∈ N+(v) is then one sector load (rarely two) instead of a binary search over
    // log2 |N+(v)| dependent probes.  nullptr = disabled (GSM_NHASH_MIN=0).
    int32_t* nh_off = nullptr;
    int32_t* nh_tab = nullptr;
    // packed N+(v) descriptor per vertex, one 16-byte load: {begin lo, begin hi, |N+(v)|, nh_off}
    // (begin = off[v] + up[v]); read by the clique kernels instead of off[v], off[v+1], up[v]
    // and nh_off[v] (three to four random sectors -> one)
    int4* nplus = nullptr;
    int64_t nh_buckets_total = 0;
    int32_t nh_min = 0;
};

// buckets of the N+(v) table of a list of length L (a power of two >= L / 4)
__host__ __device__ __forceinline__ unsigned nh_buckets(int64_t L) {
    unsigned b = 1;
    while ((int64_t)b * 4 < L) b <<= 1;
    return b;
}
__host__ __device__ __forceinline__ unsigned nh_hash(int32_t x, unsigned B) {
    return ((unsigned)x * 0x9E3779B1u) & (B - 1);  // B is a power of two
}
#ifdef __CUDACC__
__device__ __forceinline__ void nplus_load(const int4* __restrict__ np, int32_t v, int64_t& begin, int& len,
                                           int32_t& nh) {
    const int4 x = __ldg(np + v);
    begin = (int64_t)(uint32_t)x.x | ((int64_t)x.y << 32);
    len = x.z;
    nh = x.w;
}
// x ∈ N+(v), given v's table (first bucket tb) of B buckets: one 32-byte bucket per probe
__device__ __forceinline__ bool nh_find(const int32_t* __restrict__ tab, int32_t tb, unsigned B, int32_t x,
                                        unsigned& probes) {
    unsigned b = nh_hash(x, B);
    for (unsigned it = 0;; ++it) {
#ifdef GSM_DEVICE_CHECKS
        if (it >= B) {  // a table always keeps an empty slot (load <= 1/2)
            GSM_DCHECK(false, DCHK_NH);
            return false;
        }
#endif
        const int4* p = reinterpret_cast<const int4*>(tab + 8 * ((int64_t)tb + b));
        const int4 u = __ldg(p), w = __ldg(p + 1);
        ++probes;
        if ((u.x == x) | (u.y == x) | (u.z == x) | (u.w == x) | (w.x == x) | (w.y == x) | (w.z == x) | (w.w == x))
            return true;
        if (w.w < 0) return false;  // bucket not full: x would have been placed here
        b = (b + 1) & (B - 1);
    }
}
#endif

// pointer p with p[c >> 5] = the word holding column c (c > r) of hub row r
__host__ __device__ __forceinline__ const uint32_t* hub_row(const uint32_t* bits, int hw, int r) {
    const int64_t b = r >> 5;
    return bits + 32 * (b * hw - b * (b - 1) / 2) + (int64_t)(r & 31) * (hw - b) - b;
}
__host__ __device__ __forceinline__ int64_t hub_total_words(int hw) {
    return 32 * ((int64_t)hw * hw - (int64_t)hw * (hw - 1) / 2);
}

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
void clear_error();

struct Failure {
    gsm_status status;
    std::string msg;
};

[[noreturn]] inline void fail(gsm_status s, const std::string& msg) { throw Failure{s, msg}; }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    if (e == cudaErrorMemoryAllocation) fail(GSM_ERR_OUT_OF_MEMORY, buf);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) fail(GSM_ERR_NO_DEVICE, buf);
    fail(GSM_ERR_CUDA, buf);
}

#define GSM_CUDA(call) ::gsm::cuda_check((call), #call, __FILE__, __LINE__)
#define GSM_LAUNCH(what) ::gsm::cuda_check(cudaGetLastError(), what, __FILE__, __LINE__)

// ---------------------------------------------------------------- host-side trace (GSM_TRACE=1)
struct HostTrace {
    double alloc_ms = 0, alloc_bytes = 0, sync_ms = 0;
    long allocs = 0, syncs = 0;
};
extern HostTrace g_trace;

// ---------------------------------------------------------------- tuning switches
// Path/tuning switches.  Read from the environment ONCE at the start of
// every gsm_match (load_knobs) into a thread-local snapshot that every launcher reads —
// no function-static caches, so a change between calls always takes effect.  Defaults are
// the measured best; tests use the switches to force specific paths.  None of them skips
// work or changes a result.
struct Knobs {
    int clique = 1;           // GSM_CLIQUE: 0 = cliques take the breadth-first path
    int clique_warp = 32;     // GSM_CLIQUE_WARP: |N+(u)| edge of the warp-per-root kernel (0 = off)
    int clique_dsmem = 0;     // GSM_CLIQUE_DSMEM: cap of the shared-memory CTA buckets (0 = max fitting)
    int clique_dmax = 0;      // GSM_CLIQUE_DMAX: cap of the global-slab bucket (0 = max fitting)
    int clique_stream = 128;  // GSM_CLIQUE_STREAM: stream-vs-search threshold (x/32 per remaining entry)
    int clique_hash = 1;      // GSM_CLIQUE_HASH: 0 = rows by binary search only
    int clique_occ = 3;       // GSM_CLIQUE_OCC: register cap for 0 uncapped / 1 2048 / 2 1536 / 3 1280 / 4 1024 resident threads
    int pair_tail = 1;        // GSM_PAIR_TAIL
    int pair_thread_max = 16; // GSM_PAIR_THREAD_MAX
    int fused_tail = 1;       // GSM_FUSED_TAIL
    int tail_cap = 1024;      // GSM_TAIL_CAP (clamped 64..6144, even)
    int tail_block_cap = 40960;  // GSM_TAIL_BLOCK_CAP (clamped 256..49152)
    int tail_bratio = 100;    // GSM_TAIL_BRATIO_PCT
    int count_walk = 1;       // GSM_COUNT_WALK
    int expand_td = 512;      // GSM_EXPAND_TD (clamped 128..2048)
    int expand_ilp = 1;       // GSM_EXPAND_ILP (1, 2 or 4)
    int trace = 0;            // GSM_TRACE: 1 host trace, 2 per-phase cycle counters
    int member_hub = 1;       // GSM_MEMBER_HUB: pair-tail membership tests of two hubs by the hub bitmap
    int member_swap = 0;      // GSM_MEMBER_SWAP: segments longer than this may search in N(v) (0 = never; R-MAT-22 284 vs 136 ms)
    int plan_groups = 0;      // GSM_PLAN_GROUPS: row plans by lane groups (R-MAT-22 plan 19.6 vs 15.5 ms: off)
    int compress = -1;        // GSM_COMPRESS: 1/0 force the compressed partial layout on/off (-1 = flag)
    int lookahead = -1;       // GSM_LOOKAHEAD: overrides gsm_match_opts.lookahead when >= 0
    int hub_bits = 65536;     // GSM_HUB_BITS: H of the hub adjacency bitmap built at load (0 = none; R-MAT-24: 32k 378, 64k 364 ms)
    int clique_hub = 1;       // GSM_CLIQUE_HUB: clique rows of a hub pivot by bitmap lookups
    int clique_hub_ratio = 64;  // GSM_CLIQUE_HUB_RATIO: lookups when 32 nj <= ratio |N+(S[i])|
    int filter_u = 1;         // GSM_FILTER_U: K1 groups of 4 vertices per thread per pass (1, 2, 4; R-MAT-24: 0.063 / 0.086 / 0.126 ms)
    int clique_ntsel = 1;     // GSM_CLIQUE_NTSEL: CTA size per bucket from the occupancy calculator (0: shared memory only)
    int clique_lazy_ck = 1;   // GSM_CLIQUE_LAZYCK: per-root cuckoo table only when some row streams
    int clique_ranges = 0;    // GSM_CLIQUE_RANGES: K4 level 3 over the rows' nonzero word ranges (interleaved A/B on R-MAT-24: K4 269.5 on vs 260.4 ms off)
    int bigsort_min = 8192;   // GSM_BIGSORT_MIN: list length from which GSM_BIGSORT takes a list
    int bigsort = 0;          // GSM_BIGSORT (load): long lists by one radix sort (R-MAT-24 relabel 52.9 vs 50.1 ms: off)
    int filter_bps = 8;       // GSM_FILTER_BPS: K1 grid = 148 x this blocks (grid-stride beyond)
    int lidx_min = 32;        // GSM_LIDX_MIN (read at gsm_load_graph): label index for degree >= this (0 = none)
    int nhash_min = 64;       // GSM_NHASH_MIN (read at gsm_load_graph): hashed N+(v) for |N+(v)| >= this (0 = none; 8 / 16 / 64 match-time equal, 64 builds less)
    int clique_nh_stream = 64;  // GSM_CLIQUE_NH_STREAM: with a table, stream N+(S[i]) when 32 len <= this x nj
    int order = 0;            // GSM_ORDER (read at gsm_load_graph): 0 = rank by (degree, id), 1 = approximate degeneracy
};
void load_knobs();
const Knobs& knobs();

// ---------------------------------------------------------------- device memory
// Stream-ordered allocations from the device's default memory pool.
void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, cudaStream_t s);

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) dev_free(p, s);
        p = nullptr;
        n = 0;
    }
    // grow-only: contents are NOT preserved
    void ensure(size_t count, cudaStream_t stream) {
        s = stream;
        if (count <= n && p) return;
        release();
        s = stream;
        p = static_cast<T*>(dev_alloc(sizeof(T) * (count ? count : 1), stream));
        n = count;
    }
};

// ---------------------------------------------------------------- kernel launch helpers
struct KernelTimer;  // defined in gsm_match.cu

}  // namespace gsm
