// gsm_kernels.cu — the sm_100a kernels of the GSM hot path.
//
// Integer work only: no tensor cores (nothing here is a dense contraction).
// The roofline is memory: K1 streams the offsets/labels (HBM-bound); the
// expand kernel is dominated by reads of candidate lists and dependent random
// probes (cmask bytes, binary searches) into a CSR that is L2-resident for
// small graphs and HBM-resident for large ones.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gsm_kernels.h"

namespace gsm {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxGrid = 148 * 16;

inline int grid_for(int64_t items, int threads = kThreads, int cap = kMaxGrid) {
    int64_t b = (items + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

}  // namespace

// ============================================================================
// K1 candidate filter — Alg. 1 "Filter+Compute" (line 8), PAPER P:110, P:129,
// compatible = same label and degree >= deg_Q(u).  A coalesced, vectorised
// stream: each thread owns 4 consecutive vertices — two 16-byte loads of offsets
// (the 5th offset comes from the next lane by a shuffle), one 16-byte load of
// labels, one 4/8/16-byte store of the 4 masks.  |C(u)| = per-thread bit counts
// summed by one warp reduction (redux.sync) per query vertex per 128 vertices.
// ============================================================================
template <typename MaskT>
struct MaskVec4;
template <>
struct MaskVec4<uint8_t> {
    using T = uint32_t;
    __device__ static T pack(const uint32_t* m) { return m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24); }
};
template <>
struct MaskVec4<uint16_t> {
    using T = uint2;
    __device__ static T pack(const uint32_t* m) { return make_uint2(m[0] | (m[1] << 16), m[2] | (m[3] << 16)); }
};
template <>
struct MaskVec4<uint32_t> {
    using T = uint4;
    __device__ static T pack(const uint32_t* m) { return make_uint4(m[0], m[1], m[2], m[3]); }
};

template <typename MaskT, int kU>
__global__ void __launch_bounds__(kThreads, 8 / kU) k_filter(const int64_t* __restrict__ off,
                                                     const uint32_t* __restrict__ labels, int64_t n,
                                                     FilterQuery q, MaskT* __restrict__ cmask,
                                                     unsigned long long* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    unsigned long long mine = 0;  // lane u: |C(u)| of this warp's vertices
    const int64_t nvec = n >> 2;  // full groups of 4 vertices
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto mask_of = [&](int64_t d, uint32_t lab) {
        uint32_t m = 0;
        for (int u = 0; u < q.k; ++u) m |= (uint32_t)((!q.use_labels || lab == q.qlabel[u]) && d >= q.qdeg[u]) << u;
        return m;
    };
    // grid-stride over groups, kU groups per thread per pass with every load issued before any
    // use (more bytes in flight per thread: ncu showed the one-group loop at 31 % of DRAM
    // bandwidth, stalled on the shuffle that waits for the offsets); the loop bound is
    // block-uniform so the shuffles stay converged
    for (int64_t g0 = (int64_t)blockIdx.x * blockDim.x; g0 < nvec; g0 += stride * kU) {
        longlong2 A[kU], Bq[kU];
        uint4 lab[kU];
        int64_t last[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int64_t gi = g0 + j * stride + threadIdx.x;
            A[j] = make_longlong2(0, 0);
            Bq[j] = make_longlong2(0, 0);
            lab[j] = make_uint4(0, 0, 0, 0);
            last[j] = 0;
            if (gi < nvec) {
                A[j] = __ldcs(reinterpret_cast<const longlong2*>(off) + 2 * gi);
                Bq[j] = __ldcs(reinterpret_cast<const longlong2*>(off) + 2 * gi + 1);
                if (labels && q.use_labels) lab[j] = __ldcs(reinterpret_cast<const uint4*>(labels) + gi);
                if (lane == 31 || gi + 1 >= nvec) last[j] = __ldg(off + 4 * gi + 4);
            }
        }
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int64_t gi = g0 + j * stride + threadIdx.x;
            const bool live = gi < nvec;
            const int64_t nxt = __shfl_down_sync(0xffffffffu, A[j].x, 1);
            const int64_t o4 = (lane == 31 || gi + 1 >= nvec) ? last[j] : nxt;
            uint32_t m[4] = {0, 0, 0, 0};
            if (live) {
                m[0] = mask_of(A[j].y - A[j].x, lab[j].x);
                m[1] = mask_of(Bq[j].x - A[j].y, lab[j].y);
                m[2] = mask_of(Bq[j].y - Bq[j].x, lab[j].z);
                m[3] = mask_of(o4 - Bq[j].y, lab[j].w);
                reinterpret_cast<typename MaskVec4<MaskT>::T*>(cmask)[gi] = MaskVec4<MaskT>::pack(m);
            }
            for (int u = 0; u < q.k; ++u) {
                const unsigned c = ((m[0] >> u) & 1u) + ((m[1] >> u) & 1u) + ((m[2] >> u) & 1u) + ((m[3] >> u) & 1u);
                const unsigned w = __reduce_add_sync(0xffffffffu, c);
                if (lane == u) mine += w;
            }
        }
    }
    // the last n % 4 vertices
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const int64_t v = 4 * nvec + lane;
        uint32_t m = 0;
        if (v < n) {
            m = mask_of(off[v + 1] - off[v], labels ? labels[v] : 0u);
            cmask[v] = (MaskT)m;
        }
        for (int u = 0; u < q.k; ++u) {
            const unsigned w = __popc(__ballot_sync(0xffffffffu, (m >> u) & 1u));
            if (lane == u) mine += w;
        }
    }
    if (lane < q.k && mine) atomicAdd(&counts[lane], mine);
}

void launch_filter(const DevGraph& g, const FilterQuery& q, void* cmask, unsigned long long* counts,
                   cudaStream_t s) {
    // kU groups of 4 vertices per thread per pass (GSM_FILTER_U = 1, 2, 4); grid = SMs x resident blocks
    const int U = knobs().filter_u;
    const int grid = grid_for((g.n + 4 * U - 1) / (4 * U), kThreads, 148 * knobs().filter_bps / U);
    auto go = [&](auto kern, auto* mask) { kern<<<grid, kThreads, 0, s>>>(g.off, g.labels, g.n, q, mask, counts); };
    const int mb = mask_bytes_for(q.k);
    if (U == 4) {
        if (mb == 1) go(k_filter<uint8_t, 4>, (uint8_t*)cmask);
        else if (mb == 2) go(k_filter<uint16_t, 4>, (uint16_t*)cmask);
        else go(k_filter<uint32_t, 4>, (uint32_t*)cmask);
    } else if (U == 2) {
        if (mb == 1) go(k_filter<uint8_t, 2>, (uint8_t*)cmask);
        else if (mb == 2) go(k_filter<uint16_t, 2>, (uint16_t*)cmask);
        else go(k_filter<uint32_t, 2>, (uint32_t*)cmask);
    } else {
        if (mb == 1) go(k_filter<uint8_t, 1>, (uint8_t*)cmask);
        else if (mb == 2) go(k_filter<uint16_t, 1>, (uint16_t*)cmask);
        else go(k_filter<uint32_t, 1>, (uint32_t*)cmask);
    }
    GSM_LAUNCH("k_filter");
}

template <typename MaskT>
__global__ void k_mask_to_original(const MaskT* __restrict__ cmask, const int32_t* __restrict__ new2old, int64_t n,
                                   uint32_t* __restrict__ out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        out[new2old[v]] = (uint32_t)cmask[v];
}

void launch_mask_to_original(const DevGraph& g, const void* cmask, int mask_bytes, uint32_t* out, cudaStream_t s) {
    switch (mask_bytes) {
        case 1: k_mask_to_original<<<grid_for(g.n), kThreads, 0, s>>>((const uint8_t*)cmask, g.new2old, g.n, out); break;
        case 2: k_mask_to_original<<<grid_for(g.n), kThreads, 0, s>>>((const uint16_t*)cmask, g.new2old, g.n, out); break;
        default: k_mask_to_original<<<grid_for(g.n), kThreads, 0, s>>>((const uint32_t*)cmask, g.new2old, g.n, out); break;
    }
    GSM_LAUNCH("k_mask_to_original");
}

// ============================================================================
// K5 neighbourhood-encoding refinement (with the 1-step look-ahead condition
// folded in: bit u of v also needs, for every query neighbour u' of u, some
// surviving neighbour of v with bit u') — Alg. 1 line 7 "Advance+Compute: NE for
// each node in G" and line 8 "Filter ... update G's (NE, deg)" (P:108-110,
// P:134).  NE(v) = sum of the labels of v's neighbours (each label counted as
// label+1 so that it is positive; unlabeled: 1 per neighbour, i.e.
// the degree), taken — like the effective degree — over the neighbours
// that are still a candidate of some query vertex (cmask != 0), so each round
// prunes against the previous round's survivors.  Bit u of cmask[v] survives iff
// deg_eff(v) >= deg_Q(u) and NE(v) >= NE_Q(u).  Sound: an embedding's images
// keep their bits (the images of u's query neighbours are distinct alive
// neighbours of f(u) with the query's labels).  Warp per vertex over its list.
// ============================================================================
template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_refine(const int64_t* __restrict__ off,
                                                     const int32_t* __restrict__ cols,
                                                     const uint32_t* __restrict__ labels, int64_t n, FilterQuery q,
                                                     const int64_t* __restrict__ qne, const MaskT* __restrict__ in,
                                                     MaskT* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = warp; v < n; v += nwarps) {
        const uint32_t m = in[v];
        if (m == 0) {
            if (lane == 0) out[v] = 0;
            continue;
        }
        int64_t deg = 0, ne = 0;
        uint32_t nbr = 0;  // query vertices some neighbour of v can still host
        for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
            const int32_t w = cols[e];
            const uint32_t mw = in[w];
            if (mw != 0) {
                ++deg;
                ne += (labels && q.use_labels) ? (int64_t)labels[w] + 1 : 1;
                nbr |= mw;
            }
        }
        for (int o = 16; o; o >>= 1) {
            deg += __shfl_xor_sync(0xffffffffu, deg, o);
            ne += __shfl_xor_sync(0xffffffffu, ne, o);
            nbr |= __shfl_xor_sync(0xffffffffu, nbr, o);
        }
        if (lane == 0) {
            uint32_t keep = m;
            for (int u = 0; u < q.k; ++u) {
                if (!((m >> u) & 1u)) continue;
                // NE / effective degree and the 1-step look-ahead folded into the filter
                // (a state whose query neighbour has no candidate among v's
                // neighbours has no consistent descendant)
                if (deg < q.qdeg[u] || ne < qne[u] || (q.qadj[u] & ~nbr) != 0) keep &= ~(1u << u);
            }
            out[v] = (MaskT)keep;
        }
    }
}

template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_mask_counts(const MaskT* __restrict__ cmask, int64_t n, int k,
                                                          unsigned long long* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    unsigned long long mine = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t v = base + threadIdx.x;
        const uint32_t m = v < n ? (uint32_t)cmask[v] : 0u;
        for (int u = 0; u < k; ++u) {
            const unsigned b = __ballot_sync(0xffffffffu, (m >> u) & 1u);
            if (lane == u) mine += __popc(b);
        }
    }
    if (lane < k && mine) atomicAdd(&counts[lane], mine);
}

template <typename MaskT>
static void refine_t(const DevGraph& g, const FilterQuery& q, const int64_t* qne, int rounds, void* cmask, void* tmp,
                     unsigned long long* counts, cudaStream_t s) {
    MaskT* a = static_cast<MaskT*>(cmask);
    MaskT* b = static_cast<MaskT*>(tmp);
    for (int r = 0; r < rounds; ++r) {
        k_refine<MaskT><<<grid_for(g.n * 32), kThreads, 0, s>>>(g.off, g.cols, g.labels, g.n, q, qne, a, b);
        GSM_LAUNCH("k_refine");
        GSM_CUDA(cudaMemcpyAsync(a, b, sizeof(MaskT) * g.n, cudaMemcpyDeviceToDevice, s));
    }
    GSM_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * kMaxK, s));
    k_mask_counts<MaskT><<<grid_for(g.n), kThreads, 0, s>>>(a, g.n, q.k, counts);
    GSM_LAUNCH("k_mask_counts");
}

void launch_refine(const DevGraph& g, const FilterQuery& q, const int64_t* qne, int rounds, void* cmask, void* tmp,
                   unsigned long long* counts, cudaStream_t s) {
    switch (mask_bytes_for(q.k)) {
        case 1: refine_t<uint8_t>(g, q, qne, rounds, cmask, tmp, counts, s); break;
        case 2: refine_t<uint16_t>(g, q, qne, rounds, cmask, tmp, counts, s); break;
        default: refine_t<uint32_t>(g, q, qne, rounds, cmask, tmp, counts, s); break;
    }
}

// ============================================================================
// k-look-ahead tables (§3.3 "detect a state which won't have any
// consistent descendants k step ahead"; R17).  Per data vertex v and query
// vertex u: c[v][u] = |{w in N(v) : mask[w] bit u}| capped at 255 — with mask = cmask
// this is how many neighbours of v can host u (1-step); with mask = ok1 it counts the
// neighbours that can host u AND have a candidate neighbour for each later query
// neighbour of u (2-step).  Warp per vertex, one ballot per query vertex per 32 entries.
// ============================================================================
template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_la_counts(const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ cols, int64_t n, int k,
                                                        const MaskT* __restrict__ mask, uint8_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = warp; v < n; v += nwarps) {
        unsigned c = 0;  // lane u: count for query vertex u
        for (int64_t e0 = off[v]; e0 < off[v + 1]; e0 += 32) {
            const int64_t e = e0 + lane;
            const uint32_t m = e < off[v + 1] ? (uint32_t)mask[cols[e]] : 0u;
            for (int u = 0; u < k; ++u) {
                const unsigned b = __ballot_sync(0xffffffffu, (m >> u) & 1u);
                if (lane == u) c += __popc(b);
            }
            if (__all_sync(0xffffffffu, lane >= k || c >= 255)) break;
        }
        if (lane < k) out[v * k + lane] = (uint8_t)min(c, 255u);
    }
}

template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_la_ok1(const MaskT* __restrict__ cmask, const uint8_t* __restrict__ c1,
                                                     int64_t n, int k, FilterQuery dq, MaskT* __restrict__ ok1) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t m = cmask[w];
        uint32_t have = 0;  // u'' with a candidate neighbour
        for (int u = 0; u < k; ++u) have |= (uint32_t)(c1[w * k + u] != 0) << u;
        uint32_t ok = 0;
        for (int u = 0; u < k; ++u)
            if (((m >> u) & 1u) && (dq.qadj[u] & ~have) == 0) ok |= 1u << u;
        ok1[w] = (MaskT)ok;
    }
}

void launch_la_counts(const DevGraph& g, int k, int mask_bytes, const void* mask, uint8_t* out, cudaStream_t s) {
    const int grid = grid_for(g.n * 32);
    switch (mask_bytes) {
        case 1: k_la_counts<uint8_t><<<grid, kThreads, 0, s>>>(g.off, g.cols, g.n, k, (const uint8_t*)mask, out); break;
        case 2: k_la_counts<uint16_t><<<grid, kThreads, 0, s>>>(g.off, g.cols, g.n, k, (const uint16_t*)mask, out); break;
        default: k_la_counts<uint32_t><<<grid, kThreads, 0, s>>>(g.off, g.cols, g.n, k, (const uint32_t*)mask, out); break;
    }
    GSM_LAUNCH("k_la_counts");
}

void launch_la_ok1(const DevGraph& g, int k, int mask_bytes, const void* cmask, const uint8_t* c1,
                   const uint32_t* dmask_host, void* ok1, cudaStream_t s) {
    FilterQuery dq;
    std::memset(&dq, 0, sizeof(dq));
    dq.k = k;
    for (int u = 0; u < k; ++u) dq.qadj[u] = dmask_host[u];
    const int grid = grid_for(g.n);
    switch (mask_bytes) {
        case 1: k_la_ok1<uint8_t><<<grid, kThreads, 0, s>>>((const uint8_t*)cmask, c1, g.n, k, dq, (uint8_t*)ok1); break;
        case 2: k_la_ok1<uint16_t><<<grid, kThreads, 0, s>>>((const uint16_t*)cmask, c1, g.n, k, dq, (uint16_t*)ok1); break;
        default: k_la_ok1<uint32_t><<<grid, kThreads, 0, s>>>((const uint32_t*)cmask, c1, g.n, k, dq, (uint32_t*)ok1); break;
    }
    GSM_LAUNCH("k_la_ok1");
}

// ============================================================================
// Roots: level-0 frontier = C(π[0]) (Alg. 1 line 11: "All-source BFS traversal
// from c_set"), compacted in ascending (degree, id) rank; multi-GPU shard s of P
// keeps the candidates whose vertex rank v (= relabelled id) has v % P == s
// (strided over the degree order, so hubs spread round-robin, and
// independent of the query).  Stable two-pass block-scan compaction.
// ============================================================================
constexpr int kRootItems = 8;
constexpr int64_t kRootTile = (int64_t)kThreads * kRootItems;

template <typename MaskT>
__device__ __forceinline__ int root_flags(const MaskT* cmask, int64_t n, int bit, int shard, int nshards,
                                          int64_t tile, uint32_t* flags) {
    const int64_t first = tile * kRootTile + (int64_t)threadIdx.x * kRootItems;
    int c = 0;
#pragma unroll
    for (int j = 0; j < kRootItems; ++j) {
        const int64_t v = first + j;
        const uint32_t f = (v < n && (int32_t)v % nshards == shard) ? ((cmask[v] >> bit) & 1u) : 0u;
        flags[j] = f;
        c += f;
    }
    return c;
}

template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_root_count(const MaskT* __restrict__ cmask, int64_t n, int bit,
                                                         int shard, int nshards, int64_t* __restrict__ tile_counts) {
    using BlockReduce = cub::BlockReduce<int, kThreads>;
    __shared__ typename BlockReduce::TempStorage tmp;
    uint32_t flags[kRootItems];
    const int c = root_flags(cmask, n, bit, shard, nshards, blockIdx.x, flags);
    const int total = BlockReduce(tmp).Sum(c);
    if (threadIdx.x == 0) tile_counts[blockIdx.x] = total;
}

template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_root_write(const MaskT* __restrict__ cmask, int64_t n, int bit,
                                                         const int64_t* __restrict__ tile_base, int shard,
                                                         int nshards, int32_t* __restrict__ roots) {
    using BlockScan = cub::BlockScan<int, kThreads>;
    __shared__ typename BlockScan::TempStorage tmp;
    uint32_t flags[kRootItems];
    const int c = root_flags(cmask, n, bit, shard, nshards, blockIdx.x, flags);
    int excl;
    BlockScan(tmp).ExclusiveSum(c, excl);
    int64_t pos = tile_base[blockIdx.x] + excl;
    const int64_t first = (int64_t)blockIdx.x * kRootTile + (int64_t)threadIdx.x * kRootItems;
#pragma unroll
    for (int j = 0; j < kRootItems; ++j)
        if (flags[j]) roots[pos++] = (int32_t)(first + j);
}

int64_t launch_roots(const DevGraph& g, const void* cmask, int mask_bytes, int bit, int shard, int nshards,
                     int32_t* roots, cudaStream_t s) {
    const int64_t tiles = (g.n + kRootTile - 1) / kRootTile;
    DevBuf<int64_t> counts, base;
    counts.ensure(tiles, s);
    base.ensure(tiles + 1, s);
    switch (mask_bytes) {
        case 1: k_root_count<uint8_t><<<(unsigned)tiles, kThreads, 0, s>>>((const uint8_t*)cmask, g.n, bit, shard, nshards, counts.p); break;
        case 2: k_root_count<uint16_t><<<(unsigned)tiles, kThreads, 0, s>>>((const uint16_t*)cmask, g.n, bit, shard, nshards, counts.p); break;
        default: k_root_count<uint32_t><<<(unsigned)tiles, kThreads, 0, s>>>((const uint32_t*)cmask, g.n, bit, shard, nshards, counts.p); break;
    }
    GSM_LAUNCH("k_root_count");
    GSM_CUDA(cudaMemsetAsync(base.p, 0, sizeof(int64_t), s));
    size_t tb = 0;
    GSM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, counts.p, base.p + 1, tiles, s));
    DevBuf<uint8_t> tmp;
    tmp.ensure(tb, s);
    GSM_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, counts.p, base.p + 1, tiles, s));
    switch (mask_bytes) {
        case 1: k_root_write<uint8_t><<<(unsigned)tiles, kThreads, 0, s>>>((const uint8_t*)cmask, g.n, bit, base.p, shard, nshards, roots); break;
        case 2: k_root_write<uint16_t><<<(unsigned)tiles, kThreads, 0, s>>>((const uint16_t*)cmask, g.n, bit, base.p, shard, nshards, roots); break;
        default: k_root_write<uint32_t><<<(unsigned)tiles, kThreads, 0, s>>>((const uint32_t*)cmask, g.n, bit, base.p, shard, nshards, roots); break;
    }
    GSM_LAUNCH("k_root_write");
    int64_t total = 0;
    GSM_CUDA(cudaMemcpyAsync(&total, base.p + tiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GSM_CUDA(cudaStreamSynchronize(s));
    return total;
}

template <typename MaskT>
__global__ void k_root_subset(const MaskT* __restrict__ cmask, int bit, const int32_t* __restrict__ old2new, int64_t n,
                              const int32_t* __restrict__ subset, int64_t len, int32_t* __restrict__ roots,
                              unsigned long long* __restrict__ count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o = subset[i];
        if (o < 0 || o >= n) continue;
        const int32_t v = old2new[o];
        if ((cmask[v] >> bit) & 1u) roots[atomicAdd(count, 1ull)] = v;
    }
}

int64_t launch_root_subset(const DevGraph& g, const void* cmask, int mask_bytes, int bit, const int32_t* subset_old,
                           int64_t len, int32_t* roots, cudaStream_t s) {
    DevBuf<unsigned long long> cnt;
    cnt.ensure(1, s);
    GSM_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), s));
    const int grid = grid_for(len);
    switch (mask_bytes) {
        case 1: k_root_subset<uint8_t><<<grid, kThreads, 0, s>>>((const uint8_t*)cmask, bit, g.old2new, g.n, subset_old, len, roots, cnt.p); break;
        case 2: k_root_subset<uint16_t><<<grid, kThreads, 0, s>>>((const uint16_t*)cmask, bit, g.old2new, g.n, subset_old, len, roots, cnt.p); break;
        default: k_root_subset<uint32_t><<<grid, kThreads, 0, s>>>((const uint32_t*)cmask, bit, g.old2new, g.n, subset_old, len, roots, cnt.p); break;
    }
    GSM_LAUNCH("k_root_subset");
    unsigned long long h = 0;
    GSM_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    GSM_CUDA(cudaStreamSynchronize(s));
    return (int64_t)h;
}

// ============================================================================
// Per-row plan (the "Advance" source).  The paper expands from the
// spanning-tree parent; we pick, per partial result, the backward neighbour
// whose admissible list segment is shortest (same result set, less work,
// SURVEY §8(a) A4).  ID constraints restrict candidates to an open
// interval (lo, hi) of new ids; because lists are sorted, the admissible part
// of a list is a contiguous segment, located with up[a] (exact when the bound
// is a itself) or a binary search.
// ============================================================================
__device__ __forceinline__ int64_t lower_bound_cols(const int32_t* __restrict__ cols, int64_t lo, int64_t hi,
                                                    int64_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)cols[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Admissible segment of N(a) for candidates in the open interval (lov, hiv):
// up[a] splits the sorted list at a itself (exact when a bound equals a);
// otherwise an optional binary search makes it exact.
__device__ __forceinline__ void admissible_segment(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                                                   const int32_t* __restrict__ up, int64_t n, int32_t a,
                                                   int64_t lov, int64_t hiv, bool refine, int64_t& s,
                                                   int64_t& t) {
    s = off[a];
    t = off[a + 1];
    if (lov >= a || hiv <= a) {
        const int64_t split = s + up[a];
        if (lov >= a) s = split;
        if (hiv <= a) t = split;
    }
    if (refine) {
        if (lov >= 0 && lov != a) s = lower_bound_cols(cols, s, t, lov + 1);
        if (hiv < n && hiv != a) t = lower_bound_cols(cols, s, t, hiv);
    }
    if (t < s) t = s;
}

__global__ void __launch_bounds__(kThreads) k_plan_rows(const Frontier F, int64_t R, LevelPlan L,
                                                        const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ cols,
                                                        const int32_t* __restrict__ up, int64_t n,
                                                        int64_t* __restrict__ rbeg, int64_t* __restrict__ rlen,
                                                        uint8_t* __restrict__ rpiv, int64_t* __restrict__ cbeg,
                                                        int32_t* __restrict__ clen,
                                                        const int32_t* __restrict__ lidx_off,
                                                        const int32_t* __restrict__ lidx) {
    const int nb = L.nb;
    int32_t buf[kMaxK];
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* row = frontier_row(F, r, buf);
        int64_t lov = -1, hiv = n;
        for (int q = 0; q < L.nlo; ++q) lov = max(lov, (int64_t)row[L.lo[q]]);
        for (int q = 0; q < L.nhi; ++q) hiv = min(hiv, (int64_t)row[L.hi[q]]);
        const bool empty = lov + 1 >= hiv;
        int64_t ps = 0, pt = 0;
        int bq = 0;
        if (L.keyed) {
            // (label, id)-sorted lists: the admissible keys [base|lov+1, base+hiv) are one segment
            int64_t blen = INT64_MAX;
            const int64_t klo = (int64_t)L.key_base + lov + 1, khi = (int64_t)L.key_base + hiv;
            for (int q = 0; q < nb; ++q) {
                const int32_t a = row[L.bpos[q]];
                int64_t s0 = off[a], t0 = off[a + 1];
                if (!empty) {
                    const int32_t li = lidx_off ? __ldg(lidx_off + a) : -1;
                    if (li >= 0) {  // label segment from the index, ID bounds searched inside it
                        const int lab = (int)((uint32_t)L.key_base >> __popc(L.idmask));
                        const int64_t b = s0;
                        s0 = b + __ldg(lidx + li + lab);
                        t0 = b + __ldg(lidx + li + lab + 1);
                        if (lov >= 0) s0 = lower_bound_cols(cols, s0, t0, klo);
                        if (hiv < n) t0 = lower_bound_cols(cols, s0, t0, khi);
                    } else {
                        s0 = lower_bound_cols(cols, s0, t0, klo);
                        t0 = lower_bound_cols(cols, s0, t0, khi);
                    }
                } else {
                    t0 = s0;
                }
                cbeg[r * nb + q] = s0;
                clen[r * nb + q] = (int32_t)(t0 - s0);
                if (t0 - s0 < blen) { blen = t0 - s0; bq = q; ps = s0; pt = t0; }
            }
        } else {
            // pivot = shortest estimated segment (up-split only, no search yet)
            int64_t blen = INT64_MAX;
            for (int q = 0; q < nb; ++q) {
                int64_t s0, t0;
                admissible_segment(off, cols, up, n, row[L.bpos[q]], lov, hiv, false, s0, t0);
                if (t0 - s0 < blen) { blen = t0 - s0; bq = q; }
            }
            // exact segments: the pivot's (its length is the work of this row; exact bounds
            // mean the expand kernel never re-checks the ID constraints) and the membership
            // lists of the other backward neighbours (searched per candidate)
            for (int q = 0; q < nb; ++q) {
                int64_t s0, t0;
                const bool pivot = q == bq;
                admissible_segment(off, cols, up, n, row[L.bpos[q]], lov, hiv, !empty, s0, t0);
                if (empty) t0 = s0;
                cbeg[r * nb + q] = s0;
                clen[r * nb + q] = (int32_t)(t0 - s0);
                if (pivot) { ps = s0; pt = t0; }
            }
        }
        rbeg[r] = ps;
        rlen[r] = pt - ps;
        rpiv[r] = (uint8_t)bq;
    }
}

// Lane-group variant: a group of G = 2^ceil(log2 |B(i)|) lanes per row, lane q of the
// group owns backward neighbour q — the |B(i)| independent segment searches of a row run in
// parallel instead of as one thread's dependent chain (more loads in flight; the searches
// are latency-bound), the pivot choice is a shuffle-min inside the group.
template <int G>
__global__ void __launch_bounds__(kThreads) k_plan_rows_grp(const Frontier F, int64_t R, LevelPlan L,
                                                            const int64_t* __restrict__ off,
                                                            const int32_t* __restrict__ cols,
                                                            const int32_t* __restrict__ up, int64_t n,
                                                            int64_t* __restrict__ rbeg, int64_t* __restrict__ rlen,
                                                            uint8_t* __restrict__ rpiv, int64_t* __restrict__ cbeg,
                                                            int32_t* __restrict__ clen) {
    const int nb = L.nb;
    const int q = threadIdx.x & (G - 1);
    const int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    const int64_t iters = (R + ngroups - 1) / ngroups;  // uniform trip count: shuffles stay converged
    int32_t buf[kMaxK];
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t r = gid + it * ngroups;
        const bool live = r < R && q < nb;
        int64_t lov = -1, hiv = n, s0 = 0, t0 = 0;
        int32_t a = 0;
        if (r < R) {
            const int32_t* row = frontier_row(F, r, buf);
            for (int x = 0; x < L.nlo; ++x) lov = max(lov, (int64_t)row[L.lo[x]]);
            for (int x = 0; x < L.nhi; ++x) hiv = min(hiv, (int64_t)row[L.hi[x]]);
            if (live) a = row[L.bpos[q]];
        }
        const bool empty = lov + 1 >= hiv;
        int64_t est = INT64_MAX;
        if (live) {
            if (L.keyed) {
                s0 = off[a];
                t0 = off[a + 1];
                if (!empty) {
                    const int64_t klo = (int64_t)L.key_base + lov + 1, khi = (int64_t)L.key_base + hiv;
                    s0 = lower_bound_cols(cols, s0, t0, klo);
                    t0 = lower_bound_cols(cols, s0, t0, khi);
                } else {
                    t0 = s0;
                }
                est = t0 - s0;
            } else {
                admissible_segment(off, cols, up, n, a, lov, hiv, false, s0, t0);
                est = t0 - s0;
            }
        }
        // pivot = shortest (estimated) segment, lowest q on ties
        int64_t best = est;
        int bq = q;
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
            const int64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
            if (ob < best || (ob == best && oq < bq)) { best = ob; bq = oq; }
        }
        if (live && !L.keyed) {  // exact segments (ID bounds folded in), as k_plan_rows
            admissible_segment(off, cols, up, n, a, lov, hiv, !empty, s0, t0);
            if (empty) t0 = s0;
        }
        if (live) {
            cbeg[r * nb + q] = s0;
            clen[r * nb + q] = (int32_t)(t0 - s0);
            if (q == bq) {
                rbeg[r] = s0;
                rlen[r] = t0 - s0;
                rpiv[r] = (uint8_t)bq;
            }
        }
    }
}

void launch_plan_rows(const DevGraph& g, const Frontier& F, int64_t R, const LevelPlan& L, int64_t* rbeg,
                      int64_t* rlen, uint8_t* rpiv, int64_t* cbeg, int32_t* clen, cudaStream_t s) {
    const int32_t* cols = L.keyed ? g.lkeys : g.cols;
    const int nb = L.nb;
    if (knobs().plan_groups && nb >= 2 && nb <= 8) {
        const int G = nb <= 2 ? 2 : (nb <= 4 ? 4 : 8);
        const int grid = grid_for(R * G, kThreads, 148 * 8);
        if (G == 2) k_plan_rows_grp<2><<<grid, kThreads, 0, s>>>(F, R, L, g.off, cols, g.up, g.n, rbeg, rlen, rpiv, cbeg, clen);
        else if (G == 4) k_plan_rows_grp<4><<<grid, kThreads, 0, s>>>(F, R, L, g.off, cols, g.up, g.n, rbeg, rlen, rpiv, cbeg, clen);
        else k_plan_rows_grp<8><<<grid, kThreads, 0, s>>>(F, R, L, g.off, cols, g.up, g.n, rbeg, rlen, rpiv, cbeg, clen);
        GSM_LAUNCH("k_plan_rows_grp");
        return;
    }
    k_plan_rows<<<grid_for(R), kThreads, 0, s>>>(F, R, L, g.off, cols, g.up, g.n, rbeg, rlen, rpiv, cbeg, clen,
                                                 L.keyed ? g.lidx_off : nullptr, g.lidx);
    GSM_LAUNCH("k_plan_rows");
}

size_t scan_temp_bytes(int64_t R) {
    size_t b = 0;
    cub::DeviceScan::InclusiveSum(nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr, R);
    return b;
}

void launch_scan(const int64_t* rlen, int64_t R, int64_t* P, void* tmp, size_t tmp_bytes, cudaStream_t s) {
    GSM_CUDA(cudaMemsetAsync(P, 0, sizeof(int64_t), s));
    GSM_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, rlen, P + 1, R, s));
}

// ============================================================================
// Merge-path partition (the load-balancing role of Gunrock's LB advance, which
// "maps the newly traversed edges to consecutive GPU threads"): the
// merge of row ends A[r] = P[r+1] with work items 0..S-1 is cut into equal
// diagonals, so every CTA gets TD (rows + items) regardless of degree skew.
// ============================================================================
__device__ __forceinline__ int64_t merge_path(const int64_t* __restrict__ A, int64_t R, int64_t S, int64_t d) {
    int64_t lo = max((int64_t)0, d - S), hi = min(d, R);
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (A[mid] <= d - mid - 1) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void k_partition(const int64_t* __restrict__ P, int64_t R, int64_t S, int64_t D0, int64_t D1, int64_t TD,
                            int64_t ntiles, int64_t* __restrict__ tile_ra) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = min(D0 + t * TD, D1);
        tile_ra[t] = merge_path(P + 1, R, S, d);
    }
}

void launch_partition(const int64_t* P, int64_t R, int64_t S, int64_t D0, int64_t D1, int64_t TD, int64_t ntiles,
                      int64_t* tile_ra, cudaStream_t s) {
    k_partition<<<grid_for(ntiles + 1), kThreads, 0, s>>>(P, R, S, D0, D1, TD, ntiles, tile_ra);
    GSM_LAUNCH("k_partition");
}

// ============================================================================
// Expand + verify + compact — Alg. 1 lines 11-13 fused in one kernel:
//   Advance: each work item is one entry of a row's pivot segment;
//   Compute: ID bounds, cmask bit of π[i], injectivity, and
//            membership v in N(f(j)) for every other backward neighbour j
//            (binary search in the sorted CSR list) — the tree and non-tree
//            connection checks;
//   Write_to_Partial: survivors are appended to a shared-memory
//            staging tile (warp ballot + popc ranks, one shared atomic per
//            warp), then ONE global atomicAdd per tile reserves the output
//            range and the tile is copied out coalesced.  At the last level in
//            COUNT mode nothing is written: survivors are only counted.
// One CTA per merge-path tile (grid-stride); the tile's rows (entries, pivot
// segment start, work offsets) are staged in shared memory first.
// ============================================================================
__device__ __forceinline__ bool in_segment(const int32_t* __restrict__ cols, int64_t lo, int64_t hi, int32_t v,
                                           unsigned& probes) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int32_t x = cols[mid];
        ++probes;
        if (x == v) return true;
        if (x < v) lo = mid + 1; else hi = mid;
    }
    return false;
}

int64_t expand_tile(int width) {
    const int td = knobs().expand_td;
    if (width <= 4) return td;
    if (width <= 12) return std::min(td, 256);
    return 128;
}

// shared-memory layout of one expand tile (TD merge steps => <= TD+1 rows, <= TD items)
struct ExpandSmem {
    size_t P, Beg, CB, Row, CL, RowOf, Piv, LA, Out, total;
    __host__ __device__ ExpandSmem(int64_t TD, int W, int nb, bool count_only, int nla = 0) {
        const size_t R1 = (size_t)TD + 1;
        P = 0;                     // int64 [R1+1]  work offsets of the tile's rows
        Beg = P + 8 * (R1 + 1);    // int64 [R1]    pivot segment start
        CB = Beg + 8 * R1;         // int64 [R1*nb] membership segment start
        Row = CB + 8 * R1 * nb;    // int32 [R1*W]  row entries
        CL = Row + 4 * R1 * W;     // int32 [R1*nb] membership segment length
        RowOf = CL + 4 * R1 * nb;  // int32 [TD]    item -> local row (scatter + max-scan)
        Piv = RowOf + 4 * (size_t)TD;  // uint8 [R1]
        LA = Piv + R1;                 // uint8 [R1*2*nla] look-ahead exclusions per row
        Out = (LA + R1 * 2 * nla + 15) & ~(size_t)15;
        total = Out + (count_only ? 0 : 4 * (size_t)TD * (W + 1));
    }
};

// membership of v in the sorted segment a[0, len): branch-free lower bound
// (fixed trip count, predicated steps) followed by one equality test
__device__ __forceinline__ bool in_sorted(const int32_t* __restrict__ a, int len, int32_t v, unsigned& probes) {
    if (len <= 0) return false;
    const int32_t* base = a;
    int n = len;
    while (n > 1) {
        const int half = n >> 1;
        base = (base[half - 1] < v) ? base + half : base;
        n -= half;
        ++probes;
    }
    ++probes;
    return *base == v;
}

// v ∈ N(f), where seg/len is the admissible segment of f's list and v lies in its key range
// (same label and ID interval): one hub-bitmap bit when both are hubs; otherwise, when f's
// segment is long and v's whole list is shorter, f's key searched in N(v) (the graph is
// symmetric); else v's key searched in the segment.
__device__ __forceinline__ bool member(const MemberCtx& m, const int32_t* __restrict__ cols,
                                       const int32_t* seg, int len, int32_t keyv, int32_t v, int32_t f,
                                       int32_t keyf, unsigned& probes) {
    if (len <= 0) return false;
    if (m.hub_bits && v >= m.hub_base && f >= m.hub_base) {
        const int lo = min(v, f) - m.hub_base, hi = max(v, f) - m.hub_base;
        ++probes;
        return (__ldg(hub_row(m.hub_bits, m.hub_words, lo) + (hi >> 5)) >> (hi & 31)) & 1u;
    }
    if (m.swap_min > 0 && len > m.swap_min && keyf >= 0) {
        const int64_t b = m.off[v], e = m.off[v + 1];
        probes += 2;
        if (e - b < len) return in_sorted(cols + b, (int)(e - b), keyf | f, probes);
    }
    return in_sorted(seg, len, keyv, probes);
}

struct MaxOp {
    __device__ __forceinline__ int operator()(int x, int y) const { return x > y ? x : y; }
};

template <typename MaskT, bool kCountOnly, int U>
__global__ void __launch_bounds__(kThreads) k_expand(ExpandArgs a, LevelPlan L) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t TD = a.TD;
    const int W = L.width;
    const int nb = L.nb;
    const ExpandSmem lay(TD, W, nb, kCountOnly, L.nla);
    int64_t* sP = reinterpret_cast<int64_t*>(smem + lay.P);
    int64_t* sBeg = reinterpret_cast<int64_t*>(smem + lay.Beg);
    int64_t* sCB = reinterpret_cast<int64_t*>(smem + lay.CB);
    int32_t* sRow = reinterpret_cast<int32_t*>(smem + lay.Row);
    int32_t* sCL = reinterpret_cast<int32_t*>(smem + lay.CL);
    int32_t* sRowOf = reinterpret_cast<int32_t*>(smem + lay.RowOf);
    uint8_t* sPiv = smem + lay.Piv;
    uint8_t* sLA = smem + lay.LA;
    int32_t* sOut = reinterpret_cast<int32_t*>(smem + lay.Out);
    using BlockScan = cub::BlockScan<int, kThreads>;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ int sCount;
    __shared__ unsigned long long sBase;
    __shared__ unsigned long long sRed[kWarps][5];  // survivors, items, mask, probes, lists

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const MaskT* __restrict__ cmask = static_cast<const MaskT*>(a.cmask);
    const int32_t* __restrict__ cols = a.cols;
    const int per_thread = (int)((TD + kThreads - 1) / kThreads);
    unsigned long long cnt = 0;
    unsigned st_items = 0, st_mask = 0, st_probes = 0, st_lists = 0;

    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const int64_t d0 = a.D0 + t * TD;
        const int64_t d1 = min(d0 + TD, a.D1);
        const int64_t ra0 = a.tile_ra[t], ra1 = a.tile_ra[t + 1];
        const int64_t ib0 = d0 - ra0, ib1 = d1 - ra1;
        if (ib1 <= ib0) continue;  // block-uniform
        const int nitems = (int)(ib1 - ib0);
        const int64_t rlast = min(ra1, a.R - 1);
        const int nrows = (int)(rlast - ra0 + 1);
        __syncthreads();  // previous tile finished with shared memory
        // ---- stage the tile's rows; mark where each non-empty row starts
        for (int i = threadIdx.x; i < nitems; i += kThreads) sRowOf[i] = 0;
        for (int lr = threadIdx.x; lr <= nrows; lr += kThreads) sP[lr] = a.P[ra0 + lr];
        for (int lr = threadIdx.x; lr < nrows; lr += kThreads) {
            sBeg[lr] = a.rbeg[ra0 + lr];
            sPiv[lr] = a.rpiv[ra0 + lr];
        }
        {
            if (a.F.rows) {
                const int32_t* src = a.F.rows + ra0 * W;
                const int nq = nrows * W;
                for (int q = threadIdx.x; q < nq; q += kThreads) sRow[q] = src[q];
            } else {  // compressed frontier: one thread per row walks its (parent, vertex) chain
                for (int lr = threadIdx.x; lr < nrows; lr += kThreads) {
                    int64_t r = ra0 + lr;
                    int32_t* dst = sRow + lr * W;
                    for (int w = W; w > a.F.bw; --w) {
                        const int2 e = a.F.pv[w][r];
                        dst[w - 1] = e.y;
                        r = e.x;
                    }
                    for (int c = 0; c < a.F.bw; ++c) dst[c] = a.F.base[r * a.F.bw + c];
                }
            }
            const int nc = nrows * nb;
            for (int q = threadIdx.x; q < nc; q += kThreads) {
                sCB[q] = a.cbeg[ra0 * nb + q];
                sCL[q] = a.clen[ra0 * nb + q];
            }
        }
        if (threadIdx.x == 0) sCount = 0;
        __syncthreads();
        if (L.nla) {
            // look-ahead exclusions of the row: mapped vertices known to be neighbours of the new
            // image v (the f(j), j in B(i)) that are themselves candidates of target u' (or ok1)
            const MaskT* __restrict__ ok1 = static_cast<const MaskT*>(a.la_ok1);
            for (int lr = threadIdx.x; lr < nrows; lr += kThreads) {
                const int32_t* row = sRow + lr * W;
                for (int t = 0; t < L.nla; ++t) {
                    int e1 = 0, e2 = 0;
                    for (int q = 0; q < nb; ++q) {
                        const int32_t f = row[L.bpos[q]] & L.idmask;
                        e1 += (cmask[f] >> L.la_u[t]) & 1u;
                        if (L.la_depth >= 2) e2 += (ok1[f] >> L.la_u[t]) & 1u;
                    }
                    sLA[(lr * L.nla + t) * 2] = (uint8_t)e1;
                    sLA[(lr * L.nla + t) * 2 + 1] = (uint8_t)e2;
                }
            }
        }
        for (int lr = threadIdx.x; lr < nrows; lr += kThreads) {
            const int64_t s = max(sP[lr], ib0), e = min(sP[lr + 1], ib1);
            if (e > s) sRowOf[s - ib0] = lr;  // rows with items in this tile start at distinct slots
        }
        __syncthreads();
        // ---- item -> row: inclusive max-scan (each thread owns a contiguous run of slots)
        {
            const int i0 = min(nitems, (int)threadIdx.x * per_thread), i1 = min(nitems, i0 + per_thread);
            int mx = 0;
            for (int i = i0; i < i1; ++i) mx = max(mx, sRowOf[i]);
            int prefix;
            BlockScan(scan_tmp).ExclusiveScan(mx, prefix, MaxOp());
            if (threadIdx.x == 0) prefix = 0;
            for (int i = i0; i < i1; ++i) {
                prefix = max(prefix, sRowOf[i]);
                sRowOf[i] = prefix;
            }
        }
        __syncthreads();

        // ---- candidates: each thread carries U items at once (items base + j*kThreads + tid,
        //      consecutive threads read consecutive list entries) and advances their
        //      membership searches in lockstep, so U independent loads are in flight per
        //      thread instead of one dependent chain
        for (int base = 0; base < nitems; base += kThreads * U) {
            int lr[U];
            int32_t v[U];
            bool ok[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int xi = base + j * kThreads + threadIdx.x;
                ok[j] = xi < nitems;
                lr[j] = 0;
                v[j] = 0;
                if (ok[j]) {
                    ++st_items;
                    lr[j] = sRowOf[xi];
                    v[j] = cols[sBeg[lr[j]] + ((ib0 + xi) - sP[lr[j]])] & L.idmask;
                }
            }
            // (ID bounds need no test: plan_rows cut every pivot segment to the exact open
            //  interval of admissible ids; only positions neither adjacent nor bounded need
            //  an explicit injectivity compare)
            if (L.ninj) {
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    if (!ok[j]) continue;
                    const int32_t* row = sRow + lr[j] * W;
                    for (int q = 0; q < L.ninj && ok[j]; ++q) ok[j] = v[j] != row[L.inj[q]];
                }
            }
            if (L.check_mask) {
                uint32_t m[U];
#pragma unroll
                for (int j = 0; j < U; ++j)
                    if (ok[j]) { ++st_mask; m[j] = cmask[v[j]]; }
#pragma unroll
                for (int j = 0; j < U; ++j)
                    if (ok[j]) ok[j] = (m[j] >> L.qv) & 1u;
            }
            for (int q = 0; q < nb; ++q) {
                const int32_t* pb[U];
                int pn[U];
                bool act[U];
                bool more = false;
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    act[j] = ok[j] && q != sPiv[lr[j]];
                    pn[j] = 0;
                    pb[j] = cols;
                    if (act[j]) {
                        ++st_lists;
                        const int e = lr[j] * nb + q;
                        pb[j] = cols + sCB[e];
                        pn[j] = sCL[e];
                        if (pn[j] <= 0) { ok[j] = false; act[j] = false; }
                        more |= pn[j] > 1;
                    }
                }
                while (more) {  // branch-free lower bounds, advanced together
                    more = false;
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        if (pn[j] > 1) {
                            const int half = pn[j] >> 1;
                            pb[j] = (pb[j][half - 1] < (L.key_base | v[j])) ? pb[j] + half : pb[j];
                            pn[j] -= half;
                            ++st_probes;
                            more |= pn[j] > 1;
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < U; ++j)
                    if (act[j]) { ++st_probes; ok[j] = (*pb[j] == (L.key_base | v[j])); }
            }
            if (L.nla) {  // k-look-ahead: every unmapped query neighbour u' of π[i] keeps a host
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    for (int t = 0; t < L.nla && ok[j]; ++t) {
                        const int64_t x = (int64_t)v[j] * a.la_k + L.la_u[t];
                        const uint8_t* ex = sLA + (lr[j] * L.nla + t) * 2;
                        ok[j] = a.la_c1[x] > ex[0];
                        if (ok[j] && L.la_depth >= 2) ok[j] = a.la_c2[x] > ex[1];
                    }
                }
            }
            if (L.shard_p > 1) {  // level-1 sharding: this rank's (f(π[0]), f(π[1])) pairs only
#pragma unroll
                for (int j = 0; j < U; ++j)
                    if (ok[j]) ok[j] = pair_shard(sRow[lr[j] * W] & L.idmask, v[j], L.shard_p) == L.shard_s;
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                if (kCountOnly) {
                    cnt += ok[j] ? 1u : 0u;
                } else {
                    const unsigned ball = __ballot_sync(0xffffffffu, ok[j]);
                    int wbase = 0;
                    if (lane == 0 && ball) wbase = atomicAdd(&sCount, __popc(ball));
                    wbase = __shfl_sync(0xffffffffu, wbase, 0);
                    if (ok[j]) {
                        const int pos = wbase + __popc(ball & ((1u << lane) - 1u));
                        GSM_DCHECK(pos < TD && lr[j] <= (int)TD, DCHK_STAGE);
                        if (a.out_pv) {  // compressed: (input row index, vertex)
                            int32_t* o = sOut + (int64_t)pos * 2;
                            o[0] = (int32_t)(ra0 + lr[j]);
                            o[1] = v[j];
                        } else {
                            int32_t* o = sOut + (int64_t)pos * (W + 1);
                            const int32_t* row = sRow + lr[j] * W;
                            for (int c = 0; c < W; ++c) o[c] = row[c];
                            o[W] = v[j];
                        }
                    }
                }
            }
        }
        if (!kCountOnly) {
            __syncthreads();
            const int total = sCount;
            if (threadIdx.x == 0) sBase = total ? atomicAdd(a.out_count, (unsigned long long)total) : 0ull;
            __syncthreads();
            cnt += (threadIdx.x == 0) ? (unsigned long long)total : 0ull;
            const int ow = a.out_pv ? 2 : W + 1;
            int32_t* dst = a.out_pv ? reinterpret_cast<int32_t*>(a.out_pv) + sBase * 2 : a.out + sBase * (W + 1);
            const int nq = total * ow;
            for (int q = threadIdx.x; q < nq; q += kThreads) dst[q] = sOut[q];
        }
    }
    // block reduction of the counters
    unsigned long long v5[5] = {cnt, st_items, st_mask, st_probes, st_lists};
#pragma unroll
    for (int c = 0; c < 5; ++c)
        for (int o = 16; o; o >>= 1) v5[c] += __shfl_xor_sync(0xffffffffu, v5[c], o);
    __syncthreads();
    if (lane == 0)
        for (int c = 0; c < 5; ++c) sRed[warp][c] = v5[c];
    __syncthreads();
    if (threadIdx.x < 5) {
        unsigned long long s = 0;
        for (int w = 0; w < kWarps; ++w) s += sRed[w][threadIdx.x];
        if (s) {
            if (threadIdx.x == 0) {
                if (kCountOnly) atomicAdd(a.out_count, s);
                atomicAdd(&a.stats[3], s);  // survivors
            } else if (threadIdx.x < 4) {
                atomicAdd(&a.stats[threadIdx.x - 1], s);  // items, mask_checked, probes
            } else {
                atomicAdd(&a.stats[4], s);  // membership lists searched
            }
        }
    }
}

// ============================================================================
// Last position in COUNT mode: "walking" variant of the expand kernel.
// Each thread owns VT consecutive merge-path steps of the tile, found by one
// shared-memory merge-path search, and walks them serially: the candidates it
// sees inside one row are consecutive entries of the sorted pivot segment, so
// every membership test gallops forward from the previous hit (exponential
// then binary search) instead of restarting a full binary search — O(log gap)
// per candidate, no per-candidate row lookup, two barriers per tile, and only
// the tile's row ends staged in shared memory.  Nothing is written.
// ============================================================================
constexpr int kWalkVT = 16;
constexpr int kWalkMaxNb = 4;

bool use_walk(const LevelPlan& L) {
    if (!knobs().count_walk) return false;
    return L.count_only && L.nb <= kWalkMaxNb;
}

int64_t expand_tile_for(const LevelPlan& L) {
    return use_walk(L) ? (int64_t)32 * kWalkVT : expand_tile(L.width);
}

// first index in [p, e) with a[idx] >= key, galloping from p
__device__ __forceinline__ int64_t gallop(const int32_t* __restrict__ a, int64_t p, int64_t e, int32_t key,
                                          unsigned& probes) {
    if (p >= e) return e;
    ++probes;
    if (a[p] >= key) return p;
    int64_t lo = p, step = 1;  // invariant: a[lo] < key
    while (lo + step < e) {
        ++probes;
        if (a[lo + step] >= key) break;
        lo += step;
        step <<= 1;
    }
    int64_t hi = min(lo + step, e);  // answer in (lo, hi]
    ++lo;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        ++probes;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_count_walk(ExpandArgs a, LevelPlan L) {
    // warp-private tiles (TD = 32 * kWalkVT merge steps): no block barriers, so a lane
    // with a long walk only delays its own warp
    extern __shared__ __align__(16) int64_t sAall[];
    const int64_t TD = a.TD;
    const int lane_id = threadIdx.x & 31;
    int64_t* sA = sAall + (threadIdx.x >> 5) * (TD + 1);  // row ends P[r+1] of the tile's rows
    const int nb = L.nb;
    const int W = L.width;
    const MaskT* __restrict__ cmask = static_cast<const MaskT*>(a.cmask);
    const int32_t* __restrict__ cols = a.cols;
    unsigned long long cnt = 0;
    unsigned st_items = 0, st_mask = 0, st_probes = 0, st_lists = 0;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = gw; t < a.ntiles; t += nw) {
        const int64_t d0 = a.D0 + t * TD;
        const int64_t d1 = min(d0 + TD, a.D1);
        const int64_t ra0 = a.tile_ra[t], ra1 = a.tile_ra[t + 1];
        if (d1 - ra1 <= d0 - ra0) continue;  // no candidates in this tile (warp-uniform)
        const int64_t rlast = min(ra1, a.R - 1);
        const int nrows = (int)(rlast - ra0 + 1);
        __syncwarp();
        for (int i = lane_id; i < nrows; i += 32) sA[i] = a.P[ra0 + i + 1];
        __syncwarp();
        const int64_t d = d0 + (int64_t)lane_id * kWalkVT;
        if (d >= d1) continue;
        // merge-path split for diagonal d inside [ra0, ra1]
        int64_t lo = ra0, hi = min(ra1, d);
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sA[mid - ra0] <= d - mid - 1) lo = mid + 1; else hi = mid;
        }
        int64_t r = lo, x = d - lo;
        const int64_t dend = min(d + kWalkVT, d1);
        int64_t cur = -1, beg = 0, base = 0;
        int piv = 0;
        int64_t cpos[kWalkMaxNb], cend[kWalkMaxNb];
        for (int64_t step = d; step < dend; ++step) {
            if (r > rlast) break;
            if (sA[r - ra0] <= x) {  // row r ends before item x: consume the row end
                ++r;
                continue;
            }
            if (r != cur) {  // entering row r: its pivot segment and membership segments
                cur = r;
                beg = a.rbeg[r];
                base = (r == ra0) ? a.P[r] : sA[r - 1 - ra0];
                piv = a.rpiv[r];
#pragma unroll
                for (int q = 0; q < kWalkMaxNb; ++q) {
                    if (q < nb) {
                        cpos[q] = a.cbeg[r * nb + q];
                        cend[q] = cpos[q] + a.clen[r * nb + q];
                    }
                }
            }
            ++st_items;
            const int32_t v = cols[beg + (x - base)] & L.idmask;
            ++x;
            bool ok = true;
            if (L.check_mask) {
                ++st_mask;
                ok = (cmask[v] >> L.qv) & 1u;
            }
            if (ok && L.ninj) {
                int32_t buf[kMaxK];
                const int32_t* row = frontier_row(a.F, r, buf);
                for (int q = 0; q < L.ninj && ok; ++q) ok = v != row[L.inj[q]];
            }
            const int32_t key = L.key_base | v;
#pragma unroll
            for (int q = 0; q < kWalkMaxNb; ++q) {
                if (q < nb && q != piv && ok) {
                    ++st_lists;
                    cpos[q] = gallop(cols, cpos[q], cend[q], key, st_probes);
                    ok = cpos[q] < cend[q] && cols[cpos[q]] == key;
                }
            }
            cnt += ok;
        }
    }
    // block reduction of the counters (same layout as k_expand)
    __shared__ unsigned long long sRed[kWarps][5];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long v5[5] = {cnt, st_items, st_mask, st_probes, st_lists};
#pragma unroll
    for (int c = 0; c < 5; ++c)
        for (int o = 16; o; o >>= 1) v5[c] += __shfl_xor_sync(0xffffffffu, v5[c], o);
    __syncthreads();
    if (lane == 0)
        for (int c = 0; c < 5; ++c) sRed[warp][c] = v5[c];
    __syncthreads();
    if (threadIdx.x < 5) {
        unsigned long long sum = 0;
        for (int w = 0; w < kWarps; ++w) sum += sRed[w][threadIdx.x];
        if (sum) {
            if (threadIdx.x == 0) {
                atomicAdd(a.out_count, sum);
                atomicAdd(&a.stats[3], sum);
            } else if (threadIdx.x < 4) {
                atomicAdd(&a.stats[threadIdx.x - 1], sum);
            } else {
                atomicAdd(&a.stats[4], sum);
            }
        }
    }
}

template <typename MaskT>
static void launch_walk_t(const ExpandArgs& a, const LevelPlan& L, cudaStream_t s) {
    const size_t smem = sizeof(int64_t) * (size_t)(a.TD + 1) * kWarps;
    GSM_CUDA(cudaFuncSetAttribute(k_count_walk<MaskT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    int dev = 0, sms = 148, per_sm = 1;
    GSM_CUDA(cudaGetDevice(&dev));
    GSM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GSM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_count_walk<MaskT>, kThreads, smem));
    const int64_t grid =
        std::max<int64_t>(1, std::min<int64_t>((a.ntiles + kWarps - 1) / kWarps, (int64_t)sms * std::max(per_sm, 1)));
    k_count_walk<MaskT><<<(unsigned)grid, kThreads, smem, s>>>(a, L);
    GSM_LAUNCH("k_count_walk");
}

// items carried per thread (memory-level parallelism of the membership searches);
// measured: 1 beats 2/4 (issue-bound, not latency-bound)
static int expand_ilp() { return knobs().expand_ilp; }

template <typename MaskT, bool kCountOnly, int U>
static void launch_expand_u(const ExpandArgs& a, const LevelPlan& L, cudaStream_t s) {
    const size_t smem = ExpandSmem(a.TD, L.width, L.nb, kCountOnly, L.nla).total;
    // per launch: the attribute is per device, and a process may drive several devices
    GSM_CUDA(cudaFuncSetAttribute(k_expand<MaskT, kCountOnly, U>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    int dev = 0, sms = 148, per_sm = 1;
    GSM_CUDA(cudaGetDevice(&dev));
    GSM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GSM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_expand<MaskT, kCountOnly, U>, kThreads, smem));
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(a.ntiles, (int64_t)sms * std::max(per_sm, 1)));
    k_expand<MaskT, kCountOnly, U><<<(unsigned)grid, kThreads, smem, s>>>(a, L);
    GSM_LAUNCH("k_expand");
}

template <typename MaskT, bool kCountOnly>
static void launch_expand_t(const ExpandArgs& a, const LevelPlan& L, cudaStream_t s) {
    switch (expand_ilp()) {
        case 1: launch_expand_u<MaskT, kCountOnly, 1>(a, L, s); break;
        case 2: launch_expand_u<MaskT, kCountOnly, 2>(a, L, s); break;
        case 4: launch_expand_u<MaskT, kCountOnly, 4>(a, L, s); break;
        default: launch_expand_u<MaskT, kCountOnly, 1>(a, L, s); break;
    }
}

void launch_expand(const ExpandArgs& a, const LevelPlan& L, int mask_bytes, cudaStream_t s) {
    if (use_walk(L) && a.TD == (int64_t)32 * kWalkVT) {
        switch (mask_bytes) {
            case 1: launch_walk_t<uint8_t>(a, L, s); break;
            case 2: launch_walk_t<uint16_t>(a, L, s); break;
            default: launch_walk_t<uint32_t>(a, L, s); break;
        }
        return;
    }
    const bool c = L.count_only != 0;
    switch (mask_bytes) {
        case 1: c ? launch_expand_t<uint8_t, true>(a, L, s) : launch_expand_t<uint8_t, false>(a, L, s); break;
        case 2: c ? launch_expand_t<uint16_t, true>(a, L, s) : launch_expand_t<uint16_t, false>(a, L, s); break;
        default: c ? launch_expand_t<uint32_t, true>(a, L, s) : launch_expand_t<uint32_t, false>(a, L, s); break;
    }
}

// ============================================================================
// Fused tail (COUNT mode, last two positions k-2 and k-1) — candidate-set
// inheritance.  When π[k-1] is adjacent to π[k-2] and to every backward
// neighbour of π[k-2] (B(k-1) = B(k-2) ∪ {k-2}, e.g. cliques), with the same
// label and no looser ID bounds, the raw candidate set of position k-2,
//   RC(r) = ∩_{j in B(k-2)} N(f(j))  within the ID interval of position k-2,
// also contains every admissible image of π[k-1]; so one warp per partial
// result r builds RC(r) once in shared memory (Advance + Compute of position
// k-2) and counts, for every c in RC(r) that passes position k-2's
// own tests, the d in RC(r) with d ∈ N(c) (position k-1's one remaining
// connection check) — the level-(k-1) frontier is never written to HBM.
// Per c the cheaper side is enumerated: RC's entries searched in N(c) (global
// binary search), or N(c)'s admissible part searched in RC (shared memory).
// Rows whose pivot segment exceeds the per-warp buffer are handed back (overflow
// list) to the generic BFS path.
// ============================================================================
// per-warp shared memory of k_tail: RC[cap] + 64 x (int64 segment start, int32 length)
__host__ __device__ inline int tail_warp_ints(int cap) { return ((cap + 1) & ~1) + 64 * 3; }

template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_tail(TailArgs a, LevelPlan Lc, LevelPlan Ld) {
    extern __shared__ __align__(16) int32_t tail_smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    int32_t* rc = tail_smem + wib * tail_warp_ints(a.cap);  // cap is even: the int64 part stays aligned
    const MaskT* __restrict__ cmask = static_cast<const MaskT*>(a.cmask);
    const int32_t* __restrict__ cols = a.cols;
    const int W = Lc.width;
    const int nb = Lc.nb;
    const int32_t kb = Lc.key_base, idm = Lc.idmask;
    unsigned long long cnt = 0, items = 0, probes_u = 0;
    unsigned probes = 0;
    // dynamic row scheduling: row costs vary by orders of magnitude (|RC|^2), so warps
    // grab chunks of rows from a global counter instead of a static stride
    constexpr int64_t kChunk = 8;
    int64_t cbase = 0, cend = 0;
    unsigned long long cyc_p1 = 0, cyc_small = 0, cyc_big = 0, rows_small = 0, rows_big = 0;
    long long t_row = 0, t_p1 = 0;
    for (;;) {
        if (cbase >= cend) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(a.next, (unsigned long long)kChunk);
            b = __shfl_sync(0xffffffffu, b, 0);
            if ((int64_t)b >= a.R) break;
            cbase = (int64_t)b;
            cend = min(cbase + kChunk, a.R);
        }
        const int64_t r = cbase++;
        const int64_t len = a.rlen[r];
        if (len == 0) continue;
        if (len > a.cap) {
            if (lane == 0) a.overflow[atomicAdd(a.noverflow, 1ull)] = r;
            continue;
        }
        int32_t rowbuf[kMaxK];
        const int32_t* row = frontier_row(a.F, r, rowbuf);
        const int piv = a.rpiv[r];
        const int64_t beg = a.rbeg[r];
        if (a.cyc) t_row = clock64();
        // ---- phase 1: RC(r) = pivot entries present in every other backward list (order kept)
        int n = 0;
        for (int64_t base = 0; base < len; base += 32) {
            const int64_t i = base + lane;
            bool ok = i < len;
            int32_t v = ok ? (cols[beg + i] & idm) : 0;
            if (ok) ++items;
            for (int q = 0; q < nb && ok; ++q) {
                if (q == piv) continue;
                ok = in_sorted(cols + a.cbeg[r * nb + q], a.clen[r * nb + q], kb | v, probes);
            }
            const unsigned ball = __ballot_sync(0xffffffffu, ok);
            if (ok) rc[n + __popc(ball & ((1u << lane) - 1u))] = v;
            n += __popc(ball);
        }
        __syncwarp();
        if (a.cyc) {
            t_p1 = clock64();
            cyc_p1 += (unsigned long long)(t_p1 - t_row);
        }
        // ---- phase 2a: small RC with d ≻ c: the n(n-1)/2 pairs (c, d) = (RC[i], RC[j]), i < j,
        //      spread over the lanes (one independent search of d in N+(c) per lane)
        if (a.rel > 0 && !Lc.keyed && n <= 64) {
            // per-c data once per row (not once per pair): N+(c) segment, or -1 if c fails
            int64_t* cseg = reinterpret_cast<int64_t*>(rc + a.cap);
            int32_t* clen = reinterpret_cast<int32_t*>(cseg + 64);
            for (int i = lane; i < n; i += 32) {
                const int32_t c = rc[i];
                bool ok = true;
                if (Lc.check_mask) ok = (cmask[c] >> Lc.qv) & 1u;
                for (int q = 0; q < Lc.ninj && ok; ++q) ok = c != row[Lc.inj[q]];
                const int64_t s0 = a.off[c] + a.up[c];
                cseg[i] = s0;
                clen[i] = ok ? (int32_t)(a.off[c + 1] - s0) : -1;
            }
            __syncwarp();
            const int np = n * (n - 1) / 2;
            for (int pidx = lane; pidx < np; pidx += 32) {
                const float fn = 2.0f * n - 1.0f;
                int i = (int)((fn - sqrtf(fn * fn - 8.0f * pidx)) * 0.5f);
                i = max(0, min(i, n - 2));
                while (i > 0 && i * (2 * n - i - 1) / 2 > pidx) --i;
                while ((i + 1) * (2 * n - i - 2) / 2 <= pidx) ++i;
                const int j = pidx - i * (2 * n - i - 1) / 2 + i + 1;
                const int len = clen[i];
                if (len <= 0) continue;
                const int32_t d = rc[j];
                ++items;
                bool ok = true;
                if (Ld.check_mask) ok = (cmask[d] >> Ld.qv) & 1u;
                for (int q = 0; q < a.nxlo && ok; ++q) ok = d > row[a.xlo[q]];
                for (int q = 0; q < a.nxhi && ok; ++q) ok = d < row[a.xhi[q]];
                for (int q = 0; q < Ld.ninj && ok; ++q) ok = d != row[Ld.inj[q]];
                if (ok) ok = in_sorted(cols + cseg[i], len, d, probes);
                cnt += ok;
            }
            __syncwarp();
            if (a.cyc) {
                cyc_small += (unsigned long long)(clock64() - t_p1);
                ++rows_small;
            }
            continue;
        }
        // ---- phase 2b: pairs (c, d) inside RC(r), one c at a time across the warp.  The per-c
        //      data (filters, admissible part of N(c)) is fetched 32 c's at a time — lane l for
        //      c = RC[g + l] — and broadcast by shuffles, so the warp never waits on a
        //      serialized chain of per-c global loads.
        for (int g0 = 0; g0 < n; g0 += 32) {
            const int il = g0 + lane;
            bool okl = false;
            int64_t sl = 0, tl = 0;
            if (il < n) {
                const int32_t cl = rc[il];
                okl = true;
                if (Lc.check_mask) okl = (cmask[cl] >> Lc.qv) & 1u;
                for (int q = 0; q < Lc.ninj && okl; ++q) okl = cl != row[Lc.inj[q]];
                int j0 = 0, j1 = n;
                if (a.rel > 0) j0 = il + 1;
                else if (a.rel < 0) j1 = il;
                if (j1 <= j0) okl = false;
                if (okl) {
                    const int64_t cs = a.off[cl], ce = a.off[cl + 1];
                    if (!Lc.keyed && a.rel != 0) {  // d ≻ c (or ≺ c): exactly N+(c) (or N-(c)) via up[c]
                        const int64_t split = cs + a.up[cl];
                        sl = a.rel > 0 ? split : cs;
                        tl = a.rel > 0 ? ce : split;
                    } else {
                        sl = lower_bound_cols(cols, cs, ce, (int64_t)(kb | rc[j0]));
                        tl = lower_bound_cols(cols, sl, ce, (int64_t)(kb | rc[j1 - 1]) + 1);
                    }
                    if (tl <= sl) okl = false;
                }
            }
            const unsigned live = __ballot_sync(0xffffffffu, okl);
            for (int ii = 0; ii < 32; ++ii) {
                if (!((live >> ii) & 1u)) continue;  // warp-uniform
                const int i = g0 + ii;
                const int32_t c = rc[i];
                const int64_t s0 = __shfl_sync(0xffffffffu, sl, ii);
                const int64_t t0 = __shfl_sync(0xffffffffu, tl, ii);
                int j0 = 0, j1 = n;
                if (a.rel > 0) j0 = i + 1;
                else if (a.rel < 0) j1 = i;
                const int64_t nA = j1 - j0, nB = t0 - s0;
                // A (search RC's entries in N(c): global binary searches, mostly L1/L2 hits) vs
                // B (stream N(c), search each entry in RC in shared memory, stop past max RC):
                // enumerate the shorter side (measured: biasing towards B is slower)
                if (nB * 100 > (int64_t)a.bratio * nA) {
                    for (int j = j0 + lane; j < j1; j += 32) {
                        if (j == i) continue;
                        const int32_t d = rc[j];
                        ++items;
                        bool ok = true;
                        if (Ld.check_mask) ok = (cmask[d] >> Ld.qv) & 1u;
                        for (int q = 0; q < a.nxlo && ok; ++q) ok = d > row[a.xlo[q]];
                        for (int q = 0; q < a.nxhi && ok; ++q) ok = d < row[a.xhi[q]];
                        for (int q = 0; q < Ld.ninj && ok; ++q) ok = d != row[Ld.inj[q]];
                        if (ok) ok = in_sorted(cols + s0, (int)nB, kb | d, probes);
                        cnt += ok;
                    }
                } else {
                    const int32_t dmax = rc[j1 - 1];
                    for (int64_t x0 = s0; x0 < t0; x0 += 32) {
                        const int64_t x = x0 + lane;
                        const int32_t d = x < t0 ? (cols[x] & idm) : INT32_MAX;
                        if (!__any_sync(0xffffffffu, d <= dmax)) break;  // N(c) is sorted: past max RC
                        if (d > dmax) continue;
                        ++items;
                        unsigned dummy = 0;
                        bool ok = d != c && in_sorted(rc + j0, j1 - j0, d, dummy);
                        if (ok && Ld.check_mask) ok = (cmask[d] >> Ld.qv) & 1u;
                        for (int q = 0; q < a.nxlo && ok; ++q) ok = d > row[a.xlo[q]];
                        for (int q = 0; q < a.nxhi && ok; ++q) ok = d < row[a.xhi[q]];
                        for (int q = 0; q < Ld.ninj && ok; ++q) ok = d != row[Ld.inj[q]];
                        cnt += ok;
                    }
                }
            }
        }
        __syncwarp();
        if (a.cyc) {
            cyc_big += (unsigned long long)(clock64() - t_p1);
            ++rows_big;
        }
    }
    if (a.cyc && lane == 0) {
        atomicAdd(&a.cyc[0], cyc_p1);
        atomicAdd(&a.cyc[1], cyc_small);
        atomicAdd(&a.cyc[2], cyc_big);
        atomicAdd(&a.cyc[3], rows_small);
        atomicAdd(&a.cyc[4], rows_big);
    }
    probes_u = probes;
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        items += __shfl_xor_sync(0xffffffffu, items, o);
        probes_u += __shfl_xor_sync(0xffffffffu, probes_u, o);
    }
    if (lane == 0) {
        if (cnt) {
            atomicAdd(a.count, cnt);
            atomicAdd(&a.stats[3], cnt);
        }
        if (items) atomicAdd(&a.stats[0], items);
        if (probes_u) atomicAdd(&a.stats[2], probes_u);
    }
}

// Big rows of the fused tail: one CTA per row, RC(r) (up to a.cap entries) built
// block-wide in shared memory (order-preserving ballot compaction with a warp
// scan per 256-candidate round), then the 8 warps split the c's of RC(r).
constexpr int kTBThreads = 1024;  // 32 warps: the 160 KB RC buffer allows one CTA per SM
constexpr int kTBWarps = kTBThreads / 32;

template <typename MaskT>
__global__ void __launch_bounds__(kTBThreads) k_tail_block(TailArgs a, LevelPlan Lc, LevelPlan Ld) {
    extern __shared__ __align__(16) int32_t rcb[];
    __shared__ int sWarpCnt[kTBWarps];
    __shared__ int sN;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const MaskT* __restrict__ cmask = static_cast<const MaskT*>(a.cmask);
    const int32_t* __restrict__ cols = a.cols;
    const int W = Lc.width;
    const int nb = Lc.nb;
    const int32_t kb = Lc.key_base, idm = Lc.idmask;
    unsigned long long cnt = 0, items = 0;
    unsigned probes = 0;
    __shared__ unsigned long long sNext;
    for (;;) {  // dynamic: one row at a time from a global counter (rows sorted largest first)
        __syncthreads();
        if (threadIdx.x == 0) sNext = atomicAdd(a.next, 1ull);
        __syncthreads();
        const int64_t ri = (int64_t)sNext;
        if (ri >= a.R) break;
        const int64_t r = a.rows_idx ? a.rows_idx[ri] : ri;
        const int64_t len = a.rlen[r];
        if (len == 0) continue;  // block-uniform
        if (len > a.cap) {
            if (threadIdx.x == 0) a.overflow[atomicAdd(a.noverflow, 1ull)] = r;
            continue;
        }
        int32_t rowbuf[kMaxK];
        const int32_t* row = frontier_row(a.F, r, rowbuf);
        const int piv = a.rpiv[r];
        const int64_t beg = a.rbeg[r];
        __syncthreads();
        if (threadIdx.x == 0) sN = 0;
        __syncthreads();
        for (int64_t base = 0; base < len; base += kTBThreads) {
            const int64_t i = base + threadIdx.x;
            bool ok = i < len;
            const int32_t v = ok ? (cols[beg + i] & idm) : 0;
            if (ok) ++items;
            for (int q = 0; q < nb && ok; ++q) {
                if (q == piv) continue;
                ok = in_sorted(cols + a.cbeg[r * nb + q], a.clen[r * nb + q], kb | v, probes);
            }
            const unsigned ball = __ballot_sync(0xffffffffu, ok);
            if (lane == 0) sWarpCnt[warp] = __popc(ball);
            __syncthreads();
            int off = sN;
            for (int w = 0; w < warp; ++w) off += sWarpCnt[w];
            if (ok) rcb[off + __popc(ball & ((1u << lane) - 1u))] = v;
            __syncthreads();
            if (threadIdx.x == 0) {
                int tot = 0;
                for (int w = 0; w < kTBWarps; ++w) tot += sWarpCnt[w];
                sN += tot;
            }
            __syncthreads();
        }
        const int n = sN;
        // this warp's c's: i = warp, warp + 32, ...; per-c data fetched 32 c's at a time (lane l
        // for the warp's (g + l)-th c) and broadcast by shuffles
        for (int g0 = 0; warp + kTBWarps * g0 < n; g0 += 32) {
            const int il = warp + kTBWarps * (g0 + lane);
            bool okl = false;
            int64_t sl = 0, tl = 0;
            if (il < n) {
                const int32_t cl = rcb[il];
                okl = true;
                if (Lc.check_mask) okl = (cmask[cl] >> Lc.qv) & 1u;
                for (int q = 0; q < Lc.ninj && okl; ++q) okl = cl != row[Lc.inj[q]];
                int j0 = 0, j1 = n;
                if (a.rel > 0) j0 = il + 1;
                else if (a.rel < 0) j1 = il;
                if (j1 <= j0) okl = false;
                if (okl) {
                    const int64_t cs = a.off[cl], ce = a.off[cl + 1];
                    if (!Lc.keyed && a.rel != 0) {
                        const int64_t split = cs + a.up[cl];
                        sl = a.rel > 0 ? split : cs;
                        tl = a.rel > 0 ? ce : split;
                    } else {
                        sl = lower_bound_cols(cols, cs, ce, (int64_t)(kb | rcb[j0]));
                        tl = lower_bound_cols(cols, sl, ce, (int64_t)(kb | rcb[j1 - 1]) + 1);
                    }
                    if (tl <= sl) okl = false;
                }
            }
            const unsigned live = __ballot_sync(0xffffffffu, okl);
            for (int ii = 0; ii < 32; ++ii) {
                if (!((live >> ii) & 1u)) continue;  // warp-uniform
                const int i = warp + kTBWarps * (g0 + ii);
                const int32_t c = rcb[i];
                const int64_t s0 = __shfl_sync(0xffffffffu, sl, ii);
                const int64_t t0 = __shfl_sync(0xffffffffu, tl, ii);
                int j0 = 0, j1 = n;
                if (a.rel > 0) j0 = i + 1;
                else if (a.rel < 0) j1 = i;
                const int64_t nA = j1 - j0, nB = t0 - s0;
                // A (search RC's entries in N(c): global binary searches, mostly L1/L2 hits) vs
                // B (stream N(c), search each entry in RC in shared memory, stop past max RC):
                // enumerate the shorter side (measured: biasing towards B is slower)
                if (nB * 100 > (int64_t)a.bratio * nA) {
                    for (int j = j0 + lane; j < j1; j += 32) {
                        if (j == i) continue;
                        const int32_t d = rcb[j];
                        ++items;
                        bool ok = true;
                        if (Ld.check_mask) ok = (cmask[d] >> Ld.qv) & 1u;
                        for (int q = 0; q < a.nxlo && ok; ++q) ok = d > row[a.xlo[q]];
                        for (int q = 0; q < a.nxhi && ok; ++q) ok = d < row[a.xhi[q]];
                        for (int q = 0; q < Ld.ninj && ok; ++q) ok = d != row[Ld.inj[q]];
                        if (ok) ok = in_sorted(cols + s0, (int)nB, kb | d, probes);
                        cnt += ok;
                    }
                } else {
                    const int32_t dmax = rcb[j1 - 1];
                    for (int64_t x0 = s0; x0 < t0; x0 += 32) {
                        const int64_t x = x0 + lane;
                        const int32_t d = x < t0 ? (cols[x] & idm) : INT32_MAX;
                        if (!__any_sync(0xffffffffu, d <= dmax)) break;  // N(c) is sorted: past max RC
                        if (d > dmax) continue;
                        ++items;
                        unsigned dummy = 0;
                        bool ok = d != c && in_sorted(rcb + j0, j1 - j0, d, dummy);
                        if (ok && Ld.check_mask) ok = (cmask[d] >> Ld.qv) & 1u;
                        for (int q = 0; q < a.nxlo && ok; ++q) ok = d > row[a.xlo[q]];
                        for (int q = 0; q < a.nxhi && ok; ++q) ok = d < row[a.xhi[q]];
                        for (int q = 0; q < Ld.ninj && ok; ++q) ok = d != row[Ld.inj[q]];
                        cnt += ok;
                    }
                }
            }
        }
    }
    unsigned long long probes_u = probes;
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        items += __shfl_xor_sync(0xffffffffu, items, o);
        probes_u += __shfl_xor_sync(0xffffffffu, probes_u, o);
    }
    if (lane == 0) {
        if (cnt) {
            atomicAdd(a.count, cnt);
            atomicAdd(&a.stats[3], cnt);
        }
        if (items) atomicAdd(&a.stats[0], items);
        if (probes_u) atomicAdd(&a.stats[2], probes_u);
    }
}

template <typename MaskT>
static void launch_tail_block_t(const TailArgs& a, const LevelPlan& Lc, const LevelPlan& Ld, cudaStream_t s) {
    const size_t smem = sizeof(int32_t) * (size_t)a.cap;
    GSM_CUDA(cudaFuncSetAttribute(k_tail_block<MaskT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    int dev = 0, sms = 148, per_sm = 1;
    GSM_CUDA(cudaGetDevice(&dev));
    GSM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GSM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail_block<MaskT>, kTBThreads, smem));
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(a.R, (int64_t)sms * std::max(per_sm, 1)));
    k_tail_block<MaskT><<<(unsigned)grid, kTBThreads, smem, s>>>(a, Lc, Ld);
    GSM_LAUNCH("k_tail_block");
}

void launch_tail_block(const TailArgs& a, const LevelPlan& Lc, const LevelPlan& Ld, int mask_bytes, cudaStream_t s) {
    switch (mask_bytes) {
        case 1: launch_tail_block_t<uint8_t>(a, Lc, Ld, s); break;
        case 2: launch_tail_block_t<uint16_t>(a, Lc, Ld, s); break;
        default: launch_tail_block_t<uint32_t>(a, Lc, Ld, s); break;
    }
}

int tail_block_cap() { return knobs().tail_block_cap; }  // per-CTA buffer for big rows

// ============================================================================
// Pair tail (COUNT mode): the last two positions p, q are not adjacent in Q and carry
// no ID condition between them, so given a row r of the first k-2 positions their
// candidate sets (Alg. 1 line 12: label, degree, connections with the
// mapped positions, injectivity) are independent and
//     #{(x, y) : x ∈ Cp(r), y ∈ Cq(r), x != y} = |Cp| |Cq| - |Cp ∩ Cq|.
// One warp per row: lanes stride the pivot segment of p (and then of q), each candidate
// is verified against the other backward lists by binary search; |Cp ∩ Cq| re-checks
// the survivors of p against q's constraints (skipped when the labels differ).
// ============================================================================
template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_pair(PairArgs a, LevelPlan Lp, LevelPlan Lq) {
    const int lane = threadIdx.x & 31;
    const MaskT* __restrict__ cmask = static_cast<const MaskT*>(a.cmask);
    const int W = Lp.width;
    unsigned long long total = 0, items = 0;
    unsigned probes = 0;
    constexpr int64_t kChunk = 4;
    int64_t cbase = 0, cend = 0;
    for (;;) {
        if (cbase >= cend) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(a.next, (unsigned long long)kChunk);
            b = __shfl_sync(0xffffffffu, b, 0);
            if ((int64_t)b >= a.R) break;
            cbase = (int64_t)b;
            cend = min(cbase + kChunk, a.R);
        }
        const int64_t ri = cbase++;
        const int64_t r = a.rows_idx ? a.rows_idx[ri] : ri;
        int32_t rowbuf[kMaxK];
        const int32_t* row = frontier_row(a.F, r, rowbuf);
        unsigned long long cp = 0, cq = 0, cb = 0;
        {   // candidates of p
            const int64_t len = a.plen[r], beg = a.pbeg[r];
            const int piv = a.ppiv[r];
            for (int64_t x = lane; x < len; x += 32) {
                const int32_t v = a.colsp[beg + x] & Lp.idmask;
                ++items;
                bool ok = true;
                if (Lp.check_mask) ok = (cmask[v] >> Lp.qv) & 1u;
                for (int t = 0; t < Lp.ninj && ok; ++t) ok = v != row[Lp.inj[t]];
                for (int t = 0; t < Lp.nb && ok; ++t)
                    if (t != piv)
                        ok = member(a.mem, a.colsp, a.colsp + a.pcbeg[r * Lp.nb + t], a.pclen[r * Lp.nb + t],
                                    Lp.key_base | v, v, row[Lp.bpos[t]], Lp.bkey[t], probes);
                cp += ok;
                if (ok && a.need_both) {  // also a candidate of q?
                    bool o2 = true;
                    if (Lq.check_mask) o2 = (cmask[v] >> Lq.qv) & 1u;
                    for (int t = 0; t < Lq.ninj && o2; ++t) o2 = v != row[Lq.inj[t]];
                    for (int t = 0; t < Lq.nb && o2; ++t)
                        o2 = in_sorted(a.colsq + a.qcbeg[r * Lq.nb + t], a.qclen[r * Lq.nb + t], Lq.key_base | v, probes);
                    cb += o2;
                }
            }
        }
        {   // candidates of q
            const int64_t len = a.qlen[r], beg = a.qbeg[r];
            const int piv = a.qpiv[r];
            for (int64_t x = lane; x < len; x += 32) {
                const int32_t v = a.colsq[beg + x] & Lq.idmask;
                ++items;
                bool ok = true;
                if (Lq.check_mask) ok = (cmask[v] >> Lq.qv) & 1u;
                for (int t = 0; t < Lq.ninj && ok; ++t) ok = v != row[Lq.inj[t]];
                for (int t = 0; t < Lq.nb && ok; ++t)
                    if (t != piv)
                        ok = member(a.mem, a.colsq, a.colsq + a.qcbeg[r * Lq.nb + t], a.qclen[r * Lq.nb + t],
                                    Lq.key_base | v, v, row[Lq.bpos[t]], Lq.bkey[t], probes);
                cq += ok;
            }
        }
        for (int o = 16; o; o >>= 1) {
            cp += __shfl_xor_sync(0xffffffffu, cp, o);
            cq += __shfl_xor_sync(0xffffffffu, cq, o);
            cb += __shfl_xor_sync(0xffffffffu, cb, o);
        }
        total += cp * cq - cb;  // identical on every lane
    }
    unsigned long long pr = probes;
    for (int o = 16; o; o >>= 1) {
        items += __shfl_xor_sync(0xffffffffu, items, o);
        pr += __shfl_xor_sync(0xffffffffu, pr, o);
    }
    if (lane == 0) {
        if (total) {
            atomicAdd(a.count, total);
            atomicAdd(&a.stats[3], total);
        }
        if (items) atomicAdd(&a.stats[0], items);
        if (pr) atomicAdd(&a.stats[2], pr);
    }
}

// one thread per row (short segments); rows above a.thread_max candidates go to the warp pass
template <typename MaskT>
__global__ void __launch_bounds__(kThreads) k_pair_thread(PairArgs a, LevelPlan Lp, LevelPlan Lq) {
    const MaskT* __restrict__ cmask = static_cast<const MaskT*>(a.cmask);
    const int W = Lp.width;
    unsigned long long total = 0, items = 0;
    unsigned probes = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.R; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t plen = a.plen[r], qlen = a.qlen[r];
        if (plen == 0 || qlen == 0) continue;  // no candidate for p or q: nothing to count
        if (plen + qlen > a.thread_max) {
            a.overflow[atomicAdd(a.noverflow, 1ull)] = r;
            continue;
        }
        int32_t rowbuf[kMaxK];
        const int32_t* row = frontier_row(a.F, r, rowbuf);
        unsigned long long cp = 0, cq = 0, cb = 0;
        const int64_t pb = a.pbeg[r], qb = a.qbeg[r];
        const int ppv = a.ppiv[r], qpv = a.qpiv[r];
        for (int64_t x = 0; x < plen; ++x) {
            const int32_t v = a.colsp[pb + x] & Lp.idmask;
            bool ok = true;
            if (Lp.check_mask) ok = (cmask[v] >> Lp.qv) & 1u;
            for (int t = 0; t < Lp.ninj && ok; ++t) ok = v != row[Lp.inj[t]];
            for (int t = 0; t < Lp.nb && ok; ++t)
                if (t != ppv)
                    ok = member(a.mem, a.colsp, a.colsp + a.pcbeg[r * Lp.nb + t], a.pclen[r * Lp.nb + t],
                                Lp.key_base | v, v, row[Lp.bpos[t]], Lp.bkey[t], probes);
            cp += ok;
            if (ok && a.need_both) {
                bool o2 = true;
                if (Lq.check_mask) o2 = (cmask[v] >> Lq.qv) & 1u;
                for (int t = 0; t < Lq.ninj && o2; ++t) o2 = v != row[Lq.inj[t]];
                for (int t = 0; t < Lq.nb && o2; ++t)
                    o2 = in_sorted(a.colsq + a.qcbeg[r * Lq.nb + t], a.qclen[r * Lq.nb + t], Lq.key_base | v, probes);
                cb += o2;
            }
        }
        if (cp == 0) {
            items += plen;
            continue;
        }
        for (int64_t x = 0; x < qlen; ++x) {
            const int32_t v = a.colsq[qb + x] & Lq.idmask;
            bool ok = true;
            if (Lq.check_mask) ok = (cmask[v] >> Lq.qv) & 1u;
            for (int t = 0; t < Lq.ninj && ok; ++t) ok = v != row[Lq.inj[t]];
            for (int t = 0; t < Lq.nb && ok; ++t)
                if (t != qpv)
                    ok = member(a.mem, a.colsq, a.colsq + a.qcbeg[r * Lq.nb + t], a.qclen[r * Lq.nb + t],
                                Lq.key_base | v, v, row[Lq.bpos[t]], Lq.bkey[t], probes);
            cq += ok;
        }
        items += plen + qlen;
        total += cp * cq - cb;
    }
    unsigned long long pr = probes;
    for (int o = 16; o; o >>= 1) {
        total += __shfl_xor_sync(0xffffffffu, total, o);
        items += __shfl_xor_sync(0xffffffffu, items, o);
        pr += __shfl_xor_sync(0xffffffffu, pr, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (total) {
            atomicAdd(a.count, total);
            atomicAdd(&a.stats[3], total);
        }
        if (items) atomicAdd(&a.stats[0], items);
        if (pr) atomicAdd(&a.stats[2], pr);
    }
}

template <typename MaskT>
static void launch_pair_thread_t(const PairArgs& a, const LevelPlan& Lp, const LevelPlan& Lq, cudaStream_t s) {
    k_pair_thread<MaskT><<<grid_for(a.R), kThreads, 0, s>>>(a, Lp, Lq);
    GSM_LAUNCH("k_pair_thread");
}

void launch_pair_thread(const PairArgs& a, const LevelPlan& Lp, const LevelPlan& Lq, int mask_bytes, cudaStream_t s) {
    switch (mask_bytes) {
        case 1: launch_pair_thread_t<uint8_t>(a, Lp, Lq, s); break;
        case 2: launch_pair_thread_t<uint16_t>(a, Lp, Lq, s); break;
        default: launch_pair_thread_t<uint32_t>(a, Lp, Lq, s); break;
    }
}

template <typename MaskT>
static void launch_pair_t(const PairArgs& a, const LevelPlan& Lp, const LevelPlan& Lq, cudaStream_t s) {
    int dev = 0, sms = 148, per_sm = 1;
    GSM_CUDA(cudaGetDevice(&dev));
    GSM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GSM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pair<MaskT>, kThreads, 0));
    const int64_t want = (a.R + kWarps - 1) / kWarps;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1)));
    k_pair<MaskT><<<(unsigned)grid, kThreads, 0, s>>>(a, Lp, Lq);
    GSM_LAUNCH("k_pair");
}

void launch_pair(const PairArgs& a, const LevelPlan& Lp, const LevelPlan& Lq, int mask_bytes, cudaStream_t s) {
    switch (mask_bytes) {
        case 1: launch_pair_t<uint8_t>(a, Lp, Lq, s); break;
        case 2: launch_pair_t<uint16_t>(a, Lp, Lq, s); break;
        default: launch_pair_t<uint32_t>(a, Lp, Lq, s); break;
    }
}

__global__ void k_gather_len(const int64_t* __restrict__ rlen, const int64_t* __restrict__ idx, int64_t n,
                             int64_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = rlen[idx[i]];
}

void sort_rows_by_len_desc(const int64_t* rlen, int64_t* idx, int64_t n, cudaStream_t s) {
    if (n <= 1) return;
    DevBuf<int64_t> k_in, k_out, v_out;
    k_in.ensure(n, s);
    k_out.ensure(n, s);
    v_out.ensure(n, s);
    k_gather_len<<<grid_for(n), kThreads, 0, s>>>(rlen, idx, n, k_in.p);
    GSM_LAUNCH("k_gather_len");
    size_t tb = 0;
    GSM_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, k_in.p, k_out.p, idx, v_out.p, n, 0, 40, s));
    DevBuf<uint8_t> tmp;
    tmp.ensure(tb, s);
    GSM_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, k_in.p, k_out.p, idx, v_out.p, n, 0, 40, s));
    GSM_CUDA(cudaMemcpyAsync(idx, v_out.p, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, s));
}

// phase-2 strategy, in percent: stream N(c) (B) when |N(c)| <= pct/100 x |RC part|
// (measured on R-MAT-20/24: 100 beats 200, 800, 3200)
int tail_bratio() { return knobs().tail_bratio; }

// per-warp candidate buffer (even: keeps the per-warp int64 area aligned); tests force the
// overflow path with GSM_TAIL_CAP
int tail_cap() { return knobs().tail_cap; }

template <typename MaskT>
static void launch_tail_t(const TailArgs& a, const LevelPlan& Lc, const LevelPlan& Ld, cudaStream_t s) {
    const size_t smem = sizeof(int32_t) * (size_t)tail_warp_ints(a.cap) * kWarps;
    GSM_CUDA(cudaFuncSetAttribute(k_tail<MaskT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    int dev = 0, sms = 148, per_sm = 1;
    GSM_CUDA(cudaGetDevice(&dev));
    GSM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GSM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail<MaskT>, kThreads, smem));
    const int64_t want = (a.R + kWarps - 1) / kWarps;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1)));
    k_tail<MaskT><<<(unsigned)grid, kThreads, smem, s>>>(a, Lc, Ld);
    GSM_LAUNCH("k_tail");
}

void launch_tail(const TailArgs& a, const LevelPlan& Lc, const LevelPlan& Ld, int mask_bytes, cudaStream_t s) {
    switch (mask_bytes) {
        case 1: launch_tail_t<uint8_t>(a, Lc, Ld, s); break;
        case 2: launch_tail_t<uint16_t>(a, Lc, Ld, s); break;
        default: launch_tail_t<uint32_t>(a, Lc, Ld, s); break;
    }
}

__global__ void k_gather_overflow(const Frontier F, const int64_t* __restrict__ idx, int64_t n,
                                  int32_t* __restrict__ out) {
    const int W = F.W;
    int32_t buf[kMaxK];
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* row = frontier_row(F, idx[r], buf);
        for (int c = 0; c < W; ++c) out[r * W + c] = row[c];
    }
}

// rows idx[0..n) of F, materialised as plain rows (width F.W)
void launch_gather_rows(const Frontier& F, const int64_t* idx, int64_t n, int32_t* out, cudaStream_t s) {
    k_gather_overflow<<<grid_for(n), kThreads, 0, s>>>(F, idx, n, out);
    GSM_LAUNCH("k_gather_overflow");
}

// ============================================================================
// Finalize (Alg. 1 line 16: "Return ... subgraph enumeration M").
// ============================================================================
__global__ void k_to_query_order(const int32_t* __restrict__ in, int64_t N, int k, const int32_t* __restrict__ order,
                                 const int32_t* __restrict__ new2old, int32_t* __restrict__ out) {
    const int64_t total = N * k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / k;
        const int j = (int)(i - r * k);
        out[r * k + order[j]] = new2old[in[i]];
    }
}

void launch_to_query_order(const int32_t* in, int64_t N, int k, const int32_t* order, const int32_t* new2old,
                           int32_t* out, cudaStream_t s) {
    k_to_query_order<<<grid_for(N * k), kThreads, 0, s>>>(in, N, k, order, new2old, out);
    GSM_LAUNCH("k_to_query_order");
}

// all embeddings of an orbit: (f∘σ)(u) = f(σ(u))
__global__ void k_aut_expand(const int32_t* __restrict__ in, int64_t N, int k, const int8_t* __restrict__ sig,
                             int64_t num_aut, int32_t* __restrict__ out) {
    const int64_t total = N * k * num_aut;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rowid = i / k;
        const int u = (int)(i - rowid * k);
        const int64_t sidx = rowid / N;
        const int64_t r = rowid - sidx * N;
        out[i] = in[r * k + sig[sidx * k + u]];
    }
}

void launch_aut_expand(const int32_t* in, int64_t N, int k, const int8_t* sigmas, int64_t num_aut, int32_t* out,
                       cudaStream_t s) {
    k_aut_expand<<<grid_for(N * k * num_aut), kThreads, 0, s>>>(in, N, k, sigmas, num_aut, out);
    GSM_LAUNCH("k_aut_expand");
}

// Lexicographic sort: LSD over column groups packed into 64-bit keys
// (b = bits per id; floor(64/b) columns per key), CUB radix sort passes.
__global__ void k_iota(uint32_t* p, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

__global__ void k_pack_keys(const int32_t* __restrict__ rows, const uint32_t* __restrict__ perm, int64_t N, int k,
                            int c0, int c1, int b, uint64_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* r = rows + (int64_t)perm[i] * k;
        uint64_t key = 0;
        for (int c = c0; c < c1; ++c) key = (key << b) | (uint32_t)r[c];
        keys[i] = key;
    }
}

__global__ void k_gather_rows(const int32_t* __restrict__ rows, const uint32_t* __restrict__ perm, int64_t N, int k,
                              int32_t* __restrict__ out) {
    const int64_t total = N * k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / k;
        out[i] = rows[(int64_t)perm[r] * k + (i - r * k)];
    }
}

void sort_rows(const int32_t* rows, int64_t N, int k, int64_t n, int32_t* out, cudaStream_t s) {
    if (N <= 0) return;
    if (N > (int64_t)0xffffffffLL) fail(GSM_ERR_OUT_OF_MEMORY, "enumeration larger than 2^32 rows");
    int b = 1;
    while (b < 31 && ((uint64_t)(n - 1) >> b)) ++b;
    const int per = std::max(1, 64 / b);
    DevBuf<uint32_t> perm, perm2;
    DevBuf<uint64_t> keys, keys2;
    perm.ensure(N, s);
    perm2.ensure(N, s);
    keys.ensure(N, s);
    keys2.ensure(N, s);
    k_iota<<<grid_for(N), kThreads, 0, s>>>(perm.p, N);
    GSM_LAUNCH("k_iota");
    size_t tb = 0;
    GSM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys2.p, perm.p, perm2.p, N, 0, 64, s));
    DevBuf<uint8_t> tmp;
    tmp.ensure(tb, s);
    for (int c1 = k; c1 > 0; c1 -= per) {
        const int c0 = std::max(0, c1 - per);
        k_pack_keys<<<grid_for(N), kThreads, 0, s>>>(rows, perm.p, N, k, c0, c1, b, keys.p);
        GSM_LAUNCH("k_pack_keys");
        GSM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys2.p, perm.p, perm2.p, N, 0, (c1 - c0) * b, s));
        std::swap(perm.p, perm2.p);
    }
    k_gather_rows<<<grid_for(N * k), kThreads, 0, s>>>(rows, perm.p, N, k, out);
    GSM_LAUNCH("k_gather_rows");
}

}  // namespace gsm
