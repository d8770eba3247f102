// gsm_clique.cu — COUNT mode for clique queries K_k (k = 3, 4): the verify step
// on per-root local bitmaps.
//
// Which query: every position i >= 1 is adjacent to all earlier positions
// (B(i) = {0..i-1}) and the symmetry conditions (Grochow-Kellis, DESIGN R9)
// chain f(π[0]) ≺ f(π[1]) ≺ ... ≺ f(π[k-1]); unlabeled.  Then every partial
// result (u = f(π[0]), f(π[1]), ...) lives inside S(u) = N+(u) = {w ∈ N(u): w ≻ u}
// (≺ = relabelled-id order, so N+(u) is the suffix of u's sorted list at up[u]).
//
// Same search tree as Alg. 1: level 1 extends root u by a ∈ S(u);
// level i extends (u, a1, .., a_{i-1}) by the candidates of the pivot list that
// are connected to every earlier position ("connections with existing nodes
// in partial results").  What changes is the representation of the candidate
// sets: per root, the connection test "w ∈ N(S[i])" for w ∈ S(u) is evaluated
// ONCE into a bit row A[i] (bit j set iff S[j] ∈ N+(S[i]), j > i), and the
// candidate set of a partial result is the AND of the rows of its members.
// For K4 the last level counts popc(A[i] & A[j]) over the level-2 partial results
// (u, S[i], S[j]) — the width-3 frontier is never materialised, and each
// verification of two backward edges of 32 candidates is one AND + POPC.
//
// Work split (roots sorted by |S(u)| descending, dynamic scheduling):
//   d <= 32     k_clique_warp: one warp per root, lane i holds row A[i] (1 word)
//   d <= dsmem  k_clique_cta : one CTA per root, S and A in shared memory
//   larger      k_clique_cta<kGlobal>: S and A in a per-CTA global slab (L2)
// Row construction per i picks the cheaper of (a) the lanes binary-searching
// their S[j] in N+(S[i]) (global, mostly L1/L2 hits) and (b) streaming N+(S[i])
// (coalesced) and binary-searching each entry in S (shared memory).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "gsm_kernels.h"
#include "gsm_workspace.h"

namespace gsm {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// key ∈ cols[lo, hi) (sorted), by binary search
__device__ __forceinline__ bool search_list(const int32_t* __restrict__ cols, int64_t lo, int64_t hi, int32_t key,
                                            unsigned& probes) {
    int64_t l = lo, h = hi;
    while (l < h) {
        const int64_t mid = (l + h) >> 1;
        ++probes;
        if (__ldg(cols + mid) < key) l = mid + 1; else h = mid;
    }
    return l < hi && __ldg(cols + l) == key;
}

// index of key in S[lo, hi) or -1
__device__ __forceinline__ int search_local(const int32_t* S, int lo, int hi, int32_t key) {
    int l = lo, h = hi;
    while (l < h) {
        const int mid = (l + h) >> 1;
        if (S[mid] < key) l = mid + 1; else h = mid;
    }
    return (l < hi && S[l] == key) ? l : -1;
}

// Two-table cuckoo hash of S(u): vertex id -> local index.  Entry = id << 32 | index
// (all ones = empty).  A lookup is exactly two shared-memory probes, branch-free, so the
// 32 lanes of a streaming step stay converged.  Tables: 2 x P entries, P = 1.25 d rounded
// up to 32 (load <= 0.4); a 32-bit hash is mapped to [0, P) by a multiply-high.
__host__ __device__ __forceinline__ int cuckoo_slots(int dmax) {  // P
    return ((dmax + dmax / 4 + 31) / 32) * 32 + 32;
}

__device__ __forceinline__ unsigned ck_h0(int32_t v, unsigned P, unsigned seed) {
    return __umulhi((unsigned)v * (0x9E3779B1u + 2u * seed), P);
}

__device__ __forceinline__ unsigned ck_h1(int32_t v, unsigned P, unsigned seed) {
    return __umulhi(((unsigned)v + seed) * 0x85EBCA6Bu, P);
}

// Tables as two 32-bit arrays: keys Tk[2P] (-1 = empty) and local indices Tj[2P].  A lookup
// reads two 32-bit keys (half the shared-memory wavefronts of 64-bit entries); the index is
// read only on a hit.  Returns the local index of v in S(u), or -1.
__device__ __forceinline__ int ck_find(const int32_t* Tk, const int32_t* Tj, unsigned P, unsigned seed, int32_t v) {
    const unsigned s0 = ck_h0(v, P, seed), s1 = P + ck_h1(v, P, seed);
    const bool m0 = Tk[s0] == v;
    const bool m1 = Tk[s1] == v;
    return (m0 | m1) ? Tj[m0 ? s0 : s1] : -1;
}

__device__ __forceinline__ bool ck_has(const int32_t* Tk, unsigned P, unsigned seed, int32_t v) {
    return (Tk[ck_h0(v, P, seed)] == v) | (Tk[P + ck_h1(v, P, seed)] == v);
}

}  // namespace

struct BucketEdges {
    int e[7];  // |S(u)| upper edges of buckets 0..6 (6 = global slab); bucket 7 = beyond e[6]
};

// keys[r] = |N+(roots[r])| (0 if below k-1: no clique through it), vals[r] = r; bucket
// counts and the max.  Descending keys keep every bucket contiguous in the sorted order.
__global__ void k_clique_keys(const int32_t* __restrict__ roots, int64_t R, const int4* __restrict__ np,
                              int kmin, BucketEdges E, int32_t* __restrict__ keys,
                              int32_t* __restrict__ vals, unsigned long long* __restrict__ bucket, int* dmax) {
    __shared__ unsigned long long sb[8];
    __shared__ int sm, small;
    if (threadIdx.x < 8) sb[threadIdx.x] = 0;
    if (threadIdx.x == 0) sm = small = 0;
    __syncthreads();
    int lm = 0, lall = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = roots[r];
        int d = __ldg(np + u).z;
        if (d < kmin) d = 0;
        keys[r] = d;
        vals[r] = (int32_t)r;
        if (d > 0) {
            int b = 0;
            while (b < 7 && d > E.e[b]) ++b;
            atomicAdd(&sb[b], 1ull);
            if (b < 7) lm = max(lm, d);  // max over the roots this path processes
            lall = max(lall, d);
        }
    }
    atomicMax(&sm, lm);
    atomicMax(&small, lall);
    __syncthreads();
    if (threadIdx.x < 8 && sb[threadIdx.x]) atomicAdd(&bucket[threadIdx.x], sb[threadIdx.x]);
    if (threadIdx.x == 0 && sm) atomicMax(dmax, sm);
    if (threadIdx.x == 0 && small) atomicMax(dmax + 1, small);
}

struct CliqueArgs {
    const int32_t* roots;   // level-0 frontier (new ids)
    const int32_t* idx;     // roots of this launch: roots[idx[t]], t < n
    int64_t n;
    const int64_t* off;
    const int32_t* cols;
    const int32_t* up;
    const int4* np;         // DevGraph::nplus: packed {begin, |N+(v)|, nh_off} per vertex
    int32_t dmax;           // max |N+(u)| of this launch (sizes shared memory / the slab)
    int32_t stream_max;     // row construction streams N+(S[i]) when its length <= stream_max * (#j)/32
    int32_t use_hash;       // k_clique_cta: cuckoo table of S(u) (0: rows by binary search only)
    const uint32_t* hub_bits;  // hub adjacency bitmap (DevGraph::hub_bits) or nullptr
    int32_t hub_base;       // first hub rank
    int32_t hub_words;      // H / 32
    int32_t hub_ratio;      // k_clique_cta: a hub row takes bitmap lookups when 32 nj <= hub_ratio |N+(a)|
    const int32_t* nh_off;  // hashed N+(v) tables (DevGraph::nh_*) or nullptr
    const int32_t* nh_tab;
    int32_t nh_stream;      // with a table, a row streams N+(S[i]) only when 32 |N+(S[i])| <= nh_stream x nj
    int32_t ranges;         // K4: level 3 over the overlap of the rows' nonzero word ranges (else j/32..W)
    int32_t lazy_ck;        // build the per-root cuckoo table only when some row streams
    int32_t* slab;          // kGlobal: per-CTA scratch of cta_lay(..).slab_ints ints
    int32_t slab_blocks;    // kGlobal: slabs allocated (the grid must not exceed it)
    unsigned long long* next;   // dynamic root scheduler
    unsigned long long* count;  // unique cliques (atomic)
    unsigned long long* stats;  // [list entries read, global probes, bitmap words, cliques, sum |S(u)|]
    unsigned long long* cyc;    // optional (GSM_TRACE=2): warp-cycles [setup, stream rows, search rows, level 3]
};

// ---------------------------------------------------------------------------- d <= 32
template <int K>
__global__ void __launch_bounds__(256) k_clique_warp(CliqueArgs a) {
    __shared__ int32_t sS[8][32];
    __shared__ unsigned sA[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int32_t* __restrict__ cols = a.cols;
    unsigned long long cnt = 0, items = 0, sent = 0;
    unsigned probes = 0;
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t t = (int64_t)blockIdx.x * 8 + wib; t < a.n; t += nw) {
        const int32_t u = a.roots[a.idx[t]];
        int64_t s0;
        int d;
        int32_t unh;
        nplus_load(a.np, u, s0, d, unh);
        (void)unh;
        GSM_DCHECK(d <= 32, DCHK_WARP_D);
        const int32_t sv = lane < d ? cols[s0 + lane] : INT32_MAX;
        // each lane's own S entry's N+ descriptor (rows broadcast it by shuffle)
        int64_t my_b = 0;
        int my_len = 0;
        int32_t my_nh = -1;
        if (lane < d) nplus_load(a.np, sv, my_b, my_len, my_nh);
        sS[wib][lane] = sv;
        if (lane == 0) sent += d;
        __syncwarp();
        const int32_t smax = sS[wib][d - 1];
        unsigned myrow = 0;
        for (int i = 0; i < d - 1; ++i) {
            const int32_t ai = sS[wib][i];
            const int64_t ls = __shfl_sync(kFull, my_b, i);
            const int64_t le = ls + __shfl_sync(kFull, my_len, i);
            const int32_t ai_nh = __shfl_sync(kFull, my_nh, i);
            const int nj = d - 1 - i;
            unsigned bits = 0;
            if (a.hub_bits && ai >= a.hub_base) {
                // hub pivot: S[j] > S[i] >= hub_base, one bitmap word per lane (L2-resident)
                const uint32_t* hr = hub_row(a.hub_bits, a.hub_words, ai - a.hub_base);
                const bool live = lane > i && lane < d;
                bool f = false;
                if (live) {
                    const int c = sv - a.hub_base;
                    f = (__ldg(hr + (c >> 5)) >> (c & 31)) & 1u;
                }
                bits = __ballot_sync(kFull, f);
                items += live;
            } else if (ai_nh >= 0 && 32 * (le - ls) > (int64_t)a.nh_stream * nj) {
                // hashed N+(S[i]): one bucket (32-byte sector) per remaining S[j]
                const int32_t tb = ai_nh;
                const bool live = lane > i && lane < d;
                const bool f = live && nh_find(a.nh_tab, tb, nh_buckets(le - ls), sv, probes);
                bits = __ballot_sync(kFull, f);
                items += live;
            } else if (le - ls <= (int64_t)a.stream_max) {
                // stream N+(S[i]); each entry looked up in S[i+1, d) (shared memory)
                for (int64_t x0 = ls; x0 < le; x0 += 32) {
                    const int64_t x = x0 + lane;
                    const int32_t v = x < le ? cols[x] : INT32_MAX;
                    if (!__any_sync(kFull, v <= smax)) break;
                    if (v <= smax) {
                        ++items;
                        const int j = search_local(sS[wib], i + 1, d, v);
                        if (j >= 0) bits |= 1u << j;
                    }
                }
                bits = __reduce_or_sync(kFull, bits);
            } else {
                // slice of N+(S[i]) by 32 splitters (see k_clique_cta), then binary search
                const int64_t len = le - ls;
                const int64_t bl = ls + ((int64_t)lane * len) / 32;
                const int32_t spl = bl < le ? cols[bl] : INT32_MAX;
                int lo = 0, hi = 32;
#pragma unroll
                for (int st = 0; st < 5; ++st) {
                    const int mid = (lo + hi) >> 1;
                    const int32_t x = __shfl_sync(kFull, spl, mid);
                    if (x <= sv) lo = mid; else hi = mid;
                }
                const bool f = lane > i && lane < d &&
                               search_list(cols, ls + ((int64_t)lo * len) / 32, ls + ((int64_t)(lo + 1) * len) / 32, sv,
                                           probes);
                bits = __ballot_sync(kFull, f);
                items += (lane > i && lane < d);
            }
            (void)nj;
            if (lane == i) myrow = bits;
            if (K == 3 && lane == 0) cnt += __popc(bits);
        }
        if (K == 4) {
            sA[wib][lane] = myrow;
            __syncwarp();
            unsigned b = myrow & __ballot_sync(kFull, myrow != 0u);  // skip empty second rows
            while (b) {
                const int j = __ffs(b) - 1;
                b &= b - 1;
                cnt += __popc(myrow & sA[wib][j]);
            }
        }
        __syncwarp();
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(kFull, cnt, o);
        items += __shfl_xor_sync(kFull, items, o);
        probes += __shfl_xor_sync(kFull, probes, o);
    }
    if (lane == 0) {
        if (cnt) atomicAdd(a.count, cnt);
        if (cnt) atomicAdd(&a.stats[3], cnt);
        if (items) atomicAdd(&a.stats[0], items);
        if (probes) atomicAdd(&a.stats[1], (unsigned long long)probes);
        if (sent) atomicAdd(&a.stats[4], sent);
    }
}

// ---------------------------------------------------------------------------- d > 32
// Per-CTA workspace (int32 units), identical on host and device.  Shared memory always
// holds the cuckoo table T and the row-block table TB; S(u), the row
// metadata (RL: |N+(S[i])|, RB: its start) and the bit rows A are in shared memory too,
// or in a per-CTA global slab (kGlobal) for |S(u)| beyond what one CTA can hold.
// Bit rows are stored triangular: row i keeps words i/32 .. W-1 only (bits <= i are 0),
// rows of block b = i/32 have odd length (W-b)|1 (conflict-free column reads).
__host__ __device__ inline int64_t tri_words(int d) {
    const int W = (d + 31) >> 5;
    int64_t t = 0;
    for (int b = 0; b < W; ++b) t += (int64_t)min(32, d - 32 * b) * ((W - b) | 1);
    return t;
}

struct CtaLay {
    int64_t h, tb, s, rl, rh, rw, rb, A;  // offsets (int32 units) in shared memory or the slab
    int64_t smem_ints, slab_ints;
};

__host__ __device__ inline CtaLay cta_lay(int K, int dmax, bool global, bool hash, bool ranges) {
    CtaLay L;
    int64_t o = 0, g = 0;
    const int W = (dmax + 31) >> 5;
    L.h = o;  // 8-byte aligned (offset 0)
    o += hash ? 4 * (int64_t)cuckoo_slots(dmax) : 0;
    L.tb = o;
    o += 2 * (W + 1);
    int64_t& q = global ? g : o;
    q = (q + 1) & ~1LL;
    L.s = q;
    q += dmax;
    L.rl = q;
    q += dmax;
    L.rh = q;
    q += dmax;
    L.rw = q;  // K4: nonzero word range of each bit row, lo << 16 | hi (hi exclusive)
    q += (K == 4 && ranges) ? dmax : 0;  // only with GSM_CLIQUE_RANGES (keeps the 960-root CTAs 2 per SM)
    q = (q + 1) & ~1LL;  // int64 alignment
    L.rb = q;
    q += 2 * (int64_t)dmax;
    L.A = q;
    q += K == 4 ? tri_words(dmax) : 0;
    q = (q + 1) & ~1LL;
    L.smem_ints = o;
    L.slab_ints = g;
    return L;
}

template <int K, bool kGlobal, int NT, int kMinB>
__global__ void __launch_bounds__(NT, kMinB) k_clique_cta(CliqueArgs a) {
    extern __shared__ __align__(16) int32_t csm[];
    constexpr int NW = NT / 32;
    __shared__ int32_t sJ[NW][64];  // level-3 j lists / Bloom-positive queue of the row phase
    __shared__ int sRow[2];
    __shared__ unsigned long long sRoot;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int32_t* __restrict__ cols = a.cols;
    const CtaLay L = cta_lay(K, a.dmax, kGlobal, a.use_hash != 0, a.ranges != 0);
    int32_t* ws = kGlobal ? a.slab + (int64_t)blockIdx.x * L.slab_ints : csm;
    int32_t* Tk = csm + L.h;  // cuckoo keys [2P], then local indices [2P] (Tj)
    __shared__ int sFail;
    int32_t* TB = csm + L.tb;  // TB[b] = first word of row block b, TB[W + 1 + b] = its row length
    int32_t* S = ws + L.s;
    int32_t* RL = ws + L.rl;
    int32_t* RH = ws + L.rh;  // nh_off of each S entry (-1: no hashed N+)
    int32_t* RW = ws + L.rw;  // K4: nonzero word range [lo, hi) of bit row i, lo << 16 | hi
    int64_t* RB = reinterpret_cast<int64_t*>(ws + L.rb);
    unsigned* A = reinterpret_cast<unsigned*>(ws + L.A);
    unsigned long long cnt = 0;
    unsigned items = 0, words = 0, sent = 0;  // per-thread stats (32-bit: fewer registers)
    unsigned probes = 0;
    // GSM_TRACE=2 (a.cyc): phase cycles and keys per row strategy go straight to global
    // counters from lane 0 — nothing held in registers across the kernel when tracing is off
    auto trace = [&](int slot, long long cycles, unsigned long long keys, int kslot) {
        if (lane == 0) {
            atomicAdd(&a.cyc[slot], (unsigned long long)cycles);
            if (kslot >= 0) atomicAdd(&a.cyc[kslot], keys);
        }
    };
    long long tc = 0;
    for (;;) {
        if (a.cyc) tc = clock64();
        __syncthreads();
        if (threadIdx.x == 0) {
            sRoot = atomicAdd(a.next, 1ull);
            sRow[0] = 0;
            sRow[1] = 0;
        }
        __syncthreads();
        const int64_t t = (int64_t)sRoot;
        if (t >= a.n) break;
        const int32_t u = a.roots[a.idx[t]];
        int64_t s0;
        int d;
        int32_t unh;
        nplus_load(a.np, u, s0, d, unh);
        (void)unh;
#ifdef GSM_DEVICE_CHECKS
        if (d > a.dmax) {  // the launch's shared memory / slab is sized for dmax
            GSM_DCHECK(false, DCHK_CTA_D);
            continue;
        }
        GSM_DCHECK(!kGlobal || blockIdx.x < (unsigned)a.slab_blocks, DCHK_SLAB);
        const int64_t tri_lim = K == 4 ? tri_words(d) : 0;
#endif
        const int W = (d + 31) >> 5;
        const unsigned P = cuckoo_slots(d);
        if (K == 4 && threadIdx.x < W) {
            int base = 0;
            for (int b = 0; b < (int)threadIdx.x; ++b) base += 32 * ((W - b) | 1);
            TB[threadIdx.x] = base;
            TB[W + 1 + threadIdx.x] = (W - threadIdx.x) | 1;
        }
        // S(u) and, per entry, its own list N+(S[j]) (one parallel gather instead of a
        // dependent chain per row)
        int wants_stream = 0;  // some row of this root would stream N+(S[i]) (needs the cuckoo table)
        for (int j = threadIdx.x; j < d; j += NT) {
            const int32_t v = cols[s0 + j];
            S[j] = v;
            int64_t b;
            int len;
            int32_t nh;
            nplus_load(a.np, v, b, len, nh);
            RB[j] = b;
            RL[j] = len;
            RH[j] = nh;
            // the row loop's choice, given a table: hub lookups / hashed lookups / stream
            const int64_t nj = d - 1 - j;
            const bool hub = a.hub_bits && v >= a.hub_base && 32 * nj <= (int64_t)a.hub_ratio * len;
            const int64_t thr = nh >= 0 ? a.nh_stream : a.stream_max;
            wants_stream |= (nj > 0 && !hub && 32LL * len <= thr * nj) ? 1 : 0;
        }
        if (threadIdx.x == 0) sent += d;
        // cuckoo build, only if some row streams (a failed build — an eviction cycle — retries
        // with a new seed; after 4 failures the root's rows all take the binary-search strategy)
        unsigned seed = 0;
        bool use_ck = __syncthreads_or(wants_stream | !a.lazy_ck) && a.use_hash != 0;
        for (; use_ck; ++seed) {
            if (seed == 4) {
                use_ck = false;
                break;
            }
            for (int h = threadIdx.x; h < 2 * (int)P; h += NT) Tk[h] = -1;
            if (threadIdx.x == 0) sFail = 0;
            __syncthreads();
            for (int j = threadIdx.x; j < d; j += NT) {
                int32_t e = S[j];
                int tbl = 0;
                int it = 0;
                for (; it < 64; ++it) {
                    const unsigned slot = tbl ? P + ck_h1(e, P, seed) : ck_h0(e, P, seed);
                    GSM_DCHECK(slot < 2 * P, DCHK_CUCKOO);
                    e = atomicExch(&Tk[slot], e);
                    if (e == -1) break;
                    tbl ^= 1;
                }
                if (it == 64) sFail = 1;
            }
            __syncthreads();
            if (!sFail) {
                if (K == 4) {  // local indices next to the settled keys
                    int32_t* Tj = Tk + 2 * P;
                    for (int j = threadIdx.x; j < d; j += NT) {
                        const int32_t v = S[j];
                        const unsigned s0h = ck_h0(v, P, seed);
                        Tj[Tk[s0h] == v ? s0h : P + ck_h1(v, P, seed)] = j;
                    }
                }
                break;
            }
            __syncthreads();
        }
        __syncthreads();
        const int32_t smax = S[d - 1];
        if (a.cyc) {
            const long long t1 = clock64();
            trace(0, t1 - tc, 0, -1);
            tc = t1;
        }
        // ---- rows A[i] (level 1 -> 2 connection tests), warps take rows dynamically
        for (;;) {
            int i = 0;
            if (lane == 0) i = atomicAdd(&sRow[0], 1);
            i = __shfl_sync(kFull, i, 0);
            if (i >= d) break;
            const int w0 = i >> 5;
            unsigned* Ai = A + TB[w0] + (i & 31) * TB[W + 1 + w0] - w0;  // Ai[w], w >= w0
#ifdef GSM_DEVICE_CHECKS
            GSM_DCHECK(K != 4 || (Ai + w0 >= A && Ai + W <= A + tri_lim), DCHK_AROW);
#endif
            if (i == d - 1) {  // no j > i: an all-zero row (read by level 3)
                if (K == 4 && lane == 0) Ai[w0] = 0;
                continue;
            }
            const int64_t ls = RB[i];
            const int len = RL[i];
            const int64_t le = ls + len;
            const int nj = d - 1 - i;
            const int32_t ai = S[i];
            if (a.hub_bits && ai >= a.hub_base && 32LL * nj <= (int64_t)a.hub_ratio * len) {
                // hub pivot: every S[j] (j > i) is a hub too; bit j of A[i] = one word of the
                // L2-resident hub bitmap row of S[i] (replaces the stream / binary search)
                const uint32_t* hr = hub_row(a.hub_bits, a.hub_words, ai - a.hub_base);
                for (int w = w0; w < W; ++w) {
                    const int j = (w << 5) + lane;
                    const bool live = j > i && j < d;
                    bool f = false;
                    if (live) {
                        const int c = S[j] - a.hub_base;
                        f = (__ldg(hr + (c >> 5)) >> (c & 31)) & 1u;
                    }
                    items += live;
                    const unsigned bits = __ballot_sync(kFull, f);
                    if (K == 4) {
                        if (lane == 0) Ai[w] = bits;
                    } else {
                        cnt += f;
                    }
                }
                if (a.cyc) {
                    const long long t1 = clock64();
                    trace(2, t1 - tc, nj, 4);
                    tc = t1;
                }
                continue;
            }
            // hashed N+(S[i]) (load-time table): one 32-byte bucket per remaining S[j], unless
            // streaming the list is cheaper (32 len <= nh_stream x nj)
            const int32_t tb = RH[i];
            if (tb >= 0 && !(use_ck && (int64_t)len * 32 <= (int64_t)a.nh_stream * nj)) {
                const unsigned B = nh_buckets(len);
                for (int w = w0; w < W; ++w) {
                    const int j = (w << 5) + lane;
                    const bool live = j > i && j < d;
                    items += live;
                    const bool f = live && nh_find(a.nh_tab, tb, B, S[j], probes);
                    const unsigned bits = __ballot_sync(kFull, f);
                    if (K == 4) {
                        if (lane == 0) Ai[w] = bits;
                    } else {
                        cnt += f;
                    }
                }
                if (a.cyc) {
                    const long long t1 = clock64();
                    trace(2, t1 - tc, nj, 5);
                    tc = t1;
                }
                continue;
            }
            // streaming needs the cuckoo table; without it (GSM_CLIQUE_HASH=0, or 4 failed
            // builds) every row takes the binary-search strategy
            if (use_ck && (int64_t)len * 32 <= (int64_t)a.stream_max * nj) {
                if (K == 4) {
                    for (int w = w0 + lane; w < W; w += 32) Ai[w] = 0;
                    __syncwarp();
                }
                for (int64_t x0 = ls; x0 < le; x0 += 64) {  // two loads in flight per lane
                    const int64_t x = x0 + lane;
                    const int32_t v0 = x < le ? cols[x] : INT32_MAX;
                    const int32_t v1 = x + 32 < le ? cols[x + 32] : INT32_MAX;
                    if (!__any_sync(kFull, v0 <= smax)) break;
                    if (lane == 0) items += min((int64_t)64, le - x0);
                    const int j0 = K == 4 ? ck_find(Tk, Tk + 2 * P, P, seed, v0) : (ck_has(Tk, P, seed, v0) ? 0 : -1);
                    const int j1 = K == 4 ? ck_find(Tk, Tk + 2 * P, P, seed, v1) : (ck_has(Tk, P, seed, v1) ? 0 : -1);
                    if (K == 4) {
                        if (j0 >= 0) atomicOr(&Ai[j0 >> 5], 1u << (j0 & 31));
                        if (j1 >= 0) atomicOr(&Ai[j1 >> 5], 1u << (j1 & 31));
                    } else {
                        cnt += (j0 >= 0) + (j1 >= 0);
                    }
                }
                if (a.cyc) {
                    const long long t1 = clock64();
                    trace(1, t1 - tc, len, 6);
                    tc = t1;
                }
            } else {
                // 32 splitters of N+(S[i]) in one coalesced load (lane l: the first entry of
                // slice l); each key then picks its slice by a 5-step shuffle search and binary-
                // searches only that slice in global memory (5 fewer dependent global probes)
                const int64_t bl = ls + ((int64_t)lane * len) / 32;
                const int32_t spl = bl < le ? cols[bl] : INT32_MAX;
                for (int w = w0; w < W; ++w) {
                    const int j = (w << 5) + lane;
                    const bool live = j > i && j < d;
                    items += live;
                    const int32_t key = live ? S[j] : INT32_MAX;
                    int lo = 0, hi = 32;  // last slice whose first entry <= key
#pragma unroll
                    for (int st = 0; st < 5; ++st) {
                        const int mid = (lo + hi) >> 1;
                        const int32_t sv = __shfl_sync(kFull, spl, mid);
                        if (sv <= key) lo = mid; else hi = mid;
                    }
                    const int64_t sb = ls + ((int64_t)lo * len) / 32;
                    const int64_t se = ls + ((int64_t)(lo + 1) * len) / 32;
                    const bool f = live && search_list(cols, sb, se, key, probes);
                    const unsigned bits = __ballot_sync(kFull, f);
                    if (K == 4) {
                        if (lane == 0) Ai[w] = bits;
                    } else {
                        cnt += f;
                    }
                }
                if (a.cyc) {
                    const long long t1 = clock64();
                    trace(2, t1 - tc, nj, 7);
                    tc = t1;
                }
            }
        }
        if (K == 3) continue;
        __syncthreads();
        // nonzero word range of every bit row (level 3 intersects only the overlap of two
        // rows' ranges instead of every word from j/32 to the end) — for roots with W >= 8
        // words per row; shorter rows are not worth the extra pass and barrier
        const bool use_rw = a.ranges && W >= 8;
        for (int i = wib; use_rw && i < d; i += NW) {
            const int w0 = i >> 5;
            const unsigned* Ai = A + TB[w0] + (i & 31) * TB[W + 1 + w0] - w0;
            int lo = W, hi = w0;
            for (int base = w0; base < W; base += 32) {
                const int w = base + lane;
                const unsigned nz = __ballot_sync(kFull, w < W && Ai[w] != 0u);
                if (nz) {
                    if (lo == W) lo = base + __ffs(nz) - 1;
                    hi = base + 32 - __clz(nz);
                }
            }
            if (lane == 0) RW[i] = lo < hi ? (lo << 16) | hi : 0;
        }
        if (use_rw) __syncthreads();
        // ---- level 3: for every level-2 partial result (u, S[i], S[j]) (bit j of A[i]):
        //      |{l : A[i] bit l and A[j] bit l}| = popc over words of A[i] & A[j]
        // (i, j) pairs are queued per warp across rows (sJ[.][0..31] = j, [32..63] = i) and
        // processed 32 at a time, one pair per lane — rows with few bits do not leave lanes idle
        {
            int nJ = 0;
            auto flush = [&](int np) {
                __syncwarp();
                if (lane < np) {
                    const int j = sJ[wib][lane], i = sJ[wib][32 + lane];
                    const int wi = i >> 5, wj = j >> 5;
                    const unsigned* Ai = A + TB[wi] + (i & 31) * TB[W + 1 + wi] - wi;
                    const unsigned* Aj = A + TB[wj] + (j & 31) * TB[W + 1 + wj] - wj;
                    int x0 = wj, x1 = W;
                    if (use_rw) {
                        const unsigned ri = (unsigned)RW[i], rj = (unsigned)RW[j];
                        x0 = max(wj, (int)max(ri >> 16, rj >> 16));
                        x1 = (int)min(ri & 0xffffu, rj & 0xffffu);
                    }
                    unsigned c = 0;
                    for (int x = x0; x < x1; ++x) c += __popc(Ai[x] & Aj[x]);
                    cnt += c;
                    words += x1 > x0 ? x1 - x0 : 0;
                }
                __syncwarp();
            };
            for (;;) {
                int i = 0;
                if (lane == 0) i = atomicAdd(&sRow[1], 1);
                i = __shfl_sync(kFull, i, 0);
                if (i >= d - 1) break;
                const int wi = i >> 5;
                const unsigned* Ai = A + TB[wi] + (i & 31) * TB[W + 1 + wi] - wi;
                const unsigned ri = use_rw ? (unsigned)RW[i] : ((unsigned)wi << 16) | (unsigned)W;
                for (int w = max(wi, (int)(ri >> 16)); w < (int)(ri & 0xffffu); ++w) {
                    unsigned bits = Ai[w];
                    while (bits) {
                        const int take = min(__popc(bits), 32 - nJ);
                        const bool has = (bits >> lane) & 1u;
                        const int rank = __popc(bits & ((1u << lane) - 1u));
                        const bool tk = has && rank < take;
                        if (tk) {
                            GSM_DCHECK(nJ + rank < 32, DCHK_PAIRQ);
                            sJ[wib][nJ + rank] = (w << 5) + lane;
                            sJ[wib][32 + nJ + rank] = i;
                        }
                        bits &= ~__ballot_sync(kFull, tk);
                        nJ += take;
                        if (nJ == 32) {
                            flush(32);
                            nJ = 0;
                        }
                    }
                }
            }
            if (nJ > 0) flush(nJ);
        }
        if (a.cyc) trace(3, clock64() - tc, 0, -1);
    }
    unsigned long long pr = probes, it = items, wd = words;
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(kFull, cnt, o);
        it += __shfl_xor_sync(kFull, it, o);
        pr += __shfl_xor_sync(kFull, pr, o);
        wd += __shfl_xor_sync(kFull, wd, o);
    }
    if (lane == 0) {
        if (cnt) {
            atomicAdd(a.count, cnt);
            atomicAdd(&a.stats[3], cnt);
        }
        if (it) atomicAdd(&a.stats[0], it);
        if (pr) atomicAdd(&a.stats[1], pr);
        if (wd) atomicAdd(&a.stats[2], wd);
        if (sent) atomicAdd(&a.stats[4], (unsigned long long)sent);
    }
}

static int sm_count() {
    int dev = 0, sms = 148;
    GSM_CUDA(cudaGetDevice(&dev));
    GSM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
}

static int use_hash() { return knobs().clique_hash ? 1 : 0; }  // 0: every row by binary search (tests)

static size_t cta_smem(int K, int dmax, bool global) {
    return sizeof(int32_t) * (size_t)cta_lay(K, dmax, global, use_hash() != 0, knobs().clique_ranges != 0).smem_ints;
}

constexpr size_t kSmemLim = 216 * 1024;  // dynamic; + static (8 KB queues, counters) <= 227 KB

// largest |S(u)| whose whole per-root workspace fits one CTA's shared memory
int clique_dsmem(int K) {
    int d = 32;
    while (cta_smem(K, d + 32, false) <= kSmemLim) d += 32;
    if (knobs().clique_dsmem > 0) d = std::min(d, std::max(64, knobs().clique_dsmem));
    return d;
}

static int warp_max() { return knobs().clique_warp; }  // 0: no warp-per-root kernel (tests)

static int stream_max() { return knobs().clique_stream; }

template <int K, bool G, int NT, int MB>
static void launch_cta_mb(CliqueArgs a, int64_t blocks, cudaStream_t s) {
    const size_t smem = cta_smem(K, a.dmax, G);
    GSM_CUDA(cudaFuncSetAttribute(k_clique_cta<K, G, NT, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLim));
    int per_sm = 1;
    GSM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_clique_cta<K, G, NT, MB>, NT, smem));
    const int64_t cap = (int64_t)sm_count() * std::max(per_sm, 1);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(blocks, std::min<int64_t>(a.n, cap)));
    k_clique_cta<K, G, NT, MB><<<(unsigned)grid, NT, smem, s>>>(a);
    GSM_LAUNCH("k_clique_cta");
}

// Round 1: registers capped for 2048 resident threads per SM (measured on R-MAT-24 K3+K4 then:
// capped 760 ms vs uncapped 1,110 ms per step — the rows were latency-bound).
template <int K, bool G, int NT, int MB>
static int cta_occupancy_mb(size_t smem) {
    GSM_CUDA(cudaFuncSetAttribute(k_clique_cta<K, G, NT, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLim));
    int per_sm = 0;
    GSM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_clique_cta<K, G, NT, MB>, NT, smem));
    return per_sm;
}

// Round 2 (hub-bitmap / hashed rows): interleaved A/B on R-MAT-24 K3+K4 (profiles/r2_ab*.jsonl)
// — cap for 2,048 resident threads 378 ms (spills 20-40 B), uncapped 350, 1,536 337, 1,280 333,
// and 1,280 with the bucket CTA size from the occupancy calculator 323 ms (1,024: 346).
// GSM_CLIQUE_OCC: 0 = uncapped, 1 = 2,048, 2 = 1,536, 3 = 1,280 (default), 4 = 1,024 threads.
template <int K, bool G, int NT>
static void launch_cta(CliqueArgs a, int64_t blocks, cudaStream_t s) {
    switch (knobs().clique_occ) {
        case 1: launch_cta_mb<K, G, NT, 2048 / NT>(a, blocks, s); break;
        case 2: launch_cta_mb<K, G, NT, (1536 / NT > 0 ? 1536 / NT : 1)>(a, blocks, s); break;
        case 3: launch_cta_mb<K, G, NT, (1280 / NT > 0 ? 1280 / NT : 1)>(a, blocks, s); break;
        case 4: launch_cta_mb<K, G, NT, (1024 / NT > 0 ? 1024 / NT : 1)>(a, blocks, s); break;
        default: launch_cta_mb<K, G, NT, 1>(a, blocks, s); break;
    }
}

template <int K, bool G, int NT>
static int cta_occupancy(size_t smem) {
    switch (knobs().clique_occ) {
        case 1: return cta_occupancy_mb<K, G, NT, 2048 / NT>(smem);
        case 2: return cta_occupancy_mb<K, G, NT, (1536 / NT > 0 ? 1536 / NT : 1)>(smem);
        case 3: return cta_occupancy_mb<K, G, NT, (1280 / NT > 0 ? 1280 / NT : 1)>(smem);
        case 4: return cta_occupancy_mb<K, G, NT, (1024 / NT > 0 ? 1024 / NT : 1)>(smem);
        default: return cta_occupancy_mb<K, G, NT, 1>(smem);
    }
}

// bucket edges on |S(u)|: warp kernel up to kEdge[0]; CTA kernels up to each next edge
// (shared memory sized to the bucket's largest root); global slab beyond dsmem
constexpr int kNB = 8;  // 0 warp, 1-5 shared memory, 6 global slab, 7 handed back

__global__ void k_gather_roots(const int32_t* __restrict__ roots, const int32_t* __restrict__ idx, int64_t n,
                               int32_t* __restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = roots[idx[t]];
}

// largest |S(u)| the global-slab kernel takes: its cuckoo table and block table must fit
// shared memory, and 148 slabs must stay within ~4 GB (GSM_CLIQUE_DMAX lowers it: tests)
static int clique_dglob(int K) {
    int d = 1024;
    while (cta_smem(K, d + 256, true) <= kSmemLim &&
           (double)cta_lay(K, d + 256, true, true, true).slab_ints * 4.0 * 148 <= 4e9)
        d += 256;
    if (knobs().clique_dmax > 0) d = std::min(d, std::max(8, knobs().clique_dmax));
    return d;
}

template <int K>
static int64_t run_clique_k(CliqueRun& r, cudaStream_t s) {
    const int64_t R = r.R;
    const int dsmem = clique_dsmem(K);
    BucketEdges E;
    // K4: 960 keeps two 1,024-thread CTAs (2 x 105 KB) resident per SM
    const int dglob = clique_dglob(K);
    const int e[kNB - 1] = {warp_max(), 128, 256, 512, K == 4 ? 960 : 1024, dsmem, std::max(dsmem, dglob)};
    for (int b = 0; b < kNB - 1; ++b) E.e[b] = std::min(e[b], dglob);
    // a lowered shared-memory cap (GSM_CLIQUE_DSMEM, tests) also caps the smaller CTA buckets,
    // so roots above it reach the global-slab kernel
    for (int b = 1; b <= 4; ++b) E.e[b] = std::min(E.e[b], dsmem);
    Workspace& W_ = *r.ws;  // grow-only, kept with the graph (no pool round trips per call)
    DevBuf<int32_t>&keys = W_.ck_keys, &vals = W_.ck_vals, &keys2 = W_.ck_keys2, &vals2 = W_.ck_vals2,
                   &slab = W_.ck_slab;
    DevBuf<unsigned long long>&bucket = W_.ck_bucket, &sched = W_.ck_sched;
    DevBuf<int>& dmax = W_.ck_dmax;
    keys.ensure(R, s);
    vals.ensure(R, s);
    keys2.ensure(R, s);
    vals2.ensure(R, s);
    bucket.ensure(kNB, s);
    dmax.ensure(2, s);
    sched.ensure(kNB, s);
    GSM_CUDA(cudaMemsetAsync(bucket.p, 0, sizeof(unsigned long long) * kNB, s));
    GSM_CUDA(cudaMemsetAsync(dmax.p, 0, 2 * sizeof(int), s));
    GSM_CUDA(cudaMemsetAsync(sched.p, 0, sizeof(unsigned long long) * kNB, s));
    const int sms = sm_count();
    k_clique_keys<<<(unsigned)std::min<int64_t>((R + 255) / 256, (int64_t)sms * 8), 256, 0, s>>>(
        r.roots, R, r.nplus, K - 1, E, keys.p, vals.p, bucket.p, dmax.p);
    GSM_LAUNCH("k_clique_keys");
    unsigned long long hb[kNB];
    int hm[2] = {0, 0};
    GSM_CUDA(cudaMemcpyAsync(hb, bucket.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
    GSM_CUDA(cudaMemcpyAsync(hm, dmax.p, sizeof(hm), cudaMemcpyDeviceToHost, s));
    GSM_CUDA(cudaStreamSynchronize(s));
    const int hmax = hm[0];  // largest |S(u)| processed here; hm[1] = largest overall
    r.n_over = (int64_t)hb[kNB - 1];
    if (hm[1] == 0) return 1;
    int end_bit = 1;
    while (end_bit < 31 && (1 << end_bit) <= hm[1]) ++end_bit;
    size_t tb = 0;
    GSM_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, keys.p, keys2.p, vals.p, vals2.p, (int)R, 0,
                                                       end_bit, s));
    DevBuf<uint8_t>& tmp = W_.ck_tmp;
    tmp.ensure(tb, s);
    GSM_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tb, keys.p, keys2.p, vals.p, vals2.p, (int)R, 0,
                                                       end_bit, s));
    int64_t launches = 1 + 1 + (end_bit + 7) / 8;  // keys, sort (histogram + passes)
    CliqueArgs a;
    a.roots = r.roots;
    a.off = r.off;
    a.cols = r.cols;
    a.up = r.up;
    a.np = r.nplus;
    a.stream_max = stream_max();
    a.use_hash = use_hash();
    a.hub_bits = knobs().clique_hub ? r.hub_bits : nullptr;
    a.hub_base = r.hub_base;
    a.hub_words = r.hub_words;
    a.hub_ratio = knobs().clique_hub_ratio;
    a.nh_off = r.nh_off;
    a.nh_tab = r.nh_tab;
    a.nh_stream = knobs().clique_nh_stream;
    a.ranges = knobs().clique_ranges;
    a.lazy_ck = knobs().clique_lazy_ck;
    DevBuf<unsigned long long> cyc;
    a.cyc = nullptr;
    if (knobs().trace == 2) {
        cyc.ensure(8, s);
        GSM_CUDA(cudaMemsetAsync(cyc.p, 0, 8 * sizeof(unsigned long long), s));
        a.cyc = cyc.p;
    }
    a.slab = nullptr;
    a.slab_blocks = 0;
    a.count = r.count;
    a.stats = r.stats;
    // sorted descending: [bucket kNB-1 (handed back) | kNB-2 | ... | 0]
    int64_t pos = 0;
    if (r.n_over > 0) {
        k_gather_roots<<<(unsigned)std::min<int64_t>((r.n_over + 255) / 256, 1024), 256, 0, s>>>(
            r.roots, vals2.p, r.n_over, r.over_roots);
        GSM_LAUNCH("k_gather_roots");
        ++launches;
        pos = r.n_over;
    }
    for (int b = kNB - 2; b >= 0; --b) {
        const int64_t nb = (int64_t)hb[b];
        if (nb == 0) continue;
        a.idx = vals2.p + pos;
        a.n = nb;
        a.next = sched.p + b;
        a.slab = nullptr;
        pos += nb;
        a.dmax = std::min(E.e[b], hmax);
        ++launches;
        if (b == 0) {
            const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((nb + 7) / 8, (int64_t)sms * 8));
            k_clique_warp<K><<<(unsigned)grid, 256, 0, s>>>(a);
            GSM_LAUNCH("k_clique_warp");
        } else if (b == kNB - 2) {
            const int64_t blocks = std::min<int64_t>(nb, sms);
            const CtaLay L = cta_lay(K, a.dmax, true, a.use_hash != 0, a.ranges != 0);
            slab.ensure((size_t)blocks * L.slab_ints, s);
            a.slab = slab.p;
            a.slab_blocks = (int32_t)blocks;
            launch_cta<K, true, 1024>(a, blocks, s);
        } else {
            // CTA size with the most resident warps per SM for this bucket's shared memory and
            // the instantiation's registers (the runtime's occupancy calculator; ties -> smaller
            // CTAs: finer-grained root scheduling)
            const size_t sm = cta_smem(K, a.dmax, false);
            int best = 256, bestw = -1;
            for (int nt : {256, 512, 1024}) {
                const size_t per = sm + sizeof(int32_t) * 64 * (nt / 32) + 64 + 1024;  // + static + reserved
                const int ctas = !knobs().clique_ntsel ? std::min<int>(2048 / nt, (int)((228 * 1024) / per))
                               : nt == 256 ? cta_occupancy<K, false, 256>(sm)
                               : nt == 512 ? cta_occupancy<K, false, 512>(sm) : cta_occupancy<K, false, 1024>(sm);
                if (ctas * nt / 32 > bestw) {
                    bestw = ctas * nt / 32;
                    best = nt;
                }
            }
            if (best == 256) launch_cta<K, false, 256>(a, nb, s);
            else if (best == 512) launch_cta<K, false, 512>(a, nb, s);
            else launch_cta<K, false, 1024>(a, nb, s);
        }
    }
    if (a.cyc) {
        unsigned long long hc[8];
        GSM_CUDA(cudaMemcpyAsync(hc, a.cyc, sizeof(hc), cudaMemcpyDeviceToHost, s));
        GSM_CUDA(cudaStreamSynchronize(s));
        const double t = (double)(hc[0] + hc[1] + hc[2] + hc[3]) + 1e-9;
        std::fprintf(stderr, "[gsm clique K%d] k_clique_cta warp-cycles: setup %.1f%%  stream rows %.1f%%  search rows %.1f%%"
                     "  level 3 %.1f%%  (total %.3g)\n", K, 100 * hc[0] / t, 100 * hc[1] / t, 100 * hc[2] / t,
                     100 * hc[3] / t, t);
        std::fprintf(stderr, "[gsm clique K%d] k_clique_cta row keys/entries: hub bitmap %.3g  hashed N+ %.3g  "
                     "streamed %.3g  binary search %.3g\n", K, (double)hc[4], (double)hc[5], (double)hc[6],
                     (double)hc[7]);
    }
    return launches;
}

int64_t run_clique(CliqueRun& r, cudaStream_t s) {
    r.n_over = 0;
    if (r.R <= 0) return 0;
    return r.k == 3 ? run_clique_k<3>(r, s) : run_clique_k<4>(r, s);
}

}  // namespace gsm
