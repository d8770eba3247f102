// gsm_merge.cu — merge of two lexicographically sorted row blocks (SURVEY §8(a) row A9 /
// §8(e): the P-way merge of the locally pre-sorted ENUMERATE shards of P GPUs, done as a
// tree of pairwise merges instead of a re-sort of the concatenation).
//
// Merge path: output position p = diagonal p of the (na x nb) merge grid; each thread owns
// kPer consecutive outputs, finds where its diagonal crosses the merge path by a binary
// search over row comparisons, then merges its kPer rows sequentially.  Ties take `a`
// first (stable).  Rows compare as unsigned int32 tuples, the order gsm_sort_rows produces.
#include "gsm_common.h"
#include "gsm.h"

namespace gsm {

namespace {

constexpr int kPer = 8;

// row a_i < row b_j (unsigned lexicographic)
__device__ __forceinline__ bool row_less(const int32_t* __restrict__ x, const int32_t* __restrict__ y, int w) {
    for (int c = 0; c < w; ++c) {
        const uint32_t u = (uint32_t)__ldg(x + c), v = (uint32_t)__ldg(y + c);
        if (u != v) return u < v;
    }
    return false;
}

__global__ void k_merge_rows(const int32_t* __restrict__ a, int64_t na, const int32_t* __restrict__ b, int64_t nb,
                             int w, int32_t* __restrict__ out) {
    const int64_t n = na + nb;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t * kPer < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t diag = t * kPer;
        // i = number of a-rows among the first diag outputs: the smallest i in [lo, hi] with
        // NOT (b[diag - i - 1] < a[i])  ... i.e. a[i] is taken after b[diag-i-1] only if b < a
        int64_t lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
        while (lo < hi) {
            const int64_t i = (lo + hi) >> 1;
            // a[i] goes before b[diag - i - 1] unless b[diag-i-1] < a[i] (ties: a first)
            if (row_less(b + (diag - i - 1) * w, a + i * w, w)) hi = i;
            else lo = i + 1;
        }
        int64_t i = lo, j = diag - lo;
        const int64_t end = diag + kPer < n ? diag + kPer : n;
        GSM_DCHECK(i >= 0 && i <= na && j >= 0 && j <= nb, DCHK_MERGE);
        for (int64_t p = diag; p < end; ++p) {
            const bool take_a = j >= nb || (i < na && !row_less(b + j * w, a + i * w, w));
            const int32_t* src = take_a ? a + i * w : b + j * w;
            for (int c = 0; c < w; ++c) out[p * w + c] = __ldg(src + c);
            if (take_a) ++i; else ++j;
        }
    }
}

}  // namespace

void merge_rows(const int32_t* a, int64_t na, const int32_t* b, int64_t nb, int w, int32_t* out, cudaStream_t s) {
    const int64_t n = na + nb;
    if (n == 0) return;
    const int64_t threads = (n + kPer - 1) / kPer;
    int dev = 0, sms = 148;
    GSM_CUDA(cudaGetDevice(&dev));
    GSM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t grid = std::min<int64_t>((threads + 255) / 256, (int64_t)sms * 16);
    k_merge_rows<<<(unsigned)grid, 256, 0, s>>>(a, na, b, nb, w, out);
    GSM_LAUNCH("k_merge_rows");
}

}  // namespace gsm

gsm_status gsm_merge_rows(const int32_t* a, uint64_t na, const int32_t* b, uint64_t nb, int32_t width, int32_t* out,
                          int32_t device, void* stream) {
    if (na + nb == 0) return GSM_OK;
    if ((na && !a) || (nb && !b) || !out || width < 1 || width > GSM_MAX_QUERY_NODES) {
        gsm::set_error("bad arguments to gsm_merge_rows");
        return GSM_ERR_INVALID_ARGUMENT;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    try {
        gsm::clear_error();
        GSM_CUDA(cudaSetDevice(device));
        cudaStream_t s = (cudaStream_t)stream;
        gsm::merge_rows(a, (int64_t)na, b, (int64_t)nb, width, out, s);
        GSM_CUDA(cudaStreamSynchronize(s));
#ifdef GSM_DEVICE_CHECKS
        if (gsm::dcheck_collect()) gsm::fail(GSM_ERR_CUDA, "device check failed in gsm_merge_rows");
#endif
        cudaSetDevice(prev);
        return GSM_OK;
    } catch (const gsm::Failure& f) {
        cudaSetDevice(prev);
        gsm::set_error(f.msg);
        return f.status;
    } catch (...) {
        cudaSetDevice(prev);
        gsm::set_error("unexpected exception in gsm_merge_rows");
        return GSM_ERR_CUDA;
    }
}
