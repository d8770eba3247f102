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
    uint32_t max_label = 0;
    int32_t* new2old = nullptr;   // n
    int32_t* old2new = nullptr;   // n
    int32_t max_degree = 0;
};

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
