// Random-gather ceiling (SURVEY §8(d) "a measured random-gather ceiling: a microbenchmark of
// random 4 B loads over an array >> L2, giving effective sectors/s — the honest irregular
// roofline").  Not part of the product; a measurement tool.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/gather_ceiling tools/gather_ceiling.cu
//   gpurun_out/gather_ceiling [GiB]
//
// Kernels (4 B int32 array of N elements, N*4 >> 126 MB L2):
//   independent : every thread issues U independent random 4 B loads per iteration
//                 (counter-hashed indices, no dependence) — the sector-rate ceiling;
//   dependent   : every thread walks a chain idx = hash(a[idx]) — one load in flight per thread
//                 (the latency-bound shape of a binary-search probe sequence);
//   stream      : coalesced 16 B loads (the copy-style bandwidth, for comparison).
// Reported per kernel: useful bytes/s (4 B per load), sector bytes/s (32 B per load) and loads/s.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return (uint32_t)x;
}

__global__ void k_init(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)mix((uint64_t)i * 7919u);
}

template <int U>
__global__ void k_independent(const int32_t* __restrict__ a, int64_t n, int iters, unsigned long long* sink) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        int32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t idx = ((uint64_t)mix(t * 1315423911ULL + (uint64_t)it * U + u) * (uint64_t)n) >> 32;
            v[u] = __ldg(a + idx);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += (uint32_t)v[u];
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_dependent(const int32_t* __restrict__ a, int64_t n, int iters, unsigned long long* sink) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t idx = ((uint64_t)mix(t) * (uint64_t)n) >> 32;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        const uint32_t v = (uint32_t)__ldg(a + idx);
        acc += v;
        idx = ((uint64_t)mix(v ^ (t << 20) ^ it) * (uint64_t)n) >> 32;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_stream(const int4* __restrict__ a, int64_t n4, unsigned long long* sink) {
    uint32_t acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 v = __ldg(a + i);
        acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
    const double gib = argc > 1 ? std::atof(argv[1]) : 4.0;
    const int64_t n = (int64_t)(gib * (1 << 30) / 4);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int32_t* a;
    unsigned long long* sink;
    CK(cudaMalloc(&a, n * 4));
    CK(cudaMalloc(&sink, 8));
    k_init<<<sms * 16, 256>>>(a, n);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch, double loads, const char* name, double bytes_per_load) {
        launch();  // warm-up
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        const double s = best / 1e3;
        std::printf("{\"kernel\": \"%s\", \"array_gib\": %.2f, \"ms\": %.3f, \"loads_per_s\": %.4g, "
                    "\"useful_GBps\": %.1f, \"sector_GBps\": %.1f}\n",
                    name, gib, best, loads / s, loads * bytes_per_load / s / 1e9, loads * 32.0 / s / 1e9);
    };
    const int threads = 256;
    for (int occ : {8, 32}) {  // resident CTAs per SM x 256 threads
        const int blocks = sms * occ;
        const int iters = 256;
        char nm[64];
        std::snprintf(nm, sizeof(nm), "independent_u4_ctas%d", occ);
        timeit([&] { k_independent<4><<<blocks, threads>>>(a, n, iters, sink); }, (double)blocks * threads * iters * 4, nm, 4.0);
        std::snprintf(nm, sizeof(nm), "independent_u1_ctas%d", occ);
        timeit([&] { k_independent<1><<<blocks, threads>>>(a, n, iters, sink); }, (double)blocks * threads * iters, nm, 4.0);
        std::snprintf(nm, sizeof(nm), "dependent_ctas%d", occ);
        timeit([&] { k_dependent<<<blocks, threads>>>(a, n, iters, sink); }, (double)blocks * threads * iters, nm, 4.0);
    }
    timeit([&] { k_stream<<<sms * 16, 512>>>((const int4*)a, n / 4, sink); }, (double)n / 4, "stream_16B", 16.0);
    CK(cudaFree(a));
    return 0;
}
