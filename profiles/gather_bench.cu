// gather_bench.cu — random-gather ceiling of B200 (DESIGN.md §6 "What bounds the PDHG kernels";
// VERDICT r1 asked for the source of the round-1 numbers to be committed).
//
// N random int32 indices into a vector of V elements; every kernel streams the indices (coalesced)
// and gathers one element per index.  Element = 4 bytes (x-bar of the PDHG dual, fp32), 8 bytes, or
// 16 bytes (two 64-candidate words of the sample batch X read by the feasibility kernel).  Variants:
//   reg  : U indices per thread loaded first, then U gathers into registers, summed (no cp.async);
//   cpa  : the k_dual_rb / k_feas_rb recipe — chunks of CH nonzeros per CTA, one cp.async per
//          gather into shared memory, double-buffered, consumed from shared memory.
// Timing: CUDA events around 10 launches after 3 warm-ups, min over 3 repeats.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bench gather_bench.cu
// Usage: ./gather_bench [N=50000000]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <string>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <int EB> struct Elem;
template <> struct Elem<4> { using T = float; };
template <> struct Elem<8> { using T = unsigned long long; };
template <> struct Elem<16> { using T = ulonglong2; };

__device__ __forceinline__ float val(float v) { return v; }
__device__ __forceinline__ float val(unsigned long long v) { return (float)(v & 1); }
__device__ __forceinline__ float val(ulonglong2 v) { return (float)((v.x ^ v.y) & 1); }

template <int EB, int U>
__global__ void __launch_bounds__(256) k_reg(const int* __restrict__ idx, long long n, const typename Elem<EB>::T* __restrict__ v,
                                             float* __restrict__ out) {
    using T = typename Elem<EB>::T;
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x * U;
    for (long long base = (blockIdx.x * (long long)blockDim.x) * U + threadIdx.x; base < n; base += stride) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const long long p = base + (long long)u * blockDim.x; c[u] = p < n ? __ldcs(idx + p) : -1; }
        T g[U];
#pragma unroll
        for (int u = 0; u < U; ++u) if (c[u] >= 0) g[u] = __ldg(v + c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) if (c[u] >= 0) acc += val(g[u]);
    }
    out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(256) k_stream(const int* __restrict__ idx, long long n, float* __restrict__ out) {
    int acc = 0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
        acc ^= __ldcs(idx + p);
    out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = (float)acc;
}

// L2-resident streaming read (the bound of the small configs 2-4, whose per-iteration working sets
// fit in L2): every thread sums float4 loads over a buffer of B bytes, REPS passes
__global__ void __launch_bounds__(256) k_l2read(const float4* __restrict__ a, long long n4, int reps, float* __restrict__ out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(a + i);
            acc += v.x + v.y + v.z + v.w;
        }
    out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = acc;
}

template <int EB>
__device__ __forceinline__ void cpa(void* s, const void* g) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(s);
    if constexpr (EB == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(g));
    else if constexpr (EB == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(g));
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(a), "l"(g));
}

template <int EB, int CH>
__global__ void __launch_bounds__(256) k_cpa(const int* __restrict__ idx, long long n, const typename Elem<EB>::T* __restrict__ v,
                                             float* __restrict__ out) {
    using T = typename Elem<EB>::T;
    constexpr int U = CH / 256;
    __shared__ __align__(16) T sv[2][CH];
    const long long nch = (n + CH - 1) / CH;
    float acc = 0.f;
    int st = 0;
    int c[U];
    auto load = [&](long long ch) {
#pragma unroll
        for (int u = 0; u < U; ++u) { const long long p = ch * CH + u * 256 + threadIdx.x; c[u] = (ch < nch && p < n) ? __ldcs(idx + p) : -1; }
    };
    auto issue = [&](T* s) {
#pragma unroll
        for (int u = 0; u < U; ++u) if (c[u] >= 0) cpa<EB>(s + u * 256 + threadIdx.x, v + c[u]);
        asm volatile("cp.async.commit_group;");
    };
    load(blockIdx.x);
    issue(sv[0]);
    load(blockIdx.x + gridDim.x);
    for (long long ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        issue(sv[st ^ 1]);
        load(ch + 2LL * gridDim.x);
        asm volatile("cp.async.wait_group 1;");
        __syncthreads();
#pragma unroll
        for (int u = 0; u < U; ++u) acc += val(sv[st][u * 256 + threadIdx.x]);  // (garbage past n is harmless)
        __syncthreads();
        st ^= 1;
    }
    asm volatile("cp.async.wait_all;");
    out[blockIdx.x * (long long)blockDim.x + threadIdx.x] = acc;
}

template <typename K>
static double time_ms(K launch) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
        for (int w = 0; w < 3; ++w) launch();
        CK(cudaEventRecord(a));
        for (int it = 0; it < 10; ++it) launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, (double)ms / 10);
    }
    CK(cudaGetLastError());
    return best;
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 50000000LL;
    int dev = 0, sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));  // kHz
    int* d_idx; float* d_out; void* d_v;
    CK(cudaMalloc(&d_idx, n * 4));
    CK(cudaMalloc(&d_out, 64LL << 20));
    CK(cudaMalloc(&d_v, 256LL << 20));
    CK(cudaMemset(d_v, 1, 256LL << 20));
    std::vector<int> h(n);
    printf("# gather_bench: N = %lld random int32 indices, %d SMs, %.0f MHz max clock\n", n, sms, clk / 1e3);
    printf("# %-5s %-10s %-12s %10s %12s %14s\n", "elem", "vector", "variant", "us", "Ggather/s", "gathers/cyc/SM");
    const double ghz = clk / 1e6;
    const long long grid = (long long)sms * 8;
    for (int eb : {4, 8, 16}) {
        for (long long vmb : {4LL, 20LL, 80LL, 160LL}) {
            const long long V = (vmb << 20) / eb;
            unsigned long long s = 88172645463325252ULL;
            for (long long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % (unsigned long long)V); }
            CK(cudaMemcpy(d_idx, h.data(), n * 4, cudaMemcpyHostToDevice));
            auto report = [&](const char* name, double ms) {
                const double gps = n / (ms * 1e-3) / 1e9;
                printf("  %-5d %-10s %-12s %10.1f %12.1f %14.3f\n", eb, (std::to_string(vmb) + " MB").c_str(), name, ms * 1e3, gps,
                       gps / (sms * ghz));
            };
#define REG(EB, U) report("reg U=" #U, time_ms([&] { k_reg<EB, U><<<grid, 256>>>(d_idx, n, (const Elem<EB>::T*)d_v, d_out); }))
#define CPA(EB, CH) report("cpa " #CH, time_ms([&] { k_cpa<EB, CH><<<grid, 256>>>(d_idx, n, (const Elem<EB>::T*)d_v, d_out); }))
            if (eb == 4) { REG(4, 1); REG(4, 8); CPA(4, 1024); CPA(4, 2048); }
            if (eb == 8) { REG(8, 1); REG(8, 4); CPA(8, 1024); }
            if (eb == 16) { REG(16, 1); REG(16, 4); CPA(16, 512); CPA(16, 1024); }
        }
    }
    // L2-resident streaming read bandwidth (buffers well inside the 126 MB L2)
    for (long long mb : {8LL, 16LL, 32LL, 48LL}) {
        const long long n4 = (mb << 20) / 16;
        const int reps = 20;
        const double ms = time_ms([&] { k_l2read<<<grid, 256>>>((const float4*)d_v, n4, reps, d_out); });
        printf("  L2 read %lld MB x %d: %.1f us = %.2f TB/s\n", mb, reps, ms * 1e3, (double)reps * (mb << 20) / (ms * 1e-3) / 1e12);
    }
    // the index stream alone (no gathers)
    {
        const double ms = time_ms([&] { k_stream<<<grid, 256>>>(d_idx, n, d_out); });
        printf("  index stream alone: %.1f us = %.2f TB/s\n", ms * 1e3, n * 4.0 / (ms * 1e-3) / 1e12);
    }
    return 0;
}
