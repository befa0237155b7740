// push_list.cuh — list of nonzero xbar columns handed from the primal to the next dual (push_dual.cuh).
#pragma once
#include "common.cuh"

namespace gfors {

constexpr double PUSH_SCALE = 1099511627776.0;        // 2^40
constexpr double PUSH_INV = 1.0 / 1099511627776.0;

struct PushList {
    int* list[2];        // nonzero xbar columns written by the primal of parity p (buffer p^1)
    unsigned* count[2];  // list lengths (0xFFFFFFFF = unknown -> gather mode)
    unsigned thr;        // push mode iff count <= thr
    long long cap;       // list capacity (n)
    long long* acc;      // [m] int64 row accumulators, kept at 0 between uses
    unsigned* pp_rcount;            // push-primal row list length, reset by the dual (or null)
    unsigned long long* pp_wmax;    // push-primal max |w|, reset by the dual (or null)
};

// parity-selected members without dynamic indexing of the kernel-parameter arrays (which would
// copy the struct to local memory)
__device__ __forceinline__ unsigned* pl_count(const PushList& pl, int p) { return p ? pl.count[1] : pl.count[0]; }
__device__ __forceinline__ int* pl_list(const PushList& pl, int p) { return p ? pl.list[1] : pl.list[0]; }

// called by thread 0 of block 0 of whichever dual kernel is active this iteration
__device__ __forceinline__ void push_reset_next(const PushList& pl, int par) {
    *pl_count(pl, par ^ 1) = 0u;
    if (pl.pp_rcount) { *pl.pp_rcount = 0u; *pl.pp_wmax = 0ull; }
}

__device__ __forceinline__ bool push_mode(const PushList& pl, int par) {
    return pl.acc != nullptr && *(volatile unsigned*)pl_count(pl, par) <= pl.thr;
}

// block-staged append of the pass's nonzero columns (one global atomic per CTA pass); enabled is
// block-uniform.  s_list holds at most one entry per thread.
template <int NT>
__device__ __forceinline__ void push_append(const PushList& pl, int outpar, bool nz, int idx, bool enabled,
                                            unsigned* s_cnt, unsigned* s_base, int* s_list) {
    if (!enabled) return;
    if (threadIdx.x == 0) *s_cnt = 0u;
    __syncthreads();
    warp_append(nz, idx, s_cnt, s_list);
    __syncthreads();
    if (threadIdx.x == 0) *s_base = *s_cnt ? atomicAdd(pl_count(pl, outpar), *s_cnt) : 0u;
    __syncthreads();
    const unsigned c = *s_cnt, base = *s_base;
    for (unsigned t = threadIdx.x; t < c; t += NT)
        if ((long long)base + t < pl.cap) pl_list(pl, outpar)[base + t] = s_list[t];
    __syncthreads();
}

}  // namespace gfors
