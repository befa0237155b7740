// repair.cuh — repair step after the monotone relaxation (SURVEY
// §8(f) row f4; reading R26).
//
// Under the relaxation (Q = 0, c >= 0, K_u >= 0: the PDHG step treats every row as >=, the upper
// closure) sampled candidates are supersets; before EvalBest — which keeps the ORIGINAL rows —
// each lane is repaired: its 1-entries, in order of decreasing canonical cost (ties: lower index
// first), are dropped one by one while every row keeps sum_i K_ji x_i >= r_j.  One CTA per lane:
// the lane's entries are collected from the bit-sliced batch into shared memory, bitonic-sorted,
// the row sums built with shared atomics (exact integers), then one thread runs the sequential
// greedy (it is inherently ordered) over the column lists of K_u', and the dropped bits are
// cleared with atomicAnd.  Lanes with more than RP_CAP entries are left as they are (R26).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "pdhg.cuh"

namespace gfors {

constexpr int RP_CAP = 8192;   // entries per lane
constexpr int RP_NT = 512;

__host__ __device__ constexpr size_t rp_smem_bytes(long long m) {
    return (size_t)RP_CAP * (8 + 4) + (size_t)m * 4 + 64;
}

template <int KIND>
__global__ void __launch_bounds__(RP_NT) k_repair(long long n, long long m, Csr Kt, const double* __restrict__ c,
                                                   const double* __restrict__ r, uint64_t* __restrict__ X, int W) {
    extern __shared__ unsigned long long rp_sm[];
    double* key = reinterpret_cast<double*>(rp_sm);                 // [RP_CAP] cost
    int* idx = reinterpret_cast<int*>(key + RP_CAP);                // [RP_CAP] variable (<0: dropped)
    int* srow = idx + RP_CAP;                                       // [m] row sums
    __shared__ int s_cnt;
    const int l = blockIdx.x;
    const int w = l >> 6;
    const uint64_t bit = 1ull << (l & 63);
    if (threadIdx.x == 0) s_cnt = 0;
    for (long long j = threadIdx.x; j < m; j += blockDim.x) srow[j] = 0;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        if (__ldg(X + i * W + w) & bit) {
            const int t = atomicAdd(&s_cnt, 1);
            if (t < RP_CAP) { key[t] = __ldg(c + i); idx[t] = (int)i; }
        }
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (cnt > RP_CAP || cnt == 0) return;  // (block-uniform)
    int P = 1;
    while (P < cnt) P <<= 1;
    for (int t = cnt + threadIdx.x; t < P; t += blockDim.x) { key[t] = -1.0; idx[t] = 0x7fffffff; }  // sorts last
    __syncthreads();
    // bitonic sort: descending cost, ascending index
    for (int k = 2; k <= P; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int t = threadIdx.x; t < P; t += blockDim.x) {
                const int u = t ^ jj;
                if (u > t) {
                    const bool before = key[u] > key[t] || (key[u] == key[t] && idx[u] < idx[t]);  // u should precede t
                    const bool up = (t & k) == 0;
                    if (up ? before : !before) {
                        const double kk = key[t]; key[t] = key[u]; key[u] = kk;
                        const int ii = idx[t]; idx[t] = idx[u]; idx[u] = ii;
                    }
                }
            }
            __syncthreads();
        }
    }
    // row sums of the lane (exact integers)
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const int i = idx[t];
        for (long long q = __ldg(Kt.ptr + i); q < __ldg(Kt.ptr + i + 1); ++q)
            atomicAdd(&srow[__ldg(Kt.idx + q)], (int)kval<KIND>(Kt.val, q));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 0; t < cnt; ++t) {
            const int i = idx[t];
            const long long q0 = __ldg(Kt.ptr + i), q1 = __ldg(Kt.ptr + i + 1);
            bool ok = true;
            for (long long q = q0; q < q1 && ok; ++q) {
                const int row = __ldg(Kt.idx + q);
                ok = (double)(srow[row] - (int)kval<KIND>(Kt.val, q)) >= __ldg(r + row);
            }
            if (!ok) continue;
            for (long long q = q0; q < q1; ++q) srow[__ldg(Kt.idx + q)] -= (int)kval<KIND>(Kt.val, q);
            idx[t] = -1 - i;  // dropped
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const int v = idx[t];
        if (v < 0) atomicAnd(reinterpret_cast<unsigned long long*>(X + (long long)(-1 - v) * W + w), ~bit);
    }
}

}  // namespace gfors
