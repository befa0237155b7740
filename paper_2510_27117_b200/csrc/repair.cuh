// repair.cuh — repair step after the monotone relaxation (SURVEY
// §8(f) row f4; reading R26).
//
// Under the relaxation (Q = 0, c >= 0, K_u >= 0: the PDHG step treats every row as >=, the upper
// closure) sampled candidates are supersets; before EvalBest — which keeps the ORIGINAL rows —
// each lane is repaired: its 1-entries, in order of decreasing canonical cost (ties: lower index
// first), are dropped one by one while every row keeps sum_i K_ji x_i >= r_j.
//
// The drop order is the same for every lane, so it is computed once per load (`rank[i]` = position
// of variable i in the (cost desc, index asc) order, `order[t]` its inverse; host-built, see
// build_repair_order) and no lane sorts costs.  One CTA per lane:
//   1. a coalesced pass over the variables builds the lane's row sums (exact int64; shared memory
//      when m <= RP_SROWS, else a per-lane slice of global scratch) and collects the ranks of the
//      lane's 1-entries;
//   2a. <= RP_CAP entries: the ranks are bitonic-sorted in shared memory (unique int keys);
//   2b. more entries (any count, up to n): the order is scanned in chunks of RP_CHUNK ranks and each
//      chunk's 1-entries are compacted in order with a block scan;
//   3. warp 0 runs the (inherently sequential) greedy over the ordered entries — one candidate at a
//      time, its column entries checked by the lanes in parallel (ballot), column pointers of the
//      next 32 candidates prefetched one per lane — and the dropped bits are cleared with atomicAnd
//      (other CTAs own the other bits of the same words; no CTA reads another lane's bit).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "pdhg.cuh"

namespace gfors {

constexpr int RP_NT = 512;
constexpr int RP_CAP = 16384;     // entries per lane sorted in shared memory (else the ordered scan)
constexpr int RP_CHUNK = RP_NT * 8;  // ranks per chunk of the ordered scan (RP_CHUNK <= RP_CAP)
constexpr int RP_SROWS = 12288;   // row sums in shared memory up to this many rows

__host__ __device__ constexpr size_t rp_smem_bytes(long long m) {
    return (size_t)RP_CAP * 4 + (m <= RP_SROWS ? (size_t)m * 8 : 0) + 64;
}

// greedy drop over ent[0..cnt) (ranks, ascending = drop order); warp 0 only.  Dropped entries are
// marked by setting ent[t] = -1 - ent[t].
template <int KIND>
__device__ void rp_greedy_warp(int* ent, int cnt, const int* __restrict__ order, const Csr& Kt,
                               const double* __restrict__ r, long long* srow) {
    const int lane = threadIdx.x & 31;
    for (int base = 0; base < cnt; base += 32) {
        long long q0 = 0, q1 = 0;
        if (base + lane < cnt) {
            const int i = __ldg(order + ent[base + lane]);
            q0 = __ldg(Kt.ptr + i);
            q1 = __ldg(Kt.ptr + i + 1);
        }
        const int nb = min(32, cnt - base);
        for (int t = 0; t < nb; ++t) {
            const long long a = __shfl_sync(0xffffffffu, q0, t), b = __shfl_sync(0xffffffffu, q1, t);
            bool ok = true;
            for (long long q = a; q < b; q += 32) {  // column entries checked 32 at a time
                bool okq = true;
                if (q + lane < b) {
                    const int row = __ldg(Kt.idx + q + lane);
                    const long long v = (long long)kval<KIND>(Kt.val, q + lane);
                    okq = (double)(srow[row] - v) >= __ldg(r + row);
                }
                ok = __all_sync(0xffffffffu, okq) && ok;
            }
            if (!ok) continue;
            for (long long q = a + lane; q < b; q += 32) {
                const int row = __ldg(Kt.idx + q);
                srow[row] -= (long long)kval<KIND>(Kt.val, q);  // distinct rows per column: no race
            }
            __syncwarp();
            if (lane == 0) ent[base + t] = -1 - ent[base + t];
        }
    }
}

template <int KIND>
__global__ void __launch_bounds__(RP_NT) k_repair(long long n, long long m, Csr Kt, const int* __restrict__ rank,
                                                   const int* __restrict__ order, const double* __restrict__ r,
                                                   uint64_t* X, int W, long long* __restrict__ srow_g) {
    extern __shared__ unsigned long long rp_sm[];
    int* ent = reinterpret_cast<int*>(rp_sm);  // [RP_CAP] ranks of the lane's entries
    long long* srow = (m <= RP_SROWS) ? reinterpret_cast<long long*>(ent + RP_CAP)
                                      : srow_g + (long long)blockIdx.x * m;
    __shared__ int s_cnt, s_warp[RP_NT / 32];
    const int l = blockIdx.x;
    const int w = l >> 6;
    const uint64_t bit = 1ull << (l & 63);
    if (threadIdx.x == 0) s_cnt = 0;
    for (long long j = threadIdx.x; j < m; j += blockDim.x) srow[j] = 0;
    __syncthreads();
    // 1. row sums and the ranks of the lane's entries
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        if (X[i * W + w] & bit) {
            for (long long q = __ldg(Kt.ptr + i); q < __ldg(Kt.ptr + i + 1); ++q)
                atomicAdd(reinterpret_cast<unsigned long long*>(&srow[__ldg(Kt.idx + q)]),
                          (unsigned long long)(long long)kval<KIND>(Kt.val, q));
            const int t = atomicAdd(&s_cnt, 1);
            if (t < RP_CAP) ent[t] = __ldg(rank + i);
        }
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (cnt == 0) return;  // (block-uniform)
    if (cnt <= RP_CAP) {
        // 2a. bitonic sort of the ranks (unique keys, ascending)
        int P = 1;
        while (P < cnt) P <<= 1;
        for (int t = cnt + threadIdx.x; t < P; t += blockDim.x) ent[t] = 0x7fffffff;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1) {
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                for (int t = threadIdx.x; t < P; t += blockDim.x) {
                    const int u = t ^ jj;
                    if (u > t) {
                        const int a = ent[t], b = ent[u];
                        if (((t & k) == 0) ? (a > b) : (a < b)) { ent[t] = b; ent[u] = a; }
                    }
                }
                __syncthreads();
            }
        }
        if (threadIdx.x < 32) rp_greedy_warp<KIND>(ent, cnt, order, Kt, r, srow);
        __syncthreads();
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
            const int v = ent[t];
            if (v < 0) atomicAnd(reinterpret_cast<unsigned long long*>(X + (long long)__ldg(order + (-1 - v)) * W + w), ~bit);
        }
        return;
    }
    // 2b. ordered scan: chunks of RP_CHUNK ranks, each chunk's entries compacted in rank order
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    for (long long base = 0; base < n; base += RP_CHUNK) {
        unsigned f = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const long long t = base + tid * 8 + e;
            if (t < n && (X[(long long)__ldg(order + t) * W + w] & bit)) f |= 1u << e;
        }
        const int c = __popc(f);
        int incl = c;  // block-wide inclusive scan of the per-thread counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        if (tid < 32) {
            int v = tid < RP_NT / 32 ? s_warp[tid] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += u;
            }
            if (tid < RP_NT / 32) s_warp[tid] = v;  // inclusive warp totals
        }
        __syncthreads();
        int off = (wid ? s_warp[wid - 1] : 0) + incl - c;
        const int ccnt = s_warp[RP_NT / 32 - 1];
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (f >> e & 1u) ent[off++] = (int)(base + tid * 8 + e);
        __syncthreads();
        if (tid < 32) rp_greedy_warp<KIND>(ent, ccnt, order, Kt, r, srow);
        __syncthreads();
        for (int t = tid; t < ccnt; t += blockDim.x) {
            const int v = ent[t];
            if (v < 0) atomicAnd(reinterpret_cast<unsigned long long*>(X + (long long)__ldg(order + (-1 - v)) * W + w), ~bit);
        }
        __syncthreads();
    }
}

}  // namespace gfors
