// cover.cuh — cover completion of sampled candidates (customised RandSampleStep for covering rows;
// PAPER §2.4.2: "first generate a feasible candidate from the fractional solution p";
// DESIGN.md reading R27).
//
// A covering row (canonical >= row, every coefficient 1, right-hand side 1: set cover) that a lane
// violates gets the row's variable with the largest p = x_k (ties: lowest index) switched on in that
// lane.  Every decision is taken on the batch as sampled (phase 1 writes, per eligible row, its best
// variable and the lanes that violate it; phase 2 ORs them in), so the result — the union of the
// additions — is independent of the order of the rows and of the atomics.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "pdhg.cuh"

namespace gfors {

// phase 1: SUB lanes per eligible row (rows of set cover have 2..98 entries)
template <typename T, int SUB>
__global__ void __launch_bounds__(256) k_cover_scan(Csr K, const int* __restrict__ rows, long long nrows,
                                                    const T* __restrict__ xa, const T* __restrict__ xb2,
                                                    const double* __restrict__ pfix, const Ctrl* __restrict__ ctrl,
                                                    long long kint, const uint64_t* __restrict__ X, int W,
                                                    int* __restrict__ best, uint64_t* __restrict__ viol,
                                                    const unsigned char* __restrict__ ones) {
    const T* __restrict__ p = nullptr;
    if (!pfix) {
        const long long b = ctrl->blk;
        p = (((b + 1) * kint) & 1) ? xb2 : xa;  // x_k of the block (as k_sample)
    }
    constexpr int RPW = 32 / SUB;
    const int lane = threadIdx.x & (SUB - 1);
    const int gsub = (threadIdx.x & 31) / SUB;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long base = warp * RPW; base < nrows; base += nwarps * RPW) {  // warp-uniform trip count
        const long long e = base + gsub;
        const bool valid = e < nrows;
        long long q0 = 0, q1 = 0;
        if (valid) {
            const int row = rows[e];
            q0 = __ldg(K.ptr + row); q1 = __ldg(K.ptr + row + 1);
            // a variable with p = 1 (counted by the block's trigger pass) covers the row in every
            // lane: nothing violated, no gathers (same result)
            if (ones && ones[row] >= 1) { q1 = q0; }
        }
        const bool covered_all = valid && ones && q1 == q0 && ones[rows[e]] >= 1;
        double bp = -1.0;
        int bi = 0x7fffffff;
        for (int w0 = 0; w0 < W; w0 += 4) {
            uint64_t o[4] = {0ull, 0ull, 0ull, 0ull};
            for (long long q = q0 + lane; q < q1; q += SUB) {
                const int i = __ldg(K.idx + q);
                if (w0 == 0) {
                    const double pv = pfix ? pfix[i] : (double)p[i];
                    if (pv > bp || (pv == bp && i < bi)) { bp = pv; bi = i; }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (w0 + u < W) o[u] |= __ldg(X + (long long)i * W + w0 + u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
#pragma unroll
                for (int off = SUB / 2; off > 0; off >>= 1) o[u] |= __shfl_xor_sync(0xffffffffu, o[u], off, SUB);
                if (lane == 0 && valid && w0 + u < W) viol[e * W + w0 + u] = covered_all ? 0ull : ~o[u];
            }
        }
#pragma unroll
        for (int off = SUB / 2; off > 0; off >>= 1) {
            const double op = __shfl_xor_sync(0xffffffffu, bp, off, SUB);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off, SUB);
            if (op > bp || (op == bp && oi < bi)) { bp = op; bi = oi; }
        }
        if (lane == 0 && valid) best[e] = q1 > q0 ? bi : -1;
    }
}

// phase 2: OR the additions in (the last word keeps only the lanes of the batch)
__global__ void __launch_bounds__(256) k_cover_apply(long long nrows, const int* __restrict__ best,
                                                     const uint64_t* __restrict__ viol, int W, uint64_t last_mask,
                                                     uint64_t* __restrict__ X) {
    const long long total = nrows * W;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += gridDim.x * (long long)blockDim.x) {
        const long long e = t / W;
        const int w = (int)(t - e * W);
        uint64_t v = viol[t];
        if (w == W - 1) v &= last_mask;
        const int b = best[e];
        if (v && b >= 0) atomicOr(reinterpret_cast<unsigned long long*>(X + (long long)b * W + w), (unsigned long long)v);
    }
}

}  // namespace gfors
