// assign3d.cuh — customised RandSampleStep for 3D assignment (PAPER Alg. 4; SPEC
// L342-350; reading R25).
//
// Variables are the n^3 triples (i,j,k) at flat index i*n^2 + j*n + k.  Per sampling round:
//   (1) the K = ceil(gamma n) largest p = x_k (ties: lower flat index): one stable 64-bit radix
//       sort of (~bits(p), index) over the n^3 entries (CUB, captured in the loop graph);
//   (2) greedy partial non-conflict assignment over those K triples (one warp, sequential order);
//   (3) per candidate lane: Fisher-Yates shuffles of the unused j's and k's (Philox draws of the
//       lane, R25 counter layout) assign them to the unused i's (ascending);
//   (4) L pairwise interchanges (swap the j or k of two triples iff the cost sum strictly drops).
// One thread per candidate lane keeps its two permutations in shared memory (uint16); lanes are
// independent, so the batch is as parallel as k_b.  Output: the bit-sliced batch X (cleared
// first), one bit per (triple of the lane) — every lane is a feasible 3D assignment by
// construction.  The arithmetic (integer draws, two-term cost sums compared with <) is the
// oracle's exactly, so the batch is bit-identical to oracle/orc_sample_assign3d.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace gfors {

constexpr uint32_t A3_TAG_J = 0xA3D00001u, A3_TAG_K = 0xA3D00002u, A3_TAG_L = 0xA3D00003u;

// sort keys: ascending order of ~bits(p) = descending p; (+0 for -0 so equal values tie)
template <typename T>
__global__ void __launch_bounds__(256) k_a3_keys(const T* __restrict__ xa, const T* __restrict__ xb2,
                                                 const double* __restrict__ pfix, long long N,
                                                 const Ctrl* __restrict__ ctrl, long long kint, int use_fixed,
                                                 unsigned long long* __restrict__ keys, int* __restrict__ vals) {
    const T* __restrict__ p = nullptr;
    if (!use_fixed) {
        const long long b = ctrl->blk;
        p = (((b + 1) * kint) & 1) ? xb2 : xa;  // x_k of the block (as k_sample)
    }
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < N; v += gridDim.x * (long long)blockDim.x) {
        const double pv = (pfix ? pfix[v] : (double)p[v]) + 0.0;
        keys[v] = ~(unsigned long long)__double_as_longlong(pv);
        vals[v] = (int)v;
    }
}

// (2) greedy partial assignment in descending-p order; then the unused i / j / k lists (ascending).
// meta[0] = r (number of unused i's).  One warp; lane 0 runs the sequential greedy.
__global__ void __launch_bounds__(32) k_a3_greedy(const int* __restrict__ order, long long K, int n,
                                                  short* __restrict__ sj0, short* __restrict__ sk0,
                                                  short* __restrict__ Ri, short* __restrict__ Rj, short* __restrict__ Rk,
                                                  int* __restrict__ meta, unsigned char* __restrict__ used) {
    unsigned char* uj = used;
    unsigned char* uk = used + n;
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) { sj0[i] = -1; sk0[i] = -1; uj[i] = 0; uk[i] = 0; }
        const long long nn = (long long)n * n;
        for (long long t = 0; t < K; ++t) {
            const long long v = order[t];
            const int i = (int)(v / nn), j = (int)((v / n) % n), k = (int)(v % n);
            if (sj0[i] < 0 && !uj[j] && !uk[k]) { sj0[i] = (short)j; sk0[i] = (short)k; uj[j] = 1; uk[k] = 1; }
        }
        int r = 0, rj = 0, rk = 0;
        for (int i = 0; i < n; ++i) if (sj0[i] < 0) Ri[r++] = (short)i;
        for (int j = 0; j < n; ++j) if (!uj[j]) Rj[rj++] = (short)j;
        for (int k = 0; k < n; ++k) if (!uk[k]) Rk[rk++] = (short)k;
        meta[0] = r;
    }
}

__device__ __forceinline__ uint4 a3_draw(uint32_t lane, uint32_t round, uint32_t step, uint32_t tag, uint2 key) {
    return philox4x32_10(make_uint4(lane, round, step, tag), key);
}

// (3) + (4) per lane; shared memory per thread: pj, pk (r <= n), sj, sk (n) as uint16 -> 8 n bytes
__global__ void k_a3_sample(int n, const short* __restrict__ sj0, const short* __restrict__ sk0,
                            const short* __restrict__ Ri, const short* __restrict__ Rj, const short* __restrict__ Rk,
                            const int* __restrict__ meta, const double* __restrict__ cost, uint2 key,
                            const Ctrl* __restrict__ ctrl, int r_idx, int kr, unsigned round_fixed, int use_fixed,
                            long long word_off, int W, long long L, uint64_t* __restrict__ X) {
    extern __shared__ short a3_sm[];
    const int lanes = 64 * W;
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    short* pj = a3_sm + (size_t)threadIdx.x * 4 * n;
    short* pk = pj + n;
    short* sj = pk + n;
    short* sk = sj + n;
    if (l >= lanes) return;
    const unsigned round = use_fixed ? round_fixed : (unsigned)(ctrl->blk * kr + r_idx);
    const uint32_t lg = (uint32_t)(64 * word_off + l);
    const int r = meta[0];
    for (int t = 0; t < r; ++t) { pj[t] = Rj[t]; pk[t] = Rk[t]; }
    for (int t = r - 1; t >= 1; --t) {
        const uint32_t uj = a3_draw(lg, round, (uint32_t)t, A3_TAG_J, key).x;
        int q = (int)(((unsigned long long)uj * (unsigned long long)(t + 1)) >> 32);
        short tmp = pj[t]; pj[t] = pj[q]; pj[q] = tmp;
        const uint32_t uk = a3_draw(lg, round, (uint32_t)t, A3_TAG_K, key).x;
        q = (int)(((unsigned long long)uk * (unsigned long long)(t + 1)) >> 32);
        tmp = pk[t]; pk[t] = pk[q]; pk[q] = tmp;
    }
    for (int i = 0; i < n; ++i) { sj[i] = sj0[i]; sk[i] = sk0[i]; }
    for (int t = 0; t < r; ++t) { sj[Ri[t]] = pj[t]; sk[Ri[t]] = pk[t]; }
    const long long nn = (long long)n * n;
    for (long long st = 0; st < L && n >= 2; ++st) {
        const uint4 o = a3_draw(lg, round, (uint32_t)st, A3_TAG_L, key);
        const int a = (int)(((unsigned long long)o.x * (unsigned long long)n) >> 32);
        int b = (int)(((unsigned long long)o.y * (unsigned long long)(n - 1)) >> 32);
        if (b >= a) b += 1;
        const int ja = sj[a], jb = sj[b], ka = sk[a], kb = sk[b];
        const double c_a = __ldg(cost + a * nn + (long long)ja * n + ka), c_b = __ldg(cost + b * nn + (long long)jb * n + kb);
        if ((o.z & 1u) == 0u) {
            const double n_a = __ldg(cost + a * nn + (long long)jb * n + ka), n_b = __ldg(cost + b * nn + (long long)ja * n + kb);
            if (__dadd_rn(n_a, n_b) < __dadd_rn(c_a, c_b)) { sj[a] = (short)jb; sj[b] = (short)ja; }
        } else {
            const double n_a = __ldg(cost + a * nn + (long long)ja * n + kb), n_b = __ldg(cost + b * nn + (long long)jb * n + ka);
            if (__dadd_rn(n_a, n_b) < __dadd_rn(c_a, c_b)) { sk[a] = (short)kb; sk[b] = (short)ka; }
        }
    }
    const unsigned long long bit = 1ull << (l & 63);
    for (int i = 0; i < n; ++i) {
        const long long v = i * nn + (long long)sj[i] * n + sk[i];
        atomicOr(reinterpret_cast<unsigned long long*>(X + v * W + (l >> 6)), bit);
    }
}

}  // namespace gfors
