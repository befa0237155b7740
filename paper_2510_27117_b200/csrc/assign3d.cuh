// assign3d.cuh — customised RandSampleStep for 3D assignment (PAPER Alg. 4; SPEC
// L342-350; reading R25).
//
// Variables are the n^3 triples (i,j,k) at flat index i*n^2 + j*n + k.  Per sampling round:
//   (1) the K = ceil(gamma n) largest p = x_k (ties: lower flat index): one stable 64-bit radix
//       sort of (~bits(p), index) over the n^3 entries (CUB, captured in the loop graph);
//   (2) greedy partial non-conflict assignment over those K triples (sequential, from shared memory);
//   (3) per candidate lane: Fisher-Yates shuffles of the unused j's and k's (Philox draws of the
//       lane, R25 counter layout) assign them to the unused i's (ascending);
//   (4) L pairwise interchanges (swap the j or k of two triples iff the cost sum strictly drops).
// One warp per candidate lane: its random draws are made in parallel, the sequential swaps run on
// uint16 permutations in shared memory; lanes are independent.  Output: the bit-sliced batch X (cleared
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
        if (sizeof(T) == 4 && !pfix) {
            // fp32 x_k: the 32-bit key ~bits(float) orders exactly as the fp64 one (a float converts to
            // double exactly and monotonically), so the sort needs half the radix passes (end_bit 32)
            keys[v] = (unsigned long long)(~__float_as_uint((float)p[v] + 0.0f));
        } else {
            const double pv = (pfix ? pfix[v] : (double)p[v]) + 0.0;
            keys[v] = ~(unsigned long long)__double_as_longlong(pv);
        }
        vals[v] = (int)v;
    }
}

// (2) greedy partial assignment in descending-p order; then the unused i / j / k lists (ascending).
// meta[0] = r (number of unused i's).  The order is staged through shared memory in chunks by the
// whole block; thread 0 runs the (inherently sequential) greedy from shared memory.
constexpr int A3_GNT = 512, A3_GCHUNK = 4096;
__global__ void __launch_bounds__(A3_GNT) k_a3_greedy(const int* __restrict__ order, long long K, int n,
                                                      short* __restrict__ sj0, short* __restrict__ sk0,
                                                      short* __restrict__ Ri, short* __restrict__ Rj, short* __restrict__ Rk,
                                                      int* __restrict__ meta) {
    extern __shared__ int a3g_sm[];
    int* chunk = a3g_sm;                                         // [A3_GCHUNK]
    short* s_sj = reinterpret_cast<short*>(chunk + A3_GCHUNK);   // [n]
    short* s_sk = s_sj + n;                                      // [n]
    unsigned char* uj = reinterpret_cast<unsigned char*>(s_sk + n);
    unsigned char* uk = uj + n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { s_sj[i] = -1; s_sk[i] = -1; uj[i] = 0; uk[i] = 0; }
    const long long nn = (long long)n * n;
    for (long long c0 = 0; c0 < K; c0 += A3_GCHUNK) {
        const int len = (int)min((long long)A3_GCHUNK, K - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < len; t += blockDim.x) chunk[t] = __ldg(order + c0 + t);
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int t = 0; t < len; ++t) {
                const long long v = chunk[t];
                const int i = (int)(v / nn), j = (int)((v / n) % n), k = (int)(v % n);
                if (s_sj[i] < 0 && !uj[j] && !uk[k]) { s_sj[i] = (short)j; s_sk[i] = (short)k; uj[j] = 1; uk[k] = 1; }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) { sj0[i] = s_sj[i]; sk0[i] = s_sk[i]; }
    if (threadIdx.x == 0) {
        int r = 0, rj = 0, rk = 0;
        for (int i = 0; i < n; ++i) if (s_sj[i] < 0) Ri[r++] = (short)i;
        for (int j = 0; j < n; ++j) if (!uj[j]) Rj[rj++] = (short)j;
        for (int k = 0; k < n; ++k) if (!uk[k]) Rk[rk++] = (short)k;
        meta[0] = r;
    }
}
__host__ __device__ constexpr size_t a3_greedy_smem(int n) { return (size_t)A3_GCHUNK * 4 + (size_t)n * 6 + 16; }

__device__ __forceinline__ uint4 a3_draw(uint32_t lane, uint32_t round, uint32_t step, uint32_t tag, uint2 key) {
    return philox4x32_10(make_uint4(lane, round, step, tag), key);
}

// (3) + (4): one WARP per candidate lane.  The warp first draws every random number of the lane
// in parallel (Fisher-Yates targets, interchange pairs and coordinates: they do not depend on the
// state), then lane 0 runs the sequential swaps and interchanges from shared memory — keeping the
// current cost of each i in shared memory, so an interchange step costs one round trip for its two
// candidate costs — and finally the warp ORs the lane's n triples into the batch.
// Shared memory per warp: 4n (perms) + 2n (FY targets) shorts, n doubles (costs), 3L shorts (steps).
__host__ __device__ constexpr size_t a3_warp_smem(long long n, long long L) {
    return ((size_t)(6 * n + 3 * L) * 2 + 15) / 16 * 16 + (size_t)n * 8;
}
__global__ void k_a3_sample(int n, const short* __restrict__ sj0, const short* __restrict__ sk0,
                            const short* __restrict__ Ri, const short* __restrict__ Rj, const short* __restrict__ Rk,
                            const int* __restrict__ meta, const double* __restrict__ cost, uint2 key,
                            const Ctrl* __restrict__ ctrl, int r_idx, int kr, unsigned round_fixed, int use_fixed,
                            long long word_off, int W, long long L, uint64_t* __restrict__ X) {
    extern __shared__ unsigned char a3_raw[];
    const int wib = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const int lanes = 64 * W;
    const int l = blockIdx.x * (blockDim.x >> 5) + wib;
    const size_t per = a3_warp_smem(n, L);
    unsigned char* base = a3_raw + (size_t)wib * per;
    double* cur = reinterpret_cast<double*>(base);                // [n] cost of (i, sj[i], sk[i])
    short* pj = reinterpret_cast<short*>(cur + n);
    short* pk = pj + n;
    short* sj = pk + n;
    short* sk = sj + n;
    short* qj = sk + n;      // FY targets
    short* qk = qj + n;
    short* st_a = qk + n;    // interchange steps: a, b, coordinate
    short* st_b = st_a + L;
    short* st_c = st_b + L;
    if (l >= lanes) return;  // (warp-uniform)
    const unsigned round = use_fixed ? round_fixed : (unsigned)(ctrl->blk * kr + r_idx);
    const uint32_t lg = (uint32_t)(64 * word_off + l);
    const int r = meta[0];
    for (int t = ln; t < r; t += 32) { pj[t] = Rj[t]; pk[t] = Rk[t]; }
    for (int t = 1 + ln; t < r; t += 32) {
        const uint32_t uj = a3_draw(lg, round, (uint32_t)t, A3_TAG_J, key).x;
        const uint32_t uk = a3_draw(lg, round, (uint32_t)t, A3_TAG_K, key).x;
        qj[t] = (short)(((unsigned long long)uj * (unsigned long long)(t + 1)) >> 32);
        qk[t] = (short)(((unsigned long long)uk * (unsigned long long)(t + 1)) >> 32);
    }
    if (n >= 2)
        for (long long s = ln; s < L; s += 32) {
            const uint4 o = a3_draw(lg, round, (uint32_t)s, A3_TAG_L, key);
            const int a = (int)(((unsigned long long)o.x * (unsigned long long)n) >> 32);
            int b = (int)(((unsigned long long)o.y * (unsigned long long)(n - 1)) >> 32);
            if (b >= a) b += 1;
            st_a[s] = (short)a; st_b[s] = (short)b; st_c[s] = (short)(o.z & 1u);
        }
    for (int i = ln; i < n; i += 32) { sj[i] = sj0[i]; sk[i] = sk0[i]; }
    __syncwarp();
    const long long nn = (long long)n * n;
    if (ln == 0) {
        for (int t = r - 1; t >= 1; --t) {
            short tmp = pj[t]; pj[t] = pj[qj[t]]; pj[qj[t]] = tmp;
            tmp = pk[t]; pk[t] = pk[qk[t]]; pk[qk[t]] = tmp;
        }
        for (int t = 0; t < r; ++t) { sj[Ri[t]] = pj[t]; sk[Ri[t]] = pk[t]; }
    }
    __syncwarp();
    for (int i = ln; i < n; i += 32) cur[i] = __ldg(cost + i * nn + (long long)sj[i] * n + sk[i]);
    __syncwarp();
    if (ln == 0 && n >= 2) {
        for (long long s = 0; s < L; ++s) {
            const int a = st_a[s], b = st_b[s];
            const int ja = sj[a], jb = sj[b], ka = sk[a], kb = sk[b];
            const bool cj = st_c[s] == 0;
            const double n_a = __ldg(cost + a * nn + (long long)(cj ? jb : ja) * n + (cj ? ka : kb));
            const double n_b = __ldg(cost + b * nn + (long long)(cj ? ja : jb) * n + (cj ? kb : ka));
            if (__dadd_rn(n_a, n_b) < __dadd_rn(cur[a], cur[b])) {
                if (cj) { sj[a] = (short)jb; sj[b] = (short)ja; } else { sk[a] = (short)kb; sk[b] = (short)ka; }
                cur[a] = n_a; cur[b] = n_b;
            }
        }
    }
    __syncwarp();
    const unsigned long long bit = 1ull << (l & 63);
    for (int i = ln; i < n; i += 32) {
        const long long v = i * nn + (long long)sj[i] * n + sk[i];
        atomicOr(reinterpret_cast<unsigned long long*>(X + v * W + (l >> 6)), bit);
    }
}

}  // namespace gfors
