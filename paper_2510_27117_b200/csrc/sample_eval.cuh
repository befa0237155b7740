// sample_eval.cuh — RandSampleStep (Alg. 3) into a bit-sliced batch, and
// EvalBest: feasibility of K_u x vs r, objective x'Qx + c'x + c0,
// argmin with strict improvement, incumbent copy.
//
// Batch layout ("bit-sliced"): X[i*W + w] is a uint64 whose bit b is sample
// (64*(word_off + w) + b) of variable i.  One word carries 64 candidates, so a row of K is
// tested for 64 candidates with one 8-byte gather per nonzero.
#pragma once
#include "common.cuh"
#include "pdhg.cuh"

namespace gfors {

// ---------------------------------------------------------------------------------------------
// Sampler.  Contract (reading R10): u = 32-bit uniform whose bit (31-t) is bit b of plane t,
// plane pair q = Philox4x32-10(ctr = (i, global word, q, round), key = seed); planes 2q, 2q+1 =
// out0|out1<<32, out2|out3<<32.  x = [u < T], T = ceil(p 2^32).  Evaluated lazily MSB-first
// over all 64 lanes at once: a lane is decided at the first plane where u's bit differs from T's.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t bernoulli_word(double p, unsigned i, unsigned wg, unsigned round, uint2 key) {
    p = p < 0.0 ? 0.0 : (p > 1.0 ? 1.0 : p);
    const double Td = ceil(p * 4294967296.0);
    if (Td <= 0.0) return 0ull;
    if (Td >= 4294967296.0) return ~0ull;
    const uint32_t T = (uint32_t)Td;
    uint64_t res = 0ull, und = ~0ull;
#pragma unroll 1
    for (unsigned q = 0; q < 16; ++q) {
        const uint4 o = philox4x32_10(make_uint4(i, wg, q, round), key);
        const uint64_t pa = (uint64_t)o.x | ((uint64_t)o.y << 32);
        const uint64_t pb = (uint64_t)o.z | ((uint64_t)o.w << 32);
        {
            const bool tb = (T >> (31 - 2 * q)) & 1u;
            const uint64_t diff = und & (tb ? ~pa : pa);
            if (tb) res |= diff;
            und &= ~diff;
        }
        {
            const bool tb = (T >> (30 - 2 * q)) & 1u;
            const uint64_t diff = und & (tb ? ~pb : pb);
            if (tb) res |= diff;
            und &= ~diff;
        }
        if (und == 0ull) break;
    }
    return res;  // lanes with u == T stay 0 ([u < T] false)
}

// p: either a fixed vector (pfix != nullptr) or x_k of the loop (parity from ctrl).
template <typename T>
__global__ void __launch_bounds__(256) k_sample(const T* __restrict__ xa, const T* __restrict__ xb2,
                                                const double* __restrict__ pfix, long long n, int W,
                                                long long word_off, uint2 key, const Ctrl* __restrict__ ctrl,
                                                long long kint, int r, int kr, unsigned round_fixed, int use_fixed,
                                                uint64_t* __restrict__ X) {
    const T* __restrict__ p = nullptr;
    unsigned round = round_fixed;
    if (!use_fixed) {
        const long long b = ctrl->blk;
        p = (((b + 1) * kint) & 1) ? xb2 : xa;  // x_k written by iteration (b+1)*kint - 1
        round = (unsigned)(b * kr + r);
    }
    const long long total = n * (long long)W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += gridDim.x * (long long)blockDim.x) {
        const long long i = idx / W;
        const int wl = (int)(idx - i * W);
        const double pi = pfix ? pfix[i] : (double)p[i];
        X[idx] = bernoulli_word(pi, (unsigned)i, (unsigned)(word_off + wl), round, key);
    }
}

// final Alg. 1 line: round(x_k), ties -> 1 (reading R13), as a one-lane batch (W = 1, lane 0)
template <typename T>
__global__ void k_round_batch(const T* __restrict__ xa, const T* __restrict__ xb2, long long n,
                              const Ctrl* __restrict__ ctrl, long long kint, uint64_t* __restrict__ X) {
    const long long kk = ctrl->k;  // iterations completed; x_k lives in buffer (k & 1) when kint == 0
    (void)kint;
    const T* __restrict__ p = (kk & 1) ? xb2 : xa;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        X[i] = ((double)p[i] >= 0.5) ? 1ull : 0ull;
}

// ---------------------------------------------------------------------------------------------
// Feasibility, rows whose coefficients are one sign s in {+1,-1} ("count rows"): with c = #ones,
// s c >= R or s c = R becomes c >= t, c <= t or c == t.  The count is kept bit-sliced per 64-lane
// word with B <= BMAX planes saturating at 2^B - 1 >= cap (cap = t for >=, t+1 for <=/==), so
// covering rows (c >= 1) are one OR per nonzero and packing/assignment rows two planes.
// rel: 0 GE, 1 LE, 2 EQ, 3 never satisfiable.
// ---------------------------------------------------------------------------------------------
struct CountRows {
    const int* row;            // canonical row ids in this class
    const int* t;              // target
    const signed char* rel;    // relation
    const signed char* B;      // planes
    long long nrows;
};

template <int BMAX>
__device__ __forceinline__ void csa_add_bit(uint64_t (&C)[BMAX], uint64_t& sat, uint64_t v, int B) {
    uint64_t carry = v;
#pragma unroll
    for (int q = 0; q < BMAX; ++q)
        if (q < B) { const uint64_t t = C[q] & carry; C[q] ^= carry; carry = t; }
    sat |= carry;
}

template <int BMAX>
__device__ __forceinline__ void csa_add_counter(uint64_t (&C)[BMAX], uint64_t& sat, const uint64_t (&D)[BMAX],
                                                uint64_t dsat, int B) {
    uint64_t carry = 0ull;
#pragma unroll
    for (int q = 0; q < BMAX; ++q)
        if (q < B) {
            const uint64_t x = C[q] ^ D[q];
            const uint64_t s = x ^ carry;
            carry = (C[q] & D[q]) | (carry & x);
            C[q] = s;
        }
    sat |= carry | dsat;
}

// mask of lanes whose (saturated) count satisfies rel against t
template <int BMAX>
__device__ __forceinline__ uint64_t count_ok(const uint64_t (&C)[BMAX], uint64_t sat, int B, int t, int rel) {
    if (rel == 3) return 0ull;
    uint64_t gt = 0ull, eq = ~0ull;
#pragma unroll
    for (int q = BMAX - 1; q >= 0; --q)
        if (q < B) {
            if ((t >> q) & 1) eq &= C[q];
            else { gt |= eq & C[q]; eq &= ~C[q]; }
        }
    if (rel == 0) return sat | gt | eq;
    if (rel == 1) return ~sat & ~gt;
    return ~sat & eq;
}

template <int BMAX, int SUB>
__global__ void __launch_bounds__(256) k_feas_count(Csr K, CountRows cr, const uint64_t* __restrict__ X, int W,
                                                    unsigned long long* __restrict__ viol) {
    __shared__ unsigned long long s_viol[64];  // block-aggregated violations when W <= 64
    const bool use_smem = W <= 64;
    if (use_smem)
        for (int w = threadIdx.x; w < W; w += blockDim.x) s_viol[w] = 0ull;
    __syncthreads();
    constexpr int RPW = 32 / SUB;
    const int lane = threadIdx.x & (SUB - 1);
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const int gsub = (threadIdx.x & 31) / SUB;
    for (long long base = warp * RPW; base < cr.nrows; base += nwarps * RPW) {
        const long long e = base + gsub;
        const bool valid = e < cr.nrows;
        long long p0 = 0, p1 = 0;
        int B = 1, t = 0, rel = 0;
        if (valid) {
            const int row = cr.row[e];
            p0 = __ldg(K.ptr + row); p1 = __ldg(K.ptr + row + 1);
            B = cr.B[e]; t = cr.t[e]; rel = cr.rel[e];
        }
        for (int w = 0; w < W; ++w) {
            uint64_t C[BMAX];
#pragma unroll
            for (int q = 0; q < BMAX; ++q) C[q] = 0ull;
            uint64_t sat = 0ull;
            if (rel != 3)
                for (long long p = p0 + lane; p < p1; p += SUB) {
                    const uint64_t v = __ldg(X + (long long)__ldg(K.idx + p) * W + w);
                    csa_add_bit<BMAX>(C, sat, v, B);
                }
#pragma unroll
            for (int o = SUB / 2; o > 0; o >>= 1) {
                uint64_t D[BMAX];
#pragma unroll
                for (int q = 0; q < BMAX; ++q) D[q] = __shfl_xor_sync(0xffffffffu, C[q], o, SUB);
                const uint64_t dsat = __shfl_xor_sync(0xffffffffu, sat, o, SUB);
                csa_add_counter<BMAX>(C, sat, D, dsat, B);
            }
            if (lane == 0 && valid) {
                const uint64_t bad = ~count_ok<BMAX>(C, sat, B, t, rel);
                if (bad) atomicOr(use_smem ? &s_viol[w] : viol + w, (unsigned long long)bad);
            }
        }
    }
    __syncthreads();
    if (use_smem)
        for (int w = threadIdx.x; w < W; w += blockDim.x)
            if (s_viol[w]) atomicOr(viol + w, s_viol[w]);
}

// ---------------------------------------------------------------------------------------------
// Feasibility, general integer rows (integral data): exact int64 per lane.  Rows are cut in
// segments; warp = (segment, 32-lane group); partial sums are added with 64-bit integer atomics
// (exact, so the result is order independent), then a finaliser compares with r.
// ---------------------------------------------------------------------------------------------
struct IntRows {
    const int* row;            // canonical row of each int row slot
    const long long* rhs;      // r_j (canonical, integral)
    const signed char* is_eq;  // 1 for EQ rows
    const long long* seg_start;  // [2*nseg]: segment k covers nonzeros [seg_start[2k], seg_start[2k+1])
    const int* seg_slot;         // int-row slot of each segment
    long long nrows, nseg;
};

template <int KIND>
__global__ void __launch_bounds__(256) k_feas_int_partial(Csr K, IntRows ir, const uint64_t* __restrict__ X, int W,
                                                          unsigned long long* __restrict__ acc /*[nrows][64W]*/) {
    const int t = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const long long groups = 2LL * W;  // 32-lane groups
    for (long long job = warp; job < ir.nseg * groups; job += nwarps) {
        const long long sg = job / groups;
        const int gidx = (int)(job - sg * groups);
        const int w = gidx >> 1, bit = ((gidx & 1) << 5) + t;
        const long long p0 = ir.seg_start[2 * sg], p1 = ir.seg_start[2 * sg + 1];
        long long a = 0;
        for (long long p = p0; p < p1; ++p) {
            const uint64_t xw = __ldg(X + (long long)__ldg(K.idx + p) * W + w);
            if ((xw >> bit) & 1ull) a += (long long)kval<KIND>(K.val, p);
        }
        if (a) atomicAdd(acc + (long long)ir.seg_slot[sg] * 64 * W + 64LL * w + bit, (unsigned long long)a);
    }
}

__global__ void k_feas_int_final(IntRows ir, int W, const unsigned long long* __restrict__ acc,
                                 unsigned long long* __restrict__ viol) {
    const long long lanes = 64LL * W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < ir.nrows * lanes;
         idx += gridDim.x * (long long)blockDim.x) {
        const long long slot = idx / lanes;
        const long long l = idx - slot * lanes;
        const long long s = (long long)acc[idx];
        const long long r = ir.rhs[slot];
        const bool ok = ir.is_eq[slot] ? (s == r) : (s >= r);
        if (!ok) atomicOr(viol + (l >> 6), 1ull << (l & 63));
    }
}

// Real-valued rows (non-integral data): one warp per (row, 32-lane group), the row's nonzeros in
// ascending order, fp64, tolerance 1e-9 (reading R12).  Same order as the oracle.
template <int KIND>
__global__ void __launch_bounds__(256) k_feas_real(Csr K, const int* __restrict__ rows, long long nrows,
                                                   const double* __restrict__ ru, long long m1,
                                                   const uint64_t* __restrict__ X, int W,
                                                   unsigned long long* __restrict__ viol) {
    const int t = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const long long groups = 2LL * W;
    for (long long job = warp; job < nrows * groups; job += nwarps) {
        const long long e = job / groups;
        const int gidx = (int)(job - e * groups);
        const int w = gidx >> 1, bit = ((gidx & 1) << 5) + t;
        const int row = rows[e];
        double s = 0.0;
        for (long long p = K.ptr[row]; p < K.ptr[row + 1]; ++p) {
            const uint64_t xw = __ldg(X + (long long)__ldg(K.idx + p) * W + w);
            if ((xw >> bit) & 1ull) s += kval<KIND>(K.val, p);
        }
        const bool ok = row < m1 ? (ru[row] - s <= 1e-9) : (fabs(s - ru[row]) <= 1e-9);
        if (!ok) atomicOr(viol + w, 1ull << bit);
    }
}

// ---------------------------------------------------------------------------------------------
// Objective per lane: z_l = sum_i c_i x_li + sum_{(i,q) in Q} Q_iq x_li x_lq (+ c0 in the
// finaliser).  Warp = (chunk of variables, 32-lane group), exact int64 (integral data) or fp64
// chunk partials; the finaliser adds chunk partials in chunk order (deterministic).
// ---------------------------------------------------------------------------------------------
template <bool INTEGRAL, bool HASQ>
__global__ void __launch_bounds__(256) k_obj_partial(long long n, int chunk, const double* __restrict__ c,
                                                     Csr Q, const double* __restrict__ qv,
                                                     const uint64_t* __restrict__ X, int W,
                                                     void* __restrict__ zpart /*[nchunk][64W]*/) {
    const int t = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const long long groups = 2LL * W;
    const long long nchunk = (n + chunk - 1) / chunk;
    for (long long job = warp; job < nchunk * groups; job += nwarps) {
        const long long ch = job / groups;
        const int gidx = (int)(job - ch * groups);
        const int w = gidx >> 1, bit = ((gidx & 1) << 5) + t;
        const long long i0 = ch * chunk, i1 = min(n, i0 + chunk);
        long long ai = 0;
        double ad = 0.0;
        long long i = i0;
        for (; i + 3 < i1; i += 4) {
            const uint64_t x0 = __ldg(X + i * W + w), x1 = __ldg(X + (i + 1) * W + w);
            const uint64_t x2 = __ldg(X + (i + 2) * W + w), x3 = __ldg(X + (i + 3) * W + w);
            const double c0 = __ldg(c + i), c1 = __ldg(c + i + 1), c2 = __ldg(c + i + 2), c3 = __ldg(c + i + 3);
            if constexpr (INTEGRAL) {
                ai += ((x0 >> bit) & 1ull) ? (long long)c0 : 0;
                ai += ((x1 >> bit) & 1ull) ? (long long)c1 : 0;
                ai += ((x2 >> bit) & 1ull) ? (long long)c2 : 0;
                ai += ((x3 >> bit) & 1ull) ? (long long)c3 : 0;
            } else {
                ad += ((x0 >> bit) & 1ull) ? c0 : 0.0;
                ad += ((x1 >> bit) & 1ull) ? c1 : 0.0;
                ad += ((x2 >> bit) & 1ull) ? c2 : 0.0;
                ad += ((x3 >> bit) & 1ull) ? c3 : 0.0;
            }
        }
        for (; i < i1; ++i) {
            const uint64_t xi = __ldg(X + i * W + w);
            if ((xi >> bit) & 1ull) {
                if constexpr (INTEGRAL) ai += (long long)__ldg(c + i); else ad += __ldg(c + i);
            }
        }
        if constexpr (HASQ) {
            for (long long ii = i0; ii < i1; ++ii) {
                const uint64_t xi = __ldg(X + ii * W + w);
                if (!((xi >> bit) & 1ull)) continue;
                for (long long q = __ldg(Q.ptr + ii); q < __ldg(Q.ptr + ii + 1); ++q) {
                    const uint64_t xq = __ldg(X + (long long)__ldg(Q.idx + q) * W + w);
                    if ((xq >> bit) & 1ull) {
                        if constexpr (INTEGRAL) ai += (long long)__ldg(qv + q); else ad += __ldg(qv + q);
                    }
                }
            }
        }
        const long long o = ch * 64LL * W + 64LL * w + bit;
        if constexpr (INTEGRAL) reinterpret_cast<long long*>(zpart)[o] = ai;
        else reinterpret_cast<double*>(zpart)[o] = ad;
    }
}

template <bool INTEGRAL>
__global__ void k_obj_final(long long nchunk, int W, const void* __restrict__ zpart, double c0, double* __restrict__ z) {
    const long long lanes = 64LL * W;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < lanes; l += gridDim.x * (long long)blockDim.x) {
        if constexpr (INTEGRAL) {
            long long s = 0;
            for (long long ch = 0; ch < nchunk; ++ch) s += reinterpret_cast<const long long*>(zpart)[ch * lanes + l];
            z[l] = (double)(s + (long long)c0);
        } else {
            double s = 0.0;
            for (long long ch = 0; ch < nchunk; ++ch) s += reinterpret_cast<const double*>(zpart)[ch * lanes + l];
            z[l] = s + c0;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Argmin over the batch + incumbent update (reading R11): among feasible
// lanes pick min z, ties -> lowest lane; replace the incumbent iff strictly better.
// mode 0: loop round (round id from ctrl), 1: final round(x_k) (index -1), 2: hook (no update).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_argmin(const double* __restrict__ z, const unsigned long long* __restrict__ viol,
                                                long long lanes, long long word_off, Ctrl* __restrict__ ctrl,
                                                long long kint, int r, int kr, int mode) {
    __shared__ double sz[256];
    __shared__ long long sl[256];
    double bz = INFINITY;
    long long bl = -1;
    for (long long l = threadIdx.x; l < lanes; l += blockDim.x) {
        const bool feas = !((viol[l >> 6] >> (l & 63)) & 1ull);
        if (feas && (bl < 0 || z[l] < bz)) { bz = z[l]; bl = l; }
    }
    sz[threadIdx.x] = bz; sl[threadIdx.x] = bl;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const double z2 = sz[threadIdx.x + o];
            const long long l2 = sl[threadIdx.x + o];
            if (l2 >= 0 && (sl[threadIdx.x] < 0 || z2 < sz[threadIdx.x] ||
                            (z2 == sz[threadIdx.x] && l2 < sl[threadIdx.x]))) {
                sz[threadIdx.x] = z2; sl[threadIdx.x] = l2;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctrl->win_lane = -1;
        if (mode == 0) ctrl->rounds += 1;
        const long long l = sl[0];
        if (l >= 0 && sz[0] < ctrl->z_best) {
            ctrl->z_best = sz[0];
            ctrl->has_inc = 1;
            ctrl->win_lane = (int)l;
            ctrl->improved = 1;
            ctrl->found_ns = globaltimer_ns() - ctrl->t0_ns;
            if (mode == 0) {
                ctrl->found_iter = (ctrl->blk + 1) * kint;
                ctrl->found_round = ctrl->blk * kr + r;
                ctrl->found_index = 64 * word_off + l;
            } else {
                ctrl->found_iter = ctrl->k;
                ctrl->found_round = -1;
                ctrl->found_index = -1;
            }
        }
    }
}

__global__ void k_copy_best(const uint64_t* __restrict__ X, int W, long long n, const Ctrl* __restrict__ ctrl,
                            unsigned char* __restrict__ xbest) {
    const int l = ctrl->win_lane;
    if (l < 0) return;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        xbest[i] = (unsigned char)((X[i * W + (l >> 6)] >> (l & 63)) & 1ull);
}

// reset per-round accumulators (violations, integer row sums)
__global__ void k_round_reset(unsigned long long* __restrict__ viol, int W, unsigned long long* __restrict__ iacc,
                              long long niacc, unsigned long long lane_mask_last, int all_bad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < niacc; i += gridDim.x * (long long)blockDim.x)
        iacc[i] = 0ull;
    if (blockIdx.x == 0)
        for (int w = threadIdx.x; w < W; w += blockDim.x)
            viol[w] = all_bad ? ~0ull : ((w == W - 1) ? ~lane_mask_last : 0ull);
}

}  // namespace gfors
