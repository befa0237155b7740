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
#include <type_traits>

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

// Philox4x32-10 round keys precomputed on the host (round r uses key + r*(W0, W1)): kernel parameters,
// so each key is a constant-bank operand of the 3-input XOR (philox_rkw below).
struct PhiloxKeys {
    uint32_t k0[10], k1[10];
};

// 32x32 -> 64-bit product in one IMAD.WIDE.U32 (the register pair holds lo, hi)
__device__ __forceinline__ uint64_t mul_wide_u32(uint32_t a, uint32_t b) {
    uint64_t r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint4 philox_rkw(uint4 c, const PhiloxKeys& rk) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = mul_wide_u32(0xD2511F53u, c.x), p1 = mul_wide_u32(0xCD9E8D57u, c.z);
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ rk.k0[r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ rk.k1[r],
                       (uint32_t)p0);
    }
    return c;
}

// RandSampleStep pass 1: T_i = ceil(p_i 2^32) for every variable (fp64, exact).  The words of variables
// with T = 0 (p = 0) or T = 2^32 (p = 1) need no random planes and are written here (all zeros / all
// ones); the others are appended to a compact list of (i, T) (warp-aggregated atomic, any order: a
// word's value depends only on (i, word, T, round)).  p: a fixed vector (pfix) or x_k of the loop.
template <typename T>
__global__ void __launch_bounds__(256) k_sample_thr(const T* __restrict__ xa, const T* __restrict__ xb2,
                                                    const double* __restrict__ pfix, long long n, int W,
                                                    const Ctrl* __restrict__ ctrl, long long kint, int use_fixed,
                                                    uint2* __restrict__ list, unsigned* __restrict__ cnt,
                                                    uint64_t* __restrict__ X, const double* __restrict__ c_int,
                                                    unsigned long long* __restrict__ s1) {
    // c_int != null (integral c): s1 += sum of c_i over the variables with p_i = 1 (their words are all
    // ones, so k_obj_list adds this constant instead of streaming them)
    constexpr int PER = 4;  // variables per thread and chunk: one list atomic per 1024 variables
    __shared__ unsigned s_off[8], s_base;
    __shared__ long long s_one[8];
    long long one_sum = 0;
    const T* __restrict__ p = nullptr;
    if (!use_fixed) p = (((ctrl->blk + 1) * kint) & 1) ? xb2 : xa;  // x_k written by iteration (b+1)*kint - 1
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (long long c0 = (long long)blockIdx.x * 256 * PER; c0 < n; c0 += (long long)gridDim.x * 256 * PER) {
        uint32_t t[PER];
        unsigned bal[PER], tot = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const long long i = c0 + k * 256 + threadIdx.x;
            t[k] = 0;
            if (i < n) {
                double pi = pfix ? pfix[i] : (double)p[i];
                pi = pi < 0.0 ? 0.0 : (pi > 1.0 ? 1.0 : pi);
                const double Td = ceil(pi * 4294967296.0);
                if (Td <= 0.0) { for (int w = 0; w < W; ++w) X[i * W + w] = 0ull; }
                else if (Td >= 4294967296.0) {
                    for (int w = 0; w < W; ++w) X[i * W + w] = ~0ull;
                    if (c_int) one_sum += (long long)c_int[i];
                }
                else t[k] = (uint32_t)Td;
            }
            bal[k] = __ballot_sync(0xffffffffu, t[k] != 0u);
            tot += __popc(bal[k]);
        }
        if (lane == 0) s_off[wid] = tot;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned acc = 0;
            for (int w = 0; w < 8; ++w) { const unsigned v = s_off[w]; s_off[w] = acc; acc += v; }
            s_base = acc ? atomicAdd(cnt, acc) : 0u;
        }
        __syncthreads();
        unsigned o = s_base + s_off[wid];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            if (t[k]) list[o + __popc(bal[k] & ((1u << lane) - 1u))] = make_uint2((unsigned)(c0 + k * 256 + threadIdx.x), t[k]);
            o += __popc(bal[k]);
        }
        __syncthreads();  // s_off / s_base reused by the next chunk
    }
    if (c_int) {  // one integer atomic per CTA (exact, order-free)
        for (int o = 16; o > 0; o >>= 1) one_sum += __shfl_xor_sync(0xffffffffu, one_sum, o);
        if (lane == 0) s_one[wid] = one_sum;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long a = 0;
            for (int w = 0; w < 8; ++w) a += s_one[w];
            if (a) atomicAdd(s1, (unsigned long long)a);
        }
    }
}

// RandSampleStep pass 2 (Alg. 3, contract R10): the MSB-first compare decides a 64-lane word after a
// data-dependent number of plane pairs (E ~ 3.9 Philox calls for p away from 0 and 1, up to 16).  The
// work items are the words (list entry e, word w) of the listed variables, item k = e*W + w; thread t
// takes items t, t + S, t + 2S, ... (S = threads in the grid).  ONE flat loop: every trip makes two
// Philox calls (four planes; independent chains) for the thread's current word, and a thread whose
// word got decided stores it and moves on to its next item (prefetched) inside the same trip.  There
// is no inner per-word loop, so the lanes of a warp never wait at a reconvergence point for the
// slowest word: a warp runs for the max over its lanes of the SUM of their trips (~33 words each on
// config 5), not the sum over words of the max.  The last CTA to finish zeroes the list counter for
// the next round.  Identical output to bernoulli_word.
constexpr int SMP_CTAS = 5;  // resident CTAs per SM of k_sample (grid = SMP_CTAS x SMs: one wave)
__global__ void __launch_bounds__(256, SMP_CTAS) k_sample(const uint2* __restrict__ list, unsigned* __restrict__ cnt, int W,
                                                         long long word_off, const __grid_constant__ PhiloxKeys rk,
                                                         const Ctrl* __restrict__ ctrl, int r, int kr, unsigned round_fixed,
                                                         int use_fixed, uint64_t* __restrict__ X,
                                                         unsigned long long* __restrict__ s1) {
    const unsigned round = use_fixed ? round_fixed : (unsigned)(ctrl->blk * kr + r);
    const uint64_t pol = l2_policy_evict_last();  // the batch is gathered by the evaluator next
    const unsigned wbase = (unsigned)word_off;
    const long long nitems = (long long)*(volatile unsigned*)cnt * W;
    const long long S = (long long)gridDim.x * blockDim.x;
    // item k = (entry e, word w); the item S further is (e + qS, w + rS) carried over
    const long long qS = S / W;
    const unsigned rS = (unsigned)(S % W);
    long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long e = k / W;
    unsigned w = (unsigned)(k - e * W);
    auto advance = [&]() { k += S; e += qS; w += rS; if (w >= (unsigned)W) { w -= W; ++e; } };
    // current item (i, T, word) and the next one, prefetched
    uint2 cur = k < nitems ? __ldg(list + e) : make_uint2(0u, 0u);
    unsigned cwo = w;
    bool active = k < nitems;
    advance();
    uint2 nxt = k < nitems ? __ldg(list + e) : make_uint2(0u, 0u);
    unsigned nwo = w;
    bool nact = k < nitems;
    unsigned Tsh = cur.y, q = 0u, ul = ~0u, uh = ~0u, rl = 0u, rh = 0u;
    while (__any_sync(0xffffffffu, active)) {
        // planes 2q (T bit 31 - 2q), 2q + 1, 2q + 2, 2q + 3 from two Philox calls: t = 1 -> lanes with
        // u-bit 0 decide 1, und &= pl; t = 0 -> lanes with u-bit 1 decide 0, und &= ~pl (m = t ? ~0 : 0).
        // Planes after the word is decided change nothing.
        const unsigned wg = wbase + cwo;
        const uint4 o = philox_rkw(make_uint4(cur.x, wg, q, round), rk);
        const uint4 o2 = philox_rkw(make_uint4(cur.x, wg, q + 1u, round), rk);
        uint32_t m = 0u - (Tsh >> 31);
        rl |= ul & ~o.x & m; rh |= uh & ~o.y & m;
        ul &= ~(o.x ^ m);    uh &= ~(o.y ^ m);
        m = 0u - ((Tsh >> 30) & 1u);
        rl |= ul & ~o.z & m; rh |= uh & ~o.w & m;
        ul &= ~(o.z ^ m);    uh &= ~(o.w ^ m);
        m = 0u - ((Tsh >> 29) & 1u);
        rl |= ul & ~o2.x & m; rh |= uh & ~o2.y & m;
        ul &= ~(o2.x ^ m);    uh &= ~(o2.y ^ m);
        m = 0u - ((Tsh >> 28) & 1u);
        rl |= ul & ~o2.z & m; rh |= uh & ~o2.w & m;
        ul &= ~(o2.z ^ m);    uh &= ~(o2.w ^ m);
        Tsh <<= 4;
        q += 2u;
        if ((ul | uh) == 0u || q == 16u) {  // word decided (u == T lanes stay 0): store, take the next item
            if (active) st_hint_u64(X + (size_t)cur.x * W + cwo, (uint64_t)rl | ((uint64_t)rh << 32), pol);
            cur = nxt; cwo = nwo; active = nact;
            advance();
            nxt = k < nitems ? __ldg(list + e) : make_uint2(0u, 0u);
            nwo = w;
            nact = k < nitems;
            Tsh = cur.y; q = 0u; ul = uh = ~0u; rl = rh = 0u;
        }
    }
    // the last CTA out resets the list counter (every CTA read it above)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(cnt + 1, 1u) == gridDim.x - 1) {
            // the round's list length and p = 1 constant stay readable by k_obj_list (slots 2, 3 / s1[1])
            cnt[2] = cnt[0];
            if (s1) { s1[1] = s1[0]; s1[0] = 0ull; }
            cnt[0] = 0u; cnt[1] = 0u;
            __threadfence();
        }
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
    if (rel == 4) return ~0ull;  // satisfied in every lane by variables sampled with p = 1
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

template <int WV>
__device__ __forceinline__ void load_words(const uint64_t* __restrict__ p, uint64_t (&v)[WV], uint64_t pol) {
    if constexpr (WV == 1) {
        v[0] = ld_hint_u64(p, pol);
    } else if constexpr (WV == 2) {
        const ulonglong2 a = ld_hint_u64x2(p, pol);
        v[0] = a.x; v[1] = a.y;
    } else {
        const ulonglong2 a = ld_hint_u64x2(p, pol);
        const ulonglong2 b = ld_hint_u64x2(p + 2, pol);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
}

// One SUB-lane group per count row; each nonzero gathers WV words (64*WV candidates) with one
// vector load, so a covering row over 128 candidates costs one 16-byte gather per nonzero.
constexpr int FEAS_U = 1;
template <int BMAX, int SUB, int WV>
__global__ void __launch_bounds__(256) k_feas_count(Csr K, CountRows cr, const uint64_t* __restrict__ X, int W,
                                                    unsigned long long* __restrict__ viol,
                                                    const unsigned char* __restrict__ ones) {
    __shared__ unsigned long long s_viol[64];  // block-aggregated violations when W <= 64
    const bool use_smem = W <= 64;
    if (use_smem)
        for (int w = threadIdx.x; w < W; w += blockDim.x) s_viol[w] = 0ull;
    __syncthreads();
    constexpr int RPW = 32 / SUB;
    const uint64_t pfirst = l2_policy_evict_first(), plast = l2_policy_evict_last();
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
            // ones[row] = #variables of the row with p = 1 (all-ones sample words): a ">= t" row already
            // holding t of them is satisfied in every lane — no gathers
            if (ones && rel == 0 && (int)ones[row] >= t) { rel = 4; p1 = p0; }
        }
        for (int w0 = 0; w0 < W; w0 += WV) {
            uint64_t C[WV][BMAX];
            uint64_t sat[WV];
#pragma unroll
            for (int u = 0; u < WV; ++u) {
                sat[u] = 0ull;
#pragma unroll
                for (int q = 0; q < BMAX; ++q) C[u][q] = 0ull;
            }
            if (rel < 3)
                // FEAS_U nonzeros per lane in flight: all index loads, then all gathers, then the adds
                // (a zero word adds nothing, so the tail is padded with zeros)
                for (long long p = p0 + lane; p < p1; p += FEAS_U * SUB) {
                    int c[FEAS_U];
#pragma unroll
                    for (int f = 0; f < FEAS_U; ++f) c[f] = p + f * SUB < p1 ? ld_hint_i32(K.idx + p + f * SUB, pfirst) : -1;
                    uint64_t v[FEAS_U][WV];
#pragma unroll
                    for (int f = 0; f < FEAS_U; ++f) {
                        if (c[f] >= 0) load_words<WV>(X + (long long)c[f] * W + w0, v[f], plast);
                        else
#pragma unroll
                            for (int u = 0; u < WV; ++u) v[f][u] = 0ull;
                    }
#pragma unroll
                    for (int f = 0; f < FEAS_U; ++f)
#pragma unroll
                        for (int u = 0; u < WV; ++u) csa_add_bit<BMAX>(C[u], sat[u], v[f][u], B);
                }
#pragma unroll
            for (int u = 0; u < WV; ++u) {
#pragma unroll
                for (int o = SUB / 2; o > 0; o >>= 1) {
                    uint64_t D[BMAX];
#pragma unroll
                    for (int q = 0; q < BMAX; ++q) D[q] = __shfl_xor_sync(0xffffffffu, C[u][q], o, SUB);
                    const uint64_t dsat = __shfl_xor_sync(0xffffffffu, sat[u], o, SUB);
                    csa_add_counter<BMAX>(C[u], sat[u], D, dsat, B);
                }
                if (lane == 0 && valid) {
                    const uint64_t bad = ~count_ok<BMAX>(C[u], sat[u], B, t, rel);
                    if (bad) atomicOr(use_smem ? &s_viol[w0 + u] : viol + w0 + u, (unsigned long long)bad);
                }
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

// Integral linear objective by bit planes: with c'_i = c_i - cmin in [0, 2^NB),
// sum_i c_i x_li = cmin * sum_i x_li + sum_b 2^b popc(column_l & plane_b).  A warp takes 32
// consecutive variables of one word, transposes the 32x32 bit blocks (lanes 0-31 and 32-63) with
// shuffles so thread t holds sample lane t's 32 variable bits, then ANDs with the precomputed
// coefficient bit planes (planes[chunk*NB + b], bit v = bit b of c'_{32 chunk + v}) and popcounts.
__device__ __forceinline__ unsigned transpose32(unsigned x, int lane) {
    const unsigned masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int j = 16 >> k;
        const unsigned m = masks[k];
        const unsigned o = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m) | ((o & ~m) >> j)) : ((x & m) | ((o & m) << j));
    }
    return x;
}

// load time: the bit planes of c - cmin (planes[h * nb + b] bit i % 32 = bit b of c_{32h + i%32} - cmin)
__global__ void __launch_bounds__(256) k_obj_planes(const double* __restrict__ c, long long n, double cmin, int nb,
                                                    unsigned* __restrict__ planes) {
    const long long nch = (n + 31) / 32;
    for (long long h = blockIdx.x * (long long)blockDim.x + threadIdx.x; h < nch; h += gridDim.x * (long long)blockDim.x) {
        unsigned w[20] = {};
        for (int k = 0; k < 32 && h * 32 + k < n; ++k) {
            const long long cp = (long long)(c[h * 32 + k] - cmin);
#pragma unroll
            for (int b = 0; b < 20; ++b)
                if (b < nb) w[b] |= (unsigned)((cp >> b) & 1) << k;
        }
#pragma unroll
        for (int b = 0; b < 20; ++b)
            if (b < nb) planes[h * nb + b] = w[b];
    }
}

// One CTA of 8 warps per (chunk range, word group of WV words): every lane loads its variable's WV
// words with one vector load, each warp walks chunks cta*cpc + warp + 8k (two at a time, loads
// first), and the 8 warps' int64 lane sums are added in shared memory in a fixed order, giving ONE
// partial row per CTA column block: zpart[blockIdx.x][64*w + lane] (k_obj_final adds gridDim.x rows).
template <int WV>
__global__ void __launch_bounds__(256) k_obj_bits(long long n, long long cpc, const unsigned* __restrict__ planes,
                                                  int NB, long long cmin, const uint64_t* __restrict__ X, int W,
                                                  long long* __restrict__ zpart /*[gridDim.x][64W]*/,
                                                  const unsigned* __restrict__ list_cnt = nullptr, long long list_thr = 0) {
    __shared__ long long sacc[8][64 * WV];
    // list_cnt: k_obj_list serves this round when the sampler's list is short (<= list_thr)
    if (list_cnt && (long long)list_cnt[2] <= list_thr) return;
    const uint64_t pdem = l2_policy_evict_first();  // last reader of the batch: demote it in L2
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int w0 = blockIdx.y * WV;
    const long long nchunk32 = (n + 31) / 32;
    const long long c0 = blockIdx.x * cpc, c1 = min(nchunk32, c0 + cpc);
    long long alo[WV], ahi[WV];
#pragma unroll
    for (int v = 0; v < WV; ++v) alo[v] = ahi[v] = 0;
    auto load = [&](long long ch, uint64_t (&xw)[WV]) {
        const long long i = ch * 32 + lane;
        if (ch < c1 && i < n) {
            if constexpr (WV == 2) {
                const ulonglong2 a = ld_hint_u64x2(X + i * W + w0, pdem);
                xw[0] = a.x; xw[1] = a.y;
            } else {
                xw[0] = ld_hint_u64(X + i * W + w0, pdem);
            }
        } else {
#pragma unroll
            for (int v = 0; v < WV; ++v) xw[v] = 0ull;
        }
    };
    auto consume = [&](long long ch, const uint64_t (&xw)[WV]) {
        if (ch >= c1) return;
        unsigned tlo[WV], thi[WV];
#pragma unroll
        for (int v = 0; v < WV; ++v) {
            tlo[v] = transpose32((unsigned)xw[v], lane);
            thi[v] = transpose32((unsigned)(xw[v] >> 32), lane);
        }
        int slo[WV], shi[WV];
#pragma unroll
        for (int v = 0; v < WV; ++v) { slo[v] = 0; shi[v] = 0; }
        for (int b = 0; b < NB; ++b) {
            const unsigned pl = __ldg(planes + ch * NB + b);
#pragma unroll
            for (int v = 0; v < WV; ++v) {
                slo[v] += __popc(tlo[v] & pl) << b;
                shi[v] += __popc(thi[v] & pl) << b;
            }
        }
#pragma unroll
        for (int v = 0; v < WV; ++v) {
            alo[v] += (long long)slo[v] + cmin * __popc(tlo[v]);
            ahi[v] += (long long)shi[v] + cmin * __popc(thi[v]);
        }
    };
    for (long long ch = c0 + wib; ch < c1; ch += 16) {
        uint64_t xa[WV], xb[WV];
        load(ch, xa);
        load(ch + 8, xb);
        consume(ch, xa);
        consume(ch + 8, xb);
    }
#pragma unroll
    for (int v = 0; v < WV; ++v) { sacc[wib][64 * v + lane] = alo[v]; sacc[wib][64 * v + 32 + lane] = ahi[v]; }
    __syncthreads();
    if (threadIdx.x < 64 * WV) {
        long long t = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += sacc[k][threadIdx.x];
        zpart[blockIdx.x * 64LL * W + 64LL * w0 + threadIdx.x] = t;
    }
}

// The linear objective of a batch drawn by k_sample from its list: the words of the variables with
// p = 0 are zero and those with p = 1 all ones, so  z_l = c0 + s1 + sum over the LISTED variables of
// c_i x_il  (s1 = sum of c_i over p_i = 1, from k_sample_thr).  Chunks of 32 list entries per warp: the
// coefficient planes of the chunk come from ballots of (c_i - cmin) bits, the batch words are gathered
// by list index, then the same transposes and popcounts as k_obj_bits; gridDim.x partial rows, CTA 0's
// row carries s1.  Cost scales with the list (the fractional variables) instead of n.
template <int WV>
__global__ void __launch_bounds__(256) k_obj_list(const uint2* __restrict__ list, const unsigned* __restrict__ cnt,
                                                  const unsigned long long* __restrict__ s1, const double* __restrict__ c,
                                                  int NB, long long cmin, const uint64_t* __restrict__ X, int W,
                                                  long long* __restrict__ zpart /*[gridDim.x][64W]*/, long long list_thr) {
    __shared__ long long sacc[8][64 * WV];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int w0 = blockIdx.y * WV;
    const long long L = cnt[2];
    if (L > list_thr) return;  // a long list: k_obj_bits streams every variable instead
    const long long nch = (L + 31) / 32;
    long long alo[WV], ahi[WV];
#pragma unroll
    for (int v = 0; v < WV; ++v) alo[v] = ahi[v] = 0;
    for (long long ch = blockIdx.x * 8LL + wib; ch < nch; ch += gridDim.x * 8LL) {
        const long long e = ch * 32 + lane;
        uint64_t xw[WV];
        long long cv = 0;
        if (e < L) {
            const unsigned i = __ldg(list + e).x;
            if constexpr (WV == 2) {
                const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(X + (size_t)i * W + w0));
                xw[0] = a.x; xw[1] = a.y;
            } else {
                xw[0] = __ldg(X + (size_t)i * W + w0);
            }
            cv = (long long)__ldg(c + i) - cmin;
        } else {
#pragma unroll
            for (int v = 0; v < WV; ++v) xw[v] = 0ull;
        }
        unsigned tlo[WV], thi[WV];
#pragma unroll
        for (int v = 0; v < WV; ++v) {
            tlo[v] = transpose32((unsigned)xw[v], lane);
            thi[v] = transpose32((unsigned)(xw[v] >> 32), lane);
        }
        int slo[WV], shi[WV];
#pragma unroll
        for (int v = 0; v < WV; ++v) { slo[v] = 0; shi[v] = 0; }
        for (int b = 0; b < NB; ++b) {
            const unsigned pl = __ballot_sync(0xffffffffu, (cv >> b) & 1);
#pragma unroll
            for (int v = 0; v < WV; ++v) {
                slo[v] += __popc(tlo[v] & pl) << b;
                shi[v] += __popc(thi[v] & pl) << b;
            }
        }
#pragma unroll
        for (int v = 0; v < WV; ++v) {
            alo[v] += (long long)slo[v] + cmin * __popc(tlo[v]);
            ahi[v] += (long long)shi[v] + cmin * __popc(thi[v]);
        }
    }
#pragma unroll
    for (int v = 0; v < WV; ++v) { sacc[wib][64 * v + lane] = alo[v]; sacc[wib][64 * v + 32 + lane] = ahi[v]; }
    __syncthreads();
    if (threadIdx.x < 64 * WV) {
        long long t = (blockIdx.x == 0) ? (long long)s1[1] : 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += sacc[k][threadIdx.x];
        zpart[blockIdx.x * 64LL * W + 64LL * w0 + threadIdx.x] = t;
    }
}

// Quadratic term only (x'Qx per lane), exact int64, added into zpart row `slot`
template <bool INTEGRAL>
__global__ void __launch_bounds__(256) k_obj_quad(long long n, int chunk, Csr Q, const double* __restrict__ qv,
                                                  const uint64_t* __restrict__ X, int W, void* __restrict__ zpart) {
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
        const long long o = ch * 64LL * W + 64LL * w + bit;
        if constexpr (INTEGRAL) reinterpret_cast<long long*>(zpart)[o] = ai;
        else reinterpret_cast<double*>(zpart)[o] = ad;
    }
}

// z_l = sum over partial rows (fixed order) + c0.  One CTA of 1024 threads per 32 lanes: 32 row
// groups x 32 lanes, four independent accumulators per thread, then a fixed-order combine.
template <bool INTEGRAL>
__global__ void __launch_bounds__(1024) k_obj_final(long long nrows, int W, const void* __restrict__ zpart, double c0,
                                                    double* __restrict__ z) {
    using A = typename std::conditional<INTEGRAL, long long, double>::type;
    __shared__ A sh[32][33];
    const long long lanes = 64LL * W;
    const int t = threadIdx.x & 31, grp = threadIdx.x >> 5;
    const long long l = blockIdx.x * 32LL + t;
    const A* zp = reinterpret_cast<const A*>(zpart);
    A a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    long long r = grp;
    for (; r + 96 < nrows; r += 128) {
        a0 += zp[r * lanes + l]; a1 += zp[(r + 32) * lanes + l];
        a2 += zp[(r + 64) * lanes + l]; a3 += zp[(r + 96) * lanes + l];
    }
    for (; r < nrows; r += 32) a0 += zp[r * lanes + l];
    sh[grp][t] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (grp == 0) {
        A s = 0;
        for (int g = 0; g < 32; ++g) s += sh[g][t];
        if constexpr (INTEGRAL) z[l] = (double)(s + (long long)c0);
        else z[l] = s + c0;
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
