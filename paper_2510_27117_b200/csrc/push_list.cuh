// push_list.cuh — list of xbar columns handed from the primal to the next dual (push_dual.cuh).
//
// Delta push: once a push-mode dual has run, the row accumulators acc = sum_i K_u[:,i] round(xbar_i 2^40)
// are kept (not cleared) and flagged valid; the next primal then lists only the columns whose xbar
// CHANGED, and the next dual adds round(xbar_k 2^40) - round(xbar_{k-1} 2^40) for them.  Integer
// addition is exact and associative, so acc is bit-identical to a fresh push of all nonzero columns;
// near the fixed point few columns change (config 5: 0.1 % per 10 iterations after 1500), so the dual
// costs almost nothing.  A gather-mode dual clears acc (if valid) and the flag.  Flags are kept per
// parity: the dual of parity p reads dvalid[p] and writes dvalid[p^1]; the primal of parity p reads
// dvalid[p^1] (the state the next dual will see) to decide which columns to list.
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
    unsigned* dvalid;               // [2] acc holds the previous dual's xbar (delta push), per parity
};

// parity-selected members without dynamic indexing of the kernel-parameter arrays (which would
// copy the struct to local memory)
__device__ __forceinline__ unsigned* pl_count(const PushList& pl, int p) { return p ? pl.count[1] : pl.count[0]; }
__device__ __forceinline__ int* pl_list(const PushList& pl, int p) { return p ? pl.list[1] : pl.list[0]; }

// delta state the dual of parity p starts from (block-uniform)
// (dvalid == nullptr: delta push disabled, option delta_dual = 0 — accumulators cleared after each use)
__device__ __forceinline__ bool pl_valid(const PushList& pl, int p) {
    return pl.dvalid && *(volatile unsigned*)(p ? pl.dvalid + 1 : pl.dvalid) != 0u;
}
__device__ __forceinline__ void pl_set_valid(const PushList& pl, int p, bool v) {
    if (pl.dvalid) (p ? pl.dvalid[1] : pl.dvalid[0]) = v ? 1u : 0u;
}

// list criterion of the primal (parity p writes the list of the dual of parity p^1): with valid
// accumulators the changed columns, else the nonzero ones
template <typename T>
__device__ __forceinline__ bool pl_listed(bool delta, T xbn, T xbprev) { return delta ? xbn != xbprev : xbn != (T)0; }

// called by thread 0 of block 0 of whichever dual kernel is active this iteration
__device__ __forceinline__ void push_reset_next(const PushList& pl, int par) {
    *pl_count(pl, par ^ 1) = 0u;
    if (pl.pp_rcount) { *pl.pp_rcount = 0u; *pl.pp_wmax = 0ull; }
}

__device__ __forceinline__ bool push_mode(const PushList& pl, int par) {
    return pl.acc != nullptr && *(volatile unsigned*)pl_count(pl, par) <= pl.thr;
}
// iteration parity and the dual's mode read ONCE per CTA (thread 0) and broadcast through shared
// memory: when every thread read the same control words, a launch whose mode is switched off (all
// CTAs only read and exit) took ~8 us of same-address L2 requests.  Call at the top of the kernel
// (contains __syncthreads).
__device__ __forceinline__ int cta_parity(const Ctrl* ctrl, long long kint, long long j) {
    __shared__ int s_par;
    if (threadIdx.x == 0) s_par = (int)(((kint ? ctrl->blk * kint : 0) + j) & 1);
    __syncthreads();
    return s_par;
}
__device__ __forceinline__ bool cta_push_mode(const PushList& pl, int par) {
    __shared__ int s_push;
    if (threadIdx.x == 0) s_push = push_mode(pl, par) ? 1 : 0;
    __syncthreads();
    return s_push != 0;
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

// ---------------------------------------------------------------------------------------------
// Push-mode primal state (push_primal.cuh), here so the gather-mode primal (rowblock.cuh) can take
// the same device decision.  Delta push as for the dual: valid column accumulators
// accx = sum_j K_u[j,:] round(w_j 2^e) are kept between iterations with a FIXED exponent e (per
// parity pe[]), and k_wlist lists only the rows whose y changed; the window check below re-bases
// (gather iteration, accumulators cleared, fresh e) when max|w| leaves [2^-16, 2^8] of its value at
// the last re-base, so no sum can overflow and the resolution stays <= 2^-38 of max|w|*maxdeg.
// ---------------------------------------------------------------------------------------------
struct PushPrimal {
    int* rlist;                // listed rows (nonzero w, or changed y with valid accumulators)
    unsigned* rcount;          // list length (reset by the dual of the same iteration)
    unsigned rthr;             // push mode iff rcount <= rthr
    unsigned long long* wmax;  // bit pattern of max |w_j| (non-negative doubles order like uint64)
    long long* accx;           // [n] int64 column accumulators (all 0 unless pvalid)
    int maxdeg;                // largest column degree of K_u (number of terms of any a_i)
    long long m;
    unsigned* pvalid;          // [2] accx valid (delta push), per parity as for the dual
    int* pe;                   // [2] scale exponent of the valid accx
    const double* g;           // row scale (w_{k-1} recomputed from y_{k-1}, pdhg.cuh w_of)
    const signed char* rsign;
    unsigned char* xst;        // [n] stationary-column counters (k_primal_push skip), null = off
    unsigned mark_rows;        // delta scatters of <= mark_rows rows mark the columns they touch
};

constexpr int PP_HEAD = 8;     // headroom bits at a re-base
constexpr int PP_WINDOW = 16;  // max|w| may shrink by 2^16 before a re-base

struct PPMode {
    bool push;   // push-mode primal this iteration
    bool delta;  // accx valid: scatter the changes only
    int e;       // scale exponent S = 2^e
};

// b = max|w| * maxdeg < 2^eb (exponent read from the bits)
__device__ __forceinline__ int pp_bits(double b) {
    if (!(b > 0.0)) return -2000;
    return (int)((__double_as_longlong(b) >> 52) & 0x7ff) - 1022;  // b = f 2^(bexp-1023), f in [1,2)
}

__device__ __forceinline__ PPMode pp_mode(const PushPrimal& pp, int par) {
    PPMode r{false, false, 0};
    if (!pp.accx) return r;
    const unsigned cnt = *(volatile unsigned*)pp.rcount;
    const double wm = __longlong_as_double((long long)*(volatile unsigned long long*)pp.wmax);
    const int eb = pp_bits(wm * (double)pp.maxdeg);
    if (*(volatile unsigned*)(par ? pp.pvalid + 1 : pp.pvalid) != 0u) {
        r.delta = true;
        r.e = *(volatile int*)(par ? pp.pe + 1 : pp.pe);
        r.push = cnt <= pp.rthr && eb + r.e <= 62 && eb + r.e >= 62 - PP_HEAD - PP_WINDOW;
    } else {
        r.e = wm > 0.0 ? min(62 - PP_HEAD - eb, 1000) : 0;
        r.push = cnt <= pp.rthr;
    }
    return r;
}
// pp_mode read once per CTA (see cta_push_mode)
__device__ __forceinline__ PPMode cta_pp_mode(const PushPrimal& pp, int par) {
    __shared__ PPMode s_md;
    if (threadIdx.x == 0) s_md = pp_mode(pp, par);
    __syncthreads();
    return s_md;
}

// the delta scatter of this iteration marks touched columns (xst = 0), so the push primal may skip
// the columns it leaves untouched; both kernels take the decision from the same device state
__device__ __forceinline__ bool pp_marking(const PushPrimal& pp, const PPMode& md) {
    return pp.xst && md.push && md.delta && *(volatile unsigned*)pp.rcount <= pp.mark_rows;
}

// state the next primal starts from (written by thread 0 of block 0 of the active primal kernel)
__device__ __forceinline__ void pp_set_next(const PushPrimal& pp, int par, bool valid, int e) {
    (par ? pp.pvalid[0] : pp.pvalid[1]) = valid ? 1u : 0u;
    (par ? pp.pe[0] : pp.pe[1]) = e;
}
__device__ __forceinline__ bool pp_valid(const PushPrimal& pp, int par) {
    return pp.accx && *(volatile unsigned*)(par ? pp.pvalid + 1 : pp.pvalid) != 0u;
}

__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }

}  // namespace gfors
