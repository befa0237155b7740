// shard.cuh — sample-sharded EvalBest across ranks.
//
// Every rank runs the same deterministic PDHG trajectory (replicated) and draws its own global
// sample words [rank*W, (rank+1)*W).  After each sampling round a rank publishes one 32-byte record
// (best feasible z of its batch, its global sample index, valid flag) with ncclAllGather inside the
// loop graph; every rank then applies the same merge (lowest z, ties -> lowest global index,
// replace the incumbent iff strictly better — reading R11), so incumbents, improvement flags and
// therefore CheckHalt decisions are identical on all ranks.  The winning candidate's bits are not
// sent: x_k is bit-identical on all ranks, so each rank regenerates the winning lane from the
// Philox contract (one word per variable).
#pragma once
#include <dlfcn.h>

#include "common.cuh"
#include "sample_eval.cuh"

// minimal NCCL ABI (stable across 2.x): resolved at run time with dlopen so the library loads and
// runs single-rank without NCCL, and shares the NCCL already loaded by the host process (torch)
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclSuccess_ = 0 } ncclResult_t_;
typedef int ncclResult_t;
enum { ncclUint8_ = 1, ncclFloat64_ = 8 };

namespace gfors {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    void load() {
        if (ok) return;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror(); return; }
        GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
        GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        ok = GetUniqueId && CommInitRank && CommDestroy && AllGather && GetErrorString && GroupStart && GroupEnd;
        if (!ok) why = "libnccl.so.2 lacks a required symbol";
    }
};

inline NcclApi& nccl() {
    static NcclApi api;
    api.load();
    return api;
}

// rec[0] = best z of this rank's batch (+inf if none), rec[1] = its global sample index,
// rec[2] = 1 if a feasible candidate exists.  Single block of 256 threads.
// rec[3] = 1 if this rank's own time limit has passed (or a test forces it from block force_blk on):
// the flags are OR-ed by the merge, so every rank halts at the same block (CheckHalt L38-40).
__global__ void __launch_bounds__(256) k_local_record(const double* __restrict__ z, const unsigned long long* __restrict__ viol,
                                                      long long lanes, long long word_off, Ctrl* __restrict__ ctrl,
                                                      double* __restrict__ rec, int count_round, long long force_blk) {
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
            if (l2 >= 0 && (sl[threadIdx.x] < 0 || z2 < sz[threadIdx.x] || (z2 == sz[threadIdx.x] && l2 < sl[threadIdx.x]))) {
                sz[threadIdx.x] = z2; sl[threadIdx.x] = l2;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (count_round) ctrl->rounds += 1;
        const long long l = sl[0];
        rec[0] = l >= 0 ? sz[0] : INFINITY;
        rec[1] = l >= 0 ? (double)(64 * word_off + l) : -1.0;
        rec[2] = l >= 0 ? 1.0 : 0.0;
        const bool late = globaltimer_ns() >= ctrl->deadline_ns || (force_blk >= 0 && ctrl->blk >= force_blk);
        rec[3] = late ? 1.0 : 0.0;
    }
}

// identical on every rank: pick the winner record, update the incumbent iff strictly better; OR the
// time-limit flags
__global__ void k_merge_records(const double* __restrict__ all, int world, Ctrl* __restrict__ ctrl, long long kint,
                                int r, int kr, long long* __restrict__ regen /* [0]=global index or -1, [1]=round */) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int best = -1;
    for (int q = 0; q < world; ++q) {
        const double* rq = all + 4 * q;
        if (rq[3] != 0.0) ctrl->tl_any = 1;  // some rank's time limit passed: all ranks halt after this block
        if (rq[2] == 0.0) continue;
        if (best < 0 || rq[0] < all[4 * best] || (rq[0] == all[4 * best] && rq[1] < all[4 * best + 1])) best = q;
    }
    regen[0] = -1;
    ctrl->win_lane = -1;
    if (best >= 0 && all[4 * best] < ctrl->z_best) {
        ctrl->z_best = all[4 * best];
        ctrl->has_inc = 1;
        ctrl->improved = 1;
        ctrl->found_ns = globaltimer_ns() - ctrl->t0_ns;
        ctrl->found_iter = (ctrl->blk + 1) * kint;
        ctrl->found_round = ctrl->blk * kr + r;
        ctrl->found_index = (long long)all[4 * best + 1];
        regen[0] = ctrl->found_index;
        regen[1] = ctrl->found_round;
    }
}

// x_best[i] = bit (l mod 64) of the Philox word (i, l / 64, round) of x_k — the winner's candidate
template <typename T>
__global__ void k_regen_best(const T* __restrict__ xa, const T* __restrict__ xb2, long long n, const Ctrl* __restrict__ ctrl,
                             long long kint, uint2 key, const long long* __restrict__ regen,
                             unsigned char* __restrict__ xbest) {
    const long long gl = regen[0];
    if (gl < 0) return;
    const unsigned round = (unsigned)regen[1];
    const long long b = ctrl->blk;
    const T* __restrict__ p = (((b + 1) * kint) & 1) ? xb2 : xa;
    const unsigned wg = (unsigned)(gl >> 6);
    const int bit = (int)(gl & 63);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        xbest[i] = (unsigned char)((bernoulli_word((double)p[i], (unsigned)i, wg, round, key) >> bit) & 1ull);
}

// ---------------------------------------------------------------------------------------------
// Row-sharded dual (params.row_shard): rank q computes the dual of
// rows [rlo[q], rlo[q+1]) only; the y values of those rows are packed into slot q of a gather buffer
// (maxrows entries per slot, ncclAllGather in place), and every rank unpacks all slots into y and
// recomputes w_j = g_j rsign_j y_j exactly as the dual kernel does (w_of), so the replicated rest of
// the iteration sees bit-identical inputs.  At the trigger iteration the same for u = K_u xbar_{k-1}.
// The dual's output buffer is picked by the iteration parity, as in the dual kernels.
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void k_rs_pack(State<T> s, const Ctrl* __restrict__ ctrl, long long kint, long long j, long long r0,
                          long long nrows, T* __restrict__ slot, const double* __restrict__ u, double* __restrict__ uslot) {
    const int par = (int)(iter_index(ctrl, kint, j) & 1);
    const T* __restrict__ yout = par ? s.y[0] : s.y[1];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nrows; t += gridDim.x * (long long)blockDim.x) {
        slot[t] = yout[r0 + t];
        if (uslot) uslot[t] = u[r0 + t];
    }
}

template <typename T, int KIND>
__global__ void k_rs_unpack(State<T> s, const Ctrl* __restrict__ ctrl, long long kint, long long j,
                            const long long* __restrict__ rlo, int R, long long maxrows, const T* __restrict__ gath,
                            const double* __restrict__ g, const signed char* __restrict__ rsign,
                            const double* __restrict__ ugath, double* __restrict__ u) {
    const int par = (int)(iter_index(ctrl, kint, j) & 1);
    T* __restrict__ yout = par ? s.y[0] : s.y[1];
    const long long total = (long long)R * maxrows;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * (long long)blockDim.x) {
        const int q = (int)(idx / maxrows);
        const long long row = rlo[q] + (idx - (long long)q * maxrows);
        if (row >= rlo[q + 1]) continue;
        const T yt = gath[idx];
        yout[row] = yt;
        const double sg = (KIND == KV_SIGN) ? (double)rsign[row] : 1.0;
        s.w[row] = w_of(g[row], sg, yt);
        if (ugath) u[row] = ugath[idx];
    }
}

}  // namespace gfors
