// sparse_primal.cuh — primal half-step that skips the gathers of zero duals.
//
// K'y only needs w_j = g_j rsign_j y_j for the rows with y_j != 0.  On covering-type instances most
// inequality duals sit at the clamp y_j = 0 (config 5: 1 % of rows active after 100 iterations,
// 37 % after 2000), so gathering w for every nonzero wastes L1TEX wavefronts.  The dual kernel's
// output is summarised in a bitmap of nonzero w (1 bit per row, k_nzmask), every CTA stages the
// whole bitmap in shared memory (m/8 bytes; 125 KB for m = 10^6) and issues a cp.async gather only
// for nonzeros whose row bit is set — a shared-memory bit test (~bank-conflict cost) replaces a
// random L2 gather.  Skipped terms are exact zeros; reductions keep a fixed order (deterministic).
// One CTA of 1024 threads per SM; 8 nonzeros per thread per row block.
#pragma once
#include "rowblock.cuh"

namespace gfors {

constexpr int SP_NT = 1024;
constexpr int SP_NNZ = 8192;  // nonzeros per row block
constexpr int SP_U = SP_NNZ / SP_NT;

// bits[k] bit t = (w[32k + t] != 0)
template <typename T>
__global__ void k_nzmask(const T* __restrict__ w, long long m, unsigned* __restrict__ bits) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const long long nwords = (m + 31) / 32;
    for (long long k = warp; k < nwords; k += nwarps) {
        const long long j = 32 * k + lane;
        const bool nz = j < m && w[j] != (T)0;
        const unsigned b = __ballot_sync(0xffffffffu, nz);
        if (lane == 0) bits[k] = b;
    }
}

__device__ __forceinline__ void sp_load_idx(const Csr& A, const long long* __restrict__ blk_row, long long b,
                                            long long nblk, int (&rows)[SP_U]) {
    if (b < nblk) {
        const long long p0 = __ldg(A.ptr + blk_row[b]);
        const int cnt = (int)(__ldg(A.ptr + blk_row[b + 1]) - p0);
#pragma unroll
        for (int u = 0; u < SP_U; ++u) {
            const int t = u * SP_NT + threadIdx.x;
            rows[u] = t < cnt ? ldcs_i32(A.idx + p0 + t) : -1;
        }
    } else {
#pragma unroll
        for (int u = 0; u < SP_U; ++u) rows[u] = -1;
    }
}

template <typename T>
__device__ __forceinline__ void sp_issue(const int (&rows)[SP_U], const T* __restrict__ w, const unsigned* sbits, T* sv) {
#pragma unroll
    for (int u = 0; u < SP_U; ++u) {
        const int j = rows[u];
        if (j < 0) continue;
        T* dst = sv + u * SP_NT + threadIdx.x;
        if ((sbits[j >> 5] >> (j & 31)) & 1u) cp_async_elem(dst, w + j);
        else *dst = (T)0;
    }
    cp_async_commit();
}

__device__ __forceinline__ int sp_group_size(int nr) {
    int G = 32;
    while (G > 1 && G * nr > SP_NT) G >>= 1;
    return G;
}

// Row blocks hold <= SP_NT rows, so phase 2 is one pass with <= one row per G-lane group; the row
// pointers and epilogue operands of the CTA's NEXT block are loaded into registers while the current
// block is reduced (latency hidden behind a whole phase instead of exposed at its start).
struct SpRow {
    long long q0, q1;
    double xi, ci;
    int G;
    bool valid;
};

template <typename T>
__device__ __forceinline__ SpRow sp_prefetch_row(const Csr& Kt, const long long* __restrict__ blk_row, long long b,
                                                 long long nblk, const T* __restrict__ xin, const T* __restrict__ cs) {
    SpRow r{0, 0, 0.0, 0.0, 1, false};
    if (b < nblk) {
        const long long r0 = blk_row[b];
        const int nr = (int)(blk_row[b + 1] - r0);
        r.G = sp_group_size(nr);
        const int grp = threadIdx.x / r.G;
        if (grp < nr) {
            const long long i = r0 + grp;
            r.valid = true;
            r.q0 = __ldg(Kt.ptr + i);
            r.q1 = __ldg(Kt.ptr + i + 1);
            if ((threadIdx.x & (r.G - 1)) == 0) { r.xi = (double)xin[i]; r.ci = (double)cs[i]; }
        }
    }
    return r;
}

template <typename T, int KIND, bool HASQ>
__global__ void __launch_bounds__(SP_NT, 1) k_primal_sparse(Csr Kt, const long long* __restrict__ blk_row, long long nblk,
                                                            const unsigned* __restrict__ bits, long long nwords,
                                                            Csr Q, const T* __restrict__ qs, State<T> s,
                                                            const T* __restrict__ cs, const Ctrl* __restrict__ ctrl,
                                                            long long kint, long long j, PushList pl) {
    extern __shared__ __align__(16) unsigned char sp_smem[];
    __shared__ unsigned s_cnt, s_base;
    __shared__ int s_list[SP_NT];
    __shared__ bool s_en, s_dd;
    T* svb = reinterpret_cast<T*>(sp_smem);                          // [2][SP_NNZ]
    unsigned* sbits = reinterpret_cast<unsigned*>(svb + 2 * SP_NNZ);  // [nwords]
    for (long long k = threadIdx.x; k < nwords; k += SP_NT) sbits[k] = __ldg(bits + k);
    __syncthreads();
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ xin = par ? s.x[1] : s.x[0];
    T* __restrict__ xout = par ? s.x[0] : s.x[1];
    T* __restrict__ xbout = par ? s.xb[0] : s.xb[1];
    const T* __restrict__ xbprev = par ? s.xb[1] : s.xb[0];
    const double rho = ctrl->rho, tau1 = ctrl->tau1;
    int st = 0;
    int nxt[SP_U];
    sp_load_idx(Kt, blk_row, blockIdx.x, nblk, nxt);
    sp_issue<T>(nxt, s.w, sbits, svb);
    sp_load_idx(Kt, blk_row, blockIdx.x + gridDim.x, nblk, nxt);
    SpRow cur = sp_prefetch_row<T>(Kt, blk_row, blockIdx.x, nblk, xin, cs);
    for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
        sp_issue<T>(nxt, s.w, sbits, svb + (st ^ 1) * SP_NNZ);
        sp_load_idx(Kt, blk_row, b + 2LL * gridDim.x, nblk, nxt);
        const SpRow nrow = sp_prefetch_row<T>(Kt, blk_row, b + gridDim.x, nblk, xin, cs);
        if (threadIdx.x == 0) {
            s_en = pl.acc && *(volatile unsigned*)pl_count(pl, par ^ 1) <= pl.thr;
            s_dd = pl.acc && pl_valid(pl, par ^ 1);
        }
        cp_async_wait1();
        __syncthreads();
        const T* sv = svb + st * SP_NNZ;
        const long long r0 = blk_row[b];
        const long long p0 = __ldg(Kt.ptr + r0);
        const int G = cur.G;
        const int lane = threadIdx.x & (G - 1);
        const long long i = r0 + threadIdx.x / G;
        double a = 0.0, bq = 0.0;
        if (cur.valid) {
            a = rb_row_sum<T, KIND, true>(Kt, sv, p0, cur.q0, cur.q1, lane, G);
            if constexpr (HASQ) {
                if (Q.pre) {
                    if (lane == 0) bq = Q.pre[i];
                } else {
                    for (long long q = __ldg(Q.ptr + i) + lane; q < __ldg(Q.ptr + i + 1); q += G)
                        bq += (double)__ldg(qs + q) * (double)__ldg(xin + __ldg(Q.idx + q));
                }
            }
        }
        a = rb_group_sum(a, G);
        if constexpr (HASQ) bq = rb_group_sum(bq, G);
        bool nz = false;
        if (lane == 0 && cur.valid) {
            const double xi = cur.xi;
            const double delta = ((cur.ci + rho) - a) + 2.0 * bq - 2.0 * rho * xi;
            double xn = xi - tau1 * delta;
            xn = xn < 0.0 ? 0.0 : (xn > 1.0 ? 1.0 : xn);
            xout[i] = (T)xn;
            const T xbn = (T)(2.0 * xn - xi);
            xbout[i] = xbn;
            nz = pl_listed((bool)s_dd, xbn, s_dd ? xbprev[i] : (T)0);
        }
        push_append<SP_NT>(pl, par ^ 1, nz, (int)i, s_en, &s_cnt, &s_base, s_list);
        __syncthreads();
        st ^= 1;
        cur = nrow;
    }
    asm volatile("cp.async.wait_all;");
}

template <typename T>
inline size_t sparse_primal_smem(long long m) {
    return 2 * SP_NNZ * sizeof(T) + ((m + 31) / 32) * sizeof(unsigned);
}

}  // namespace gfors
