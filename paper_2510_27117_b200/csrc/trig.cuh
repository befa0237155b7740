// trig.cuh — trigger-time indicator row pass on CTA row blocks with
// cp.async double-buffered gathers of the two vectors it needs (x_k and xbar_{k-1}).
//   v_j = (K_u x_k)_j      -> (K x_k + r)_j = rh_j - g_j rsign_j v_j       (primal feasibility gap)
//   d_j = (K_u (x_k - xbar_{k-1}))_j -> s^y_j = (y_{k-1} - y_k)_j / tau2 + g_j rsign_j d_j
// Dynamic shared memory: [2 stages][2 vectors][RB_NNZ] elements of T.
#pragma once
#include "rowblock.cuh"

namespace gfors {

template <typename T>
__device__ __forceinline__ void trig_issue(const Csr& A, const long long* __restrict__ blk_row, long long b,
                                           long long nblk, const T* __restrict__ v1, const T* __restrict__ v2,
                                           T* s1, T* s2) {
    if (b < nblk) {
        const long long p0 = __ldg(A.ptr + blk_row[b]);
        const int cnt = (int)(__ldg(A.ptr + blk_row[b + 1]) - p0);
        int cols[RB_U];
#pragma unroll
        for (int u = 0; u < RB_U; ++u) {
            const int t = u * RB_NT + threadIdx.x;
            cols[u] = t < cnt ? ldcs_i32(A.idx + p0 + t) : -1;
        }
#pragma unroll
        for (int u = 0; u < RB_U; ++u)
            if (cols[u] >= 0) {
                cp_async_elem(s1 + u * RB_NT + threadIdx.x, v1 + cols[u]);
                cp_async_elem(s2 + u * RB_NT + threadIdx.x, v2 + cols[u]);
            }
    }
    cp_async_commit();
}

template <typename T, int KIND>
__global__ void __launch_bounds__(RB_NT) k_trig_rows_cp(Csr K, const long long* __restrict__ blk_row, long long nblk,
                                                        State<T> s, const double* __restrict__ g,
                                                        const double* __restrict__ rh,
                                                        const signed char* __restrict__ rsign, long long m1,
                                                        const Ctrl* __restrict__ ctrl, long long kint, long long j,
                                                        double* __restrict__ part1) {
    extern __shared__ __align__(16) unsigned char trig_smem[];
    T* base = reinterpret_cast<T*>(trig_smem);  // [stage][vec][RB_NNZ]
    __shared__ double sh[32];
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ xk = par ? s.x[0] : s.x[1];
    const T* __restrict__ xbp = par ? s.xb[1] : s.xb[0];
    const T* __restrict__ yprev = par ? s.y[1] : s.y[0];
    const T* __restrict__ ynew = par ? s.y[0] : s.y[1];
    const double tau2 = ctrl->tau2;
    double ge = 0.0, eq = 0.0, sy2 = 0.0;
    int st = 0;
    trig_issue<T>(K, blk_row, blockIdx.x, nblk, xk, xbp, base, base + RB_NNZ);
    for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
        T* nx = base + (st ^ 1) * 2 * RB_NNZ;
        trig_issue<T>(K, blk_row, b + gridDim.x, nblk, xk, xbp, nx, nx + RB_NNZ);
        cp_async_wait1();
        __syncthreads();
        const T* sx = base + st * 2 * RB_NNZ;
        const T* sb = sx + RB_NNZ;
        const long long r0 = blk_row[b], r1 = blk_row[b + 1];
        const long long p0 = __ldg(K.ptr + r0);
        const int nr = (int)(r1 - r0);
        const int G = rb_group_size(nr);
        const int lane = threadIdx.x & (G - 1), grp = threadIdx.x / G, ngr = RB_NT / G;
        for (int rb = 0; rb < nr; rb += ngr) {
            const int rr = rb + grp;
            const long long row = r0 + rr;
            double v = 0.0, d = 0.0;
            if (rr < nr) {
                const long long q1 = __ldg(K.ptr + row + 1);
                for (long long q = __ldg(K.ptr + row) + lane; q < q1; q += G) {
                    const double kv = kval<KIND>(K.val, q);
                    const double a = (double)sx[q - p0];
                    v += kv * a;
                    d += kv * (a - (double)sb[q - p0]);
                }
            }
            v = rb_group_sum(v, G);
            d = rb_group_sum(d, G);
            if (lane == 0 && rr < nr) {
                const double sg = (KIND == KV_SIGN) ? (double)rsign[row] : 1.0;
                const double gj = g[row];
                const double gap = rh[row] - gj * (sg * v);
                if (row < m1) ge = fmax(ge, fmax(gap, 0.0)); else eq = fmax(eq, fabs(gap));
                const double sy = ((double)yprev[row] - (double)ynew[row]) / tau2 + gj * (sg * d);
                sy2 += sy * sy;
            }
        }
        __syncthreads();
        st ^= 1;
    }
    asm volatile("cp.async.wait_all;");
    const double a = block_max<RB_NT>(ge, sh);
    const double bb = block_max<RB_NT>(eq, sh);
    const double c = block_sum<RB_NT>(sy2, sh);
    if (threadIdx.x == 0) { part1[3 * blockIdx.x] = a; part1[3 * blockIdx.x + 1] = bb; part1[3 * blockIdx.x + 2] = c; }
}

template <typename T, int KIND>
inline size_t trig_cp_smem() { return 4 * RB_NNZ * sizeof(T); }

}  // namespace gfors
