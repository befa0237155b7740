// push_dual.cuh — dual half-step from the nonzero columns of xbar ("push" mode).
//
// As rho grows the iterate binarises and most xbar_i = 2x_k - x_{k-1} become exactly 0 (config 5:
// 49 % after 500 iterations, 95 % after 2000).  K_u xbar then only involves the nonzero columns, so
// instead of one random gather per nonzero of K (gather mode, k_dual_rb) the primal kernel of the
// previous iteration appends its nonzero columns to a list, and this mode scatters
// xbar_i (fixed point, 2^-40 resolution) into int64 row accumulators with integer atomics through
// the transposed CSR — integer addition is associative, so the result does not depend on the
// order of the atomics (deterministic) — then a row pass applies the dual update and clears the
// accumulators.  The mode is chosen on the device from the list length (<= thr -> push), so the
// captured graph runs both kernels and the unused one exits at once.  Used for +-1 pattern
// matrices (bounded row sums: |sum| <= 2 * 2^20 * 2^40 < 2^63).  Delta push: see push_list.cuh.
#pragma once
#include "rowblock.cuh"
#include "push_list.cuh"

namespace gfors {

// scatter round(xbar_i 2^40) of the listed columns into the row accumulators of K_u rows (push mode
// only); with valid accumulators (delta push) the change round(xbar_k 2^40) - round(xbar_{k-1} 2^40)
template <typename T>
__global__ void __launch_bounds__(256) k_push_scatter(Csr Kt, PushList pl, State<T> s, const Ctrl* __restrict__ ctrl,
                                                      long long kint, long long j) {
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    if (!push_mode(pl, par)) return;
    const bool delta = pl_valid(pl, par);
    const T* __restrict__ xb = par ? s.xb[1] : s.xb[0];      // xbar_{k-1}
    const T* __restrict__ xbp = par ? s.xb[0] : s.xb[1];     // xbar_{k-2} (delta push only)
    const long long cnt = *pl_count(pl, par);
    const int* __restrict__ list = pl_list(pl, par);
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * (long long)blockDim.x) {
        const int i = list[k];
        long long v = __double2ll_rn((double)xb[i] * PUSH_SCALE);
        if (delta) v -= __double2ll_rn((double)xbp[i] * PUSH_SCALE);
        if (v == 0) continue;
        const long long q1 = __ldg(Kt.ptr + i + 1);
        for (long long q = __ldg(Kt.ptr + i); q < q1; ++q)
            atomicAdd(reinterpret_cast<unsigned long long*>(pl.acc + __ldg(Kt.idx + q)), (unsigned long long)v);
    }
}

// dual update from the accumulators (push mode only); keeps them (valid for the next delta push) and
// resets the next list
template <typename T>
__global__ void __launch_bounds__(256) k_push_rows(long long m, PushList pl, State<T> s, const double* __restrict__ g,
                                                   const double* __restrict__ rh, const signed char* __restrict__ rsign,
                                                   long long m1, const Ctrl* __restrict__ ctrl, long long kint, long long j,
                                                   double* __restrict__ u_out) {
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    if (!push_mode(pl, par)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) { push_reset_next(pl, par); pl_set_valid(pl, par ^ 1, true); }
    const T* __restrict__ yin = par ? s.y[1] : s.y[0];
    T* __restrict__ yout = par ? s.y[0] : s.y[1];
    const double tau2 = ctrl->tau2;
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < m; row += gridDim.x * (long long)blockDim.x) {
        const long long a = pl.acc[row];
        if (!pl.dvalid && a) pl.acc[row] = 0;
        const double sg = (double)rsign[row];
        const double u = sg * ((double)a * PUSH_INV);  // (K_u xbar_{k-1})_j
        const double gj = g[row];
        double yn = (double)yin[row] + tau2 * (rh[row] - gj * u);
        if (row < m1 && yn < 0.0) yn = 0.0;
        const T yt = (T)yn;
        yout[row] = yt;
        s.w[row] = w_of(gj, sg, yt);
        if (u_out) u_out[row] = u;
    }
}

}  // namespace gfors
