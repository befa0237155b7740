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
    const int par = cta_parity(ctrl, kint, j);
    if (!cta_push_mode(pl, par)) return;
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

constexpr int PP_U4 = 4;
template <typename T>
__device__ __forceinline__ void ld4t(const T* __restrict__ p, T (&o)[PP_U4]) {
    if constexpr (sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
        const double2 v0 = reinterpret_cast<const double2*>(p)[0], v1 = reinterpret_cast<const double2*>(p)[1];
        o[0] = v0.x; o[1] = v0.y; o[2] = v1.x; o[3] = v1.y;
    }
}
template <typename T>
__device__ __forceinline__ void st4t(T* __restrict__ p, const T (&v)[PP_U4]) {
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
        reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
    }
}

// dual update from the accumulators (push mode only); keeps them (valid for the next delta push) and
// resets the next list
template <typename T>
__global__ void __launch_bounds__(256) k_push_rows(long long m, PushList pl, State<T> s, const double* __restrict__ g,
                                                   const double* __restrict__ rh, const signed char* __restrict__ rsign,
                                                   long long m1, const Ctrl* __restrict__ ctrl, long long kint, long long j,
                                                   double* __restrict__ u_out) {
    const int par = cta_parity(ctrl, kint, j);
    if (!cta_push_mode(pl, par)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) { push_reset_next(pl, par); pl_set_valid(pl, par ^ 1, true); }
    const T* __restrict__ yin = par ? s.y[1] : s.y[0];
    T* __restrict__ yout = par ? s.y[0] : s.y[1];
    const double tau2 = ctrl->tau2;
    auto one = [&](long long row, long long a, double sg, double gj, double rj, double yi, T& yt, T& wt) {
        const double u = sg * ((double)a * PUSH_INV);  // (K_u xbar_{k-1})_j
        double yn = yi + tau2 * (rj - gj * u);
        if (row < m1 && yn < 0.0) yn = 0.0;
        yt = (T)yn;
        wt = w_of(gj, sg, yt);
        if (u_out) u_out[row] = u;
    };
    // 4 consecutive rows per thread with 16-byte loads/stores (the row pass streams ~29 B per row)
    const long long m4 = (m / 4) * 4;
    for (long long r0 = 4 * (blockIdx.x * (long long)blockDim.x + threadIdx.x); r0 < m4;
         r0 += 4 * (gridDim.x * (long long)blockDim.x)) {
        const longlong2 a01 = *reinterpret_cast<const longlong2*>(pl.acc + r0);
        const longlong2 a23 = *reinterpret_cast<const longlong2*>(pl.acc + r0 + 2);
        const long long a[4] = {a01.x, a01.y, a23.x, a23.y};
        if (!pl.dvalid && (a[0] | a[1] | a[2] | a[3])) {
            *reinterpret_cast<longlong2*>(pl.acc + r0) = make_longlong2(0, 0);
            *reinterpret_cast<longlong2*>(pl.acc + r0 + 2) = make_longlong2(0, 0);
        }
        const char4 sg4 = *reinterpret_cast<const char4*>(rsign + r0);
        const double sg[4] = {(double)sg4.x, (double)sg4.y, (double)sg4.z, (double)sg4.w};
        const double2 g01 = __ldg(reinterpret_cast<const double2*>(g + r0)), g23 = __ldg(reinterpret_cast<const double2*>(g + r0 + 2));
        const double2 h01 = __ldg(reinterpret_cast<const double2*>(rh + r0)), h23 = __ldg(reinterpret_cast<const double2*>(rh + r0 + 2));
        const double gg[4] = {g01.x, g01.y, g23.x, g23.y}, hh[4] = {h01.x, h01.y, h23.x, h23.y};
        T yi[PP_U4], yo[PP_U4], wo[PP_U4];
        ld4t(yin + r0, yi);
#pragma unroll
        for (int u = 0; u < 4; ++u) one(r0 + u, a[u], sg[u], gg[u], hh[u], (double)yi[u], yo[u], wo[u]);
        st4t(yout + r0, yo);
        st4t(s.w + r0, wo);
    }
    for (long long row = m4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; row < m; row += gridDim.x * (long long)blockDim.x) {
        const long long a = pl.acc[row];
        if (!pl.dvalid && a) pl.acc[row] = 0;
        T yt, wt;
        one(row, a, (double)rsign[row], g[row], rh[row], (double)yin[row], yt, wt);
        yout[row] = yt;
        s.w[row] = wt;
    }
}

}  // namespace gfors
