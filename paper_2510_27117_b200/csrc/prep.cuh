// prep.cuh — Preprocess on the device: row 2-norms of K, spectral norms of Q
// and of the row-normalised K by power iteration (readings R4-R6), deterministic reductions.
#pragma once
#include "common.cuh"
#include "pdhg.cuh"

namespace gfors {

// s_j = ||K_u row j||_2 (exact for integer data); zero rows -> 1
template <int KIND>
__global__ void k_row_norms(Csr K, double* __restrict__ s, unsigned long long* __restrict__ zero_rows) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < K.rows; j += gridDim.x * (long long)blockDim.x) {
        double a = 0.0;
        for (long long p = K.ptr[j]; p < K.ptr[j + 1]; ++p) { const double v = kval<KIND>(K.val, p); a += v * v; }
        a = sqrt(a);
        if (a == 0.0) { a = 1.0; atomicAdd(zero_rows, 1ull); }
        s[j] = a;
    }
}

// w_j = rowscale_j * sum_p val_p * v[idx_p]   (rowscale may be null; SIGN rows use rsign)
template <int KIND>
__global__ void __launch_bounds__(256) k_spmv_rows(Csr A, const signed char* __restrict__ rsign,
                                                   const double* __restrict__ rowscale, const double* __restrict__ v,
                                                   double* __restrict__ w) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long j = warp; j < A.rows; j += nwarps) {
        double a = 0.0;
        for (long long p = A.ptr[j] + lane; p < A.ptr[j + 1]; p += 32) a += kval<KIND>(A.val, p) * v[A.idx[p]];
        a = warp_sum(a);
        if (lane == 0) {
            if (KIND == KV_SIGN && rsign) a *= (double)rsign[j];
            if (rowscale) a /= rowscale[j];
            w[j] = a;
        }
    }
}

// the per-row factor of the transposed product, once per row: w'_j = (w_j / s_j) * rsign_j (the same
// operations, in the same order, as k_spmv_cols applies per nonzero: identical terms)
template <int KIND>
__global__ void __launch_bounds__(256) k_prescale(const double* __restrict__ w, const double* __restrict__ rowscale,
                                                  const signed char* __restrict__ rsign, long long m,
                                                  double* __restrict__ out) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < m; j += gridDim.x * (long long)blockDim.x) {
        double wj = w[j];
        if (rowscale) wj /= rowscale[j];
        if (KIND == KV_SIGN && rsign) wj *= (double)rsign[j];
        out[j] = wj;
    }
}

// u_i = sum_j val_ji * w'_j with G lanes per column (short columns: a whole warp per column left most
// lanes idle); every lane of the warp runs the same trip count (the shuffles need all 32)
template <int KIND, int G>
__global__ void __launch_bounds__(256) k_spmv_cols_g(Csr At, const double* __restrict__ wp, double* __restrict__ u) {
    constexpr int PER = 32 / G;  // columns per warp and trip
    const int lane = threadIdx.x & 31, sub = lane & (G - 1);
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long i0 = warp * PER; i0 < At.rows; i0 += nwarps * PER) {
        const long long i = i0 + lane / G;
        double a = 0.0;
        if (i < At.rows)
            for (long long p = At.ptr[i] + sub; p < At.ptr[i + 1]; p += G) a += kval<KIND>(At.val, p) * wp[At.idx[p]];
        for (int o = G >> 1; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o, G);
        if (sub == 0 && i < At.rows) u[i] = a;
    }
}

// transposed product through the explicit transpose CSR: u_i = sum_j val_ji * (w_j / s_j) * rsign_j
template <int KIND>
__global__ void __launch_bounds__(256) k_spmv_cols(Csr At, const signed char* __restrict__ rsign,
                                                   const double* __restrict__ rowscale, const double* __restrict__ w,
                                                   double* __restrict__ u) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long i = warp; i < At.rows; i += nwarps) {
        double a = 0.0;
        for (long long p = At.ptr[i] + lane; p < At.ptr[i + 1]; p += 32) {
            const int j = At.idx[p];
            double wj = w[j];
            if (rowscale) wj /= rowscale[j];
            if (KIND == KV_SIGN && rsign) wj *= (double)rsign[j];
            a += kval<KIND>(At.val, p) * wj;
        }
        a = warp_sum(a);
        if (lane == 0) u[i] = a;
    }
}

// fixed-order sum of squares: per-block partials then one block
__global__ void __launch_bounds__(256) k_sumsq_partial(const double* __restrict__ v, long long n, double* __restrict__ part) {
    __shared__ double sh[32];
    double a = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        a += v[i] * v[i];
    a = block_sum<256>(a, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = a;
}
__global__ void __launch_bounds__(256) k_sum_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
    __shared__ double sh[32];
    double a = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[b];
    a = block_sum<256>(a, sh);
    if (threadIdx.x == 0) *out = sqrt(a);
}
// v = u / nrm
__global__ void k_scale_vec(const double* __restrict__ u, const double* __restrict__ nrm, long long n, double* __restrict__ v) {
    const double s = *nrm;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        v[i] = u[i] / s;
}
__global__ void k_fill(double* __restrict__ v, long long n, double val) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        v[i] = val;
}
// Philox restart vector of reading R5: v_i = (out0 + 0.5) 2^-32, key (0x9E3779B9, 0), ctr (i,0,0,0)
__global__ void k_philox_vec(double* __restrict__ v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x) {
        const uint4 o = philox4x32_10(make_uint4((unsigned)i, 0u, 0u, 0u), make_uint2(0x9E3779B9u, 0u));
        v[i] = ((double)o.x + 0.5) * (1.0 / 4294967296.0);
    }
}

// Loop data in iterate precision: g_j = 1/(s_j kappa), rh_j = (r_j/s_j)/kappa; cs = c/omega; qs = Q/omega
template <typename T>
__global__ void k_make_rowdata(long long m, const double* __restrict__ s, const double* __restrict__ ru, double kappa,
                               T* __restrict__ g, T* __restrict__ rh) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < m; j += gridDim.x * (long long)blockDim.x) {
        g[j] = (T)((1.0 / s[j]) / kappa);
        rh[j] = (T)((ru[j] / s[j]) / kappa);
    }
}
template <typename T>
__global__ void k_scale_to(const double* __restrict__ a, long long n, double omega, T* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        out[i] = (T)(a[i] / omega);
}

// state init: x = xbar = 0.5, y = 0 (reading R14) in buffer 0
template <typename T>
__global__ void k_init_state(State<T> s, long long n, long long m) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x) {
        s.x[0][i] = (T)0.5; s.xb[0][i] = (T)0.5; s.x[1][i] = (T)0.5; s.xb[1][i] = (T)0.5;
    }
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < m; j += gridDim.x * (long long)blockDim.x) {
        s.y[0][j] = (T)0; s.y[1][j] = (T)0; s.w[j] = (T)0;
    }
}
template <typename T>
__global__ void k_to_T(const double* __restrict__ a, long long n, T* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        out[i] = (T)a[i];
}
template <typename T>
__global__ void k_from_T(const T* __restrict__ a, long long n, double* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x)
        out[i] = (double)a[i];
}

}  // namespace gfors
