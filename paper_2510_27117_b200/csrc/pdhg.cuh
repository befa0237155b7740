// pdhg.cuh — Alg. 2 as two fused HBM-streaming kernels per iteration,
// plus the trigger-time indicator passes.
//
// Notation: the library keeps the canonical USER matrix K_u (rows GE first)
// and a per-row scale g_j = 1/(s_j kappa), so the scaled saddle matrix is K = -diag(g) K_u and
// r = diag(g) r_u.  State vectors are ping-ponged by iteration parity:
// iteration kk reads buffer (kk&1) and writes buffer (kk&1)^1, so x_{k-1}, xbar_{k-1} and
// y_{k-1} survive the step for free (needed by the Thm. 2 residuals) and Q x_{k-1} never races
// with the write of x_k.
#pragma once
#include "common.cuh"

namespace gfors {

template <typename T>
struct State {
    T* x[2];
    T* xb[2];
    T* y[2];
    T* w;  // w_j = g_j * (rsign_j) * y_j  (so K'y = -K_u' w)
};

// w_j from the STORED dual y_j (already rounded to T), so w is a function of the stored y alone and
// the delta push (push_primal.cuh) can recompute w_{k-1} bit-exactly from y_{k-1}
template <typename T>
__device__ __forceinline__ T w_of(double gj, double sg, T yt) { return (T)(gj * sg * (double)yt); }

struct Csr {
    const long long* ptr;  // int64 [rows+1]
    const int* idx;        // int32 [nnz]
    const void* val;       // by KKind (nullptr for SIGN)
    long long rows;
    const double* pre = nullptr;  // Q only: precomputed row products (dense-Q path, dense_q.cuh)
};

// Row-segment plan for long rows: segment s covers nonzeros [seg_start[s], seg_start[s+1]),
// row r owns segments [row_seg[r], row_seg[r+1]).
struct SegPlan {
    const long long* seg_start;
    const int* seg_row;
    const long long* row_seg;
    long long nseg;
};

__device__ __forceinline__ long long iter_index(const Ctrl* ctrl, long long kint, long long j) {
    return (kint ? ctrl->blk * kint : 0) + j;
}

// ---------------------------------------------------------------------------------------------
// Dual half-step: y_k = Pi( y_{k-1} + tau2 (K xbar_{k-1} + r) ), Pi clamps GE rows
// at 0; fused: w_j = g_j rsign_j y_j for the primal gather.  SUB lanes per row, rows handed out
// warp-uniformly so every shuffle has all 32 lanes present.
// ---------------------------------------------------------------------------------------------
template <typename T, int KIND, int SUB>
__global__ void __launch_bounds__(256) k_dual(Csr K, State<T> s, const double* __restrict__ g,
                                              const double* __restrict__ rh, const signed char* __restrict__ rsign,
                                              long long m1, const Ctrl* __restrict__ ctrl,
                                              long long kint, long long j) {
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ xb = (par ? s.xb[1] : s.xb[0]);
    const T* __restrict__ yin = (par ? s.y[1] : s.y[0]);
    T* __restrict__ yout = (par ? s.y[0] : s.y[1]);
    const double tau2 = ctrl->tau2;
    constexpr int RPW = 32 / SUB;  // rows per warp
    const int lane = threadIdx.x & (SUB - 1);
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const int gsub = (threadIdx.x & 31) / SUB;
    for (long long base = warp * RPW; base < K.rows; base += nwarps * RPW) {
        const long long row = base + gsub;
        double acc = 0.0;
        if (row < K.rows) {
            const long long p0 = __ldg(K.ptr + row), p1 = __ldg(K.ptr + row + 1);
            long long p = p0 + lane;
            for (; p + 3 * SUB < p1; p += 4 * SUB) {
                const int c0 = __ldg(K.idx + p), c1 = __ldg(K.idx + p + SUB);
                const int c2 = __ldg(K.idx + p + 2 * SUB), c3 = __ldg(K.idx + p + 3 * SUB);
                const double v0 = (double)__ldg(xb + c0), v1 = (double)__ldg(xb + c1);
                const double v2 = (double)__ldg(xb + c2), v3 = (double)__ldg(xb + c3);
                if constexpr (KIND == KV_SIGN) acc += (v0 + v1) + (v2 + v3);
                else acc += (kval<KIND>(K.val, p) * v0 + kval<KIND>(K.val, p + SUB) * v1) +
                            (kval<KIND>(K.val, p + 2 * SUB) * v2 + kval<KIND>(K.val, p + 3 * SUB) * v3);
            }
            for (; p < p1; p += SUB) acc += kval<KIND>(K.val, p) * (double)__ldg(xb + __ldg(K.idx + p));
        }
        acc = group_sum<SUB>(acc);
        if (lane == 0 && row < K.rows) {
            const double sg = (KIND == KV_SIGN) ? (double)rsign[row] : 1.0;
            const double gj = (double)g[row];
            const double u = sg * acc;  // (K_u xbar)_j
            double yn = (double)yin[row] + tau2 * ((double)rh[row] - gj * u);
            if (row < m1 && yn < 0.0) yn = 0.0;
            const T yt = (T)yn;
            yout[row] = yt;
            s.w[row] = w_of(gj, sg, yt);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Primal half-step:  delta = c + rho + K'y_k + 2Qx_{k-1} - 2 rho x_{k-1},
// x_k = Pi_[0,1](x_{k-1} - tau1 delta), xbar_k = 2x_k - x_{k-1}.  One SUB-lane group per column
// over the transposed CSR of K_u (and the CSR row of Q).
// ---------------------------------------------------------------------------------------------
template <typename T, int KIND, int SUB, bool HASQ>
__global__ void __launch_bounds__(256) k_primal(Csr Kt, Csr Q, const T* __restrict__ qs, State<T> s,
                                                const T* __restrict__ cs, const Ctrl* __restrict__ ctrl,
                                                long long kint, long long j) {
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ xin = (par ? s.x[1] : s.x[0]);
    T* __restrict__ xout = (par ? s.x[0] : s.x[1]);
    T* __restrict__ xbout = (par ? s.xb[0] : s.xb[1]);
    const T* __restrict__ w = s.w;
    const double rho = ctrl->rho, tau1 = ctrl->tau1;
    constexpr int RPW = 32 / SUB;
    const int lane = threadIdx.x & (SUB - 1);
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const int gsub = (threadIdx.x & 31) / SUB;
    for (long long base = warp * RPW; base < Kt.rows; base += nwarps * RPW) {
        const long long i = base + gsub;
        double a = 0.0, b = 0.0;
        if (i < Kt.rows) {
            const long long p0 = __ldg(Kt.ptr + i), p1 = __ldg(Kt.ptr + i + 1);
            long long p = p0 + lane;
            for (; p + 3 * SUB < p1; p += 4 * SUB) {
                const int r0 = __ldg(Kt.idx + p), r1 = __ldg(Kt.idx + p + SUB);
                const int r2 = __ldg(Kt.idx + p + 2 * SUB), r3 = __ldg(Kt.idx + p + 3 * SUB);
                const double v0 = (double)__ldg(w + r0), v1 = (double)__ldg(w + r1);
                const double v2 = (double)__ldg(w + r2), v3 = (double)__ldg(w + r3);
                if constexpr (KIND == KV_SIGN) a += (v0 + v1) + (v2 + v3);
                else a += (kval<KIND>(Kt.val, p) * v0 + kval<KIND>(Kt.val, p + SUB) * v1) +
                          (kval<KIND>(Kt.val, p + 2 * SUB) * v2 + kval<KIND>(Kt.val, p + 3 * SUB) * v3);
            }
            for (; p < p1; p += SUB) a += kval<KIND>(Kt.val, p) * (double)__ldg(w + __ldg(Kt.idx + p));
            if constexpr (HASQ) {
                if (Q.pre) {
                    if (lane == 0) b = Q.pre[i];
                } else {
                    const long long q0 = __ldg(Q.ptr + i), q1 = __ldg(Q.ptr + i + 1);
                    for (long long q = q0 + lane; q < q1; q += SUB)
                        b += (double)__ldg(qs + q) * (double)__ldg(xin + __ldg(Q.idx + q));
                }
            }
        }
        a = group_sum<SUB>(a);
        if constexpr (HASQ) b = group_sum<SUB>(b);
        if (lane == 0 && i < Kt.rows) {
            const double xi = (double)xin[i];
            // K'y = -a  (K = -diag(g) K_u, w = g y)
            const double delta = (((double)cs[i] + rho) - a) + 2.0 * b - 2.0 * rho * xi;
            double xn = xi - tau1 * delta;
            xn = xn < 0.0 ? 0.0 : (xn > 1.0 ? 1.0 : xn);
            xout[i] = (T)xn;
            xbout[i] = (T)(2.0 * xn - xi);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Long-row path: one warp per fixed-length segment writes a partial sum (deterministic), a
// second kernel combines a row's partials in segment order.  Used for rows/columns too long or
// too few for the group kernels (e.g. the 50 x 50k multi-knapsack rows).
// part[s] = sum_{p in seg s} val_p * (va[idx_p] - (vb ? vb[idx_p] : 0))
// ---------------------------------------------------------------------------------------------
template <typename T, int KIND>
__global__ void __launch_bounds__(256) k_seg_partial(Csr A, SegPlan sp, const T* __restrict__ va0,
                                                     const T* __restrict__ va1, const T* __restrict__ vb0,
                                                     const T* __restrict__ vb1, int sel_mode,
                                                     const Ctrl* __restrict__ ctrl, long long kint, long long j,
                                                     double* __restrict__ part) {
    // sel_mode 0: va = va0 (no parity); 1: va = va{par} (input side); 2: va = va{par^1} (output side);
    // vb (optional) always the input side of its pair
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ va = sel_mode == 0 ? va0 : (sel_mode == 1 ? (par ? va1 : va0) : (par ? va0 : va1));
    const T* __restrict__ vb = vb0 ? (par ? vb1 : vb0) : nullptr;
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long sgi = warp; sgi < sp.nseg; sgi += nwarps) {
        const long long p0 = __ldg(sp.seg_start + sgi), p1 = __ldg(sp.seg_start + sgi + 1);
        double acc = 0.0;
        long long p = p0 + lane;
        for (; p + 96 < p1; p += 128) {
            const int c0 = __ldg(A.idx + p), c1 = __ldg(A.idx + p + 32);
            const int c2 = __ldg(A.idx + p + 64), c3 = __ldg(A.idx + p + 96);
            double v0 = (double)__ldg(va + c0), v1 = (double)__ldg(va + c1);
            double v2 = (double)__ldg(va + c2), v3 = (double)__ldg(va + c3);
            if (vb) {
                v0 -= (double)__ldg(vb + c0); v1 -= (double)__ldg(vb + c1);
                v2 -= (double)__ldg(vb + c2); v3 -= (double)__ldg(vb + c3);
            }
            acc += (kval<KIND>(A.val, p) * v0 + kval<KIND>(A.val, p + 32) * v1) +
                   (kval<KIND>(A.val, p + 64) * v2 + kval<KIND>(A.val, p + 96) * v3);
        }
        for (; p < p1; p += 32) {
            const int c = __ldg(A.idx + p);
            double v = (double)__ldg(va + c);
            if (vb) v -= (double)__ldg(vb + c);
            acc += kval<KIND>(A.val, p) * v;
        }
        acc = warp_sum(acc);
        if (lane == 0) part[sgi] = acc;
    }
}

template <typename T, int KIND>
__global__ void __launch_bounds__(256) k_dual_seg_final(long long rows, SegPlan sp, const double* __restrict__ part,
                                                        State<T> s, const double* __restrict__ g, const double* __restrict__ rh,
                                                        const signed char* __restrict__ rsign, long long m1,
                                                        const Ctrl* __restrict__ ctrl, long long kint, long long j) {
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const double tau2 = ctrl->tau2;
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < rows;
         row += gridDim.x * (long long)blockDim.x) {
        double acc = 0.0;
        for (long long q = sp.row_seg[row]; q < sp.row_seg[row + 1]; ++q) acc += part[q];
        const double sg = (KIND == KV_SIGN) ? (double)rsign[row] : 1.0;
        const double gj = (double)g[row];
        double yn = (double)(par ? s.y[1] : s.y[0])[row] + tau2 * ((double)rh[row] - gj * (sg * acc));
        if (row < m1 && yn < 0.0) yn = 0.0;
        const T yt = (T)yn;
        (par ? s.y[0] : s.y[1])[row] = yt;
        s.w[row] = w_of(gj, sg, yt);
    }
}

template <typename T, bool HASQ>
__global__ void __launch_bounds__(256) k_primal_seg_final(long long n, SegPlan sp, const double* __restrict__ part,
                                                          Csr Q, const T* __restrict__ qs, State<T> s,
                                                          const T* __restrict__ cs, const Ctrl* __restrict__ ctrl,
                                                          long long kint, long long j) {
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const double rho = ctrl->rho, tau1 = ctrl->tau1;
    const T* __restrict__ xin = (par ? s.x[1] : s.x[0]);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x) {
        double a = 0.0, b = 0.0;
        for (long long q = sp.row_seg[i]; q < sp.row_seg[i + 1]; ++q) a += part[q];
        if constexpr (HASQ) {
            if (Q.pre) b = Q.pre[i];
            else
                for (long long q = Q.ptr[i]; q < Q.ptr[i + 1]; ++q) b += (double)qs[q] * (double)xin[Q.idx[q]];
        }
        const double xi = (double)xin[i];
        const double delta = (((double)cs[i] + rho) - a) + 2.0 * b - 2.0 * rho * xi;
        double xn = xi - tau1 * delta;
        xn = xn < 0.0 ? 0.0 : (xn > 1.0 ? 1.0 : xn);
        (par ? s.x[0] : s.x[1])[i] = (T)xn;
        (par ? s.xb[0] : s.xb[1])[i] = (T)(2.0 * xn - xi);
    }
}

// ---------------------------------------------------------------------------------------------
// Trigger indicators (reading R9), fixed-order block partials.
// Row pass:  v_j = (K_u x_k)_j, d_j = (K_u (x_k - xbar_{k-1}))_j
//   (K x_k + r)_j = rh_j - g_j v_j      -> primal gap (max over GE of max(.,0), max over EQ |.|)
//   s^y_j = (y_{k-1} - y_k)_j / tau2 + g_j d_j
// part1[3*b + {0,1,2}] = {max GE gap, max EQ gap, sum s^y^2} of block b.
// ---------------------------------------------------------------------------------------------
template <typename T, int KIND, int SUB, bool SEG>
__global__ void __launch_bounds__(256) k_trig_rows(Csr K, SegPlan sp, const double* __restrict__ pv,
                                                   const double* __restrict__ pd, State<T> s,
                                                   const double* __restrict__ g, const double* __restrict__ rh,
                                                   const signed char* __restrict__ rsign, long long m1,
                                                   const Ctrl* __restrict__ ctrl, long long kint, long long j,
                                                   double* __restrict__ part1) {
    __shared__ double sh[32];
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ xk = (par ? s.x[0] : s.x[1]);
    const T* __restrict__ xbp = (par ? s.xb[1] : s.xb[0]);
    const double tau2 = ctrl->tau2;
    constexpr int RPW = 32 / SUB;
    const int lane = threadIdx.x & (SUB - 1);
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    const int gsub = (threadIdx.x & 31) / SUB;
    double ge = 0.0, eq = 0.0, sy2 = 0.0;
    for (long long base = warp * RPW; base < K.rows; base += nwarps * RPW) {
        const long long row = base + gsub;
        double v = 0.0, d = 0.0;
        if (row < K.rows) {
            if constexpr (SEG) {
                if (lane == 0)
                    for (long long q = sp.row_seg[row]; q < sp.row_seg[row + 1]; ++q) { v += pv[q]; d += pd[q]; }
            } else {
                for (long long p = K.ptr[row] + lane; p < K.ptr[row + 1]; p += SUB) {
                    const int c = __ldg(K.idx + p);
                    const double kv = kval<KIND>(K.val, p);
                    const double xv = (double)xk[c];
                    v += kv * xv;
                    d += kv * (xv - (double)xbp[c]);
                }
            }
        }
        if constexpr (!SEG) { v = group_sum<SUB>(v); d = group_sum<SUB>(d); }
        if (lane == 0 && row < K.rows) {
            const double sg = (KIND == KV_SIGN) ? (double)rsign[row] : 1.0;
            const double gj = (double)g[row];
            const double gap = (double)rh[row] - gj * (sg * v);
            if (row < m1) ge = fmax(ge, fmax(gap, 0.0)); else eq = fmax(eq, fabs(gap));
            const double sy = ((double)(par ? s.y[1] : s.y[0])[row] - (double)(par ? s.y[0] : s.y[1])[row]) / tau2 + gj * (sg * d);
            sy2 += sy * sy;
        }
    }
    const double a = block_max<256>(ge, sh);
    const double b = block_max<256>(eq, sh);
    const double c = block_sum<256>(sy2, sh);
    if (threadIdx.x == 0) { part1[3 * blockIdx.x] = a; part1[3 * blockIdx.x + 1] = b; part1[3 * blockIdx.x + 2] = c; }
}

// Column pass: e_i = (Q (x_k - x_{k-1}))_i; s^x_i = (x_{k-1} - x_k)_i/tau1 + 2e_i - 2 rho (x_k - x_{k-1})_i;
// binary gap term x_i (1 - x_i).  part2[2*b + {0,1}] = {sum s^x^2, sum x(1-x)}.
template <typename T, bool HASQ>
__global__ void __launch_bounds__(256) k_trig_cols(long long n, Csr Q, const T* __restrict__ qs, State<T> s,
                                                   const Ctrl* __restrict__ ctrl, long long kint, long long j,
                                                   double* __restrict__ part2) {
    __shared__ double sh[32];
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ xk = (par ? s.x[0] : s.x[1]);
    const T* __restrict__ xp = (par ? s.x[1] : s.x[0]);
    const double rho = ctrl->rho, tau1 = ctrl->tau1;
    double sx2 = 0.0, bg = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x) {
        const double xi = (double)xk[i], xo = (double)xp[i];
        double e = 0.0;
        if constexpr (HASQ) {
            if (Q.pre) e = Q.pre[i];  // dense-Q path: Q~(x_k - x_{k-1}) precomputed
            else
                for (long long q = Q.ptr[i]; q < Q.ptr[i + 1]; ++q) {
                    const int c = Q.idx[q];
                    e += (double)qs[q] * ((double)xk[c] - (double)xp[c]);
                }
        }
        const double sx = (xo - xi) / tau1 + 2.0 * e - 2.0 * rho * (xi - xo);
        sx2 += sx * sx;
        bg += xi * (1.0 - xi);
    }
    const double a = block_sum<256>(sx2, sh);
    const double b = block_sum<256>(bg, sh);
    if (threadIdx.x == 0) { part2[2 * blockIdx.x] = a; part2[2 * blockIdx.x + 1] = b; }
}

// fixed-order combination of the block partials -> ind[4] (single block of 256 threads)
__device__ __forceinline__ void reduce_indicators(const double* part1, int nb1, const double* part2, int nb2,
                                                  long long n, double* sh, double* ind) {
    double ge = 0.0, eq = 0.0, sy2 = 0.0, sx2 = 0.0, bg = 0.0;
    for (int b = threadIdx.x; b < nb1; b += blockDim.x) {
        ge = fmax(ge, part1[3 * b]); eq = fmax(eq, part1[3 * b + 1]); sy2 += part1[3 * b + 2];
    }
    for (int b = threadIdx.x; b < nb2; b += blockDim.x) { sx2 += part2[2 * b]; bg += part2[2 * b + 1]; }
    ge = block_max<256>(ge, sh);
    eq = block_max<256>(eq, sh);
    sy2 = block_sum<256>(sy2, sh);
    sx2 = block_sum<256>(sx2, sh);
    bg = block_sum<256>(bg, sh);
    if (threadIdx.x == 0) {
        ind[0] = ge + eq;
        ind[1] = sqrt(sx2);
        ind[2] = sqrt(sy2);
        ind[3] = bg / (double)n;
    }
}

template <int DUMMY = 0>
__global__ void k_indicators_only(const double* part1, int nb1, const double* part2, int nb2, long long n,
                                  double* out) {
    __shared__ double sh[32];
    reduce_indicators(part1, nb1, part2, nb2, n, sh, out);
}

}  // namespace gfors
