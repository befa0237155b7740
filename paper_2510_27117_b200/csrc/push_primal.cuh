// push_primal.cuh — primal half-step from the nonzero duals ("push" mode).
//
// K'y = -K_u' w with w_j = g_j rsign_j y_j, and on covering-type instances most inequality duals sit
// at the clamp y_j = 0 (config 5: 1 % / 7 % / 37 % nonzero after 100 / 500 / 2000 iterations).  When
// few rows are active the product is computed from them: k_wlist lists the rows with w_j != 0 (and
// the max |w|), k_push_scatter_cols adds w_j in fixed point (scale S = 2^e chosen from max|w| and the
// largest column degree so no sum can overflow int64) into int64 column accumulators through the row
// CSR with integer atomics — order-independent, hence deterministic — and k_primal_push applies the
// box-projected update column by column (coalesced).  The accumulators are then kept (delta push,
// push_list.cuh): later iterations list and scatter only the rows whose y changed.  With many listed
// rows the gather kernel (k_primal_rb) runs instead and clears them; the choice is made on the device
// from the list length (pp_mode), every kernel of the unused mode exits at once.
#pragma once
#include "push_list.cuh"
#include "rowblock.cuh"

namespace gfors {

// lists the rows for the push-mode primal of parity par: valid accumulators -> rows whose y changed
// this iteration, else rows with w != 0; and max |w|
constexpr int WL_CAP = 4096;  // staged list entries per CTA between global flushes
template <typename T>
__global__ void __launch_bounds__(256) k_wlist(State<T> s, PushPrimal pp, const Ctrl* __restrict__ ctrl, long long kint,
                                               long long jj) {
    // each CTA scans a contiguous range of rows in 256-row passes and stages its list in shared
    // memory; one global atomic per WL_CAP staged rows (the single list counter was the contended
    // resource of the per-pass flush: ~4000 same-address atomics per launch on config 5)
    __shared__ unsigned s_cnt, s_base;
    __shared__ int s_list[WL_CAP];
    __shared__ double sh[32];
    const int par = (int)(iter_index(ctrl, kint, jj) & 1);
    const bool delta = pp_valid(pp, par);
    const T* __restrict__ ynew = par ? s.y[0] : s.y[1];
    const T* __restrict__ yold = par ? s.y[1] : s.y[0];
    double mx = 0.0;
    const long long m = pp.m;
    constexpr int WU = 4;  // rows per thread and pass (their loads in flight together)
    const long long per = ((m + gridDim.x - 1) / gridDim.x + 256 * WU - 1) / (256 * WU) * (256 * WU);
    const long long r0 = blockIdx.x * per, r1 = min(m, r0 + per);
    if (threadIdx.x == 0) s_cnt = 0u;
    __syncthreads();
    auto flush = [&]() {
        __syncthreads();
        if (threadIdx.x == 0) s_base = s_cnt ? atomicAdd(pp.rcount, s_cnt) : 0u;
        __syncthreads();
        const unsigned c = s_cnt, b = s_base;
        for (unsigned t = threadIdx.x; t < c; t += 256)
            if ((long long)b + t < m) pp.rlist[b + t] = s_list[t];
        __syncthreads();
        if (threadIdx.x == 0) s_cnt = 0u;
        __syncthreads();
    };
    for (long long b0 = r0; b0 < r1; b0 += 256 * WU) {  // block-uniform trip count
        double v[WU];
        bool listed[WU];
#pragma unroll
        for (int u = 0; u < WU; ++u) {
            const long long j = b0 + u * 256 + threadIdx.x;
            v[u] = j < r1 ? (double)s.w[j] : 0.0;
            listed[u] = delta ? (j < r1 && ynew[j] != yold[j]) : v[u] != 0.0;
        }
#pragma unroll
        for (int u = 0; u < WU; ++u) {
            mx = fmax(mx, fabs(v[u]));
            warp_append(listed[u], (int)(b0 + u * 256 + threadIdx.x), &s_cnt, s_list);
        }
        __syncthreads();
        if (s_cnt > WL_CAP - 256 * WU) flush();  // (block-uniform: read after the barrier)
    }
    flush();
    mx = block_max<256>(mx, sh);
    if (threadIdx.x == 0 && mx > 0.0) atomicMax(pp.wmax, (unsigned long long)__double_as_longlong(mx));
}

// push mode: accx[i] += round(w_j S) for every nonzero (j, i) of the listed rows; delta push adds
// round(w_j S) - round(w_j^prev S) with w^prev recomputed from y_{k-1} exactly as the dual made it
template <typename T>
__global__ void __launch_bounds__(256) k_push_scatter_cols(Csr K, PushPrimal pp, State<T> s, const Ctrl* __restrict__ ctrl,
                                                           long long kint, long long jj) {
    const int par = cta_parity(ctrl, kint, jj);
    const PPMode md = cta_pp_mode(pp, par);
    if (!md.push) return;
    const bool mark = pp_marking(pp, md);
    const double S = pow2(md.e);
    const T* __restrict__ yold = par ? s.y[1] : s.y[0];
    const long long cnt = *pp.rcount;
    // a warp per listed row: rows have 2..98 nonzeros on the set-cover workloads
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long k = warp; k < cnt; k += nwarps) {
        const int jr = pp.rlist[k];
        long long v = __double2ll_rn((double)s.w[jr] * S);
        if (md.delta) v -= __double2ll_rn((double)w_of(pp.g[jr], (double)pp.rsign[jr], yold[jr]) * S);
        if (v == 0) continue;
        const long long q1 = __ldg(K.ptr + jr + 1);
        for (long long q = __ldg(K.ptr + jr) + lane; q < q1; q += 32) {
            const int i = __ldg(K.idx + q);
            atomicAdd(reinterpret_cast<unsigned long long*>(pp.accx + i), (unsigned long long)v);
            if (mark) pp.xst[i] = 0;
        }
    }
}

// Stationary columns.  The update of column i is a function xn_k = F(x_{k-1}, a_k, rho) (double,
// before rounding to T), x_k = (T)xn_k, xbar_k = (T)(2 xn_k - x_{k-1}).  Iteration k has "the same
// inputs" as k-1 when rho is unchanged (not the first iteration of a loop block, not hook mode),
// a_k = a_{k-1} (delta push with the same exponent, and the marking scatter left accx_i alone — a
// touched column has xst_i cleared) and there is no Q (b depends on other columns).  xst_i = 2
// certifies x_k = x_{k-1} = x_{k-2} and xn_k = xn_{k-1} (same inputs at k); then, if iteration k+1
// has the same inputs again, xn_{k+1} = xn_k, so x_{k+1} = x_{k-1} and xbar_{k+1} = xbar_{k-1} —
// exactly what the output buffers of iteration k+1 already hold — and the column is skipped:
// bit-identical, 1 byte read instead of 24-28.  xst_i = 1: x_k = x_{k-1} only; 0: changed/touched.
// Skipping also needs: not the trigger iteration (it pushes every x_k), and no value of a skipped
// column for the next dual's list (delta list, where an unchanged column is not listed, or none).
// push mode: x_k = Pi(x_{k-1} - tau1 (c + rho - a + 2 Q x_{k-1} - 2 rho x_{k-1})), xbar_k = 2x_k - x_{k-1},
// with a = accx / S (accumulators kept for the next delta push); also hands the nonzero (or, with
// valid dual accumulators, the changed) xbar columns to the next dual (PushList).  A pure stream over
// the columns (c, x_{k-1}, accx in; x_k, xbar_k out): each thread owns PP_U = 4 CONSECUTIVE columns
// and moves them with 16-byte vector loads/stores (one instruction per array for fp32), the
// block-staged list append is amortised over 256*PP_U columns.
constexpr int PP_U = 4;
constexpr int PP_LPASSES = 4;  // passes staged in shared memory between list flushes
constexpr int PP_OCC32 = 5, PP_OCC64 = 4;  // resident CTAs per SM (launch bounds, persistent grid)

template <typename T>
__device__ __forceinline__ void ld4(const T* __restrict__ p, T (&o)[PP_U]) {
    if constexpr (sizeof(T) == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
        const double2 v0 = __ldg(reinterpret_cast<const double2*>(p)), v1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
        o[0] = v0.x; o[1] = v0.y; o[2] = v1.x; o[3] = v1.y;
    }
}
template <typename T>
__device__ __forceinline__ void st4(T* __restrict__ p, const T (&v)[PP_U]) {
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
        reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
    }
}

// persistent grid (one wave at the occupancy the launch bounds give): the per-CTA prologue (mode,
// flags — a chain of dependent loads) is paid once, not per 1024 columns; matters when most columns
// are skipped
template <typename T>
inline int pp_grid(long long n, int occ = 0) {
    const long long passes = (n + 256 * PP_U - 1) / (256 * PP_U);
    if (occ <= 0) occ = sizeof(T) == 4 ? PP_OCC32 : PP_OCC64;
    return (int)std::max<long long>(1, std::min<long long>(passes, (long long)sm_count() * occ));
}

template <typename T, bool HASQ, int OCC = (sizeof(T) == 4 ? PP_OCC32 : PP_OCC64)>
__global__ void __launch_bounds__(256, OCC) k_primal_push(long long n, PushPrimal pp, Csr Q, const T* __restrict__ qs,
                                                     State<T> s, const T* __restrict__ cs, const Ctrl* __restrict__ ctrl,
                                                     long long kint, long long j, PushList pl, Csr Kt,
                                                     long long* __restrict__ accv, unsigned* __restrict__ ones_cnt,
                                                     unsigned* __restrict__ trig_flag) {
    __shared__ unsigned s_cnt, s_base;
    __shared__ int s_list[PP_LPASSES * 256 * PP_U];
    __shared__ bool s_en;
    const int par = cta_parity(ctrl, kint, j);
    const PPMode md = cta_pp_mode(pp, par);
    if (!md.push) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // trigger iteration: also push x_k into the row accumulators of the indicator pass (k_trig_rows_push).
        // (Measured on config 5, blocks 1-20: even with a dense x_k this beats the gather-mode trigger pass,
        // 0.75 vs 0.88 ms per block for push column pass + trigger rows.)
        if (accv) *trig_flag = 1u;
        const double wm = __longlong_as_double((long long)*(volatile unsigned long long*)pp.wmax);
        pp_set_next(pp, par, wm > 0.0, md.e);  // accumulators kept (nothing was scattered if w == 0)
    }
    const double invS = pow2(-md.e);
    const T* __restrict__ xin = par ? s.x[1] : s.x[0];
    T* __restrict__ xout = par ? s.x[0] : s.x[1];
    T* __restrict__ xbout = par ? s.xb[0] : s.xb[1];
    const T* __restrict__ xbprev = par ? s.xb[1] : s.xb[0];  // xbar_{k-1} (delta list of the next dual)
    const double rho = ctrl->rho, tau1 = ctrl->tau1;
    const bool dd = pl.acc && pl_valid(pl, par ^ 1);  // constant during the kernel
    const bool track = !HASQ && kint > 0 && j > 0 && pp_marking(pp, md);  // same inputs as iteration k-1
    const bool skip = track && accv == nullptr && (pl.acc == nullptr || dd);
    unsigned char* __restrict__ xst = pp.xst;
    const int per = 256 * PP_U;
    const int nbase = (int)((n + per - 1) / per);
    const long long* __restrict__ accx = pp.accx;
    // list the columns of the next dual while it can still be short (read once; the list has room
    // for every column, so appending past the threshold only wastes a little work)
    if (threadIdx.x == 0) {
        s_en = pl.acc && *(volatile unsigned*)pl_count(pl, par ^ 1) <= pl.thr;
        s_cnt = 0u;
    }
    __syncthreads();
    bool en = s_en;  // (re-read after each flush: stops once the list is already too long for a push)
    uchar4 st_next = make_uchar4(0, 0, 0, 0);
    if (xst && (long long)blockIdx.x * per + PP_U * (threadIdx.x + 1) <= n)
        st_next = *reinterpret_cast<const uchar4*>(xst + (long long)blockIdx.x * per + PP_U * threadIdx.x);
    int npass = 0;
    for (int bb = blockIdx.x; bb < nbase; bb += gridDim.x) {  // block-uniform trip count
        const int i0 = bb * per + PP_U * threadIdx.x;
        const uchar4 st4v = st_next;  // loaded one pass ahead
        {
            const long long i1 = (long long)(bb + gridDim.x) * per + PP_U * threadIdx.x;
            if (xst && i1 + PP_U <= n) st_next = *reinterpret_cast<const uchar4*>(xst + i1);
        }
        // the 4 columns are stationary and untouched: nothing to compute or write (see above)
        const bool skip4 = skip && i0 + PP_U <= n && st4v.x == 2 && st4v.y == 2 && st4v.z == 2 && st4v.w == 2;
        T xb[PP_U] = {}, xbp[PP_U] = {};
        if (!skip4) {
            long long ai[PP_U];
            T xi[PP_U], ci[PP_U], xk[PP_U];
            if (i0 + PP_U <= n) {
                const longlong2 a01 = __ldg(reinterpret_cast<const longlong2*>(accx + i0));
                const longlong2 a23 = __ldg(reinterpret_cast<const longlong2*>(accx + i0) + 1);
                ai[0] = a01.x; ai[1] = a01.y; ai[2] = a23.x; ai[3] = a23.y;
                ld4(xin + i0, xi);
                ld4(cs + i0, ci);
                if (dd) ld4(xbprev + i0, xbp);
            } else {
#pragma unroll
                for (int u = 0; u < PP_U; ++u) {
                    const int i = i0 + u;
                    ai[u] = i < n ? accx[i] : 0;
                    xi[u] = i < n ? xin[i] : (T)0;
                    ci[u] = i < n ? cs[i] : (T)0;
                    xbp[u] = (dd && i < n) ? xbprev[i] : (T)0;
                }
            }
#pragma unroll
            for (int u = 0; u < PP_U; ++u) {
                double b = 0.0;
                if constexpr (HASQ)
                    if (i0 + u < n) {
                        if (Q.pre) b = Q.pre[i0 + u];
                        else
                            for (long long q = __ldg(Q.ptr + i0 + u); q < __ldg(Q.ptr + i0 + u + 1); ++q)
                                b += (double)__ldg(qs + q) * (double)__ldg(xin + __ldg(Q.idx + q));
                    }
                const double x0 = (double)xi[u];
                const double delta = (((double)ci[u] + rho) - (double)ai[u] * invS) + 2.0 * b - 2.0 * rho * x0;
                double xn = x0 - tau1 * delta;
                xn = xn < 0.0 ? 0.0 : (xn > 1.0 ? 1.0 : xn);
                xk[u] = (T)xn;
                xb[u] = (T)(2.0 * xn - x0);
            }
            if (xst) {
                // stationarity state of the computed columns (a gather-mode primal does not keep it:
                // the iteration after one is never "same inputs", so xst restarts at <= 1)
                unsigned char sv[PP_U] = {st4v.x, st4v.y, st4v.z, st4v.w};
                if (i0 + PP_U > n)
                    for (int u = 0; u < PP_U; ++u) sv[u] = i0 + u < n ? xst[i0 + u] : 0;
                bool ch = false;
                for (int u = 0; u < PP_U; ++u) {
                    const unsigned char nv = xk[u] != xi[u] ? 0 : ((track && sv[u] >= 1) ? 2 : 1);
                    ch |= nv != sv[u];
                    sv[u] = nv;
                }
                if (ch) {
                    if (i0 + PP_U <= n) *reinterpret_cast<uchar4*>(xst + i0) = make_uchar4(sv[0], sv[1], sv[2], sv[3]);
                    else for (int u = 0; u < PP_U; ++u) if (i0 + u < n) xst[i0 + u] = sv[u];
                }
            }
            if (i0 + PP_U <= n) {
                st4(xout + i0, xk);
                st4(xbout + i0, xb);
            } else {
#pragma unroll
                for (int u = 0; u < PP_U; ++u)
                    if (i0 + u < n) { xout[i0 + u] = xk[u]; xbout[i0 + u] = xb[u]; }
            }
            if (accv) {
#pragma unroll
                for (int u = 0; u < PP_U; ++u) {
                    if (i0 + u >= n || xk[u] == (T)0) continue;
                    const long long v = __double2ll_rn((double)xk[u] * 1099511627776.0);  // 2^40 fixed point
                    const bool one = xk[u] == (T)1;
                    const long long q1 = __ldg(Kt.ptr + i0 + u + 1);
                    for (long long q = __ldg(Kt.ptr + i0 + u); q < q1; ++q) {
                        const int r = __ldg(Kt.idx + q);
                        atomicAdd(reinterpret_cast<unsigned long long*>(accv + r), (unsigned long long)v);
                        if (one) atomicAdd(ones_cnt + r, 1u);
                    }
                }
            }
        }
        if (en) {
#pragma unroll
            for (int u = 0; u < PP_U; ++u)
                warp_append(!skip4 && i0 + u < n && pl_listed(dd, xb[u], xbp[u]), i0 + u, &s_cnt, s_list);
        }
        // flush the staged list every PP_LPASSES passes and at the end (block-uniform decision)
        if (en && (++npass == PP_LPASSES || bb + (int)gridDim.x >= nbase)) {
            npass = 0;
            __syncthreads();
            if (threadIdx.x == 0) {
                s_base = atomicAdd(pl_count(pl, par ^ 1), s_cnt);
                // once the list holds more than the push threshold the next dual gathers anyway: stop
                // listing (the count only grows, so it stays above the threshold; in a dense phase every
                // column changes and listing them all cost ~15 % of this kernel)
                s_en = (unsigned long long)s_base + s_cnt <= (unsigned long long)pl.thr;
            }
            __syncthreads();
            const unsigned c = s_cnt, base = s_base;
            for (unsigned t = threadIdx.x; t < c; t += 256)
                if ((long long)base + t < pl.cap) pl_list(pl, par ^ 1)[base + t] = s_list[t];
            __syncthreads();
            if (threadIdx.x == 0) s_cnt = 0u;
            en = s_en;
            __syncthreads();
        }
    }
}

// Trigger row pass from the pushed x_k (no gathers): v_j = (K_u x_k)_j from the fixed-point row
// accumulators, d_j = v_j - (K_u xbar_{k-1})_j; same partial layout as k_trig_rows_rb.  Runs iff the
// primal of the trigger iteration pushed (trig_flag), clears accumulators and flag.  +-1 rows.
template <typename T>
__global__ void __launch_bounds__(256) k_trig_rows_push(long long m, State<T> s, const double* __restrict__ g,
                                                        const double* __restrict__ rh,
                                                        const signed char* __restrict__ rsign, long long m1,
                                                        const double* __restrict__ u_prev, const Ctrl* __restrict__ ctrl,
                                                        long long kint, long long j, double* __restrict__ part1,
                                                        unsigned char* __restrict__ ones_out, long long* __restrict__ accv,
                                                        unsigned* __restrict__ ones_cnt, unsigned* __restrict__ trig_flag) {
    __shared__ double sh[32];
    __shared__ int s_on;  // (read once per CTA, see cta_push_mode)
    if (threadIdx.x == 0) s_on = *(volatile unsigned*)trig_flag != 0u;
    __syncthreads();
    if (!s_on) return;
    const int par = cta_parity(ctrl, kint, j);
    const T* __restrict__ yprev = par ? s.y[1] : s.y[0];
    const T* __restrict__ ynew = par ? s.y[0] : s.y[1];
    const double tau2 = ctrl->tau2;
    double ge = 0.0, eq = 0.0, sy2 = 0.0;
    for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < m; row += gridDim.x * (long long)blockDim.x) {
        const long long a = accv[row];
        if (a) accv[row] = 0;
        const unsigned c1 = ones_cnt[row];
        if (c1) ones_cnt[row] = 0u;
        if (ones_out) ones_out[row] = (unsigned char)min(c1, 255u);
        const double sg = (double)rsign[row];
        const double gj = g[row];
        const double ku = sg * ((double)a * (1.0 / 1099511627776.0));  // (K_u x_k)_j
        const double gap = rh[row] - gj * ku;
        if (row < m1) ge = fmax(ge, fmax(gap, 0.0)); else eq = fmax(eq, fabs(gap));
        const double sy = ((double)yprev[row] - (double)ynew[row]) / tau2 + gj * (ku - u_prev[row]);
        sy2 += sy * sy;
    }
    const double aa = block_max<256>(ge, sh);
    const double bb = block_max<256>(eq, sh);
    const double cc = block_sum<256>(sy2, sh);
    if (threadIdx.x == 0) { part1[3 * blockIdx.x] = aa; part1[3 * blockIdx.x + 1] = bb; part1[3 * blockIdx.x + 2] = cc; }
    // every block has read the flag at entry (it is cleared only by a later kernel: k_trig_clear)
}

__global__ void k_trig_clear(unsigned* trig_flag) { *trig_flag = 0u; }

}  // namespace gfors
