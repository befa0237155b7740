// push_primal.cuh — primal half-step from the nonzero duals ("push" mode).
//
// K'y = -K_u' w with w_j = g_j rsign_j y_j, and on covering-type instances most inequality duals sit
// at the clamp y_j = 0 (config 5: 1 % / 7 % / 37 % nonzero after 100 / 500 / 2000 iterations).  When
// few rows are active the product is computed from them: k_wlist lists the rows with w_j != 0 (and
// the max |w|), k_push_scatter_cols adds w_j in fixed point (scale S = 2^e chosen from max|w| and the
// largest column degree so no sum can overflow int64) into int64 column accumulators through the row
// CSR with integer atomics — order-independent, hence deterministic — and k_primal_push applies the
// box-projected update column by column (coalesced) and clears the accumulators.  With many active
// rows the gather kernel (k_primal_rb) runs instead; the choice is made on the device from the list
// length, every kernel of the unused mode exits at once.
#pragma once
#include "push_list.cuh"
#include "rowblock.cuh"

namespace gfors {

struct PushPrimal {
    int* rlist;                // rows with w_j != 0
    unsigned* rcount;          // list length (reset by the dual of the same iteration)
    unsigned rthr;             // push mode iff rcount <= rthr
    unsigned long long* wmax;  // bit pattern of max |w_j| (non-negative doubles order like uint64)
    long long* accx;           // [n] int64 column accumulators, kept at 0 between uses
    int maxdeg;                // largest column degree of K_u (number of terms of any a_i)
    long long m;
};

__device__ __forceinline__ bool pprimal_mode(const PushPrimal& pp) {
    return pp.accx != nullptr && *(volatile unsigned*)pp.rcount <= pp.rthr;
}

// fixed-point scale S = 2^e with (max|w| * maxdeg) * 2^e < 2^62 (exponent read from the bits;
// capped at 2^1000 for vanishing w); returns e, S and 1/S are then exact powers of two
__device__ __forceinline__ int pprimal_exp(const PushPrimal& pp) {
    const double wm = __longlong_as_double((long long)*(volatile unsigned long long*)pp.wmax);
    if (!(wm > 0.0)) return 0;
    const double b = wm * (double)pp.maxdeg;
    const int bexp = (int)((__double_as_longlong(b) >> 52) & 0x7ff);  // b = f 2^(bexp-1023), f in [1,2)
    return min(62 - (bexp - 1022), 1000);                               // b < 2^(bexp-1022)
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }

template <typename T>
__global__ void __launch_bounds__(256) k_wlist(const T* __restrict__ w, PushPrimal pp) {
    __shared__ unsigned s_cnt, s_base;
    __shared__ int s_list[256];
    __shared__ double sh[32];
    double mx = 0.0;
    const long long m = pp.m;
    const long long nbase = (m + 255) / 256;
    for (long long bb = blockIdx.x; bb < nbase; bb += gridDim.x) {  // block-uniform trip count
        const long long j = bb * 256 + threadIdx.x;
        const double v = j < m ? (double)w[j] : 0.0;
        mx = fmax(mx, fabs(v));
        if (threadIdx.x == 0) s_cnt = 0u;
        __syncthreads();
        warp_append(v != 0.0, (int)j, &s_cnt, s_list);
        __syncthreads();
        if (threadIdx.x == 0) s_base = s_cnt ? atomicAdd(pp.rcount, s_cnt) : 0u;
        __syncthreads();
        for (unsigned t = threadIdx.x; t < s_cnt; t += 256)
            if ((long long)s_base + t < m) pp.rlist[s_base + t] = s_list[t];
        __syncthreads();
    }
    mx = block_max<256>(mx, sh);
    if (threadIdx.x == 0 && mx > 0.0) atomicMax(pp.wmax, (unsigned long long)__double_as_longlong(mx));
}

// push mode: accx[i] += round(w_j * S) for every nonzero (j, i) of the listed rows
template <typename T>
__global__ void __launch_bounds__(256) k_push_scatter_cols(Csr K, PushPrimal pp, const T* __restrict__ w) {
    if (!pprimal_mode(pp)) return;
    const double S = pow2(pprimal_exp(pp));
    const long long cnt = *pp.rcount;
    // a warp per listed row: rows have 2..98 nonzeros on the set-cover workloads
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long k = warp; k < cnt; k += nwarps) {
        const int jr = pp.rlist[k];
        const long long v = __double2ll_rn((double)w[jr] * S);
        const long long q1 = __ldg(K.ptr + jr + 1);
        for (long long q = __ldg(K.ptr + jr) + lane; q < q1; q += 32)
            atomicAdd(reinterpret_cast<unsigned long long*>(pp.accx + __ldg(K.idx + q)), (unsigned long long)v);
    }
}

// push mode: x_k = Pi(x_{k-1} - tau1 (c + rho - a + 2 Q x_{k-1} - 2 rho x_{k-1})), xbar_k = 2x_k - x_{k-1},
// with a = accx / S; also hands the nonzero xbar columns to the next dual (PushList).  Each thread
// handles PP_U consecutive columns per pass so the block-staged append is amortised over
// 256*PP_U columns.
constexpr int PP_U = 4;

template <typename T, bool HASQ>
__global__ void __launch_bounds__(256, 6) k_primal_push(long long n, PushPrimal pp, Csr Q, const T* __restrict__ qs,
                                                     State<T> s, const T* __restrict__ cs, const Ctrl* __restrict__ ctrl,
                                                     long long kint, long long j, PushList pl, Csr Kt,
                                                     long long* __restrict__ accv, unsigned* __restrict__ ones_cnt,
                                                     unsigned* __restrict__ trig_flag) {
    __shared__ unsigned s_cnt, s_base;
    __shared__ int s_list[256 * PP_U];
    __shared__ bool s_en;
    if (!pprimal_mode(pp)) return;
    // trigger iteration: also push x_k into the row accumulators of the indicator pass (k_trig_rows_push)
    if (accv && blockIdx.x == 0 && threadIdx.x == 0) *trig_flag = 1u;
    const double invS = pow2(-pprimal_exp(pp));
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
    const T* __restrict__ xin = par ? s.x[1] : s.x[0];
    T* __restrict__ xout = par ? s.x[0] : s.x[1];
    T* __restrict__ xbout = par ? s.xb[0] : s.xb[1];
    const double rho = ctrl->rho, tau1 = ctrl->tau1;
    const long long per = 256LL * PP_U;
    const long long nbase = (n + per - 1) / per;
    long long* __restrict__ accx = pp.accx;
    for (long long bb = blockIdx.x; bb < nbase; bb += gridDim.x) {  // block-uniform trip count
        if (threadIdx.x == 0) { s_en = pl.acc && *(volatile unsigned*)pl_count(pl, par ^ 1) <= pl.thr; s_cnt = 0u; }
        __syncthreads();
        const bool en = s_en;
        // all loads of the PP_U columns first (independent, in flight together), then the updates
        long long ai[PP_U];
        double xi[PP_U], ci[PP_U];
#pragma unroll
        for (int u = 0; u < PP_U; ++u) {
            const long long i = bb * per + u * 256 + threadIdx.x;
            ai[u] = 0; xi[u] = 0.0; ci[u] = 0.0;
            if (i < n) { ai[u] = __ldcs(accx + i); xi[u] = (double)xin[i]; ci[u] = (double)__ldg(cs + i); }
        }
#pragma unroll
        for (int u = 0; u < PP_U; ++u) {
            const long long i = bb * per + u * 256 + threadIdx.x;
            bool nzb = false;
            T xk = (T)0;
            if (i < n) {
                if (ai[u]) accx[i] = 0;
                const double a = (double)ai[u] * invS;
                double b = 0.0;
                if constexpr (HASQ)
                    for (long long q = __ldg(Q.ptr + i); q < __ldg(Q.ptr + i + 1); ++q)
                        b += (double)__ldg(qs + q) * (double)__ldg(xin + __ldg(Q.idx + q));
                const double delta = ((ci[u] + rho) - a) + 2.0 * b - 2.0 * rho * xi[u];
                double xn = xi[u] - tau1 * delta;
                xn = xn < 0.0 ? 0.0 : (xn > 1.0 ? 1.0 : xn);
                xk = (T)xn;
                xout[i] = xk;
                const T xbn = (T)(2.0 * xn - xi[u]);
                xbout[i] = xbn;
                nzb = xbn != (T)0;
            }
            if (en) warp_append(nzb, (int)i, &s_cnt, s_list);
            if (accv && xk != (T)0) {
                const long long v = __double2ll_rn((double)xk * 1099511627776.0);  // 2^40 fixed point
                const bool one = xk == (T)1;
                const long long q1 = __ldg(Kt.ptr + i + 1);
                for (long long q = __ldg(Kt.ptr + i); q < q1; ++q) {
                    const int r = __ldg(Kt.idx + q);
                    atomicAdd(reinterpret_cast<unsigned long long*>(accv + r), (unsigned long long)v);
                    if (one) atomicAdd(ones_cnt + r, 1u);
                }
            }
        }
        __syncthreads();
        if (en) {
            if (threadIdx.x == 0) s_base = s_cnt ? atomicAdd(pl_count(pl, par ^ 1), s_cnt) : 0u;
            __syncthreads();
            const unsigned c = s_cnt, base = s_base;
            for (unsigned t = threadIdx.x; t < c; t += 256)
                if ((long long)base + t < pl.cap) pl_list(pl, par ^ 1)[base + t] = s_list[t];
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
    if (*(volatile unsigned*)trig_flag == 0u) return;
    const long long kk = iter_index(ctrl, kint, j);
    const int par = (int)(kk & 1);
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
