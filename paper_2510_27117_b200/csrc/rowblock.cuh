// rowblock.cuh — nonzero-balanced "row-block" SpMV kernels for the PDHG step (B200 design).
//
// The PDHG products K xbar (rows of K_u) and K' w (rows of the transposed CSR) have short rows
// (2..98 and ~10 nonzeros on config 5) and random column indices, so each iteration is a stream of
// int32 indices from HBM plus one random L2 gather per nonzero.  Measured on B200, random 4-8 byte
// gathers saturate at ~0.9 per cycle per SM (one L1TEX wavefront each) whatever the cache policy,
// so the kernels are built to keep that pipe full:
//   * one CTA owns a contiguous range of rows holding <= RB_NNZ nonzeros (planned on the host);
//   * phase 1 streams the block's indices (coalesced, evict-first) and issues one cp.async (LDGSTS)
//     gather per nonzero straight into shared memory — no registers held by in-flight loads, so
//     occupancy stays at 2048 threads/SM — double-buffered: the gathers of the CTA's next row block
//     are in flight while the current one is reduced;
//   * phase 2 reduces rows from shared memory with groups of G threads (G = 32..1 from the block's
//     row count, fixed order => deterministic) and runs the fused epilogue (dual clamp, or primal
//     box projection + extrapolation) with coalesced vector traffic.
#pragma once
#include "common.cuh"
#include "pdhg.cuh"
#include "push_list.cuh"

namespace gfors {

// Nonzeros per row block: 2048 (8 per thread) for fp32, 1024 for fp64.  The double-buffered
// gather tile takes 2*RB_NNZ*sizeof(T) of shared memory per CTA and the rest of the SM's 256 KB
// L1/shared array is the L1 that tracks the in-flight gathers: at 32 KB per CTA (fp64, 2048) the
// carve-out leaves too few L1 lines and the gather rate halves (measured: 0.42 vs 0.87 gathers per
// cycle per SM, scratch microbenchmark), at 16 KB it does not (config 5 fp64 dual 0.47 -> 0.27 ms).
constexpr int RB_NNZ32 = 2048;
constexpr int RB_NNZ64 = 1024;
constexpr int RB_NT = 256;
template <typename T>
constexpr int RB_NNZ_OF = sizeof(T) == 8 ? RB_NNZ64 : RB_NNZ32;

// the index stream is read once: not allocated in L1, whose capacity tracks the in-flight 4-byte
// cp.async.ca gathers (measured: dual 2.496 -> 2.470 ms per dense block against ld.global.cs)
__device__ __forceinline__ int ldcs_i32(const int* p) {
    int v;
    asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* g) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (sizeof(T) == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(g));
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;"); }

// phase 1 of row block b, split in two so the index loads of block b+2*grid are in flight while
// block b is reduced: rb_load_idx (registers, evict-first) then rb_issue (cp.async gathers)
template <int U>
__device__ __forceinline__ void rb_load_idx(const Csr& A, const long long* __restrict__ blk_row, long long b,
                                            long long nblk, int (&cols)[U]) {
    if (b < nblk) {
        const long long p0 = __ldg(A.ptr + blk_row[b]);
        const int cnt = (int)(__ldg(A.ptr + blk_row[b + 1]) - p0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = u * RB_NT + threadIdx.x;
            cols[u] = t < cnt ? ldcs_i32(A.idx + p0 + t) : -1;
        }
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) cols[u] = -1;
    }
}

template <typename T, int U>
__device__ __forceinline__ void rb_issue(const int (&cols)[U], const T* __restrict__ v, T* sv) {
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (cols[u] >= 0) cp_async_elem(sv + u * RB_NT + threadIdx.x, v + cols[u]);
    cp_async_commit();
}

__device__ __forceinline__ int rb_group_size(int nr) {
    int G = 32;
    while (G > 1 && G * nr > RB_NT) G >>= 1;
    return G;
}

__device__ __forceinline__ double rb_group_sum(double v, int G) {
    for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
    return v;
}

// sum of val_q * sv[q - p0] over the row's nonzeros [q0, q1) by the G lanes of a group.
// ILP4: four independent accumulators combined as ((a0 + a1) + (a2 + a3)) (fixed order) so the
// shared-memory loads of a long per-thread row overlap; costs registers, used where G is small.
template <typename T, int KIND, bool ILP4 = false>
__device__ __forceinline__ double rb_row_sum(const Csr& A, const T* sv, long long p0, long long q0, long long q1,
                                             int lane, int G) {
    const int i1 = (int)(q1 - p0);
    int i = (int)(q0 - p0) + lane;
    if constexpr (!ILP4) {
        double acc = 0.0;
        for (; i < i1; i += G) {
            if constexpr (KIND == KV_SIGN) acc += (double)sv[i];
            else acc += kval<KIND>(A.val, p0 + i) * (double)sv[i];
        }
        return acc;
    } else {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if constexpr (KIND == KV_SIGN) {
            for (; i + 3 * G < i1; i += 4 * G) {
                a0 += (double)sv[i]; a1 += (double)sv[i + G]; a2 += (double)sv[i + 2 * G]; a3 += (double)sv[i + 3 * G];
            }
            for (; i < i1; i += G) a0 += (double)sv[i];
        } else {
            for (; i + 3 * G < i1; i += 4 * G) {
                a0 += kval<KIND>(A.val, p0 + i) * (double)sv[i];
                a1 += kval<KIND>(A.val, p0 + i + G) * (double)sv[i + G];
                a2 += kval<KIND>(A.val, p0 + i + 2 * G) * (double)sv[i + 2 * G];
                a3 += kval<KIND>(A.val, p0 + i + 3 * G) * (double)sv[i + 3 * G];
            }
            for (; i < i1; i += G) a0 += kval<KIND>(A.val, p0 + i) * (double)sv[i];
        }
        return (a0 + a1) + (a2 + a3);
    }
}

// ---------------------------------------------------------------------------------------------
// Dual half-step on row blocks of K_u:
//   y_k = Pi( y_{k-1} + tau2 (K xbar_{k-1} + r) ),  K = -diag(g) K_u,  w = g rsign y_k
// Nothing on the issue path waits on a dependent load: each row block has a 16-byte descriptor
// {first row, rows | log2(G) << 16, first nonzero, nonzeros} (host-built, int32: nnz < 2^31); a CTA loads the
// descriptor of unit b + 3*grid and the column indices of b + 2*grid while it reduces unit b, and at
// the top of each iteration issues unit b + grid at once: one cp.async per nonzero (x-bar gather),
// plus cp.async copies of the block's row pointers and sign bytes, so the reduction reads only shared
// memory; the per-row y, g, r-hat loads of the epilogue are issued before the row's reduction.  The
// shared-memory footprint stays ~18 KB per CTA: the L1 left over tracks the in-flight 4-byte gathers
// (at ~26 KB per CTA x 8 CTAs the dual ran 1.8x slower).
// ---------------------------------------------------------------------------------------------
constexpr int RB_RMAX = 192;  // rows per row block (the plans cap them; per-row data lives in smem)

template <typename T>
struct DualBuf {  // (ordered so every member is naturally aligned for its cp.async)
    T tile[RB_NNZ_OF<T>];
    int4 d;                    // the unit's descriptor
    int rp[RB_RMAX + 1];
    int sgw[RB_RMAX / 4 + 2];  // sign bytes, 4-byte aligned window starting at row (r0 & ~3)
};

__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g));
}

template <typename T, int KIND>
__global__ void __launch_bounds__(RB_NT, 8) k_dual_rb(Csr K, const int4* __restrict__ desc, const int* __restrict__ ptr32,
                                                   long long nblk, State<T> s, const double* __restrict__ g,
                                                   const double* __restrict__ rh, const signed char* __restrict__ rsign,
                                                   long long m1, const Ctrl* __restrict__ ctrl, long long kint,
                                                   long long j, double* __restrict__ u_out, PushList pl) {
    constexpr int NZ = RB_NNZ_OF<T>;
    constexpr int U = NZ / RB_NT;
    __shared__ __align__(16) DualBuf<T> buf[2];
    const int par = cta_parity(ctrl, kint, j);
    if (cta_push_mode(pl, par)) return;  // sparse xbar: k_push_scatter/k_push_rows do this iteration
    const bool clear_acc = pl.acc && pl_valid(pl, par);
    if (pl.acc && blockIdx.x == 0 && threadIdx.x == 0) { push_reset_next(pl, par); pl_set_valid(pl, par ^ 1, false); }
    const T* __restrict__ xb = par ? s.xb[1] : s.xb[0];
    const T* __restrict__ yin = par ? s.y[1] : s.y[0];
    T* __restrict__ yout = par ? s.y[0] : s.y[1];
    const double tau2 = ctrl->tau2;
    const long long G0 = gridDim.x;
    auto ldesc = [&](long long b) { return b < nblk ? __ldg(desc + b) : make_int4(0, 0, 0, 0); };
    int cols[U];
    auto load = [&](const int4& d) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = u * RB_NT + threadIdx.x;
            cols[u] = t < d.w ? ldcs_i32(K.idx + d.z + t) : -1;
        }
    };
    auto issue = [&](long long b, const int4& d, int bi) {
        DualBuf<T>& B = buf[bi];
        if (b < nblk) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (cols[u] >= 0) cp_async_elem(B.tile + u * RB_NT + threadIdx.x, xb + cols[u]);
            const int nr = d.y & 0xffff, r0 = d.x, t = threadIdx.x;
            if (t <= nr) cp_async4(&B.rp[t], ptr32 + r0 + t);
            if constexpr (KIND == KV_SIGN) {
                const int a0 = r0 & ~3;
                if (t < ((r0 + nr - a0) + 3) / 4) cp_async4(&B.sgw[t], rsign + a0 + 4 * t);
            }
            if (t == 0) B.d = d;
        }
        asm volatile("cp.async.commit_group;");
    };
    const long long b0 = blockIdx.x;
    int4 d1 = ldesc(b0), d2 = ldesc(b0 + G0), d3;
    load(d1);
    issue(b0, d1, 0);
    load(d2);
    d1 = d2;
    d2 = ldesc(b0 + 2 * G0);
    int st = 0;
    for (long long b = b0; b < nblk; b += G0) {
        issue(b + G0, d1, st ^ 1);
        load(d2);
        d3 = ldesc(b + 3 * G0);
        cp_async_wait1();
        __syncthreads();
        const DualBuf<T>& B = buf[st];
        const int4 d = B.d;
        const int nr = d.y & 0xffff, lg = d.y >> 16, G = 1 << lg;
        const long long r0 = d.x;
        const int p0 = d.z;
        const int lane = threadIdx.x & (G - 1), grp = threadIdx.x >> lg, ngr = RB_NT >> lg;
        for (int rb = 0; rb < nr; rb += ngr) {
            const int rr = rb + grp;
            const long long row = r0 + rr;
            double acc = 0.0, gj = 0.0, rhj = 0.0, yj = 0.0;
            if (rr < nr) {
                if (lane == 0) { gj = g[row]; rhj = rh[row]; yj = (double)yin[row]; }  // in flight during the sum
                acc = rb_row_sum<T, KIND>(K, B.tile, p0, B.rp[rr], B.rp[rr + 1], lane, G);
            }
            acc = rb_group_sum(acc, G);
            if (lane == 0 && rr < nr) {
                double sg = 1.0;
                if constexpr (KIND == KV_SIGN)
                    sg = (double)reinterpret_cast<const signed char*>(B.sgw)[(r0 & 3) + rr];
                double yn = yj + tau2 * (rhj - gj * (sg * acc));
                if (row < m1 && yn < 0.0) yn = 0.0;
                const T yt = (T)yn;
                yout[row] = yt;
                s.w[row] = w_of(gj, sg, yt);
                if (u_out) u_out[row] = sg * acc;  // (K_u xbar_{k-1})_j, kept for the trigger pass
                if (clear_acc) pl.acc[row] = 0;    // delta-push accumulators are stale after a gather
            }
        }
        __syncthreads();
        d1 = d2;
        d2 = d3;
        st ^= 1;
    }
    asm volatile("cp.async.wait_all;");
}

// ---------------------------------------------------------------------------------------------
// Primal half-step on row blocks of K_u' (one "row" = one variable i):
//   delta = c + rho + K'y_k + 2Q x_{k-1} - 2 rho x_{k-1};  x_k = Pi_[0,1](x_{k-1} - tau1 delta);
//   xbar_k = 2 x_k - x_{k-1}
// ---------------------------------------------------------------------------------------------
template <typename T, int KIND, bool HASQ>
__global__ void __launch_bounds__(RB_NT, 6) k_primal_rb(Csr Kt, const long long* __restrict__ blk_row, long long nblk,
                                                     Csr Q, const T* __restrict__ qs, State<T> s,
                                                     const T* __restrict__ cs, const Ctrl* __restrict__ ctrl,
                                                     long long kint, long long j, PushList pl, PushPrimal pp) {
    constexpr int NZ = RB_NNZ_OF<T>;
    __shared__ __align__(16) T sv[2][NZ];
    __shared__ unsigned s_cnt, s_base;
    __shared__ int s_list[RB_NT];
    __shared__ bool s_en, s_dd;
    const int par = cta_parity(ctrl, kint, j);
    if (cta_pp_mode(pp, par).push) return;  // push-mode primal runs instead
    const bool clear_accx = pp_valid(pp, par);  // delta-push accumulators are stale after a gather
    if (pp.accx && blockIdx.x == 0 && threadIdx.x == 0) pp_set_next(pp, par, false, 0);
    const T* __restrict__ xin = par ? s.x[1] : s.x[0];
    T* __restrict__ xout = par ? s.x[0] : s.x[1];
    T* __restrict__ xbout = par ? s.xb[0] : s.xb[1];
    const T* __restrict__ xbprev = par ? s.xb[1] : s.xb[0];
    const double rho = ctrl->rho, tau1 = ctrl->tau1;
    int st = 0;
    int nxt[NZ / RB_NT];
    rb_load_idx(Kt, blk_row, blockIdx.x, nblk, nxt);
    rb_issue(nxt, s.w, sv[0]);
    rb_load_idx(Kt, blk_row, blockIdx.x + gridDim.x, nblk, nxt);
    for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
        rb_issue(nxt, s.w, sv[st ^ 1]);
        rb_load_idx(Kt, blk_row, b + 2LL * gridDim.x, nblk, nxt);
        if (threadIdx.x == 0) {
            s_en = pl.acc && *(volatile unsigned*)pl_count(pl, par ^ 1) <= pl.thr;
            s_dd = pl.acc && pl_valid(pl, par ^ 1);
        }
        cp_async_wait1();
        __syncthreads();
        const long long r0 = blk_row[b], r1 = blk_row[b + 1];
        const long long p0 = __ldg(Kt.ptr + r0);
        const int nr = (int)(r1 - r0);
        const int G = rb_group_size(nr);
        const int lane = threadIdx.x & (G - 1), grp = threadIdx.x / G, ngr = RB_NT / G;
        const bool en = s_en, dd = s_dd;
        for (int rb = 0; rb < nr; rb += ngr) {
            const int rr = rb + grp;
            const long long i = r0 + rr;
            double a = 0.0, bq = 0.0, xi = 0.0, ci = 0.0;
            if (rr < nr) {
                if (lane == 0) { xi = (double)xin[i]; ci = (double)cs[i]; }  // issued before the reduction
                a = rb_row_sum<T, KIND, true>(Kt, sv[st], p0, __ldg(Kt.ptr + i), __ldg(Kt.ptr + i + 1), lane, G);
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
            if (lane == 0 && rr < nr) {
                const double delta = ((ci + rho) - a) + 2.0 * bq - 2.0 * rho * xi;
                double xn = xi - tau1 * delta;
                xn = xn < 0.0 ? 0.0 : (xn > 1.0 ? 1.0 : xn);
                xout[i] = (T)xn;
                const T xbn = (T)(2.0 * xn - xi);
                xbout[i] = xbn;
                nz = pl_listed(dd, xbn, dd ? xbprev[i] : (T)0);
                if (clear_accx) pp.accx[i] = 0;
            }
            push_append<RB_NT>(pl, par ^ 1, nz, (int)i, en, &s_cnt, &s_base, s_list);
        }
        __syncthreads();
        st ^= 1;
    }
    asm volatile("cp.async.wait_all;");
}

// ---------------------------------------------------------------------------------------------
// Trigger row pass on row blocks: v = K_u x_k (one gather per nonzero), and
// d = K_u (x_k - xbar_{k-1}) = v - u with u = K_u xbar_{k-1} stored by the last dual of the block.
// ---------------------------------------------------------------------------------------------
template <typename T, int KIND>
__global__ void __launch_bounds__(RB_NT) k_trig_rows_rb(Csr K, const long long* __restrict__ blk_row, long long nblk,
                                                        State<T> s, const double* __restrict__ g,
                                                        const double* __restrict__ rh,
                                                        const signed char* __restrict__ rsign, long long m1,
                                                        const double* __restrict__ u_prev, const Ctrl* __restrict__ ctrl,
                                                        long long kint, long long j, double* __restrict__ part1,
                                                        unsigned char* __restrict__ ones_out,
                                                        const unsigned* __restrict__ trig_flag) {
    constexpr int NZ = RB_NNZ_OF<T>;
    __shared__ __align__(16) T sv[2][NZ];
    __shared__ double sh[32];
    __shared__ int s_skip;  // (read once per CTA, see cta_push_mode)
    if (threadIdx.x == 0) s_skip = (trig_flag && *(volatile const unsigned*)trig_flag) ? 1 : 0;
    __syncthreads();
    if (s_skip) return;  // x_k was pushed: k_trig_rows_push
    const int par = cta_parity(ctrl, kint, j);
    const T* __restrict__ xk = par ? s.x[0] : s.x[1];
    const T* __restrict__ yprev = par ? s.y[1] : s.y[0];
    const T* __restrict__ ynew = par ? s.y[0] : s.y[1];
    const double tau2 = ctrl->tau2;
    double ge = 0.0, eq = 0.0, sy2 = 0.0;
    int st = 0;
    int nxt[NZ / RB_NT];
    rb_load_idx(K, blk_row, blockIdx.x, nblk, nxt);
    rb_issue(nxt, xk, sv[0]);
    rb_load_idx(K, blk_row, blockIdx.x + gridDim.x, nblk, nxt);
    for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
        rb_issue(nxt, xk, sv[st ^ 1]);
        rb_load_idx(K, blk_row, b + 2LL * gridDim.x, nblk, nxt);
        cp_async_wait1();
        __syncthreads();
        const long long r0 = blk_row[b], r1 = blk_row[b + 1];
        const long long p0 = __ldg(K.ptr + r0);
        const int nr = (int)(r1 - r0);
        const int G = rb_group_size(nr);
        const int lane = threadIdx.x & (G - 1), grp = threadIdx.x / G, ngr = RB_NT / G;
        for (int rb = 0; rb < nr; rb += ngr) {
            const int rr = rb + grp;
            const long long row = r0 + rr;
            double v = 0.0;
            int c1 = 0;  // entries of the row with x_k == 1 exactly (sampled as 1 in every lane)
            if (rr < nr) {
                const long long q0 = __ldg(K.ptr + row), q1 = __ldg(K.ptr + row + 1);
                v = rb_row_sum<T, KIND>(K, sv[st], p0, q0, q1, lane, G);
                if (ones_out)
                    for (long long q = q0 + lane; q < q1; q += G) c1 += sv[st][q - p0] == (T)1;
            }
            v = rb_group_sum(v, G);
            if (ones_out)
                for (int o = G >> 1; o > 0; o >>= 1) c1 += __shfl_xor_sync(0xffffffffu, c1, o, G);
            if (lane == 0 && rr < nr) {
                if (ones_out) ones_out[row] = (unsigned char)min(c1, 255);
                const double sg = (KIND == KV_SIGN) ? (double)rsign[row] : 1.0;
                const double gj = g[row];
                const double ku = sg * v;  // (K_u x_k)_j
                const double gap = rh[row] - gj * ku;
                if (row < m1) ge = fmax(ge, fmax(gap, 0.0)); else eq = fmax(eq, fabs(gap));
                const double sy = ((double)yprev[row] - (double)ynew[row]) / tau2 + gj * (ku - u_prev[row]);
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

}  // namespace gfors
