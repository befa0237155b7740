// feas_rb.cuh — EvalBest feasibility of the one-sign "count rows" (covering, packing, assignment,
// small-rhs 0/1 rows) as a nonzero-balanced row-block kernel
// (evaluator).
//
// Same counters as k_feas_count (sample_eval.cuh): per row, a bit-sliced saturating count over the
// 64-candidate words of its variables.  What changes is how the random gathers are issued — the
// k_dual_rb recipe (rowblock.cuh) — and that nothing on the issue path waits on a dependent load:
//   * each count class has its own CSR (an alias of K's when the class is a contiguous row range,
//     else a compacted copy) cut into blocks of <= FB_NNZ nonzeros and <= FB_ROWS rows, described by
//     one 16-byte record per block {first entry, rows | log2(G) << 8, first nonzero, nonzeros} (int32:
//     nnz < 2^31; G = lanes per row, the largest power of two <= 32 with G * rows <= FB_NT);
//   * a CTA (blockIdx.y = its group of WV words) walks blocks u, u + grid, ...; the record of block
//     u + 3*grid is loaded while unit u is reduced, the column indices (and row-in-block bytes) of
//     u + 2*grid likewise, so at the top of each iteration unit u + grid can be issued at once:
//     ONE cp.async per nonzero moving the WV words (WV = 2: 16 bytes = 128 candidates) of that
//     variable into shared memory, plus cp.async copies of the block's row pointers and packed row
//     targets — double-buffered, the reduction of u reads only shared memory;
//   * the reduction: each row by a group of G lanes (csa_add_bit per word, csa_add_counter across
//     the group: exact, order-free; a plain OR for the one-plane class, BMAX = 1); violated lanes
//     OR-ed into per-CTA shared words, flushed with one atomicOr per word at the end.
// Rows already satisfied in every lane by variables sampled with p = 1 (`skip`, from the trigger
// pass's count of exact ones) gather nothing: their flags are staged in shared memory one iteration
// ahead and a nonzero finds its row through the per-nonzero row-in-block byte `rib`.
#pragma once
#include "common.cuh"
#include "pdhg.cuh"
#include "sample_eval.cuh"

namespace gfors {

constexpr int FB_NNZ = 1024;   // nonzeros per row block, k_b <= 128 per unit (2 words: 16 KB of 16-byte gathers per buffer)
constexpr int FB_NNZ8 = 256;   // nonzeros per row block of the wide plan: 8 words (64 bytes) per nonzero, 16 KB per buffer
constexpr int FB_NT = 256;
constexpr int FB_ROWS = 255;   // rows per block (row-in-block index is a byte)

struct ClassCsr {
    const int* ptr;             // [nrows+1] class-local row pointers into idx (int32: nnz < 2^31)
    const int* idx;             // column indices
    const unsigned char* rib;   // row-in-block of each nonzero (indexed like idx)
    const int4* desc;           // [nblk] {first entry, rows | log2(G) << 8, first nonzero, nonzeros}
    const int* info;            // [nrows] packed target: t | rel << 16 | B << 20
    long long nblk;
};

__host__ __device__ constexpr int fb_pack_info(int t, int rel, int B) { return t | (rel << 16) | (B << 20); }

__device__ __forceinline__ void fb_cp4(void* smem, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g));
}
template <int WV>
__device__ __forceinline__ void fb_cp_async(uint64_t* smem, const uint64_t* g, uint64_t pol) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (WV == 2) asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(g), "l"(pol));
    else asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(s), "l"(g), "l"(pol));
}

template <int WV, int NNZ>
struct FbBuf {
    uint64_t tile[NNZ * WV];
    int rp[FB_ROWS + 1];
    int info[FB_ROWS];
    int nr;
};

// WV words per nonzero and unit: 1 or 2 (one 8/16-byte cp.async per nonzero, plan of FB_NNZ), or 8
// (k_b >= 512: the 64-byte piece of the sample row is moved by 4 consecutive lanes with 16 bytes each —
// one cache line per nonzero per warp instruction instead of 4 separate gathers; plan of FB_NNZ8)
template <int BMAX, int WV, int NNZ, bool SKIP>
__global__ void __launch_bounds__(FB_NT, 6) k_feas_rb(ClassCsr cc, const unsigned char* __restrict__ skip,
                                                   const uint64_t* __restrict__ X, int W,
                                                   unsigned long long* __restrict__ viol) {
    constexpr int LPN = WV >= 2 ? WV / 2 : 1;  // lanes per nonzero (16 bytes each)
    constexpr int U = NNZ * LPN / FB_NT;
    extern __shared__ __align__(16) unsigned char fb_smem[];  // two FbBuf (dynamic: > 48 KB for FB_NNZ)
    FbBuf<WV, NNZ>* buf = reinterpret_cast<FbBuf<WV, NNZ>*>(fb_smem);
    __shared__ unsigned long long s_viol[64];
    __shared__ unsigned char s_skip[2][FB_NT];  // skip flags of the rows of the next unit to issue (ring of 2)
    const bool use_smem = W <= 64;
    for (int w = threadIdx.x; w < 64; w += FB_NT) s_viol[w] = 0ull;
    const long long nunits = cc.nblk;
    const long long G0 = gridDim.x;
    const int w0 = blockIdx.y * WV;
    const uint64_t pf = l2_policy_evict_first(), pl = l2_policy_evict_last();
    auto desc = [&](long long u) { return u < nunits ? __ldg(cc.desc + u) : make_int4(0, 0, 0, 0); };
    // phase 1a for a unit whose descriptor d is in registers: indices, row-in-block bytes, skip flag
    int cols[U];
    unsigned char ribs[U];
    unsigned char skf = 0;
    auto load = [&](const int4& d) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int t = (k * FB_NT + threadIdx.x) / LPN;
            cols[k] = t < d.w ? ld_hint_i32(cc.idx + d.z + t, pf) : -1;
            if (SKIP) ribs[k] = t < d.w ? ld_hint_u8(cc.rib + d.z + t, pf) : 0;
        }
        skf = (SKIP && (int)threadIdx.x < (d.y & 0xff)) ? __ldg(skip + d.x + threadIdx.x) : 0;
    };
    // phase 1b: gathers + row metadata of unit u into buffer bi
    auto issue = [&](long long u, const int4& d, int bi) {
        FbBuf<WV, NNZ>& B = buf[bi];
        if (u < nunits) {
            const int nr = d.y & 0xff;
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (cols[k] >= 0 && !(SKIP && s_skip[bi][ribs[k]])) {
                    const int pq = k * FB_NT + threadIdx.x, t = pq / LPN, c = pq % LPN;
                    fb_cp_async<WV == 1 ? 1 : 2>(B.tile + t * WV + 2 * c, X + (long long)cols[k] * W + w0 + 2 * c, pl);
                }
            if ((int)threadIdx.x <= nr) fb_cp4(&B.rp[threadIdx.x], cc.ptr + d.x + threadIdx.x);
            if ((int)threadIdx.x < nr) fb_cp4(&B.info[threadIdx.x], cc.info + d.x + threadIdx.x);
            if (threadIdx.x == 0) B.nr = d.y;
        }
        asm volatile("cp.async.commit_group;");
    };
    const long long u0 = blockIdx.x;
    int4 d1 = desc(u0), d2 = desc(u0 + G0), d3;
    load(d1);
    s_skip[0][threadIdx.x] = skf;
    __syncthreads();
    issue(u0, d1, 0);
    load(d2);
    s_skip[1][threadIdx.x] = skf;
    d1 = d2;                 // descriptor of the unit issued next (u + grid)
    d2 = desc(u0 + 2 * G0);  // ... and of the one loaded next (u + 2*grid)
    __syncthreads();
    int st = 0;
    for (long long u = u0; u < nunits; u += G0) {
        issue(u + G0, d1, st ^ 1);
        load(d2);                 // unit u + 2*grid: consumed by the next iteration's issue
        d3 = desc(u + 3 * G0);    // unit u + 3*grid: consumed by the next iteration's load
        asm volatile("cp.async.wait_group 1;");
        __syncthreads();
        // phase 2: unit u from buffer st
        const FbBuf<WV, NNZ>& B = buf[st];
        const int nr = B.nr & 0xff, lgG = B.nr >> 8, G = 1 << lgG;
        const int p0 = B.rp[0];
        const int lane = threadIdx.x & (G - 1), grp = threadIdx.x >> lgG, ngr = FB_NT >> lgG;
        if constexpr (WV == 8) {
            // 8-word units: one thread per (row, word) walks the row's nonzeros with that word's counter
            // (a plain OR for the one-plane class); consecutive threads read consecutive words of a
            // nonzero (no bank conflicts) and no cross-lane reduction is needed.  The per-row lane groups
            // below (8 shuffle reductions per row) executed ~30x more instructions for these units.
            for (int task = threadIdx.x; task < nr * WV; task += FB_NT) {
                const int rr = task / WV, v = task % WV;
                const int in = B.info[rr];
                const int t = in & 0xffff, rel = (in >> 16) & 0xf, Bp = (in >> 20) & 0xf;
                if (SKIP && s_skip[st][rr]) continue;  // satisfied in every lane
                const int q0 = B.rp[rr] - p0, q1 = B.rp[rr + 1] - p0;
                uint64_t Cn[BMAX], sat = 0ull;
                if constexpr (BMAX == 1) {
                    uint64_t o0 = 0ull, o1 = 0ull;
                    int i = q0;
                    for (; i + 1 < q1; i += 2) { o0 |= B.tile[i * WV + v]; o1 |= B.tile[(i + 1) * WV + v]; }
                    if (i < q1) o0 |= B.tile[i * WV + v];
                    Cn[0] = o0 | o1;
                } else {
#pragma unroll
                    for (int q = 0; q < BMAX; ++q) Cn[q] = 0ull;
                    for (int i = q0; i < q1; ++i) csa_add_bit<BMAX>(Cn, sat, B.tile[i * WV + v], Bp);
                }
                const uint64_t bad = ~count_ok<BMAX>(Cn, sat, Bp, t, rel);
                if (bad) atomicOr(use_smem ? &s_viol[w0 + v] : viol + w0 + v, (unsigned long long)bad);
            }
        } else {
        // VB words per pass over the rows (both words for k_b = 128; one at a time for the 8-word units,
        // whose counters would not fit in registers)
        constexpr int VB = WV <= 2 ? WV : 1;
        for (int v0 = 0; v0 < WV; v0 += VB)
        for (int rb = 0; rb < nr; rb += ngr) {
            const int rr = rb + grp;
            const bool valid = rr < nr;
            int Bp = 1, t = 0, rel = 3, q0 = 0, q1 = 0;
            if (valid) {
                const int in = B.info[rr];
                t = in & 0xffff; rel = (in >> 16) & 0xf; Bp = (in >> 20) & 0xf;
                q0 = B.rp[rr] - p0; q1 = B.rp[rr + 1] - p0;
                if (SKIP && s_skip[st][rr]) { rel = 4; q1 = q0; }
            }
            uint64_t Cn[VB][BMAX], sat[VB];
#pragma unroll
            for (int v = 0; v < VB; ++v) {
                sat[v] = 0ull;
#pragma unroll
                for (int q = 0; q < BMAX; ++q) Cn[v][q] = 0ull;
            }
            if constexpr (BMAX == 1) {
                // one plane (B = 1, count capped at 1): the count is the OR of the words
                uint64_t o[VB];
#pragma unroll
                for (int v = 0; v < VB; ++v) o[v] = 0ull;
                if (rel < 3)
                    for (int i = q0 + lane; i < q1; i += G) {
#pragma unroll
                        for (int v = 0; v < VB; ++v) o[v] |= B.tile[i * WV + v0 + v];
                    }
#pragma unroll
                for (int v = 0; v < VB; ++v) {
                    for (int sh = G >> 1; sh > 0; sh >>= 1) o[v] |= __shfl_xor_sync(0xffffffffu, o[v], sh, G);
                    Cn[v][0] = o[v];
                }
            } else {
                if (rel < 3)
                    for (int i = q0 + lane; i < q1; i += G) {
#pragma unroll
                        for (int v = 0; v < VB; ++v) csa_add_bit<BMAX>(Cn[v], sat[v], B.tile[i * WV + v0 + v], Bp);
                    }
#pragma unroll
                for (int v = 0; v < VB; ++v)
                    for (int o = G >> 1; o > 0; o >>= 1) {
                        uint64_t D[BMAX];
#pragma unroll
                        for (int q = 0; q < BMAX; ++q) D[q] = __shfl_xor_sync(0xffffffffu, Cn[v][q], o, G);
                        const uint64_t dsat = __shfl_xor_sync(0xffffffffu, sat[v], o, G);
                        csa_add_counter<BMAX>(Cn[v], sat[v], D, dsat, Bp);
                    }
            }
            if (lane == 0 && valid) {
#pragma unroll
                for (int v = 0; v < VB; ++v) {
                    const uint64_t bad = ~count_ok<BMAX>(Cn[v], sat[v], Bp, t, rel);
                    if (bad) atomicOr(use_smem ? &s_viol[w0 + v0 + v] : viol + w0 + v0 + v, (unsigned long long)bad);
                }
            }
        }
        }  // (per-row lane groups)
        __syncthreads();                  // buffer st and s_skip[st] are free
        s_skip[st][threadIdx.x] = skf;    // flags of unit u + 2*grid (issued next iteration into st)
        d1 = d2;
        d2 = d3;
        st ^= 1;
    }
    asm volatile("cp.async.wait_all;");
    __syncthreads();
    if (use_smem)
        for (int w = threadIdx.x; w < W; w += FB_NT)
            if (s_viol[w]) atomicOr(viol + w, s_viol[w]);
}

// skip[e] = 1: class entry e is a ">= t" row already holding t variables sampled with p = 1 (every
// lane satisfies it, no gathers needed).  ones[] is the trigger pass's per-row count of x_k == 1.
__global__ void k_feas_skip(CountRows cr, const unsigned char* __restrict__ ones, unsigned char* __restrict__ skip) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < cr.nrows; e += gridDim.x * (long long)blockDim.x)
        skip[e] = (cr.rel[e] == 0 && (int)ones[cr.row[e]] >= cr.t[e]) ? 1 : 0;
}

// load time: the row-in-block byte of every nonzero of a plan, from its descriptors (one warp per row;
// rib is indexed like idx, i.e. from position base of the class's nonzeros)
__global__ void __launch_bounds__(256) k_fb_rib(const int4* __restrict__ desc, const int* __restrict__ ptr, long long nblk,
                                                long long base, unsigned char* __restrict__ rib) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
        const int4 d = desc[b];
        const int nr = d.y & 0xff;
        for (int r = wid; r < nr; r += blockDim.x >> 5)
            for (long long q = ptr[d.x + r] + lane; q < ptr[d.x + r + 1]; q += 32) rib[q - base] = (unsigned char)r;
    }
}

}  // namespace gfors
