// gfors.cu — C ABI (include/gfors.h) and device runtime of the B200 GFORS hot path.
//
// Host side: validation + canonicalisation + layout planning (once per gfors_load), the device
// Preprocess driver, and the loop driver, which captures one Alg. 1 sampling block
// (k_int PDHG iterations, indicators, k_r x [sample, evaluate, argmin], CheckHalt) into the body
// of a CUDA-graph WHILE node whose condition is set on the device by the CheckHalt kernel, so
// a whole gfors_run is one graph launch with no host synchronisation inside the loop.
#include <cuda_runtime.h>
#include <math.h>
#include <cmath>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <map>
#include <tuple>
#include <mutex>
#include <thread>
#include <condition_variable>
#include <functional>
#include <cub/cub.cuh>
#include <cstdarg>
#include <memory>
#include <string>
#include <vector>

#include "../../include/gfors.h"
#include "common.cuh"
#include "pdhg.cuh"
#include "prep.cuh"
#include "sample_eval.cuh"
#include "rowblock.cuh"
#include "sparse_primal.cuh"
#include "shard.cuh"
#include "push_dual.cuh"
#include "push_primal.cuh"
#include "dense_q.cuh"
#include "assign3d.cuh"
#include "repair.cuh"
#include "feas_rb.cuh"
#include "cover.cuh"
#include <cudaTypedefs.h>
#include <cstdlib>

using namespace gfors;

namespace {

constexpr int NT = 256;
inline int rb_grid() { return sm_count() * 8; }  // persistent row-block kernels: 8 CTAs per SM

struct Err {
    gfors_status st;
    std::string msg;
};

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e__ = (call);                                                             \
        if (e__ != cudaSuccess)                                                               \
            throw Err{e__ == cudaErrorMemoryAllocation ? GFORS_E_OOM : GFORS_E_CUDA,          \
                      std::string(#call) + ": " + cudaGetErrorString(e__)};                   \
    } while (0)

[[noreturn]] void input_error(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Err{GFORS_E_INPUT, buf};
}

// Device memory comes from a PRIVATE stream-ordered pool per device (the device's default pool,
// which other libraries share, is left untouched) with an unbounded release threshold: memory a
// closed solver frees stays mapped while other solvers live, so the next load reuses it instead of
// paying the page mapping again (measured: the K upload + transpose phase of a config-5 load varies
// 42-300 ms with plain cudaMalloc/cudaFree); gfors_release_memory trims it on request.
// Allocation runs on a private non-blocking stream and is made synchronous (allocate + sync); frees
// are stream-ordered on that stream after the owning context's stream is drained.  A caller
// allocator (gfors_device_opts.alloc/free) replaces all of this for its context.
// optional caller allocator of the context whose API call runs on this thread (gfors_device_opts)
struct AllocHooks {
    void* (*alloc)(size_t, void*) = nullptr;
    void (*free)(void*, void*) = nullptr;
    void* ctx = nullptr;
};
static thread_local AllocHooks tls_hooks;
struct HookScope {  // installs a context's hooks for the duration of one API call
    AllocHooks prev;
    explicit HookScope(const AllocHooks& h) : prev(tls_hooks) { tls_hooks = h; }
    ~HookScope() { tls_hooks = prev; }
};

static cudaMemPool_t& pool_of(int dev) {
    static cudaMemPool_t pools[64] = {};
    return pools[dev];
}
static cudaStream_t alloc_stream() {
    static std::mutex mu;
    static cudaStream_t st[64] = {};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!st[dev]) {
        // a PRIVATE pool (the device's default pool, which other libraries share, is left untouched)
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        CK(cudaMemPoolCreate(&pool_of(dev), &props));
        unsigned long long thr = ~0ull;
        CK(cudaMemPoolSetAttribute(pool_of(dev), cudaMemPoolAttrReleaseThreshold, &thr));
        CK(cudaStreamCreateWithFlags(&st[dev], cudaStreamNonBlocking));
    }
    return st[dev];
}

// contexts alive per device (create +1, destroy -1); returns the new count
static int live_contexts(int dev, int delta) {
    static std::mutex mu;
    static int live[64] = {};
    if (dev < 0 || dev >= 64) return 1;
    std::lock_guard<std::mutex> g(mu);
    live[dev] = std::max(0, live[dev] + delta);
    return live[dev];
}

// The private pool keeps what it has mapped when solvers close: trimming it after the last solver and
// re-mapping for the next one made a config-5 load take 0.12-2.3 s instead of a steady 0.11 s (the
// driver's page mapping; measured with profiles/exp_e2e.py).  gfors_release_memory(device) returns the
// pool's unused memory to the system on request.
static void pool_release(int dev) {
    if (dev < 0 || dev >= 64 || !pool_of(dev)) return;
    cudaMemPoolTrimTo(pool_of(dev), 0);
    cudaGetLastError();
}

template <typename X>
X* dalloc(size_t count) {
    if (count == 0) count = 1;
    void* p = nullptr;
    if (tls_hooks.alloc) {
        p = tls_hooks.alloc(count * sizeof(X), tls_hooks.ctx);
        if (!p) throw Err{GFORS_E_OOM, "device_opts.alloc returned NULL"};
        return reinterpret_cast<X*>(p);
    }
    cudaStream_t as = alloc_stream();
    if (as) {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaMallocFromPoolAsync(&p, count * sizeof(X), pool_of(dev), as));
        CK(cudaStreamSynchronize(as));
    } else {
        CK(cudaMalloc(&p, count * sizeof(X)));
    }
    return reinterpret_cast<X*>(p);
}
// allocator whose resize() leaves new elements uninitialised: the large host copies of K are then
// first touched by the parallel copy loops instead of a serial value-initialisation pass
template <typename T>
struct DefaultInitAlloc : std::allocator<T> {
    template <typename U> struct rebind { using other = DefaultInitAlloc<U>; };
    DefaultInitAlloc() = default;
    template <typename U> DefaultInitAlloc(const DefaultInitAlloc<U>&) {}
    template <typename U> void construct(U* p) noexcept { ::new ((void*)p) U; }
    template <typename U, typename... A> void construct(U* p, A&&... a) { ::new ((void*)p) U(std::forward<A>(a)...); }
};
template <typename T> using hvec = std::vector<T, DefaultInitAlloc<T>>;

template <typename X>
X* dupload_raw(const X* p, size_t count, cudaStream_t s) {
    X* d = dalloc<X>(count);
    if (count) CK(cudaMemcpyAsync(d, p, count * sizeof(X), cudaMemcpyHostToDevice, s));
    return d;
}

template <typename X, typename Al>
X* dupload(const std::vector<X, Al>& v, cudaStream_t s) {
    X* p = dalloc<X>(v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice, s));
    return p;
}

int grid_for(long long work, int per_thread = 1) {
    long long b = (work / per_thread + NT - 1) / NT;
    if (b < 1) b = 1;
    if (b > sm_count() * 8) b = sm_count() * 8;
    return (int)b;
}

int pick_sub(double mean_len) {
    if (mean_len <= 2.5) return 2;
    if (mean_len <= 6) return 4;
    if (mean_len <= 12) return 8;
    if (mean_len <= 24) return 16;
    return 32;
}

struct HostSeg {
    std::vector<long long> seg_start, row_seg;
    std::vector<int> seg_row;
};

// split each row of a CSR into segments of at most seg nonzeros
HostSeg make_segments(const std::vector<int64_t>& ptr, long long rows, long long seg) {
    HostSeg h;
    h.row_seg.resize(rows + 1);
    h.row_seg[0] = 0;
    for (long long r = 0; r < rows; ++r) {
        const long long len = ptr[r + 1] - ptr[r];
        const long long ns = len == 0 ? 0 : (len + seg - 1) / seg;
        for (long long k = 0; k < ns; ++k) {
            h.seg_start.push_back(ptr[r] + k * seg);
            h.seg_row.push_back((int)r);
        }
        h.row_seg[r + 1] = h.row_seg[r] + ns;
    }
    h.seg_start.push_back(ptr[rows]);
    return h;
}

struct DevSeg {
    long long* seg_start = nullptr;
    int* seg_row = nullptr;
    long long* row_seg = nullptr;
    long long nseg = 0;
    SegPlan plan() const { return SegPlan{seg_start, seg_row, row_seg, nseg}; }
};

struct DirPlan {  // how one product direction (K rows or K' columns) is computed
    int sub = 32;
    bool seg = false;        // long rows: fixed-length segments + ordered combine
    bool rb = false;         // row blocks of <= RB_NNZ_OF<T> nonzeros per CTA
    long long seg_len = 1024;
    DevSeg ds;
    long long* blk_row = nullptr;
    long long nblk = 0;
    int4* desc = nullptr;    // per row block {first row, rows | log2(G) << 16, first nonzero, nonzeros} (k_dual_rb)
    int* ptr32 = nullptr;    // int32 copy of the row pointers (nnz < 2^31)
    std::vector<long long> hblk;  // host copy of the block boundaries (row-sharded dual)
};

// greedy nonzero-balanced row blocks: consecutive rows, <= cap nonzeros each (rows <= cap long)
// rows per row block at most (empty rows, e.g. every column when m = 0, would otherwise pile into
// one CTA: max cut's primal took 84 us per launch for n = 20480 in a single block)
constexpr long long RB_ROWS_MAX = RB_RMAX;  // per-row data of a block is staged in smem (k_dual_rb)

static std::vector<long long> make_rowblocks_from(const std::vector<int64_t>& ptr, long long rows, long long cap,
                                                  long long cap_rows = LLONG_MAX) {
    std::vector<long long> b;
    b.push_back(0);
    long long r = 0;
    while (r < rows) {
        long long e = r;
        while (e < rows && ptr[e + 1] - ptr[r] <= cap && e - r < cap_rows) ++e;
        if (e == r) e = r + 1;  // (not reached when every row is <= cap)
        b.push_back(e);
        r = e;
    }
    return b;
}
static std::vector<long long> make_rowblocks(const std::vector<int64_t>& ptr, long long rows, long long cap,
                                             long long cap_rows = LLONG_MAX) {
    return make_rowblocks_from(ptr, rows, cap, cap_rows);
}

// descriptors of the row blocks for k_dual_rb (G = 2^lg lanes per row, the largest power of two <= 32
// with G * rows <= RB_NT)
int4* upload_desc(const std::vector<long long>& b, const std::vector<int64_t>& ptr, cudaStream_t s,
                  std::vector<void*>& owned) {
    const long long nb = (long long)b.size() - 1;
    std::vector<int4> desc((size_t)std::max<long long>(nb, 1));
    for (long long k = 0; k < nb; ++k) {
        const int nr = (int)(b[k + 1] - b[k]);
        int lg = 5;
        while (lg > 0 && (1 << lg) * nr > RB_NT) --lg;
        desc[k] = make_int4((int)b[k], nr | (lg << 16), (int)ptr[b[k]], (int)(ptr[b[k + 1]] - ptr[b[k]]));
    }
    int4* dd = dupload(desc, s);
    owned.push_back(dd);
    return dd;
}

// int32 copy of a row-pointer array on the device (nnz < 2^31)
__global__ void k_ptr32(const long long* __restrict__ p64, long long len, int* __restrict__ p32) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += gridDim.x * (long long)blockDim.x)
        p32[i] = (int)p64[i];
}

// maxlen: the longest row (precomputed by the load); dptr64: the device copy of ptr
DirPlan plan_direction(const std::vector<int64_t>& ptr, long long rows, cudaStream_t s,
                       std::vector<void*>& owned, long long maxlen, const long long* dptr64) {
    DirPlan d;
    const long long nnz = ptr[rows];
    const double mean = rows ? (double)nnz / (double)rows : 0.0;
    d.sub = pick_sub(mean);
    // long or few rows: fixed-length segments, one warp each (>= 8 warps per SM of work)
    const long long groups = rows;
    d.seg = (maxlen > 4096) || (groups * 32 < (long long)sm_count() * 2048 && nnz > (long long)sm_count() * 1024);
    if (maxlen <= RB_NNZ32) {
        d.seg = false;
        d.rb = true;
    }
    if (d.rb) {
        std::vector<long long> b = make_rowblocks(ptr, rows, RB_NNZ32, RB_ROWS_MAX);
        d.nblk = (long long)b.size() - 1;
        d.blk_row = dupload(b, s);
        owned.push_back(d.blk_row);
        d.desc = upload_desc(b, ptr, s, owned);
        d.hblk = b;
        d.ptr32 = dalloc<int>(rows + 1);
        owned.push_back(d.ptr32);
        k_ptr32<<<grid_for(rows + 1), NT, 0, s>>>(dptr64, rows + 1, d.ptr32);
        CK(cudaGetLastError());
    }
    if (d.seg) {
        long long L = 1024;
        while (L > 128 && nnz / L < (long long)sm_count() * 16) L /= 2;
        d.seg_len = L;
        HostSeg h = make_segments(ptr, rows, L);
        d.ds.seg_start = dupload(h.seg_start, s);
        d.ds.seg_row = dupload(h.seg_row, s);
        d.ds.row_seg = dupload(h.row_seg, s);
        d.ds.nseg = (long long)h.seg_row.size();
        owned.push_back(d.ds.seg_start);
        owned.push_back(d.ds.seg_row);
        owned.push_back(d.ds.row_seg);
    }
    return d;
}

// the fp64 plan: row blocks of <= RB_NNZ64 nonzeros; rows longer than that take the short-row kernels
DirPlan plan_direction64(const DirPlan& d32, const std::vector<int64_t>& ptr, long long rows, cudaStream_t s,
                         std::vector<void*>& owned) {
    DirPlan d = d32;
    if (!d32.rb) return d;
    long long maxlen = 0;
    for (long long r = 0; r < rows; ++r) maxlen = std::max<long long>(maxlen, ptr[r + 1] - ptr[r]);
    if (maxlen > RB_NNZ64) {
        d.rb = false;
        d.blk_row = nullptr;
        d.nblk = 0;
        return d;
    }
    std::vector<long long> b = make_rowblocks(ptr, rows, RB_NNZ64, RB_ROWS_MAX);
    d.nblk = (long long)b.size() - 1;
    d.blk_row = dupload(b, s);
    owned.push_back(d.blk_row);
    d.desc = upload_desc(b, ptr, s, owned);
    d.hblk = b;
    return d;
}

const char* kClassNames[] = {"pdhg_dual", "pdhg_primal", "trig_rows", "trig_cols", "sample", "feas", "obj",
                             "argmin", "halt", "pdhg_dual_push", "pdhg_primal_push", "pdhg_qx", "obj_tc", "cover",
                             "pdhg_primal_col"};
enum KClass { KC_DUAL = 0, KC_PRIMAL, KC_TRIGR, KC_TRIGC, KC_SAMPLE, KC_FEAS, KC_OBJ, KC_ARGMIN, KC_HALT, KC_DUAL_PUSH,
              KC_PRIMAL_PUSH, KC_QX, KC_OBJ_TC, KC_COVER, KC_PRIMAL_COL, KC_N };  // PRIMAL_COL: k_primal_push alone

}  // namespace

// opt a kernel into the largest dynamic shared memory it can have next to its static shared memory
constexpr size_t SMEM_PER_BLOCK_MAX = 227 * 1024;
constexpr size_t SP_DYN_MAX = SMEM_PER_BLOCK_MAX - 8 * 1024;  // k_primal_sparse: static part < 8 KB
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: remember, per (kernel, device), the
// largest size set so far (thread-safe); a second solver on another GPU sets its own
static void smem_attr(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    size_t& cur = done[{fn, dev}];
    if (bytes <= cur) return;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
}
// one wave: the grid of a grid-stride kernel capped at its resident CTAs (occupancy x SMs), so no CTA
// waits for a second wave — which matters most when the kernel's mode is switched off on the device
// and every CTA only reads the mode and exits
static int fit_grid(const void* fn, long long want, int block, size_t smem = 0) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, size_t>, int> occ;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int per = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = occ.find({fn, dev, block, smem});
        if (it != occ.end()) per = it->second;
    }
    if (!per) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, block, smem));
        per = std::max(per, 1);
        std::lock_guard<std::mutex> g(mu);
        occ[{fn, dev, block, smem}] = per;
    }
    return (int)std::max<long long>(1, std::min<long long>(want, (long long)sms * per));
}
static void set_max_dyn_smem(const void* fn) {
    cudaFuncAttributes a;
    CK(cudaFuncGetAttributes(&a, fn));
    smem_attr(fn, SMEM_PER_BLOCK_MAX - a.sharedSizeBytes);
}

// 2-D TMA map of a row-major int8 matrix [rows][ld] with (128-byte x box_rows) boxes and the 128-byte
// swizzle the UMMA descriptors of dense_q.cuh expect; cuTensorMapEncodeTiled is taken from the driver
// through the runtime's entry-point query (no libcuda link dependency)
static CUtensorMap make_tmap_i8(const void* base, long long ld, long long rows, int box_rows, int box_cols = 128,
                                bool swz128 = true) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw Err{GFORS_E_CUDA, "cuTensorMapEncodeTiled not available"};
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Err{GFORS_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r)};
    return m;
}

// =============================================================================================
// CheckHalt + UpdatePenalty + loop control, one block of 256 threads
// =============================================================================================
__global__ void __launch_bounds__(256) k_halt(Ctrl* __restrict__ ctrl, HaltPar hp, const double* __restrict__ part1,
                                              int nb1, const double* __restrict__ part2, int nb2, long long n,
                                              double* __restrict__ hist, const double* __restrict__ rho_tab,
                                              long long nrho, double* __restrict__ trace,
                                              cudaGraphConditionalHandle handle, int use_handle) {
    __shared__ double sh[32];
    __shared__ double ind[4];
    reduce_indicators(part1, nb1, part2, nb2, n, sh, ind);
    __syncthreads();
    if (threadIdx.x != 0) return;
    const double pg = ind[0], dg = ind[1] + ind[2], bg = ind[3];
    for (int a = 0; a < 4; ++a) ctrl->ind[a] = ind[a];
    const int improved = ctrl->improved;
    ctrl->improved = 0;
    ctrl->since_improve = improved ? 0 : ctrl->since_improve + 1;
    const int W = hp.window;
    const long long slot = ctrl->checks % W;
    hist[slot] = pg; hist[W + slot] = dg; hist[2 * W + slot] = bg;
    ctrl->checks += 1;
    int halt = 0;
    if (!isfinite(pg) || !isfinite(dg) || !isfinite(bg)) {
        halt = 4;
    } else {
        const double v[3] = {pg, dg, bg};
        bool all_ok = true;
        for (int a = 0; a < 3; ++a) {
            bool ok = v[a] <= hp.tol[a];
            if (!ok && ctrl->checks >= W) {
                double mx = hist[a * W], mn = hist[a * W];
                for (int s = 1; s < W; ++s) { mx = fmax(mx, hist[a * W + s]); mn = fmin(mn, hist[a * W + s]); }
                const double den = fabs(mx) > 1e-300 ? fabs(mx) : 1e-300;
                ok = (mx - mn) / den < hp.stall_rel;
            }
            all_ok = all_ok && ok;
        }
        if (all_ok && ctrl->since_improve >= W) halt = 1;
        else if (hp.sharded ? ctrl->tl_any != 0 : globaltimer_ns() >= ctrl->deadline_ns) halt = 3;
        else if (ctrl->blk + 1 >= ctrl->max_blocks) halt = 2;
    }
    const long long k = (ctrl->blk + 1) * hp.k_int;
    if (hp.trace_cap > 0) {
        double* row = trace + 8 * (ctrl->n_trace % hp.trace_cap);
        row[0] = (double)k; row[1] = ctrl->rho; row[2] = pg; row[3] = ind[1]; row[4] = ind[2];
        row[5] = bg; row[6] = ctrl->z_best; row[7] = improved;
    }
    ctrl->n_trace += 1;
    ctrl->blk += 1;
    ctrl->k = k;
    ctrl->rho = rho_tab[ctrl->blk < nrho ? ctrl->blk : nrho - 1];
    ctrl->halt = halt;
    if (use_handle) cudaGraphSetConditional(handle, halt ? 0u : 1u);
}

__global__ void k_loop_start(Ctrl* ctrl, double time_limit_s) {
    const unsigned long long t = globaltimer_ns();
    ctrl->t0_ns = t;
    const double lim = time_limit_s * 1e9;
    ctrl->deadline_ns = lim >= 1.8e19 ? ~0ull : t + (unsigned long long)lim;
}

// =============================================================================================
// Context
// =============================================================================================
struct gfors_ctx {
    int device = 0;
    int num_sms = NUM_SMS_B200;  // queried at create
    bool counted = false;        // counted in live_contexts (the device pool is trimmed after the last)
    cudaStream_t stream = nullptr, cap_stream = nullptr;
    bool own_stream = false;
    int rank = 0, world = 1;
    std::string err;
    int stage = 0;  // 0 created, 1 loaded, 2 preprocessed

    // ---- canonical problem (host) ----
    long long n = 0, m = 0, m1 = 0, m2 = 0, nnz = 0, qnnz = 0;
    long long m1p = 0;      // rows [0,m1p) are inequalities for the PDHG step (m under the relaxation, R26)
    bool repair = false;    // repair lanes before EvalBest (repair.cuh)
    AllocHooks hooks;          // optional caller allocator (device_opts.alloc/free)
    long long maxrowdeg = 0;   // longest row of K (load)
    double* kval_dev = nullptr;  // load-time only: the caller's values copied by the device validation
    long long maxcoldeg_raw = 0;  // longest column of K (load)
    bool kcan_pinned = false;  // d_kcol was uploaded straight from the caller's pinned K columns (load)
    bool complete = false;  // cover completion before EvalBest (cover.cuh)
    int* d_cover_rows = nullptr;      // eligible covering rows (prep-owned, built on first use)
    long long n_cover = -1;
    int* d_rp_rank = nullptr;         // repair drop order (repair.cuh): rank of each variable, built on first use
    int* d_rp_order = nullptr;        // its inverse
    long long* d_rp_srow = nullptr;   // per-lane row sums when m > RP_SROWS
    long long rp_srow_len = 0;
    uint2* d_slist = nullptr;         // RandSampleStep list of (i, ceil(p_i 2^32)) with 0 < p_i < 1
    unsigned* d_scnt = nullptr;       // its length, the k_sample exit ticket, the last round's length
    unsigned long long* d_s1 = nullptr;  // [2] sum of c over p = 1 (accumulating / last round's), for k_obj_list
    int* d_cover_best = nullptr;
    uint64_t* d_cover_viol = nullptr;
    long long cover_viol_len = 0;
    bool maximize = false, integral = false, hasq = false;
    double c0 = 0.0;
    std::vector<int64_t> kptr, ktptr, qptr;
    hvec<int32_t> kcol;  // canonical K on the host: filled by the load only when it permutes or negates
    hvec<double> kval;   // rows, else on first use from the device copies (ensure_host_k)
    bool khost = false;
    std::vector<int32_t> ktrow, qcol;
    std::vector<double> ktval, qval, ru;
    hvec<double> c;  // first touched by the parallel copy in the load
    std::vector<int64_t> perm;
    std::vector<signed char> rsign;
    int kkind = KV_F64;

    // ---- TUReformulate lift data (tu_impl.inc) ----
    struct TuLift {
        bool active = false;
        long long n_orig = 0;
        bool maximize = false;          // sense of the ORIGINAL problem (the reduced one is canonical)
        std::vector<int> keep;          // reduced variable -> original column (Ibar, ascending)
        std::vector<int> icol;          // eliminated columns I
        std::vector<double> s;          // x_I = s + S x_Ibar
        std::vector<int64_t> sptr;
        std::vector<int32_t> scol;
        std::vector<double> sval;
    } tu;

    // ---- customised 3D-assignment sampler (assign3d.cuh) ----
    struct A3 {
        int sampler = 0;        // of the current run / hook call
        long long n = 0, K = 0, L = 0;
        unsigned long long* keys[2] = {nullptr, nullptr};
        int* vals[2] = {nullptr, nullptr};
        void* tmp = nullptr;
        size_t tmp_bytes = 0;
        short *sj0 = nullptr, *sk0 = nullptr, *Ri = nullptr, *Rj = nullptr, *Rk = nullptr;
        int* meta = nullptr;
        long long alloc_n = 0;
    } a3;

    // ---- dense-Q path (dense_q.cuh) ----
    bool qdense = false;           // Q stored as dense int8 Qd[qld][qld]
    long long qld = 0;             // padded dimension (multiple of 128)
    int8_t* d_qd = nullptr;        // problem-owned
    CUtensorMap tmQ{};             // TMA map of Qd (128 x 128 byte boxes, 128B swizzle)
    CUtensorMap tmQ64{};           // TMA map of Qd for the GEMV (256-byte x 64-row boxes, no swizzle)
    bool qx_fix = true;            // fp32 iterates: exact fixed-point dp4a GEMV (option qx_fix = 0: fp64 FMA)
    bool qx_reuse = true;          // fp32 loop: the trigger's product of x_k serves the next block's first primal (option qx_reuse)
    double* d_qxpart2 = nullptr;   // [nchunk][qld] partials of the trigger's product (prep-owned)
    long long* d_qreuse = nullptr; // block index whose first primal may reuse d_qxpart2 (prep-owned)
    TcItem* d_tcitems = nullptr;   // objective work items, grouped per CTA
    int* d_tcoff = nullptr;        // [tc_grid + 1]
    int tc_grid = 0;
    double* d_qx = nullptr;        // [n] Q~ x of the primal input (prep-owned)
    double* d_qdx = nullptr;       // [n] Q~ (x_k - x_{k-1}) for the trigger residual
    double* d_qxpart = nullptr;    // [nchunk][qld] GEMV column-chunk partials
    int8_t* d_Xs = nullptr;        // [64W][xld] unpacked samples (prep-owned)
    long long xld = 0;             // leading dimension of the unpacked samples (n rounded up to 128)
    // dense integer rows of K (MKP's K.X on tensor cores): the general integer rows
    // as int8 Kd[ceil128(n_int)][xld], split-K work items of the FEAS instance of k_obj_dense_tc
    bool kdense = false;
    int8_t* d_kd = nullptr;
    CUtensorMap tmK{};
    TcItem* d_kitems = nullptr;
    int* d_koff = nullptr;
    int k_tc_grid = 0;
    int* d_kS = nullptr;           // [n_int][lanes] int32 row sums (kept zero between rounds)
    long long kS_len = 0;
    long long Xs_lanes = 0;
    CUtensorMap tmX{};

    // ---- device problem ----
    long long *d_kptr = nullptr, *d_ktptr = nullptr, *d_qptr = nullptr;
    int *d_kcol = nullptr, *d_ktrow = nullptr, *d_qcol = nullptr;
    void *d_kval = nullptr, *d_ktval = nullptr;
    double *d_qval = nullptr, *d_c = nullptr, *d_ru = nullptr;
    signed char* d_rsign = nullptr;
    DirPlan pd, pp;  // dual (rows of K), primal (rows of K') for the preprocessed precision
    DirPlan pdv[2], ppv[2];  // [0] fp32, [1] fp64 plans (row-block size differs)
    bool plans64 = false;    // pdv[1], ppv[1] built (on the first fp64 Preprocess)
    bool push_dual_ok = false, push_primal_ok = false;  // push modes allowed by the matrix
    bool delta_dual = true;                             // delta push of the dual (option delta_dual)
    bool xskip = true;                                  // stationary-column skip (option xskip)
    unsigned mark_rows = 0;
    unsigned char* d_xst = nullptr;                     // [n] stationarity counters (push_primal.cuh)
    bool capturing = false;                             // enqueueing into the graph capture (branch())
    bool cond_branch = false;                           // conditional-node mode branches (option cond_branch)
    bool dry = false;                                   // LAUNCH counts only
    cudaStream_t cap_stream2 = nullptr;                 // captures the conditional branch bodies
    long long gstatic = 0;                              // unconditional launches per block of the graph
    bool sparse_primal = false;     // primal skips gathers of zero duals (sparse_primal.cuh)
    long long* sp_blk_row = nullptr;
    long long sp_nblk = 0;
    unsigned* d_nzbits = nullptr;
    bool push_dual = false;          // sparse-xbar dual (push_dual.cuh)
    bool push_primal = false;        // sparse-dual primal (push_primal.cuh)
    unsigned rthr = 0;
    int* d_rlist = nullptr;
    unsigned* d_rcount = nullptr;
    unsigned long long* d_wmax = nullptr;
    long long* d_accx = nullptr;
    long long* d_accv = nullptr;       // [m] pushed K_u x_k (trigger)
    unsigned* d_ones_cnt = nullptr;    // [m] pushed #(x_k == 1) per row (trigger)
    unsigned* d_trig_flag = nullptr;
    int maxcoldeg = 0;
    unsigned push_thr = 0;
    int* d_plist[2] = {nullptr, nullptr};
    unsigned* d_pcount = nullptr;    // [2]
    unsigned* d_pflags = nullptr;    // delta push: [0,1] dual acc valid, [2,3] primal accx valid, [4,5] primal exponent
    long long* d_acc = nullptr;      // [m]
    double* d_segpart = nullptr;
    double* d_segpart2 = nullptr;
    double* d_u = nullptr;  // K_u xbar of the block's last iteration (trigger pass, rb path)
    unsigned char* d_ones = nullptr;  // per row: #entries with x_k == 1 at the last trigger (rb path)
    long long segpart_len = 0;
    // evaluator plan
    struct CountList {
        int* row = nullptr;
        int* t = nullptr;
        signed char* rel = nullptr;
        signed char* B = nullptr;
        long long nrows = 0;
        int sub = 32;
    } cnt[3];  // BMAX 1, 2, 8: rows longer than FB_NNZ (k_feas_count)
    struct CountRb {               // rows <= FB_NNZ nonzeros of each class (k_feas_rb, feas_rb.cuh)
        CountList rows;
        ClassCsr cc{};                  // blocks of FB_NNZ nonzeros (units of 1-2 words)
        ClassCsr cc8{};                 // blocks of FB_NNZ8 nonzeros (units of 8 words, k_b % 512 == 0)
        unsigned char* skip = nullptr;  // [nrows] per-round "satisfied by p = 1 variables" flags
    } cntrb[3];
    int* d_int_row = nullptr;
    long long* d_int_rhs = nullptr;
    signed char* d_int_eq = nullptr;
    long long* d_int_seg_start = nullptr;
    int* d_int_seg_slot = nullptr;
    long long n_int = 0, n_int_seg = 0;
    int* d_real_row = nullptr;
    long long n_real = 0;
    bool never_feasible = false;
    std::vector<void*> owned;

    // ---- Preprocess ----
    double* d_s = nullptr;
    double omega = 1.0, kappa = 1.0;
    long long zero_rows = 0;
    int precision = 64;
    void *d_g = nullptr, *d_rh = nullptr, *d_cs = nullptr, *d_qs = nullptr;
    void *d_x[2] = {nullptr, nullptr}, *d_xb[2] = {nullptr, nullptr}, *d_y[2] = {nullptr, nullptr}, *d_w = nullptr;
    double* d_tmp[4] = {nullptr, nullptr, nullptr, nullptr};
    double* d_red = nullptr;  // reduction partials
    double* d_scalar = nullptr;

    // ---- loop ----
    Ctrl* d_ctrl = nullptr;
    double* d_part1 = nullptr;
    double* d_part2 = nullptr;
    int nb1 = 1, nb2 = 1;
    double* d_hist = nullptr;
    double* d_rho = nullptr;
    long long nrho = 0, rho_cap = 0;
    double* d_trace = nullptr;
    int trace_cap = 0;
    unsigned char* d_xbest = nullptr;
    uint64_t* d_X = nullptr;
    long long X_words = 0;
    unsigned long long* d_viol = nullptr;
    unsigned long long* d_iacc = nullptr;
    long long iacc_len = 0;
    void* d_zpart = nullptr;
    long long zpart_len = 0;
    double* d_z = nullptr;
    long long z_len = 0;
    int obj_chunk = 2048;
    bool obj_bits = false;        // integral c with a small range: bit-plane objective kernel
    unsigned* d_planes = nullptr;  // [ceil(n/32)][obj_nb] coefficient bit planes of c - cmin
    int obj_nb = 0;
    long long obj_cmin = 0;
    long long hk = 0;  // iterations done in hook mode (parity)
    bool have_run = false;
    gfors_run_info last_info{};

    // graph cache
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    gfors_params gkey{};
    int gkey_W = -1;
    bool gvalid = false;

    // sample sharding over NCCL (shard.cuh)
    ncclComm_t comm = nullptr;
    bool sharded = false;
    bool loopback = false;         // world simulated ranks in this context (test mode, no NCCL)
    // row-sharded dual (params.row_shard; shard.cuh): rank q owns dual row blocks [rs_blo[q], rs_blo[q+1])
    bool rs_on = false;
    int rs_key = -1;                      // precision the partition below was made for
    std::vector<long long> rs_blo, rs_rlo;
    long long rs_maxrows = 0;
    long long* d_rs_rlo = nullptr;
    void* d_rs_y = nullptr;               // [world][maxrows] y gather buffer (iterate type)
    double* d_rs_u = nullptr;             // [world][maxrows] u gather buffer

    // options set through gfors_set_option (tests, benchmarks); defaults are the production path
    struct Options {
        long long force_deadline_rank = -1;   // this (simulated) rank reports its time limit as passed ...
        long long force_deadline_block = -1;  // ... from this block on (tests of the halt agreement)
        long long force_capture_fail = 0;     // sharded: make the graph capture fail (eager fallback test)
        // load-time choices (applied by the next gfors_load; -1 = automatic)
        long long dense_q = -1;       // dense int8 Q storage (dense_q.cuh): 1 force, 0 off
        long long dense_k = -1;       // dense int8 integer rows of K on tensor cores: 1 force, 0 off
        long long qx_fix = 1;         // fp32 iterates: exact fixed-point dp4a GEMV (0: fp64 FMA GEMV)
        long long qx_reuse = 1;       // fp32 loop: the trigger's product of x_k serves the next block's first primal
        long long push_dual = -1;     // sparse-xbar dual (push_dual.cuh): 1 force, 0 off
        long long push_primal = -1;   // sparse-y primal (push_primal.cuh): 1 force, 0 off
        long long delta_dual = 1;     // delta push of the dual
        long long xskip = 1;          // stationary-column skip of the push primal
        long long cond_branch = 0;    // graph conditional nodes run only the chosen mode's kernels
        long long sparse_primal = -1; // zero-dual-skipping gather primal (sparse_primal.cuh): 1 force, 0 off
        long long obj_bits = 1;       // bit-plane objective kernel for integral c (0: exact per-lane kernel)
        long long load_timing = 0;    // print the load phases (host timer)
        long long obj_list = 1;       // linear objective over the sampler's list only (k_obj_list; 0: every variable)
    } opt;
    double* d_rec = nullptr;       // [4] local record + [4*world] gathered records
    long long* d_regen = nullptr;  // [2] winner global index, round
    std::string graph_note;        // why the graph fell back to the eager loop, if it did
    bool gno = false;              // graph capture failed for gkey: use the eager loop

    // profiling
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_ev;
    std::vector<double> prof_active_ms, prof_active_n;  // per class, last gfors_profile_blocks
    long long launches = 0;

    ~gfors_ctx();
    void free_problem();
    void free_prep();
};

// Every API call leaves the context's stream idle (the calls are synchronous), and the free-batches
// (free_prep / free_problem) synchronise that stream first, so no kernel of this context still uses p;
// the free is ordered on the allocation stream before any later allocation from the pool.
static void dfree(void* p) {
    if (!p) return;
    if (tls_hooks.free) { tls_hooks.free(p, tls_hooks.ctx); return; }
    cudaStream_t as = alloc_stream();
    if (as) cudaFreeAsync(p, as); else cudaFree(p);
}

void gfors_ctx::free_problem() {
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : owned) dfree(p);
    owned.clear();
    d_kptr = d_ktptr = d_qptr = nullptr;
    d_kcol = d_ktrow = d_qcol = nullptr;
    d_kval = d_ktval = nullptr;
    d_qval = d_c = d_ru = nullptr;
    d_rsign = nullptr;
    d_qd = nullptr; d_tcitems = nullptr; d_tcoff = nullptr; qdense = false; tc_grid = 0;
    kdense = false; d_kd = nullptr; d_kitems = nullptr; d_koff = nullptr; k_tc_grid = 0; xld = 0;
    for (auto& c : cnt) c = CountList{};
    for (auto& c : cntrb) c = CountRb{};
    d_int_row = nullptr; d_int_rhs = nullptr; d_int_eq = nullptr; d_int_seg_start = nullptr; d_int_seg_slot = nullptr;
    d_real_row = nullptr;
    d_planes = nullptr;
    sp_blk_row = nullptr;
    d_nzbits = nullptr;
    sparse_primal = false;
    obj_bits = false;
    pd = DirPlan{}; pp = DirPlan{};
}

void gfors_ctx::free_prep() {
    if (stream) cudaStreamSynchronize(stream);
    void** ps[] = {(void**)&d_s, &d_g, &d_rh, &d_cs, &d_qs, &d_x[0], &d_x[1], &d_xb[0], &d_xb[1], &d_y[0], &d_y[1],
                   &d_w, (void**)&d_tmp[0], (void**)&d_tmp[1], (void**)&d_tmp[2], (void**)&d_tmp[3],
                   (void**)&d_red, (void**)&d_scalar, (void**)&d_segpart, (void**)&d_segpart2, (void**)&d_u, (void**)&d_ones, (void**)&d_rec, (void**)&d_regen, (void**)&d_plist[0], (void**)&d_plist[1], (void**)&d_pcount, (void**)&d_pflags, (void**)&d_acc, (void**)&d_rlist, (void**)&d_rcount, (void**)&d_wmax, (void**)&d_accx, (void**)&d_xst, (void**)&d_accv, (void**)&d_ones_cnt, (void**)&d_trig_flag, (void**)&d_part1,
                   (void**)&d_part2, (void**)&d_hist, (void**)&d_rho, (void**)&d_trace, (void**)&d_xbest,
                   (void**)&d_X, (void**)&d_viol, (void**)&d_iacc, &d_zpart, (void**)&d_z, (void**)&d_ctrl,
                   (void**)&d_qx, (void**)&d_qdx, (void**)&d_qxpart, (void**)&d_Xs, (void**)&d_kS,
                   (void**)&d_qxpart2, (void**)&d_qreuse, (void**)&d_cover_rows, (void**)&d_cover_best,
                   (void**)&d_cover_viol, (void**)&d_rp_rank, (void**)&d_rp_order, (void**)&d_rp_srow, (void**)&d_slist, (void**)&d_scnt, (void**)&d_s1,
                   (void**)&d_rs_rlo, &d_rs_y, (void**)&d_rs_u};
    for (void** p : ps) { dfree(*p); *p = nullptr; }
    X_words = iacc_len = zpart_len = z_len = Xs_lanes = kS_len = 0;
    n_cover = -1;
    cover_viol_len = 0;
    rp_srow_len = 0;
    rs_key = -1;
    rs_on = false;
    for (int b = 0; b < 2; ++b) { dfree(a3.keys[b]); dfree(a3.vals[b]); }
    for (void* q : {(void*)a3.tmp, (void*)a3.sj0, (void*)a3.sk0, (void*)a3.Ri, (void*)a3.Rj, (void*)a3.Rk,
                    (void*)a3.meta})
        dfree(q);
    a3 = A3{};
    rho_cap = 0;
    trace_cap = 0;
    if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
    if (graph) { cudaGraphDestroy(graph); graph = nullptr; }
    gvalid = false;
}

gfors_ctx::~gfors_ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    free_prep();
    free_problem();
    // the pool keeps the freed memory for the next solver (gfors_release_memory returns it)
    if (counted) live_contexts(device, -1);
    if (comm) nccl().CommDestroy(comm);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (cap_stream2) cudaStreamDestroy(cap_stream2);
    if (own_stream && stream) cudaStreamDestroy(stream);
}

// host copies of the canonical K (kcol, kval) from the device ones, for the host-side consumers
// (relaxation checks, cover rows, TUReformulate) when the load did not need to make them
void ensure_host_k(gfors_ctx* C) {
    if (C->khost) return;
    const long long nnz = C->nnz;
    C->kcol.resize(nnz);
    C->kval.resize(nnz);
    if (nnz) {
        CK(cudaStreamSynchronize(C->stream));
        CK(cudaMemcpy(C->kcol.data(), C->d_kcol, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (C->kkind == KV_F64) {
            CK(cudaMemcpy(C->kval.data(), C->d_kval, nnz * sizeof(double), cudaMemcpyDeviceToHost));
        } else if (C->kkind == KV_I8) {
            std::vector<signed char> a(nnz);
            CK(cudaMemcpy(a.data(), C->d_kval, nnz, cudaMemcpyDeviceToHost));
            for (long long p = 0; p < nnz; ++p) C->kval[p] = (double)a[p];
        } else {  // one +-1 value per row
            for (long long j = 0; j < C->m; ++j)
                for (long long p = C->kptr[j]; p < C->kptr[j + 1]; ++p) C->kval[p] = (double)C->rsign[j];
        }
    }
    C->khost = true;
}

#include "load_impl.inc"
#include "tu_impl.inc"

// =============================================================================================
// Typed dispatch helpers
// =============================================================================================
namespace {

struct LaunchCtx {
    gfors_ctx* C;
    cudaStream_t s;
    int cls;
};

inline void prof_begin(gfors_ctx* C, cudaStream_t s, int cls, cudaEvent_t* a) {
    C->launches++;
    if (!C->profiling) return;
    CK(cudaEventCreate(a));
    CK(cudaEventRecord(*a, s));
    (void)cls;
}
inline void prof_end(gfors_ctx* C, cudaStream_t s, int cls, cudaEvent_t a) {
    if (!C->profiling) return;
    cudaEvent_t b;
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(b, s));
    C->prof_ev.push_back({cls, {a, b}});
}
#define LAUNCH(C, s, cls, ...)                                   \
    do {                                                         \
        if ((C)->dry) { (C)->launches++; break; } /* count only */ \
        cudaEvent_t ev_a__ = nullptr;                            \
        prof_begin((C), (s), (cls), &ev_a__);                    \
        __VA_ARGS__;                                             \
        CK(cudaGetLastError());                                  \
        prof_end((C), (s), (cls), ev_a__);                       \
    } while (0)

// Mode branch (dual: gather vs push; primal: gather vs push; trigger pass: gather vs pushed).  By
// default both branches are launched and every kernel checks the device decision itself and exits
// at once when it is not the chosen one.  Option cond_branch = 1: in the graph capture a one-thread
// decide kernel sets the handle of an IF/ELSE conditional node instead, so only the chosen kernels
// run (counted on the device, ctrl->dyn_launches) — measured SLOWER on config 5 (2.66 vs 2.55 ms
// per block: 31 conditional nodes per block cost more than the early exits they replace).
template <class Dec, class A, class B>
void branch(gfors_ctx* C, cudaStream_t s, Dec decide, A then_, B else_) {
    if (!C->capturing || C->dry || !C->cond_branch) {
        else_(s);  // (trigger pass: the gather branch's partial fill must precede the pushed pass)
        then_(s);
        return;
    }
    const long long l0 = C->launches;
    C->dry = true;
    then_(s);
    const int nthen = (int)(C->launches - l0);
    else_(s);
    const int nelse = (int)(C->launches - l0) - nthen;
    C->dry = false;
    C->launches = l0;
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
    decide(s, h, nthen, nelse);
    C->launches++;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 2;  // [0] then, [1] else
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, cg, deps, nd, &cp));
    cudaGraph_t bodies[2] = {cp.conditional.phGraph_out[0], cp.conditional.phGraph_out[1]};
    if (!C->cap_stream2) CK(cudaStreamCreateWithFlags(&C->cap_stream2, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        CK(cudaStreamBeginCaptureToGraph(C->cap_stream2, bodies[b], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        if (b == 0) then_(C->cap_stream2); else else_(C->cap_stream2);
        cudaGraph_t g2;
        CK(cudaStreamEndCapture(C->cap_stream2, &g2));
    }
    C->launches = l0 + 1;  // the branch kernels are counted on the device
    CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
}

__global__ void k_decide_dual(PushList pl, Ctrl* ctrl, long long kint, long long j, cudaGraphConditionalHandle h,
                              int nthen, int nelse) {
    const bool push = push_mode(pl, (int)(iter_index(ctrl, kint, j) & 1));
    ctrl->dyn_launches += push ? nthen : nelse;
    cudaGraphSetConditional(h, push ? 1u : 0u);
}
__global__ void k_decide_primal(PushPrimal pp, Ctrl* ctrl, long long kint, long long j, cudaGraphConditionalHandle h,
                                int nthen, int nelse) {
    const bool push = pp_mode(pp, (int)(iter_index(ctrl, kint, j) & 1)).push;
    ctrl->dyn_launches += push ? nthen : nelse;
    cudaGraphSetConditional(h, push ? 1u : 0u);
}
__global__ void k_decide_flag(const unsigned* flag, Ctrl* ctrl, cudaGraphConditionalHandle h, int nthen, int nelse) {
    const bool on = *flag != 0u;
    ctrl->dyn_launches += on ? nthen : nelse;
    cudaGraphSetConditional(h, on ? 1u : 0u);
}

template <typename T>
State<T> state_of(gfors_ctx* C) {
    State<T> st;
    for (int b = 0; b < 2; ++b) { st.x[b] = (T*)C->d_x[b]; st.xb[b] = (T*)C->d_xb[b]; st.y[b] = (T*)C->d_y[b]; }
    st.w = (T*)C->d_w;
    return st;
}
inline Csr csr_K(gfors_ctx* C) { return Csr{C->d_kptr, C->d_kcol, C->d_kval, C->m}; }
inline Csr csr_Kt(gfors_ctx* C) { return Csr{C->d_ktptr, C->d_ktrow, C->d_ktval, C->n}; }
inline Csr csr_Q(gfors_ctx* C, const double* pre = nullptr) { return Csr{C->d_qptr, C->d_qcol, C->d_qval, C->n, pre}; }

// dense-Q GEMV (dense_q.cuh): out = Q~ (a - b), a/b picked on the device by iteration parity
// (ctrl != nullptr) or taken directly (ctrl == nullptr, omega = 1: Preprocess power iteration)
template <typename TX>
void enqueue_qx(gfors_ctx* C, cudaStream_t s, QxSrc<TX> src, bool diff, double omega, double* out) {
    const long long n = C->n;
    const long long nchunk = (n + QX_CW - 1) / QX_CW;
    if constexpr (sizeof(TX) == 4) {
        if (C->qx_fix) {  // fp32 iterates: exact dp4a products on the fixed-point image of x
            const long long units = (n + QT_ROWS - 1) / QT_ROWS * nchunk;
            // 4-stage ring x 3 CTAs per SM (sweep in round 1: 78.6 us vs 83.1 for 6x2 at n = 20480)
            const int grid = (int)std::min<long long>(units, (long long)C->num_sms * 3);
            // product reuse across loop blocks (qx_reuse): the trigger computes S(x_k) (not the
            // difference) into d_qxpart2; the next block's first primal skips its GEMV and reads it
            // (k_int > 1: with one iteration per block the skipped GEMV would be the trigger's x_{k-1} product)
            const bool trig_reuse = diff && C->qx_reuse && src.ctrl && src.kint > 1;
            const bool prim_reuse = !diff && C->qx_reuse && src.ctrl && src.kint > 1 && src.j == 0;
            double* dst = trig_reuse ? C->d_qxpart2 : C->d_qxpart;
            const long long* reuse = prim_reuse ? C->d_qreuse : nullptr;
            if (trig_reuse) {
                diff = false;
                src = QxSrc<TX>{{src.a[0], src.a[1]}, {nullptr, nullptr}, src.ctrl, src.kint, src.j};
            }
#define QXF_LAUNCH(STV, MBV)                                                                                          \
    {                                                                                                                 \
        const size_t smb = qt_smem_bytes(STV);                                                                        \
        if (diff) smem_attr((const void*)k_qx_tma_fix<true, STV, MBV>, smb);                                         \
        else smem_attr((const void*)k_qx_tma_fix<false, STV, MBV>, smb);                                             \
        if (diff)                                                                                                     \
            LAUNCH(C, s, KC_QX, (k_qx_tma_fix<true, STV, MBV><<<grid, QT_NT, smb, s>>>(C->tmQ64, n, C->qld, src, dst, reuse))); \
        else                                                                                                          \
            LAUNCH(C, s, KC_QX, (k_qx_tma_fix<false, STV, MBV><<<grid, QT_NT, smb, s>>>(C->tmQ64, n, C->qld, src, dst, reuse))); \
    }
            QXF_LAUNCH(4, 3)
#undef QXF_LAUNCH
            if (trig_reuse)
                LAUNCH(C, s, KC_QX, (k_qx_diff_final<<<grid_for(n), 256, 0, s>>>(n, C->qld, nchunk, C->d_qxpart2, C->d_qxpart,
                                                                                omega, out, C->d_qreuse, src.ctrl)));
            else if (prim_reuse)
                LAUNCH(C, s, KC_QX, (k_qx_final_sel<<<grid_for(n), 256, 0, s>>>(n, C->qld, nchunk, C->d_qxpart, C->d_qxpart2,
                                                                               C->d_qreuse, src.ctrl, src.kint, src.j, omega, out)));
            else
                LAUNCH(C, s, KC_QX, (k_qx_final<<<grid_for(n), 256, 0, s>>>(n, C->qld, nchunk, C->d_qxpart, omega, out)));
            return;
        }
    }
    {
        const long long units = (n + QT_ROWS - 1) / QT_ROWS * nchunk;
        const int grid = (int)std::min<long long>(units, sm_count() * 2LL);
        if (diff) smem_attr((const void*)k_qx_tma<TX, true>, qt_smem_bytes());
        else smem_attr((const void*)k_qx_tma<TX, false>, qt_smem_bytes());
        if (diff)
            LAUNCH(C, s, KC_QX, (k_qx_tma<TX, true><<<grid, QT_NT, qt_smem_bytes(), s>>>(C->tmQ64, n, C->qld, src, C->d_qxpart)));
        else
            LAUNCH(C, s, KC_QX, (k_qx_tma<TX, false><<<grid, QT_NT, qt_smem_bytes(), s>>>(C->tmQ64, n, C->qld, src, C->d_qxpart)));
    }
    LAUNCH(C, s, KC_QX, (k_qx_final<<<grid_for(n), 256, 0, s>>>(n, C->qld, nchunk, C->d_qxpart, omega, out)));
}

#define SUB_SWITCH(sub, ...)                                  \
    switch (sub) {                                            \
        case 2: { constexpr int SUBV = 2; __VA_ARGS__; } break;  \
        case 4: { constexpr int SUBV = 4; __VA_ARGS__; } break;  \
        case 8: { constexpr int SUBV = 8; __VA_ARGS__; } break;  \
        case 16: { constexpr int SUBV = 16; __VA_ARGS__; } break; \
        default: { constexpr int SUBV = 32; __VA_ARGS__; } break; \
    }
#define KIND_SWITCH(kind, ...)                                           \
    switch (kind) {                                                      \
        case KV_SIGN: { constexpr int KINDV = KV_SIGN; __VA_ARGS__; } break; \
        case KV_I8: { constexpr int KINDV = KV_I8; __VA_ARGS__; } break;     \
        default: { constexpr int KINDV = KV_F64; __VA_ARGS__; } break;       \
    }

// one PDHG iteration (dual + primal); kint/j select the parity (see pdhg.cuh)
// row-sharded dual: pack this rank's y (and u) rows, all-gather, unpack every rank's rows + w (shard.cuh)
template <typename T>
void enqueue_rs_exchange(gfors_ctx* C, cudaStream_t s, State<T> st, long long kint, long long j, bool with_u) {
    const long long MR = C->rs_maxrows;
    T* gy = (T*)C->d_rs_y;
    double* gu = with_u ? C->d_rs_u : nullptr;
    for (int r = 0; r < C->world; ++r) {
        if (!C->loopback && r != C->rank) continue;
        const long long r0 = C->rs_rlo[r], nr = C->rs_rlo[r + 1] - r0;
        if (nr <= 0) continue;
        LAUNCH(C, s, KC_DUAL, (k_rs_pack<T><<<grid_for(nr), NT, 0, s>>>(st, C->d_ctrl, kint, j, r0, nr, gy + r * MR,
                                                                        C->d_u, gu ? gu + r * MR : nullptr)));
    }
    if (!C->loopback && !C->dry) {
        NcclApi& api = nccl();
        int rc = api.GroupStart();
        if (!rc) rc = api.AllGather(gy + C->rank * MR, gy, MR * sizeof(T), ncclUint8_, C->comm, s);
        if (!rc && gu) rc = api.AllGather(gu + C->rank * MR, gu, MR, ncclFloat64_, C->comm, s);
        if (!rc) rc = api.GroupEnd();
        if (rc != 0) throw Err{GFORS_E_NCCL, std::string("ncclAllGather (row-sharded dual): ") + api.GetErrorString(rc)};
    }
    KIND_SWITCH(C->kkind, LAUNCH(C, s, KC_DUAL, (k_rs_unpack<T, KINDV><<<grid_for(C->world * MR), NT, 0, s>>>(
        st, C->d_ctrl, kint, j, C->d_rs_rlo, C->world, MR, gy, (const double*)C->d_g, C->d_rsign, gu, C->d_u))));
}

// params.row_shard: validate, and split the dual's row blocks over the ranks by nonzeros
void set_row_shard(gfors_ctx* C, int on, int prec) {
    C->rs_on = false;
    if (!on) return;
    if (!C->sharded) input_error("params.row_shard: needs world > 1 (an NCCL id or the loopback communicator)");
    if (C->m <= 0 || !C->pd.rb) input_error("params.row_shard: needs the row-block dual (every row <= %d nonzeros)", RB_NNZ_OF<float>);
    if (C->rs_key != prec) {
        const auto& hb = C->pd.hblk;
        const long long nb = (long long)hb.size() - 1, R = C->world;
        const long long total = C->kptr[C->m];
        C->rs_blo.assign(R + 1, nb);
        C->rs_blo[0] = 0;
        long long b = 0;
        for (long long q = 1; q < R; ++q) {  // first block whose start reaches q/R of the nonzeros
            const long long target = total * q / R;
            while (b < nb && C->kptr[hb[b]] < target) ++b;
            C->rs_blo[q] = b;
        }
        C->rs_rlo.resize(R + 1);
        C->rs_maxrows = 1;
        for (long long q = 0; q <= R; ++q) C->rs_rlo[q] = hb[C->rs_blo[q]];
        for (long long q = 0; q < R; ++q) C->rs_maxrows = std::max(C->rs_maxrows, C->rs_rlo[q + 1] - C->rs_rlo[q]);
        dfree(C->d_rs_rlo); dfree(C->d_rs_y); dfree(C->d_rs_u);
        C->d_rs_rlo = dupload(C->rs_rlo, C->stream);
        C->d_rs_y = dalloc<double>(R * C->rs_maxrows);  // (large enough for either iterate type)
        C->d_rs_u = dalloc<double>(R * C->rs_maxrows);
        C->rs_key = prec;
        C->gvalid = false;
    }
    C->rs_on = true;
}

template <typename T>
void enqueue_iter(gfors_ctx* C, cudaStream_t s, long long kint, long long j) {
    State<T> st = state_of<T>(C);
    PushList pl{{nullptr, nullptr}, {nullptr, nullptr}, 0u, 0, nullptr, nullptr, nullptr};
    if (C->push_dual)
        pl = PushList{{C->d_plist[0], C->d_plist[1]}, {C->d_pcount, C->d_pcount + 1}, C->push_thr, C->n, C->d_acc,
                      C->push_primal ? C->d_rcount : nullptr, C->push_primal ? C->d_wmax : nullptr, C->delta_dual ? C->d_pflags : nullptr};
    PushPrimal ppr{};
    if (C->push_primal)
        ppr = PushPrimal{C->d_rlist, C->d_rcount, C->rthr, C->d_wmax, C->d_accx, C->maxcoldeg, C->m,
                         C->d_pflags + 2, reinterpret_cast<int*>(C->d_pflags + 4), (const double*)C->d_g, C->d_rsign,
                         C->d_xst, C->mark_rows};
    const Ctrl* ctrl = C->d_ctrl;
    const double* g = (const double*)C->d_g;
    const double* rh = (const double*)C->d_rh;
    if (C->m > 0) {
        if (C->pd.rb) {
            const int grid = (int)std::min<long long>(C->pd.nblk, rb_grid());
            double* u_out = (kint == 0 || j == kint - 1) ? C->d_u : nullptr;
            auto gather = [&](cudaStream_t q) {
                if (!C->rs_on) {
                    KIND_SWITCH(C->kkind, LAUNCH(C, q, KC_DUAL,
                        (k_dual_rb<T, KINDV><<<grid, RB_NT, 0, q>>>(csr_K(C), C->pd.desc, C->pd.ptr32, C->pd.nblk, st, g, rh,
                                                                    C->d_rsign, C->m1p, ctrl, kint, j, u_out, pl))));
                    return;
                }
                // row-sharded: this rank's blocks only (loopback: every simulated rank's range in turn)
                for (int r = 0; r < C->world; ++r) {
                    if (!C->loopback && r != C->rank) continue;
                    const long long b0 = C->rs_blo[r], nb = C->rs_blo[r + 1] - b0;
                    if (nb <= 0) continue;
                    const int gr = (int)std::min<long long>(nb, rb_grid());
                    KIND_SWITCH(C->kkind, LAUNCH(C, q, KC_DUAL,
                        (k_dual_rb<T, KINDV><<<gr, RB_NT, 0, q>>>(csr_K(C), C->pd.desc + b0, C->pd.ptr32, nb, st, g, rh,
                                                                  C->d_rsign, C->m1p, ctrl, kint, j, u_out, pl))));
                }
            };
            if (C->push_dual) {
                // sparse xbar: scatter the listed columns into the row accumulators, then the rows
                auto push = [&](cudaStream_t q) {
                    LAUNCH(C, q, KC_DUAL_PUSH, (k_push_scatter<T><<<fit_grid((const void*)k_push_scatter<T>, grid_for(C->n), NT), NT, 0, q>>>(csr_Kt(C), pl, st, ctrl, kint, j)));
                    LAUNCH(C, q, KC_DUAL_PUSH, (k_push_rows<T><<<fit_grid((const void*)k_push_rows<T>, grid_for(C->m), NT), NT, 0, q>>>(C->m, pl, st, g, rh, C->d_rsign, C->m1p,
                                                                                      ctrl, kint, j, u_out)));
                };
                branch(C, s, [&](cudaStream_t q, cudaGraphConditionalHandle h, int a, int b) {
                    k_decide_dual<<<1, 1, 0, q>>>(pl, C->d_ctrl, kint, j, h, a, b);
                    CK(cudaGetLastError());
                }, push, gather);
            } else {
                gather(s);
            }
            if (C->rs_on) enqueue_rs_exchange<T>(C, s, st, kint, j, u_out != nullptr);
        } else if (!C->pd.seg) {
            const int grid = grid_for(C->m * (long long)C->pd.sub);
            KIND_SWITCH(C->kkind, SUB_SWITCH(C->pd.sub, LAUNCH(C, s, KC_DUAL,
                (k_dual<T, KINDV, SUBV><<<grid, NT, 0, s>>>(csr_K(C), st, g, rh, C->d_rsign, C->m1p, ctrl, kint, j)))));
        } else {
            const int grid = grid_for(C->pd.ds.nseg * 32);
            const int grid2 = grid_for(C->m);
            KIND_SWITCH(C->kkind, LAUNCH(C, s, KC_DUAL,
                (k_seg_partial<T, KINDV><<<grid, NT, 0, s>>>(csr_K(C), C->pd.ds.plan(), st.xb[0], st.xb[1], nullptr,
                                                             nullptr, 1, ctrl, kint, j, C->d_segpart));
                (k_dual_seg_final<T, KINDV><<<grid2, NT, 0, s>>>(C->m, C->pd.ds.plan(), C->d_segpart, st, g, rh,
                                                                 C->d_rsign, C->m1p, ctrl, kint, j))));
        }
    }
    if (C->qdense)  // 2 Q~ x term of the primal gradient by the dense GEMV
        enqueue_qx<T>(C, s, QxSrc<T>{{st.x[0], st.x[1]}, {nullptr, nullptr}, ctrl, kint, j}, false, C->omega, C->d_qx);
    const Csr Q = csr_Q(C, C->qdense ? C->d_qx : nullptr);
    const T* qs = (const T*)C->d_qs;
    const T* cs = (const T*)C->d_cs;
    // K' values: SIGN rows fold the sign into w, so the transpose carries no values
    const int tkind = C->kkind;
    // trigger iteration of a loop block: the push-mode primal also pushes x_k for the indicator pass
    const bool trig_push = C->push_primal && kint > 0 && j == kint - 1;
    auto gather = [&](cudaStream_t q) {
        if (C->sparse_primal && !C->push_primal && sparse_primal_smem<T>(C->m) <= SP_DYN_MAX) {
            const long long nwords = (C->m + 31) / 32;
            LAUNCH(C, q, KC_PRIMAL, (k_nzmask<T><<<grid_for(nwords * 32), NT, 0, q>>>(st.w, C->m, C->d_nzbits)));
            const size_t sm = sparse_primal_smem<T>(C->m);
            const int grid = (int)std::min<long long>(C->sp_nblk, (long long)sm_count());
            if (C->hasq) {
                KIND_SWITCH(tkind, {
                    set_max_dyn_smem((const void*)k_primal_sparse<T, KINDV, true>);
                    LAUNCH(C, q, KC_PRIMAL, (k_primal_sparse<T, KINDV, true><<<grid, SP_NT, sm, q>>>(csr_Kt(C), C->sp_blk_row, C->sp_nblk,
                        C->d_nzbits, nwords, Q, qs, st, cs, ctrl, kint, j, pl)));
                });
            } else {
                KIND_SWITCH(tkind, {
                    set_max_dyn_smem((const void*)k_primal_sparse<T, KINDV, false>);
                    LAUNCH(C, q, KC_PRIMAL, (k_primal_sparse<T, KINDV, false><<<grid, SP_NT, sm, q>>>(csr_Kt(C), C->sp_blk_row, C->sp_nblk,
                        C->d_nzbits, nwords, Q, qs, st, cs, ctrl, kint, j, pl)));
                });
            }
        } else if (C->pp.rb) {
            const long long want = std::min<long long>(C->pp.nblk, rb_grid());
            if (C->hasq) {
                KIND_SWITCH(tkind, {
                    const int grid = fit_grid((const void*)k_primal_rb<T, KINDV, true>, want, RB_NT);
                    LAUNCH(C, q, KC_PRIMAL, (k_primal_rb<T, KINDV, true><<<grid, RB_NT, 0, q>>>(csr_Kt(C), C->pp.blk_row,
                        C->pp.nblk, Q, qs, st, cs, ctrl, kint, j, pl, ppr)));
                });
            } else {
                KIND_SWITCH(tkind, {
                    const int grid = fit_grid((const void*)k_primal_rb<T, KINDV, false>, want, RB_NT);
                    LAUNCH(C, q, KC_PRIMAL, (k_primal_rb<T, KINDV, false><<<grid, RB_NT, 0, q>>>(csr_Kt(C), C->pp.blk_row,
                        C->pp.nblk, Q, qs, st, cs, ctrl, kint, j, pl, ppr)));
                });
            }
        } else if (!C->pp.seg) {
            const int grid = grid_for(C->n * (long long)C->pp.sub);
            if (C->hasq) {
                KIND_SWITCH(tkind, SUB_SWITCH(C->pp.sub, LAUNCH(C, q, KC_PRIMAL,
                    (k_primal<T, KINDV, SUBV, true><<<grid, NT, 0, q>>>(csr_Kt(C), Q, qs, st, cs, ctrl, kint, j)))));
            } else {
                KIND_SWITCH(tkind, SUB_SWITCH(C->pp.sub, LAUNCH(C, q, KC_PRIMAL,
                    (k_primal<T, KINDV, SUBV, false><<<grid, NT, 0, q>>>(csr_Kt(C), Q, qs, st, cs, ctrl, kint, j)))));
            }
        } else {
            const int grid = grid_for(C->pp.ds.nseg * 32);
            const int grid2 = grid_for(C->n);
            KIND_SWITCH(tkind, LAUNCH(C, q, KC_PRIMAL,
                (k_seg_partial<T, KINDV><<<grid, NT, 0, q>>>(csr_Kt(C), C->pp.ds.plan(), st.w, st.w, nullptr, nullptr, 0,
                                                             ctrl, kint, j, C->d_segpart2))));
            if (C->hasq)
                LAUNCH(C, q, KC_PRIMAL, (k_primal_seg_final<T, true><<<grid2, NT, 0, q>>>(
                                            C->n, C->pp.ds.plan(), C->d_segpart2, Q, qs, st, cs, ctrl, kint, j)));
            else
                LAUNCH(C, q, KC_PRIMAL, (k_primal_seg_final<T, false><<<grid2, NT, 0, q>>>(
                                            C->n, C->pp.ds.plan(), C->d_segpart2, Q, qs, st, cs, ctrl, kint, j)));
        }
    };
    if (C->push_primal) {
        // list the active duals (or the changed ones); the push kernels run iff the list is short
        LAUNCH(C, s, KC_PRIMAL_PUSH, (k_wlist<T><<<(int)std::min<long long>((C->m + 255) / 256, sm_count() * 4LL), NT, 0, s>>>(
                                          st, ppr, ctrl, kint, j)));
        auto push = [&](cudaStream_t q) {
            LAUNCH(C, q, KC_PRIMAL_PUSH, (k_push_scatter_cols<T><<<fit_grid((const void*)k_push_scatter_cols<T>, grid_for(C->m * 32LL), NT), NT, 0, q>>>(csr_K(C), ppr, st, ctrl, kint, j)));
            if (C->hasq)
                LAUNCH(C, q, KC_PRIMAL_COL, (k_primal_push<T, true><<<pp_grid<T>(C->n), NT, 0, q>>>(C->n, ppr, Q, qs, st, cs, ctrl, kint, j, pl,
                    csr_Kt(C), trig_push ? C->d_accv : nullptr, C->d_ones_cnt, C->d_trig_flag)));
            else
                LAUNCH(C, q, KC_PRIMAL_COL, (k_primal_push<T, false><<<pp_grid<T>(C->n), NT, 0, q>>>(C->n, ppr, Q, qs, st, cs, ctrl, kint, j, pl,
                    csr_Kt(C), trig_push ? C->d_accv : nullptr, C->d_ones_cnt, C->d_trig_flag)));
        };
        branch(C, s, [&](cudaStream_t q, cudaGraphConditionalHandle h, int a, int b) {
            k_decide_primal<<<1, 1, 0, q>>>(ppr, C->d_ctrl, kint, j, h, a, b);
            CK(cudaGetLastError());
        }, push, gather);
    } else {
        gather(s);
    }
}

// trigger indicator passes after iteration j of the block
template <typename T>
void enqueue_trigger(gfors_ctx* C, cudaStream_t s, long long kint, long long j) {
    State<T> st = state_of<T>(C);
    const Ctrl* ctrl = C->d_ctrl;
    const double* g = (const double*)C->d_g;
    const double* rh = (const double*)C->d_rh;
    if (C->m > 0) {
        if (C->pd.rb) {
            int grid = 1;
            KIND_SWITCH(C->kkind, grid = fit_grid((const void*)k_trig_rows_rb<T, KINDV>,
                                                  std::min<long long>(C->pd.nblk, (long long)C->nb1), RB_NT));
            auto gather = [&](cudaStream_t q) {
                KIND_SWITCH(C->kkind, LAUNCH(C, q, KC_TRIGR,
                    (k_trig_rows_rb<T, KINDV><<<grid, RB_NT, 0, q>>>(csr_K(C), C->pd.blk_row, C->pd.nblk, st, g, rh,
                                                                     C->d_rsign, C->m1p, C->d_u, ctrl, kint, j, C->d_part1,
                                                                     C->d_ones, C->push_primal ? C->d_trig_flag : nullptr))));
                if (grid < C->nb1)
                    LAUNCH(C, q, KC_TRIGR, (k_fill<<<1, NT, 0, q>>>(C->d_part1 + 3LL * grid, 3LL * (C->nb1 - grid), 0.0)));
            };
            if (C->push_primal) {
                // x_k pushed by the trigger iteration's primal: gather-free pass over the rows (writes all nb1 partials)
                auto pushed = [&](cudaStream_t q) {
                    LAUNCH(C, q, KC_TRIGR, (k_trig_rows_push<T><<<C->nb1, NT, 0, q>>>(C->m, st, g, rh, C->d_rsign, C->m1p, C->d_u,
                        ctrl, kint, j, C->d_part1, C->d_ones, C->d_accv, C->d_ones_cnt, C->d_trig_flag)));
                };
                branch(C, s, [&](cudaStream_t q, cudaGraphConditionalHandle h, int a, int b) {
                    k_decide_flag<<<1, 1, 0, q>>>(C->d_trig_flag, C->d_ctrl, h, a, b);
                    CK(cudaGetLastError());
                }, pushed, gather);
                LAUNCH(C, s, KC_TRIGR, (k_trig_clear<<<1, 1, 0, s>>>(C->d_trig_flag)));
            } else {
                gather(s);
            }
        } else if (!C->pd.seg) {
            KIND_SWITCH(C->kkind, SUB_SWITCH(C->pd.sub, LAUNCH(C, s, KC_TRIGR,
                (k_trig_rows<T, KINDV, SUBV, false><<<C->nb1, NT, 0, s>>>(csr_K(C), C->pd.ds.plan(), nullptr, nullptr,
                    st, g, rh, C->d_rsign, C->m1p, ctrl, kint, j, C->d_part1)))));
        } else {
            const int grid = grid_for(C->pd.ds.nseg * 32);
            KIND_SWITCH(C->kkind, LAUNCH(C, s, KC_TRIGR,
                (k_seg_partial<T, KINDV><<<grid, NT, 0, s>>>(csr_K(C), C->pd.ds.plan(), st.x[0], st.x[1], nullptr,
                                                             nullptr, 2, ctrl, kint, j, C->d_segpart));
                (k_seg_partial<T, KINDV><<<grid, NT, 0, s>>>(csr_K(C), C->pd.ds.plan(), st.x[0], st.x[1], st.xb[0],
                                                             st.xb[1], 2, ctrl, kint, j, C->d_segpart2));
                (k_trig_rows<T, KINDV, 32, true><<<C->nb1, NT, 0, s>>>(csr_K(C), C->pd.ds.plan(), C->d_segpart,
                    C->d_segpart2, st, g, rh, C->d_rsign, C->m1p, ctrl, kint, j, C->d_part1))));
        }
    } else {
        LAUNCH(C, s, KC_TRIGR, (k_fill<<<1, NT, 0, s>>>(C->d_part1, 3LL * C->nb1, 0.0)));
    }
    if (C->qdense)  // Q~(x_k - x_{k-1}) of s^x: x_k = par ? x[0] : x[1], x_{k-1} = par ? x[1] : x[0]
        enqueue_qx<T>(C, s, QxSrc<T>{{st.x[1], st.x[0]}, {st.x[0], st.x[1]}, ctrl, kint, j}, true, C->omega, C->d_qdx);
    if (C->hasq)
        LAUNCH(C, s, KC_TRIGC, (k_trig_cols<T, true><<<C->nb2, NT, 0, s>>>(C->n, csr_Q(C, C->qdense ? C->d_qdx : nullptr), (const T*)C->d_qs, st, ctrl,
                                                                            kint, j, C->d_part2)));
    else
        LAUNCH(C, s, KC_TRIGC, (k_trig_cols<T, false><<<C->nb2, NT, 0, s>>>(C->n, csr_Q(C), (const T*)C->d_qs, st, ctrl,
                                                                             kint, j, C->d_part2)));
}

// k_obj_bits launch shape: gx CTAs per word group (<= 8 per SM in total, >= 16 chunks each)
struct ObjBitsShape { int wv; int nwg; long long gx; long long cpc; };
ObjBitsShape obj_bits_shape(const gfors_ctx* C, int W) {
    ObjBitsShape o;
    o.wv = (W % 2 == 0) ? 2 : 1;
    o.nwg = W / o.wv;
    const long long nchunk32 = (C->n + 31) / 32;
    long long gx = std::max<long long>(1, (long long)C->num_sms * 8 / o.nwg);
    gx = std::min<long long>(gx, (nchunk32 + 15) / 16);
    o.cpc = (nchunk32 + gx - 1) / gx;
    o.gx = (nchunk32 + o.cpc - 1) / o.cpc;
    return o;
}

// x_l' Q x_l of every lane of the batch by the tcgen05 int8 kernel (dense_q.cuh): unpack the bit-sliced
// samples to int8 rows, then tc_grid partial rows of int64 lane sums at zrows
// unpack the round's batch into sample-major int8 rows (the B operand of the tensor-core kernels) and
// encode its tensor map; once per round when both dense paths run
void enqueue_unpack(gfors_ctx* C, cudaStream_t s, int W) {
    const long long lanes = 64LL * W;
    LAUNCH(C, s, KC_OBJ_TC, (k_unpack_samples<<<grid_for(C->xld / 16 * W * 8), NT, 0, s>>>(C->d_X, W, C->n, C->xld, C->d_Xs)));
    // the map of this batch width (host encode, ~1 us; captured by value into a graph node)
    if (!C->dry) C->tmX = make_tmap_i8(C->d_Xs, C->xld, lanes, (int)std::min<long long>(TC_NMAX, lanes));
}

void enqueue_obj_dense(gfors_ctx* C, cudaStream_t s, int W, long long* zrows, bool unpacked) {
    const long long lanes = 64LL * W;
    if (!unpacked) enqueue_unpack(C, s, W);
    const int nbox = (int)std::min<long long>(TC_NMAX, lanes);
    const size_t sm = tc_smem_bytes(nbox, (int)lanes);
    LAUNCH(C, s, KC_OBJ_TC, (k_obj_dense_tc<false><<<C->tc_grid, TC_NT, sm, s>>>(C->tmQ, C->tmX, C->d_tcitems, C->d_tcoff,
                                                                                (int)lanes, nbox, C->d_X, W, C->n, zrows, nullptr)));
}

// K.X for the dense integer rows on tensor cores (split-K), then the row test
void enqueue_feas_dense(gfors_ctx* C, cudaStream_t s, int W) {
    const long long lanes = 64LL * W;
    enqueue_unpack(C, s, W);
    const int nbox = (int)std::min<long long>(TC_NMAX, lanes);
    const size_t sm = tc_smem_bytes(nbox, (int)lanes);
    LAUNCH(C, s, KC_FEAS, (k_obj_dense_tc<true><<<C->k_tc_grid, TC_NT, sm, s>>>(C->tmK, C->tmX, C->d_kitems, C->d_koff,
                                                                               (int)lanes, nbox, C->d_X, W, C->n_int, nullptr, C->d_kS)));
    LAUNCH(C, s, KC_FEAS, (k_feas_dense_final<<<grid_for(C->n_int * lanes), NT, 0, s>>>(C->d_kS, C->n_int, (int)lanes, C->d_int_rhs,
                                                                                        C->d_int_eq, C->d_viol)));
}

// evaluation of the batch in d_X (W words per variable); viol/iacc must have been reset
// list_batch: the batch is exactly what k_sample drew from its list this round (no repair / completion):
// the linear objective then only visits the listed (fractional) variables (k_obj_list)
void enqueue_eval(gfors_ctx* C, cudaStream_t s, int W, const unsigned char* ones = nullptr, bool list_batch = false) {
    const Csr K = csr_K(C);
    for (int li = 0; li < 3; ++li) {
        auto& rb = C->cntrb[li];
        if (!rb.rows.nrows) continue;
        CountRows cr{rb.rows.row, rb.rows.t, rb.rows.rel, rb.rows.B, rb.rows.nrows};
        if (ones) LAUNCH(C, s, KC_FEAS, (k_feas_skip<<<grid_for(cr.nrows), NT, 0, s>>>(cr, ones, rb.skip)));
        const unsigned char* sk = ones ? rb.skip : nullptr;
        const int wv = (W % 8 == 0) ? 8 : ((W % 2 == 0) ? 2 : 1);
        const int nwg = W / wv;
        const ClassCsr& cc = wv == 8 ? rb.cc8 : rb.cc;
        // grid: the resident CTAs per SM (shared memory bound) x SMs, over all word groups
        auto feas_grid = [&](const void* fn, size_t smb) {
            smem_attr(fn, smb);
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, FB_NT, smb));
            return dim3((unsigned)std::max<long long>(1, std::min<long long>(cc.nblk, (long long)C->num_sms * std::max(per_sm, 1) / nwg)),
                        (unsigned)nwg);
        };
#define FEAS_LAUNCH(BM, WVV, NNZV, SK)                                                                            \
        {                                                                                                       \
            const size_t smb = 2 * sizeof(FbBuf<WVV, NNZV>);                                                    \
            const dim3 grid = feas_grid((const void*)k_feas_rb<BM, WVV, NNZV, SK>, smb);                        \
            LAUNCH(C, s, KC_FEAS, (k_feas_rb<BM, WVV, NNZV, SK><<<grid, FB_NT, smb, s>>>(cc, sk, C->d_X, W, C->d_viol))); \
        }
#define FEAS_RB2(BM, SK) \
        if (wv == 8) FEAS_LAUNCH(BM, 8, FB_NNZ8, SK) \
        else if (wv == 2) FEAS_LAUNCH(BM, 2, FB_NNZ, SK) \
        else FEAS_LAUNCH(BM, 1, FB_NNZ, SK)
#define FEAS_RB(BM) if (sk) { FEAS_RB2(BM, true) } else { FEAS_RB2(BM, false) }
        if (li == 0) { FEAS_RB(1) } else if (li == 1) { FEAS_RB(2) } else { FEAS_RB(8) }
#undef FEAS_RB
#undef FEAS_RB2
#undef FEAS_LAUNCH
    }
    for (int li = 0; li < 3; ++li) {
        auto& cl = C->cnt[li];
        if (!cl.nrows) continue;
        CountRows cr{cl.row, cl.t, cl.rel, cl.B, cl.nrows};
        const int grid = grid_for(cl.nrows * (long long)cl.sub);
        const size_t sm = 0;
        const int wv = (W % 4 == 0) ? 4 : ((W % 2 == 0) ? 2 : 1);
#define FEAS_WV(BM)                                                                                                \
    if (wv == 4) { SUB_SWITCH(cl.sub, LAUNCH(C, s, KC_FEAS, (k_feas_count<BM, SUBV, 4><<<grid, NT, sm, s>>>(K, cr, C->d_X, W, C->d_viol, ones)))); } \
    else if (wv == 2) { SUB_SWITCH(cl.sub, LAUNCH(C, s, KC_FEAS, (k_feas_count<BM, SUBV, 2><<<grid, NT, sm, s>>>(K, cr, C->d_X, W, C->d_viol, ones)))); } \
    else { SUB_SWITCH(cl.sub, LAUNCH(C, s, KC_FEAS, (k_feas_count<BM, SUBV, 1><<<grid, NT, sm, s>>>(K, cr, C->d_X, W, C->d_viol, ones)))); }
        if (li == 0) {
            FEAS_WV(1)
        } else if (li == 1) {
            FEAS_WV(2)
        } else {
            FEAS_WV(8)
        }
#undef FEAS_WV
    }
    bool unpacked = false;
    if (C->n_int && C->kdense) {
        enqueue_feas_dense(C, s, W);
        unpacked = true;
    } else if (C->n_int) {
        IntRows ir{C->d_int_row, C->d_int_rhs, C->d_int_eq, C->d_int_seg_start, C->d_int_seg_slot, C->n_int, C->n_int_seg};
        const int grid = grid_for(C->n_int_seg * 2LL * W * 32);
        KIND_SWITCH(C->kkind, LAUNCH(C, s, KC_FEAS, (k_feas_int_partial<KINDV><<<grid, NT, 0, s>>>(K, ir, C->d_X, W, C->d_iacc))));
        LAUNCH(C, s, KC_FEAS, (k_feas_int_final<<<grid_for(C->n_int * 64LL * W), NT, 0, s>>>(ir, W, C->d_iacc, C->d_viol)));
    }
    if (C->n_real) {
        const int grid = grid_for(C->n_real * 2LL * W * 32);
        KIND_SWITCH(C->kkind, LAUNCH(C, s, KC_FEAS, (k_feas_real<KINDV><<<grid, NT, 0, s>>>(K, C->d_real_row, C->n_real, C->d_ru,
                                                                                             C->m1, C->d_X, W, C->d_viol))));
    }
    const long long nchunk = (C->n + C->obj_chunk - 1) / C->obj_chunk;
    const int grid = grid_for(nchunk * 2LL * W * 32);
    const Csr Q = csr_Q(C);
    if (C->obj_bits) {
        // linear term by coefficient bit planes, quadratic term (if any) appended as extra partial rows
        const ObjBitsShape ob = obj_bits_shape(C, W);
        const long long jpw = ob.gx;
        const dim3 og((unsigned)ob.gx, (unsigned)ob.nwg);
        if (list_batch && C->opt.obj_list && C->d_slist && !C->hasq && !C->qdense) {
            // the list kernel when at most half the variables are fractional (converged blocks), else the
            // streaming one (it reads consecutive variables; measured 0.094 vs 0.106 ms on a full list);
            // the one not chosen reads the list length and exits
            const long long thr = C->n / 2;
            if (ob.wv == 2) {
                LAUNCH(C, s, KC_OBJ, (k_obj_list<2><<<og, 256, 0, s>>>(C->d_slist, C->d_scnt, C->d_s1, C->d_c, C->obj_nb,
                                                                      C->obj_cmin, C->d_X, W, (long long*)C->d_zpart, thr)));
                LAUNCH(C, s, KC_OBJ, (k_obj_bits<2><<<og, 256, 0, s>>>(C->n, ob.cpc, C->d_planes, C->obj_nb, C->obj_cmin,
                                                                      C->d_X, W, (long long*)C->d_zpart, C->d_scnt, thr)));
            } else {
                LAUNCH(C, s, KC_OBJ, (k_obj_list<1><<<og, 256, 0, s>>>(C->d_slist, C->d_scnt, C->d_s1, C->d_c, C->obj_nb,
                                                                      C->obj_cmin, C->d_X, W, (long long*)C->d_zpart, thr)));
                LAUNCH(C, s, KC_OBJ, (k_obj_bits<1><<<og, 256, 0, s>>>(C->n, ob.cpc, C->d_planes, C->obj_nb, C->obj_cmin,
                                                                      C->d_X, W, (long long*)C->d_zpart, C->d_scnt, thr)));
            }
        } else if (ob.wv == 2)
            LAUNCH(C, s, KC_OBJ, (k_obj_bits<2><<<og, 256, 0, s>>>(C->n, ob.cpc, C->d_planes, C->obj_nb, C->obj_cmin,
                                                                  C->d_X, W, (long long*)C->d_zpart)));
        else
            LAUNCH(C, s, KC_OBJ, (k_obj_bits<1><<<og, 256, 0, s>>>(C->n, ob.cpc, C->d_planes, C->obj_nb, C->obj_cmin,
                                                                  C->d_X, W, (long long*)C->d_zpart)));
        long long rows = jpw;
        if (C->qdense) {
            enqueue_obj_dense(C, s, W, (long long*)C->d_zpart + jpw * 64LL * W, unpacked);
            rows += C->tc_grid;
        } else if (C->hasq) {
            long long* zq = (long long*)C->d_zpart + jpw * 64LL * W;
            LAUNCH(C, s, KC_OBJ, (k_obj_quad<true><<<grid, NT, 0, s>>>(C->n, C->obj_chunk, Q, C->d_qval, C->d_X, W, zq)));
            rows += nchunk;
        }
        LAUNCH(C, s, KC_OBJ, (k_obj_final<true><<<2 * W, 1024, 0, s>>>(rows, W, C->d_zpart, C->c0, C->d_z)));
    } else if (C->integral) {
        if (C->qdense) {
            LAUNCH(C, s, KC_OBJ, (k_obj_partial<true, false><<<grid, NT, 0, s>>>(C->n, C->obj_chunk, C->d_c, Q, C->d_qval, C->d_X, W, C->d_zpart)));
            enqueue_obj_dense(C, s, W, (long long*)C->d_zpart + nchunk * 64LL * W, unpacked);
            LAUNCH(C, s, KC_OBJ, (k_obj_final<true><<<2 * W, 1024, 0, s>>>(nchunk + C->tc_grid, W, C->d_zpart, C->c0, C->d_z)));
            return;
        }
        if (C->hasq)
            LAUNCH(C, s, KC_OBJ, (k_obj_partial<true, true><<<grid, NT, 0, s>>>(C->n, C->obj_chunk, C->d_c, Q, C->d_qval, C->d_X, W, C->d_zpart)));
        else
            LAUNCH(C, s, KC_OBJ, (k_obj_partial<true, false><<<grid, NT, 0, s>>>(C->n, C->obj_chunk, C->d_c, Q, C->d_qval, C->d_X, W, C->d_zpart)));
        LAUNCH(C, s, KC_OBJ, (k_obj_final<true><<<2 * W, 1024, 0, s>>>(nchunk, W, C->d_zpart, C->c0, C->d_z)));
    } else {
        if (C->hasq)
            LAUNCH(C, s, KC_OBJ, (k_obj_partial<false, true><<<grid, NT, 0, s>>>(C->n, C->obj_chunk, C->d_c, Q, C->d_qval, C->d_X, W, C->d_zpart)));
        else
            LAUNCH(C, s, KC_OBJ, (k_obj_partial<false, false><<<grid, NT, 0, s>>>(C->n, C->obj_chunk, C->d_c, Q, C->d_qval, C->d_X, W, C->d_zpart)));
        LAUNCH(C, s, KC_OBJ, (k_obj_final<false><<<2 * W, 1024, 0, s>>>(nchunk, W, C->d_zpart, C->c0, C->d_z)));
    }
}

void enqueue_reset(gfors_ctx* C, cudaStream_t s, int W, unsigned long long last_mask) {
    const long long niacc = C->n_int * 64LL * W;
    LAUNCH(C, s, KC_ARGMIN, (k_round_reset<<<grid_for(std::max<long long>(niacc, 1)), NT, 0, s>>>(
                                C->d_viol, W, C->d_iacc, niacc, last_mask, C->never_feasible ? 1 : 0)));
}

// make sure the batch buffers fit W words per variable
void ensure_batch(gfors_ctx* C, int W) {
    const long long words = C->n * (long long)W;
    if (words > C->X_words) {
        dfree(C->d_X); C->d_X = nullptr;
        C->d_X = dalloc<uint64_t>(words);
        C->X_words = words;
        dfree(C->d_viol); C->d_viol = dalloc<unsigned long long>(W);
        C->gvalid = false;
    }
    if (!C->d_slist) {
        C->d_slist = dalloc<uint2>(C->n);
        C->d_scnt = dalloc<unsigned>(4);
        CK(cudaMemset(C->d_scnt, 0, 4 * sizeof(unsigned)));
        C->d_s1 = dalloc<unsigned long long>(2);
        CK(cudaMemset(C->d_s1, 0, 2 * sizeof(unsigned long long)));
        C->gvalid = false;
    }
    const long long niacc = C->n_int * 64LL * W;
    if (niacc > C->iacc_len) {
        dfree(C->d_iacc); C->d_iacc = dalloc<unsigned long long>(niacc); C->iacc_len = niacc; C->gvalid = false;
    }
    if (!C->d_iacc) { C->d_iacc = dalloc<unsigned long long>(1); C->iacc_len = 1; }
    const long long nchunk = (C->n + C->obj_chunk - 1) / C->obj_chunk;
    long long zrows = nchunk;
    if (C->obj_bits) {
        zrows = obj_bits_shape(C, W).gx + (C->qdense ? C->tc_grid : (C->hasq ? nchunk : 0));
    } else if (C->qdense) {
        zrows = nchunk + C->tc_grid;
    }
    if ((C->qdense || C->kdense) && 64LL * W > C->Xs_lanes) {  // grow-only: smaller batches (final round) reuse it
        if (64LL * W > 4096) input_error("params.k_b: the dense tensor-core evaluation supports k_b <= 4096 per rank");
        dfree(C->d_Xs);
        C->d_Xs = dalloc<int8_t>(64LL * W * C->xld);
        C->Xs_lanes = 64LL * W;
        C->gvalid = false;
    }
    if (C->kdense && C->n_int * 64LL * W > C->kS_len) {
        dfree(C->d_kS);
        C->d_kS = dalloc<int>(C->n_int * 64LL * W);
        CK(cudaMemsetAsync(C->d_kS, 0, C->n_int * 64LL * W * sizeof(int), C->stream));
        C->kS_len = C->n_int * 64LL * W;
        C->gvalid = false;
    }
    const long long zp = zrows * 64LL * W;
    if (zp > C->zpart_len) { dfree(C->d_zpart); C->d_zpart = dalloc<double>(zp); C->zpart_len = zp; C->gvalid = false; }
    if (64LL * W > C->z_len) { dfree(C->d_z); C->d_z = dalloc<double>(64LL * W); C->z_len = 64LL * W; C->gvalid = false; }
}

void ensure_a3(gfors_ctx* C, long long a3n);

// monotone relaxation (R26): every row acts as >= in the PDHG step / indicators; EvalBest unchanged
void set_relax(gfors_ctx* C, int relax, int repair) {
    if (relax) ensure_host_k(C);
    if (repair && !relax) input_error("params.repair: needs relax = 1");
    if (relax) {
        if (C->hasq) input_error("params.relax: the monotone relaxation needs Q = 0");
        for (long long i = 0; i < C->n; ++i)
            if (C->c[i] < 0.0) input_error("params.relax: needs c >= 0 (canonical; c[%lld] < 0)", i);
        for (double v : C->kval)
            if (v < 0.0) input_error("params.relax: needs K_u >= 0 (canonical)");
    }
    if (repair) {
        if (!C->integral) input_error("params.repair: needs integral data");
        if (C->sharded) input_error("params.repair: not with the NCCL-sharded loop (winner regeneration)");
    }
    if (C->m1p != (relax ? C->m : C->m1)) C->gvalid = false;
    C->m1p = relax ? C->m : C->m1;
    C->repair = repair != 0;
    if (C->repair && !C->d_rp_rank) {
        // the drop order of every lane: decreasing canonical cost, ties lower index first (R26)
        std::vector<int> order((size_t)C->n), rank((size_t)C->n);
        for (long long i = 0; i < C->n; ++i) order[i] = (int)i;
        std::sort(order.begin(), order.end(), [&](int a, int b) {
            return C->c[a] > C->c[b] || (C->c[a] == C->c[b] && a < b);
        });
        for (long long t = 0; t < C->n; ++t) rank[order[t]] = (int)t;
        C->d_rp_order = dupload(order, C->stream);
        C->d_rp_rank = dupload(rank, C->stream);
    }
}

// cover completion (cover.cuh, R27): eligible rows built once, phase buffers sized for W
void set_complete(gfors_ctx* C, int complete, int W) {
    C->complete = complete != 0;
    if (!complete) return;
    if (C->sharded) input_error("params.complete: not with the NCCL-sharded loop (winner regeneration)");
    if (C->n_cover < 0) {
        ensure_host_k(C);
        std::vector<int> rows;
        for (long long j = 0; j < C->m1; ++j) {
            bool ok = C->ru[j] == 1.0 && C->kptr[j + 1] > C->kptr[j];
            for (long long q = C->kptr[j]; q < C->kptr[j + 1] && ok; ++q) ok = C->kval[q] == 1.0;
            if (ok) rows.push_back((int)j);
        }
        C->n_cover = (long long)rows.size();
        dfree(C->d_cover_rows);
        C->d_cover_rows = dupload(rows, C->stream);
        dfree(C->d_cover_best);
        C->d_cover_best = dalloc<int>(std::max<long long>(C->n_cover, 1));
        C->gvalid = false;
    }
    if (C->n_cover * (long long)W > C->cover_viol_len) {
        dfree(C->d_cover_viol);
        C->d_cover_viol = dalloc<uint64_t>(std::max<long long>(C->n_cover * (long long)W, 1));
        C->cover_viol_len = C->n_cover * (long long)W;
        C->gvalid = false;
    }
}

template <typename T>
void enqueue_cover(gfors_ctx* C, cudaStream_t s, const double* pfix, int W, long long kint,
                   const unsigned char* ones = nullptr) {
    if (C->n_cover <= 0) return;
    LAUNCH(C, s, KC_COVER, (k_cover_scan<T, 8><<<grid_for(C->n_cover * 8LL), NT, 0, s>>>(csr_K(C), C->d_cover_rows, C->n_cover,
        (const T*)C->d_x[0], (const T*)C->d_x[1], pfix, C->d_ctrl, kint, C->d_X, W, C->d_cover_best, C->d_cover_viol, ones)));
    LAUNCH(C, s, KC_COVER, (k_cover_apply<<<grid_for(C->n_cover * (long long)W), NT, 0, s>>>(C->n_cover, C->d_cover_best,
        C->d_cover_viol, W, ~0ull, C->d_X)));
}

void enqueue_repair(gfors_ctx* C, cudaStream_t s, int W) {
    const size_t sm = rp_smem_bytes(C->m);
    if (C->m > RP_SROWS && 64LL * W * C->m > C->rp_srow_len) {
        dfree(C->d_rp_srow);
        C->d_rp_srow = dalloc<long long>(64LL * W * C->m);
        C->rp_srow_len = 64LL * W * C->m;
        C->gvalid = false;
    }
    KIND_SWITCH(C->kkind, {
        smem_attr((const void*)k_repair<KINDV>, rp_smem_bytes(RP_SROWS));
        LAUNCH(C, s, KC_SAMPLE, (k_repair<KINDV><<<64 * W, RP_NT, sm, s>>>(C->n, C->m, csr_Kt(C), C->d_rp_rank, C->d_rp_order,
                                                                         C->d_ru, C->d_X, W, C->d_rp_srow)));
    });
}

// select the RandSampleStep of a run / hook (validates Alg. 4's parameters against the problem)
void set_sampler(gfors_ctx* C, int sampler, long long a3n, double gamma, long long ls) {
    C->a3.sampler = sampler;
    if (sampler != 1) return;
    if (a3n < 1 || a3n > 4096 || a3n * a3n * a3n != C->n)
        input_error("params.a3_n: sampler 1 needs n = a3_n^3 variables (a3_n = %lld, n = %lld)", a3n, C->n);
    if (!(gamma > 0.0)) input_error("params.a3_gamma: must be > 0");
    if (C->sharded) input_error("params.sampler: the Alg. 4 sampler is not combined with the NCCL-sharded loop "
                                "(its winner regeneration replays the Bernoulli contract)");
    ensure_a3(C, a3n);
    C->a3.n = a3n;
    C->a3.K = std::min<long long>(C->n, (long long)std::ceil(gamma * (double)a3n));
    C->a3.L = ls < 0 ? 2 * a3n : ls;
}

// buffers of the Alg. 4 sampler for a3_n (grow-only; the radix-sort temp storage is sized for n^3)
void ensure_a3(gfors_ctx* C, long long a3n) {
    auto& A = C->a3;
    if (a3n <= A.alloc_n) return;
    const long long N = C->n;
    for (int b = 0; b < 2; ++b) { dfree(A.keys[b]); dfree(A.vals[b]); A.keys[b] = dalloc<unsigned long long>(N); A.vals[b] = dalloc<int>(N); }
    dfree(A.tmp); A.tmp = nullptr;
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, A.keys[0], A.keys[1], A.vals[0], A.vals[1], (int)N));
    A.tmp = dalloc<unsigned char>(bytes);
    A.tmp_bytes = bytes;
    for (short** q : {&A.sj0, &A.sk0, &A.Ri, &A.Rj, &A.Rk}) { dfree(*q); *q = dalloc<short>(a3n); }
    dfree(A.meta); A.meta = dalloc<int>(1);
    A.alloc_n = a3n;
    C->gvalid = false;
}

// Alg. 4 (assign3d.cuh): sort -> greedy partial assignment -> per-lane completion + interchanges
template <typename T>
void enqueue_sample_a3(gfors_ctx* C, cudaStream_t s, const double* pfix, int W, long long word_off, uint64_t seed,
                       long long kint, int r, int kr, unsigned round_fixed, int use_fixed) {
    auto& A = C->a3;
    const long long N = C->n;
    const uint2 key = make_uint2((unsigned)(seed & 0xffffffffu), (unsigned)(seed >> 32));
    if (!C->dry) CK(cudaMemsetAsync(C->d_X, 0, N * (long long)W * sizeof(uint64_t), s));
    LAUNCH(C, s, KC_SAMPLE, (k_a3_keys<T><<<grid_for(N), NT, 0, s>>>((const T*)C->d_x[0], (const T*)C->d_x[1], pfix, N,
                                                                   C->d_ctrl, kint, use_fixed, A.keys[0], A.vals[0])));
    if (!C->dry) {
        size_t bytes = A.tmp_bytes;
        const int end_bit = (sizeof(T) == 4 && !pfix) ? 32 : 64;  // 32-bit keys for fp32 x_k (k_a3_keys)
        CK(cub::DeviceRadixSort::SortPairs(A.tmp, bytes, A.keys[0], A.keys[1], A.vals[0], A.vals[1], (int)N, 0, end_bit, s));
    }
    // (the CUB radix-sort kernels are library launches: not counted in gfors_run_info.launches)
    const size_t gsm = a3_greedy_smem((int)A.n);
    if (gsm > 48 * 1024) smem_attr((const void*)k_a3_greedy, gsm);
    LAUNCH(C, s, KC_SAMPLE, (k_a3_greedy<<<1, A3_GNT, gsm, s>>>(A.vals[1], A.K, (int)A.n, A.sj0, A.sk0, A.Ri, A.Rj, A.Rk,
                                                                  A.meta)));
    const int lanes = 64 * W;
    const size_t per = a3_warp_smem(A.n, A.L);
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per));
    const size_t sm = per * wpb;
    if (sm > 48 * 1024) smem_attr((const void*)k_a3_sample, sm);
    LAUNCH(C, s, KC_SAMPLE, (k_a3_sample<<<(lanes + wpb - 1) / wpb, 32 * wpb, sm, s>>>((int)A.n, A.sj0, A.sk0, A.Ri, A.Rj,
        A.Rk, A.meta, C->d_c, key, C->d_ctrl, r, kr, round_fixed, use_fixed, word_off, W, A.L, C->d_X)));
}

template <typename T>
void enqueue_sample(gfors_ctx* C, cudaStream_t s, const double* pfix, int W, long long word_off, uint64_t seed,
                    long long kint, int r, int kr, unsigned round_fixed, int use_fixed) {
    if (C->a3.sampler == 1) {
        enqueue_sample_a3<T>(C, s, pfix, W, word_off, seed, kint, r, kr, round_fixed, use_fixed);
        return;
    }
    PhiloxKeys rk;
    for (int t = 0; t < 10; ++t) {  // round t uses key + t*(W0, W1) (mod 2^32)
        rk.k0[t] = (uint32_t)(seed & 0xffffffffu) + (uint32_t)t * 0x9E3779B9u;
        rk.k1[t] = (uint32_t)(seed >> 32) + (uint32_t)t * 0xBB67AE85u;
    }
    LAUNCH(C, s, KC_SAMPLE, (k_sample_thr<T><<<grid_for(C->n), NT, 0, s>>>((const T*)C->d_x[0], (const T*)C->d_x[1], pfix,
                                C->n, W, C->d_ctrl, kint, use_fixed, C->d_slist, C->d_scnt, C->d_X,
                                C->obj_bits ? C->d_c : nullptr, C->d_s1)));
    LAUNCH(C, s, KC_SAMPLE, (k_sample<<<C->num_sms * SMP_CTAS, NT, 0, s>>>(C->d_slist, C->d_scnt, W, word_off, rk, C->d_ctrl, r, kr,
                                round_fixed, use_fixed, C->d_X, C->d_s1)));
}

// one whole Alg. 1 sampling block (graph body)
template <typename T>
void enqueue_block(gfors_ctx* C, cudaStream_t s, const gfors_params* p, int W, HaltPar hp,
                   cudaGraphConditionalHandle h, int use_handle) {
    const long long kint = p->k_int;
    for (long long j = 0; j < kint; ++j) enqueue_iter<T>(C, s, kint, j);
    enqueue_trigger<T>(C, s, kint, kint - 1);
    // loopback (test mode): all `world` ranks run here one after another, records written straight
    // into the gathered slots; otherwise this rank's own word range and an ncclAllGather
    const int nsim = C->loopback ? C->world : 1;
    for (int r = 0; r < p->k_r; ++r) {
        for (int q = 0; q < nsim; ++q) {
            const int rank = C->loopback ? q : C->rank;
            const long long word_off = (long long)rank * W;
            enqueue_reset(C, s, W, ~0ull);
            enqueue_sample<T>(C, s, nullptr, W, word_off, p->seed, kint, r, p->k_r, 0u, 0);
            if (C->repair) enqueue_repair(C, s, W);
            if (C->complete) enqueue_cover<T>(C, s, nullptr, W, kint, (C->m > 0 && C->pd.rb) ? C->d_ones : nullptr);
            // the trigger pass of this block counted the p = 1 entries of every row (rb path)
            enqueue_eval(C, s, W, (C->m > 0 && C->pd.rb) ? C->d_ones : nullptr,
                         C->a3.sampler != 1 && !C->repair && !C->complete);
            if (!C->sharded) {
                LAUNCH(C, s, KC_ARGMIN, (k_argmin<<<1, NT, 0, s>>>(C->d_z, C->d_viol, 64LL * W, word_off, C->d_ctrl, kint, r, p->k_r, 0)));
                LAUNCH(C, s, KC_ARGMIN, (k_copy_best<<<grid_for(C->n), NT, 0, s>>>(C->d_X, W, C->n, C->d_ctrl, C->d_xbest)));
                continue;
            }
            // record (-> ncclAllGather) -> identical merge on every rank -> regenerate the winner's bits
            const long long fb = (C->opt.force_deadline_rank == rank) ? C->opt.force_deadline_block : -1;
            double* rec = C->loopback ? C->d_rec + 4 + 4 * q : C->d_rec;
            LAUNCH(C, s, KC_ARGMIN, (k_local_record<<<1, NT, 0, s>>>(C->d_z, C->d_viol, 64LL * W, word_off, C->d_ctrl, rec,
                                                                   q == 0, fb)));
        }
        if (C->sharded) {
            if (C->capturing && C->opt.force_capture_fail) throw Err{GFORS_E_CUDA, "forced capture failure (test option)"};
            if (!C->loopback) {
                const int rc = C->dry ? 0 : nccl().AllGather(C->d_rec, C->d_rec + 4, 4, ncclFloat64_, C->comm, s);
                if (rc != 0) throw Err{GFORS_E_NCCL, std::string("ncclAllGather: ") + nccl().GetErrorString(rc)};
            }
            LAUNCH(C, s, KC_ARGMIN, (k_merge_records<<<1, 32, 0, s>>>(C->d_rec + 4, C->world, C->d_ctrl, kint, r, p->k_r, C->d_regen)));
            const uint2 key = make_uint2((unsigned)(p->seed & 0xffffffffu), (unsigned)(p->seed >> 32));
            LAUNCH(C, s, KC_ARGMIN, (k_regen_best<T><<<grid_for(C->n), NT, 0, s>>>((const T*)C->d_x[0], (const T*)C->d_x[1], C->n,
                                                                                  C->d_ctrl, kint, key, C->d_regen, C->d_xbest)));
        }
    }
    LAUNCH(C, s, KC_HALT, (k_halt<<<1, NT, 0, s>>>(C->d_ctrl, hp, C->d_part1, C->nb1, C->d_part2, C->nb2, C->n, C->d_hist,
                                                  C->d_rho, C->nrho, C->d_trace, h, use_handle)));
}

}  // namespace

// =============================================================================================
// Preprocess (a2) on the device
// =============================================================================================
static double dev_norm(gfors_ctx* C, const double* v, long long len) {
    cudaStream_t s = C->stream;
    const int nb = std::min(grid_for(len), 1024);
    k_sumsq_partial<<<nb, NT, 0, s>>>(v, len, C->d_red);
    CK(cudaGetLastError());
    k_sum_final<<<1, NT, 0, s>>>(C->d_red, nb, C->d_scalar);
    CK(cudaGetLastError());
    double h = 0.0;
    CK(cudaMemcpyAsync(&h, C->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
}

// power iteration on M'M (readings R5, R6).  isq: M = Q (symmetric) else
// M = D^-1 K_u (row scale s).
static double power_iteration(gfors_ctx* C, bool isq, double tol, int max_iter) {
    cudaStream_t s = C->stream;
    const long long cols = C->n, rows = isq ? C->n : C->m;
    if (rows == 0) return 0.0;
    double* v = C->d_tmp[0];
    double* w = C->d_tmp[1];
    double* u = C->d_tmp[2];
    k_fill<<<grid_for(cols), NT, 0, s>>>(v, cols, 1.0 / std::sqrt((double)cols));
    CK(cudaGetLastError());
    double sigma = 0.0, sigma_prev = 0.0;
    bool restarted = false;
    const int gr = grid_for(rows * 32LL), gc = grid_for(cols * 32LL);
    for (int t = 1; t <= max_iter; ++t) {
        if (isq && C->qdense) {
            enqueue_qx<double>(C, s, QxSrc<double>{{v, v}, {nullptr, nullptr}, nullptr, 0, 0}, false, 1.0, w);
        } else if (isq) {
            k_spmv_rows<KV_F64><<<gr, NT, 0, s>>>(csr_Q(C), nullptr, nullptr, v, w);
        } else {
            KIND_SWITCH(C->kkind, (k_spmv_rows<KINDV><<<gr, NT, 0, s>>>(csr_K(C), C->d_rsign, C->d_s, v, w)));
        }
        CK(cudaGetLastError());
        sigma = dev_norm(C, w, rows);
        if (isq && C->qdense) {
            enqueue_qx<double>(C, s, QxSrc<double>{{w, w}, {nullptr, nullptr}, nullptr, 0, 0}, false, 1.0, u);
        } else if (isq) {
            k_spmv_rows<KV_F64><<<gc, NT, 0, s>>>(csr_Q(C), nullptr, nullptr, w, u);
        } else {
            // w' once per row, then G lanes per column (G from the mean column length)
            const int G = pick_sub(cols ? (double)C->nnz / (double)cols : 1.0);
            const int gcg = grid_for(cols * (long long)G);
            KIND_SWITCH(C->kkind, {
                k_prescale<KINDV><<<grid_for(rows), NT, 0, s>>>(w, C->d_s, C->d_rsign, rows, C->d_tmp[3]);
                SUB_SWITCH(G, (k_spmv_cols_g<KINDV, SUBV><<<gcg, NT, 0, s>>>(csr_Kt(C), C->d_tmp[3], u)));
            });
        }
        CK(cudaGetLastError());
        const double nu = dev_norm(C, u, cols);
        if (nu == 0.0) {
            if (t == 1 && !restarted) {
                k_philox_vec<<<grid_for(cols), NT, 0, s>>>(v, cols);
                CK(cudaGetLastError());
                const double nv = dev_norm(C, v, cols);
                CK(cudaMemcpyAsync(C->d_scalar, &nv, sizeof(double), cudaMemcpyHostToDevice, s));
                k_scale_vec<<<grid_for(cols), NT, 0, s>>>(v, C->d_scalar, cols, v);
                CK(cudaGetLastError());
                restarted = true;
                t = 0;
                continue;
            }
            break;
        }
        // v = u / ||u||  (the norm is already in d_scalar)
        k_scale_vec<<<grid_for(cols), NT, 0, s>>>(u, C->d_scalar, cols, v);
        CK(cudaGetLastError());
        if (t > 1 && std::fabs(sigma - sigma_prev) <= tol * sigma) break;
        sigma_prev = sigma;
    }
    return sigma;
}

// push-mode state at the start of a run / after set_state: lists unknown (gather first), delta-push
// accumulators cleared and invalid
static void reset_push(gfors_ctx* C, cudaStream_t s) {
    if (C->push_dual) {
        CK(cudaMemsetAsync(C->d_pcount, 0xff, 2 * sizeof(unsigned), s));
        CK(cudaMemsetAsync(C->d_acc, 0, std::max<long long>(C->m, 1) * sizeof(long long), s));
        CK(cudaMemsetAsync(C->d_pflags, 0, 8 * sizeof(unsigned), s));
    }
    if (C->push_primal) {
        CK(cudaMemsetAsync(C->d_rcount, 0, sizeof(unsigned), s));
        CK(cudaMemsetAsync(C->d_accx, 0, C->n * sizeof(long long), s));
        if (C->d_xst) CK(cudaMemsetAsync(C->d_xst, 0, C->n, s));
    }
}

// the product plans and push modes of the preprocessed precision (row-block size is per precision)
static void select_plans(gfors_ctx* C) {
    const int v = C->precision == 64 ? 1 : 0;
    if (v == 1 && !C->plans64) {
        C->pdv[1] = plan_direction64(C->pdv[0], C->kptr, C->m, C->stream, C->owned);
        C->ppv[1] = plan_direction64(C->ppv[0], C->ktptr, C->n, C->stream, C->owned);
        C->plans64 = true;
    }
    C->pd = C->pdv[v];
    C->pp = C->ppv[v];
    C->push_dual = C->push_dual_ok && C->pd.rb && C->pp.rb;
    C->push_primal = C->push_primal_ok && C->push_dual;
}

template <typename T>
static void alloc_loop_data(gfors_ctx* C) {
    const long long n = C->n, m = C->m;
    C->d_g = dalloc<double>(m); C->d_rh = dalloc<double>(m); C->d_cs = dalloc<T>(n); C->d_qs = dalloc<T>(C->qdense ? 1 : C->qnnz);
    for (int b = 0; b < 2; ++b) { C->d_x[b] = dalloc<T>(n); C->d_xb[b] = dalloc<T>(n); C->d_y[b] = dalloc<T>(m); }
    C->d_w = dalloc<T>(m);
    cudaStream_t s = C->stream;
    k_make_rowdata<double><<<grid_for(m), NT, 0, s>>>(m, C->d_s, C->d_ru, C->kappa, (double*)C->d_g, (double*)C->d_rh);
    CK(cudaGetLastError());
    k_scale_to<T><<<grid_for(n), NT, 0, s>>>(C->d_c, n, C->omega, (T*)C->d_cs);
    CK(cudaGetLastError());
    if (C->qnnz && !C->qdense) {
        k_scale_to<T><<<grid_for(C->qnnz), NT, 0, s>>>(C->d_qval, C->qnnz, C->omega, (T*)C->d_qs);
        CK(cudaGetLastError());
    }
    k_init_state<T><<<grid_for(std::max(n, m)), NT, 0, s>>>(state_of<T>(C), n, m);
    CK(cudaGetLastError());
}

static void do_preprocess(gfors_ctx* C, const gfors_prep_opts* o, gfors_scaling* out) {
    if (C->stage < 1) throw Err{GFORS_E_STATE, "gfors_preprocess: call gfors_load first"};
    gfors_prep_opts d;
    gfors_prep_opts_default(&d);
    if (!o) o = &d;
    if (o->precision != 32 && o->precision != 64) input_error("prep_opts.precision: must be 32 or 64");
    if (!(o->tol > 0.0)) input_error("prep_opts.tol: must be > 0");
    if (o->max_iter < 1) input_error("prep_opts.max_iter: must be >= 1");
    CK(cudaSetDevice(C->device));
    C->free_prep();
    cudaStream_t s = C->stream;
    const long long n = C->n, m = C->m;
    const long long big = std::max(n, m);
    for (int k = 0; k < 4; ++k) C->d_tmp[k] = dalloc<double>(big);
    C->d_red = dalloc<double>(2048);
    C->d_scalar = dalloc<double>(1);
    C->d_s = dalloc<double>(m);
    if (C->qdense) {
        C->d_qx = dalloc<double>(n);
        C->d_qdx = dalloc<double>(n);
        C->d_qxpart = dalloc<double>((n + QX_CW - 1) / QX_CW * C->qld);
        C->d_qxpart2 = dalloc<double>((n + QX_CW - 1) / QX_CW * C->qld);
        C->d_qreuse = dalloc<long long>(1);
        CK(cudaMemsetAsync(C->d_qreuse, 0xff, sizeof(long long), s));  // -1: nothing to reuse
    }
    unsigned long long* d_zr = dalloc<unsigned long long>(1);
    CK(cudaMemsetAsync(d_zr, 0, sizeof(unsigned long long), s));
    // step 1: row 2-norms of K
    if (m) {
        KIND_SWITCH(C->kkind, (k_row_norms<KINDV><<<grid_for(m), NT, 0, s>>>(csr_K(C), C->d_s, d_zr)));
        CK(cudaGetLastError());
    }
    unsigned long long zr = 0;
    CK(cudaMemcpyAsync(&zr, d_zr, sizeof zr, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    dfree(d_zr);
    C->zero_rows = (long long)zr;
    // step 2: omega = ||Q||_2 + ||c||_2
    const double qn = C->qnnz ? power_iteration(C, true, o->tol, o->max_iter) : 0.0;
    const double cn = dev_norm(C, C->d_c, n);
    const double omega = qn + cn;
    C->omega = omega > 0.0 ? omega : 1.0;
    // step 3: kappa = ||D^-1 K||_2
    const double kap = m ? power_iteration(C, false, o->tol, o->max_iter) : 0.0;
    C->kappa = kap > 0.0 ? kap : 1.0;
    C->precision = o->precision;
    select_plans(C);
    if (C->precision == 64) alloc_loop_data<double>(C); else alloc_loop_data<float>(C);
    // loop workspaces
    C->nb1 = 1024;
    C->nb2 = std::max(1, std::min(grid_for(n), 1024));
    C->d_part1 = dalloc<double>(3LL * C->nb1);
    C->d_part2 = dalloc<double>(2LL * C->nb2);
    C->segpart_len = std::max<long long>(std::max(C->pd.ds.nseg, C->pp.ds.nseg), 1);
    C->d_segpart = dalloc<double>(C->segpart_len);
    C->d_segpart2 = dalloc<double>(C->segpart_len);
    C->d_u = dalloc<double>(std::max<long long>(m, 1));
    C->d_ones = dalloc<unsigned char>(std::max<long long>(m, 1));
    C->d_rec = dalloc<double>(4 + 4LL * C->world);
    if (C->push_dual) {
        C->d_plist[0] = dalloc<int>(n);
        C->d_plist[1] = dalloc<int>(n);
        C->d_pcount = dalloc<unsigned>(2);
        C->d_acc = dalloc<long long>(std::max<long long>(m, 1));
        C->d_pflags = dalloc<unsigned>(8);
        CK(cudaMemsetAsync(C->d_pcount, 0xff, 2 * sizeof(unsigned), s));
        CK(cudaMemsetAsync(C->d_acc, 0, std::max<long long>(m, 1) * sizeof(long long), s));
        CK(cudaMemsetAsync(C->d_pflags, 0, 8 * sizeof(unsigned), s));
    }
    if (C->push_primal) {
        C->d_rlist = dalloc<int>(std::max<long long>(m, 1));
        C->d_rcount = dalloc<unsigned>(1);
        C->d_wmax = dalloc<unsigned long long>(1);
        C->d_accx = dalloc<long long>(n);
        if (C->xskip) {
            C->d_xst = dalloc<unsigned char>(n + 4);
            CK(cudaMemsetAsync(C->d_xst, 0, n + 4, s));
        }
        CK(cudaMemsetAsync(C->d_rcount, 0xff, sizeof(unsigned), s));
        CK(cudaMemsetAsync(C->d_wmax, 0, sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(C->d_accx, 0, n * sizeof(long long), s));
        C->d_accv = dalloc<long long>(std::max<long long>(m, 1));
        C->d_ones_cnt = dalloc<unsigned>(std::max<long long>(m, 1));
        C->d_trig_flag = dalloc<unsigned>(1);
        CK(cudaMemsetAsync(C->d_accv, 0, std::max<long long>(m, 1) * sizeof(long long), s));
        CK(cudaMemsetAsync(C->d_ones_cnt, 0, std::max<long long>(m, 1) * sizeof(unsigned), s));
        CK(cudaMemsetAsync(C->d_trig_flag, 0, sizeof(unsigned), s));
    }
    C->d_regen = dalloc<long long>(2);
    C->d_ctrl = dalloc<Ctrl>(1);
    C->d_hist = dalloc<double>(3 * 1024);
    C->d_xbest = dalloc<unsigned char>(n);
    CK(cudaMemsetAsync(C->d_ctrl, 0, sizeof(Ctrl), s));
    CK(cudaMemsetAsync(C->d_xbest, 0, n, s));
    CK(cudaStreamSynchronize(s));
    C->hk = 0;
    C->have_run = false;
    C->stage = 2;
    if (out) { out->obj_scale = C->omega; out->k_scale = C->kappa; out->zero_rows = C->zero_rows; }
}

// =============================================================================================
// Run (Alg. 1)
// =============================================================================================
static void host_rho_table(const gfors_params* p, long long count, std::vector<double>& rho) {
    // UpdatePenalty (readings R7, R8): rho_t = clip(rho_min(1+t/T)^p, rho_{t-1}+delta, rho_max)
    rho.resize(count);
    double prev = p->rho_min;
    for (long long t = 0; t < count; ++t) {
        const double tilde = p->rho_min * std::pow(1.0 + (double)t / p->growth_T, p->growth_p);
        const double lo = prev + p->rho_delta;
        double v = tilde < lo ? lo : tilde;
        v = v > p->rho_max ? p->rho_max : v;
        rho[t] = v;
        prev = v;
    }
}

static void validate_params(const gfors_params* p) {
    if (!(p->sigma > 0.0 && p->sigma < 1.0)) input_error("params.sigma: must be in (0,1)");
    if (p->k_int < 1) input_error("params.k_int: must be >= 1");
    if (p->k_r < 1) input_error("params.k_r: must be >= 1");
    if (p->k_b < 64 || p->k_b % 64) input_error("params.k_b: must be a positive multiple of 64");
    if (p->k_b / 64 > (1 << 20)) input_error("params.k_b: too large");
    if (p->stall_window < 1 || p->stall_window > 1024) input_error("params.stall_window: must be in [1,1024]");
    if (p->max_iters < 0) input_error("params.max_iters: must be >= 0");
    if (!(p->growth_T > 0.0)) input_error("params.growth_T: must be > 0");
    if (!(p->time_limit_s > 0.0)) input_error("params.time_limit_s: must be > 0");
    if (!(p->rho_min >= 0.0) || !(p->rho_max >= p->rho_min)) input_error("params.rho_min/rho_max: need 0 <= rho_min <= rho_max");
    if (p->trace_cap < 0) input_error("params.trace_cap: must be >= 0");
    if (p->sampler != 0 && p->sampler != 1) input_error("params.sampler: must be 0 (Bernoulli) or 1 (3D assignment)");
}

static bool same_graph_key(const gfors_params& a, const gfors_params& b) {
    return a.sigma == b.sigma && a.k_int == b.k_int && a.k_r == b.k_r && a.k_b == b.k_b && a.tol_primal == b.tol_primal &&
           a.tol_dual == b.tol_dual && a.tol_binary == b.tol_binary && a.stall_rel == b.stall_rel &&
           a.stall_window == b.stall_window && a.seed == b.seed && a.trace_cap == b.trace_cap &&
           a.sampler == b.sampler && a.a3_n == b.a3_n && a.a3_gamma == b.a3_gamma && a.a3_ls == b.a3_ls &&
           a.relax == b.relax && a.repair == b.repair && a.complete == b.complete && a.row_shard == b.row_shard;
}

template <typename T>
static void run_tail_and_final(gfors_ctx* C, long long k_done, long long tail, int W) {
    cudaStream_t s = C->stream;
    for (long long t = 0; t < tail; ++t) enqueue_iter<T>(C, s, 0, k_done + t);
    // x_k parity for the final round: ctrl->k = k_done + tail
    const long long kfinal = k_done + tail;
    CK(cudaMemcpyAsync(&C->d_ctrl->k, &kfinal, sizeof(long long), cudaMemcpyHostToDevice, s));
    // final EvalBest(round(x_k)): one-lane batch
    enqueue_reset(C, s, 1, 1ull);
    LAUNCH(C, s, KC_SAMPLE, (k_round_batch<T><<<grid_for(C->n), NT, 0, s>>>((const T*)C->d_x[0], (const T*)C->d_x[1], C->n,
                                                                           C->d_ctrl, 0, C->d_X)));
    enqueue_eval(C, s, 1);
    LAUNCH(C, s, KC_ARGMIN, (k_argmin<<<1, NT, 0, s>>>(C->d_z, C->d_viol, 1, 0, C->d_ctrl, 0, 0, 1, 1)));
    LAUNCH(C, s, KC_ARGMIN, (k_copy_best<<<grid_for(C->n), NT, 0, s>>>(C->d_X, 1, C->n, C->d_ctrl, C->d_xbest)));
    (void)W;
}

template <typename T>
static void do_run_t(gfors_ctx* C, const gfors_params* p, gfors_run_info* out) {
    cudaStream_t s = C->stream;
    const int W = (int)(p->k_b / 64);
    ensure_batch(C, W);
    set_sampler(C, p->sampler, p->a3_n, p->a3_gamma, p->a3_ls);
    set_relax(C, p->relax, p->repair);
    set_complete(C, p->complete, W);
    set_row_shard(C, p->row_shard, C->precision);
    const long long max_blocks = p->max_iters / p->k_int;
    const long long tail = p->max_iters % p->k_int;
    // rho table (host pow, like the oracle; reading R7)
    const long long nrho = max_blocks + 2;
    std::vector<double> rho;
    host_rho_table(p, nrho, rho);
    if (nrho > C->rho_cap) {
        dfree(C->d_rho);
        C->d_rho = dalloc<double>(nrho);
        C->rho_cap = nrho;
        C->gvalid = false;
    }
    C->nrho = nrho;
    CK(cudaMemcpyAsync(C->d_rho, rho.data(), nrho * sizeof(double), cudaMemcpyHostToDevice, s));
    const int tcap = std::max(1, p->trace_cap);
    if (tcap > C->trace_cap) { dfree(C->d_trace); C->d_trace = dalloc<double>(8LL * tcap); C->trace_cap = tcap; C->gvalid = false; }
    // reset state and control
    const long long l0 = C->launches;
    k_init_state<T><<<grid_for(std::max(C->n, C->m)), NT, 0, s>>>(state_of<T>(C), C->n, C->m);
    CK(cudaGetLastError());
    C->launches++;
    reset_push(C, s);
    Ctrl h{};
    h.blk = 0; h.k = 0; h.rho = rho[0]; h.tau1 = std::sqrt(p->sigma); h.tau2 = std::sqrt(p->sigma);
    h.max_blocks = max_blocks; h.z_best = INFINITY; h.found_iter = h.found_round = h.found_index = -1; h.win_lane = -1;
    CK(cudaMemcpyAsync(C->d_ctrl, &h, sizeof h, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(C->d_xbest, 0, C->n, s));
    CK(cudaMemsetAsync(C->d_hist, 0, 3 * 1024 * sizeof(double), s));
    HaltPar hp{{p->tol_primal, p->tol_dual, p->tol_binary}, p->stall_rel, p->stall_window, p->trace_cap,
               p->k_int, p->k_r, p->k_b * (long long)C->world, C->sharded ? 1 : 0};
    k_loop_start<<<1, 1, 0, s>>>(C->d_ctrl, p->time_limit_s);
    CK(cudaGetLastError());
    C->launches++;

    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    bool used_graph = false;
    if (max_blocks > 0) {
        if (p->use_graph) {
            const bool same = same_graph_key(C->gkey, *p) && C->gkey_W == W;
            if (!(C->gvalid && same) && !(C->gno && same)) {
                if (C->gexec) { cudaGraphExecDestroy(C->gexec); C->gexec = nullptr; }
                if (C->graph) { cudaGraphDestroy(C->graph); C->graph = nullptr; }
                CK(cudaGraphCreate(&C->graph, 0));
                cudaGraphConditionalHandle handle;
                CK(cudaGraphConditionalHandleCreate(&handle, C->graph, 1, cudaGraphCondAssignDefault));
                cudaGraphNodeParams cp = {};
                cp.type = cudaGraphNodeTypeConditional;
                cp.conditional.handle = handle;
                cp.conditional.type = cudaGraphCondTypeWhile;
                cp.conditional.size = 1;
                cudaGraphNode_t node;
                CK(cudaGraphAddNode(&node, C->graph, nullptr, 0, &cp));
                cudaGraph_t body = cp.conditional.phGraph_out[0];
                if (!C->cap_stream) CK(cudaStreamCreateWithFlags(&C->cap_stream, cudaStreamNonBlocking));
                CK(cudaStreamBeginCaptureToGraph(C->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
                bool cap_ok = true;
                const long long c0 = C->launches;
                C->capturing = true;
                try {
                    enqueue_block<T>(C, C->cap_stream, p, W, hp, handle, 1);
                } catch (const Err& e) {
                    cap_ok = false;
                    C->graph_note = "capture failed: " + e.msg;
                }
                C->capturing = false;
                C->dry = false;
                C->gstatic = C->launches - c0;  // unconditional kernels per block (branch kernels: on the device)
                C->launches = c0;
                cudaGraph_t g2;
                const cudaError_t ec = cudaStreamEndCapture(C->cap_stream, &g2);
                if (ec != cudaSuccess) { cap_ok = false; C->graph_note = std::string("end capture: ") + cudaGetErrorString(ec); }
                if (cap_ok) {
                    const cudaError_t ei = cudaGraphInstantiate(&C->gexec, C->graph, 0);
                    if (ei != cudaSuccess) { cap_ok = false; C->graph_note = std::string("instantiate: ") + cudaGetErrorString(ei); }
                }
                cudaGetLastError();
                if (!cap_ok) {
                    // e.g. a collective that cannot live in a conditional body: fall back to the eager loop
                    if (C->gexec) { cudaGraphExecDestroy(C->gexec); C->gexec = nullptr; }
                    if (C->graph) { cudaGraphDestroy(C->graph); C->graph = nullptr; }
                    if (!C->sharded) throw Err{GFORS_E_CUDA, C->graph_note};
                }
                C->gkey = *p;
                C->gkey_W = W;
                C->gvalid = cap_ok;
                C->gno = !cap_ok;
            }
        }
        used_graph = p->use_graph && C->gvalid;
        if (used_graph) {
            CK(cudaGraphLaunch(C->gexec, s));
        } else {
            // eager: one block at a time, host reads the halt flag (debug / fallback path)
            for (long long b = 0; b < max_blocks; ++b) {
                enqueue_block<T>(C, s, p, W, hp, cudaGraphConditionalHandle{}, 0);
                int hf = 0;
                CK(cudaMemcpyAsync(&hf, &C->d_ctrl->halt, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                if (hf) break;
            }
        }
    }
    CK(cudaMemcpyAsync(&h, C->d_ctrl, sizeof h, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (used_graph) C->launches += h.blk * C->gstatic + h.dyn_launches;
    long long k_done = max_blocks > 0 ? h.k : 0;
    int reason = max_blocks > 0 ? h.halt : 2;
    long long tail_run = 0;
    if (reason == 2) tail_run = (max_blocks > 0 ? p->max_iters - k_done : p->max_iters);
    if (reason != 4) run_tail_and_final<T>(C, k_done, tail_run, W);
    CK(cudaEventRecord(e1, s));
    CK(cudaMemcpyAsync(&h, C->d_ctrl, sizeof h, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    gfors_run_info info{};
    info.iters = k_done + tail_run;
    info.rounds = h.rounds;
    info.candidates = h.rounds * p->k_b * (long long)C->world;
    info.halt_reason = reason;
    info.elapsed_s = ms * 1e-3;
    info.n_trace = h.n_trace;
    info.launches = C->launches - l0;
    C->last_info = info;
    C->have_run = true;
    C->hk = info.iters;
    if (out) *out = info;
    C->rs_on = false;  // hooks after the run are unsharded
    if (reason == 4) throw Err{GFORS_E_DIVERGED, "diverged: non-finite indicator at iteration " + std::to_string(h.k)};
}

// =============================================================================================
// C ABI
// =============================================================================================
#define API_BEGIN(C)                                 \
    if (!(C)) return GFORS_E_STATE;                  \
    HookScope hook_scope_((C)->hooks);               \
    try {                                            \
        cudaSetDevice((C)->device);
#define API_END(C)                                   \
    }                                                \
    catch (const Err& e) {                           \
        (C)->err = e.msg;                            \
        return e.st;                                 \
    }                                                \
    catch (const std::exception& e) {                \
        (C)->err = e.what();                         \
        return GFORS_E_CUDA;                         \
    }                                                \
    (C)->err.clear();                                \
    return GFORS_OK;

template <typename T>
static void set_state_t(gfors_ctx* C, const double* x, const double* xbar, const double* y) {
    cudaStream_t s = C->stream;
    double* t = C->d_tmp[3];
    if (x) { CK(cudaMemcpyAsync(t, x, C->n * 8, cudaMemcpyHostToDevice, s)); k_to_T<T><<<grid_for(C->n), NT, 0, s>>>(t, C->n, (T*)C->d_x[0]); CK(cudaStreamSynchronize(s)); }
    if (xbar) { CK(cudaMemcpyAsync(t, xbar, C->n * 8, cudaMemcpyHostToDevice, s)); k_to_T<T><<<grid_for(C->n), NT, 0, s>>>(t, C->n, (T*)C->d_xb[0]); CK(cudaStreamSynchronize(s)); }
    if (y && C->m) { CK(cudaMemcpyAsync(t, y, C->m * 8, cudaMemcpyHostToDevice, s)); k_to_T<T><<<grid_for(C->m), NT, 0, s>>>(t, C->m, (T*)C->d_y[0]); CK(cudaStreamSynchronize(s)); }
    CK(cudaGetLastError());
    reset_push(C, s);
    CK(cudaStreamSynchronize(s));
    C->hk = 0;
}

template <typename T>
static void get_state_t(gfors_ctx* C, double* x, double* xbar, double* y) {
    cudaStream_t s = C->stream;
    const int b = (int)(C->hk & 1);
    double* t = C->d_tmp[3];
    if (x) { k_from_T<T><<<grid_for(C->n), NT, 0, s>>>((T*)C->d_x[b], C->n, t); CK(cudaMemcpyAsync(x, t, C->n * 8, cudaMemcpyDeviceToHost, s)); CK(cudaStreamSynchronize(s)); }
    if (xbar) { k_from_T<T><<<grid_for(C->n), NT, 0, s>>>((T*)C->d_xb[b], C->n, t); CK(cudaMemcpyAsync(xbar, t, C->n * 8, cudaMemcpyDeviceToHost, s)); CK(cudaStreamSynchronize(s)); }
    if (y && C->m) { k_from_T<T><<<grid_for(C->m), NT, 0, s>>>((T*)C->d_y[b], C->m, t); CK(cudaMemcpyAsync(y, t, C->m * 8, cudaMemcpyDeviceToHost, s)); CK(cudaStreamSynchronize(s)); }
    CK(cudaGetLastError());
}

extern "C" {

void gfors_params_default(gfors_params* p) {
    // SPEC L293, L667 defaults; k_b = 128 per rank
    memset(p, 0, sizeof *p);
    p->sigma = 0.99; p->k_int = 10; p->k_r = 1; p->k_b = 128;
    p->rho_min = 1e-3; p->rho_max = 10.0; p->growth_T = 100.0; p->growth_p = 2.0; p->rho_delta = 1e-6;
    p->tol_primal = 1e-6; p->tol_dual = 1e-6; p->tol_binary = 1e-6; p->stall_rel = 1e-8; p->stall_window = 50;
    p->max_iters = 100000; p->time_limit_s = 1800.0; p->seed = 20251030ull; p->use_graph = 1; p->trace_cap = 4096;
    p->sampler = 0; p->a3_ls = -1; p->a3_n = 0; p->a3_gamma = 4.0;
    p->relax = 0; p->repair = 0; p->complete = 0;
}

void gfors_prep_opts_default(gfors_prep_opts* p) {
    p->tol = 1e-7; p->max_iter = 500; p->precision = 64;
}

gfors_status gfors_create(gfors_ctx** out, const gfors_device_opts* opts) {
    if (!out) return GFORS_E_INPUT;
    *out = nullptr;
    auto* C = new gfors_ctx();
    try {
        if (opts) { C->device = opts->device; C->rank = opts->rank; C->world = opts->world; }
        if (opts && (!!opts->alloc != !!opts->free)) input_error("device_opts: alloc and free go together");
        if (opts && opts->alloc) C->hooks = AllocHooks{opts->alloc, opts->free, opts->alloc_ctx};
        HookScope hs(C->hooks);
        if (C->world < 1 || C->rank < 0 || C->rank >= C->world) input_error("device_opts: need 0 <= rank < world");
        if (opts && opts->loopback) {
            if (opts->nccl_id || C->rank != 0) input_error("device_opts.loopback: needs rank = 0 and nccl_id = NULL");
            C->loopback = true;
            C->sharded = true;  // the exchange protocol (record, merge, regeneration, halt flags) without NCCL
        }
        // nccl_id == NULL with world > 1: independent sample shard (rank r draws global words
        // [r*W, (r+1)*W)); the caller merges incumbents with gfors_merge_records.  nccl_id != NULL:
        // in-loop record exchange over NCCL every sampling round (shard.cuh).
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (C->device < 0 || C->device >= ndev) input_error("device_opts.device: %d not in [0,%d)", C->device, ndev);
        CK(cudaSetDevice(C->device));
        CK(cudaDeviceGetAttribute(&C->num_sms, cudaDevAttrMultiProcessorCount, C->device));
        live_contexts(C->device, +1);
        C->counted = true;
        if (opts && opts->nccl_id) {
            NcclApi& api = nccl();
            if (!api.ok) throw Err{GFORS_E_NCCL, api.why};
            ncclUniqueId id;
            memcpy(&id, opts->nccl_id, sizeof id);
            const int rc = api.CommInitRank(&C->comm, C->world, id, C->rank);
            if (rc != 0) throw Err{GFORS_E_NCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(rc)};
            C->sharded = true;
        }
        if (opts && opts->stream) {
            C->stream = (cudaStream_t)opts->stream;
        } else {
            CK(cudaStreamCreateWithFlags(&C->stream, cudaStreamNonBlocking));
            C->own_stream = true;
        }
    } catch (const Err& e) {
        gfors_status st = e.st;
        delete C;
        return st;
    }
    *out = C;
    return GFORS_OK;
}

gfors_status gfors_set_option(gfors_ctx* C, const char* key, int64_t value) {
    API_BEGIN(C)
    if (!key) input_error("gfors_set_option: key is NULL");
    const std::string k(key);
    if (k == "force_deadline_rank") C->opt.force_deadline_rank = value;
    else if (k == "force_deadline_block") C->opt.force_deadline_block = value;
    else if (k == "force_capture_fail") C->opt.force_capture_fail = value;
    else if (k == "dense_q") C->opt.dense_q = value;
    else if (k == "dense_k") C->opt.dense_k = value;
    else if (k == "qx_fix") C->opt.qx_fix = value;
    else if (k == "qx_reuse") C->opt.qx_reuse = value;
    else if (k == "push_dual") C->opt.push_dual = value;
    else if (k == "push_primal") C->opt.push_primal = value;
    else if (k == "delta_dual") C->opt.delta_dual = value;
    else if (k == "xskip") C->opt.xskip = value;
    else if (k == "cond_branch") C->opt.cond_branch = value;
    else if (k == "sparse_primal") C->opt.sparse_primal = value;
    else if (k == "obj_bits") C->opt.obj_bits = value;
    else if (k == "load_timing") C->opt.load_timing = value;
    else if (k == "obj_list") C->opt.obj_list = value;
    else input_error("gfors_set_option: unknown key '%s'", key);
    C->gvalid = false;
    C->gno = false;
    API_END(C)
}

gfors_status gfors_load(gfors_ctx* C, const gfors_problem* prob) {
    API_BEGIN(C)
    C->tu = gfors_ctx::TuLift{};
    do_load(C, prob);
    API_END(C)
}

gfors_status gfors_tu_reformulate(gfors_ctx* C, const int64_t* rows_J, const int32_t* cols_I, int64_t count) {
    API_BEGIN(C)
    do_tu_reformulate(C, rows_J, cols_I, count);
    API_END(C)
}

gfors_status gfors_dims(gfors_ctx* C, int64_t* n, int64_t* m, int64_t* n_orig) {
    API_BEGIN(C)
    if (C->stage < 1) throw Err{GFORS_E_STATE, "gfors_dims: call gfors_load first"};
    if (n) *n = C->n;
    if (m) *m = C->m;
    if (n_orig) *n_orig = C->tu.active ? C->tu.n_orig : C->n;
    API_END(C)
}

gfors_status gfors_preprocess(gfors_ctx* C, const gfors_prep_opts* o, gfors_scaling* out) {
    API_BEGIN(C)
    do_preprocess(C, o, out);
    API_END(C)
}

gfors_status gfors_run(gfors_ctx* C, const gfors_params* p, gfors_run_info* out) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_run: call gfors_preprocess first"};
    gfors_params d;
    gfors_params_default(&d);
    if (!p) p = &d;
    validate_params(p);
    if (C->precision == 64) do_run_t<double>(C, p, out); else do_run_t<float>(C, p, out);
    API_END(C)
}

gfors_status gfors_best_incumbent(gfors_ctx* C, double* z, uint8_t* x, gfors_incumbent_info* info) {
    if (!C) return GFORS_E_STATE;
    try {
        cudaSetDevice(C->device);
        if (!C->have_run) throw Err{GFORS_E_STATE, "gfors_best_incumbent: call gfors_run first"};
        Ctrl h;
        CK(cudaMemcpyAsync(&h, C->d_ctrl, sizeof h, cudaMemcpyDeviceToHost, C->stream));
        std::vector<uint8_t> xr;
        if (x && C->tu.active) xr.resize(C->n);
        if (x) CK(cudaMemcpyAsync(C->tu.active ? xr.data() : x, C->d_xbest, C->n, cudaMemcpyDeviceToHost, C->stream));
        CK(cudaStreamSynchronize(C->stream));
        if (x && C->tu.active) tu_lift(C, xr.data(), x);  // x_I = s + S x_Ibar
        const bool maxi = C->tu.active ? C->tu.maximize : C->maximize;
        const double zz = h.has_inc ? (maxi ? -h.z_best : h.z_best) : INFINITY;
        if (z) *z = zz;
        if (info) {
            info->found_iter = h.found_iter; info->found_round = h.found_round; info->found_index = h.found_index;
            info->found_time_s = h.found_ns * 1e-9; info->has_incumbent = h.has_inc;
        }
        C->err.clear();
        return h.has_inc ? GFORS_OK : GFORS_NO_INCUMBENT;
    } catch (const Err& e) {
        C->err = e.msg;
        return e.st;
    }
}

const char* gfors_last_error(const gfors_ctx* C) { return C ? C->err.c_str() : "null context"; }

gfors_status gfors_release_memory(int32_t device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return GFORS_E_INPUT;
    if (cudaSetDevice(device) != cudaSuccess) return GFORS_E_CUDA;
    if (live_contexts(device, 0) > 0) return GFORS_E_STATE;
    cudaStream_t as = alloc_stream();
    if (as) cudaStreamSynchronize(as);
    pool_release(device);
    return GFORS_OK;
}

void gfors_destroy(gfors_ctx* C) {
    if (!C) return;
    HookScope hs(C->hooks);  // the context's buffers go back to the allocator they came from
    delete C;
}

gfors_status gfors_get_scaled(gfors_ctx* C, double* row_scale, double* r_scaled, double* c_scaled) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_get_scaled: call gfors_preprocess first"};
    std::vector<double> s(C->m);
    if (C->m) CK(cudaMemcpy(s.data(), C->d_s, C->m * sizeof(double), cudaMemcpyDeviceToHost));
    if (row_scale) memcpy(row_scale, s.data(), C->m * sizeof(double));
    if (r_scaled)
        for (long long j = 0; j < C->m; ++j) r_scaled[j] = (C->ru[j] / s[j]) / C->kappa;
    if (c_scaled)
        for (long long i = 0; i < C->n; ++i) c_scaled[i] = C->c[i] / C->omega;
    API_END(C)
}

gfors_status gfors_sample(gfors_ctx* C, const double* p, uint64_t seed, uint32_t round_id, int64_t word_begin,
                          int64_t n_words, uint64_t* bits) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_sample: call gfors_preprocess first"};
    if (!p || !bits) input_error("gfors_sample: p and bits required");
    if (n_words < 1 || n_words > (1 << 20)) input_error("gfors_sample: n_words out of range");
    if (word_begin < 0 || word_begin + n_words > (1LL << 32)) input_error("gfors_sample: word range exceeds 2^32");
    for (long long i = 0; i < C->n; ++i)
        if (!(p[i] >= 0.0 && p[i] <= 1.0)) input_error("gfors_sample: p[%lld] not in [0,1]", i);
    ensure_batch(C, (int)n_words);
    set_sampler(C, 0, 0, 0.0, 0);
    cudaStream_t s = C->stream;
    double* dp = C->d_tmp[3];
    CK(cudaMemcpyAsync(dp, p, C->n * sizeof(double), cudaMemcpyHostToDevice, s));
    if (C->precision == 64)
        enqueue_sample<double>(C, s, dp, (int)n_words, word_begin, seed, 1, 0, 1, round_id, 1);
    else
        enqueue_sample<float>(C, s, dp, (int)n_words, word_begin, seed, 1, 0, 1, round_id, 1);
    CK(cudaMemcpyAsync(bits, C->d_X, C->n * n_words * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    API_END(C)
}

gfors_status gfors_sample_assign3d(gfors_ctx* C, const double* p, uint64_t seed, uint32_t round_id, int64_t word_begin,
                                   int64_t n_words, int64_t a3_n, double a3_gamma, int64_t a3_ls, uint64_t* bits) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_sample_assign3d: call gfors_preprocess first"};
    if (!p || !bits) input_error("gfors_sample_assign3d: p and bits required");
    if (n_words < 1 || n_words > (1 << 14)) input_error("gfors_sample_assign3d: n_words out of range");
    if (word_begin < 0 || 64 * (word_begin + n_words) > (1LL << 32)) input_error("gfors_sample_assign3d: lane range exceeds 2^32");
    ensure_batch(C, (int)n_words);
    set_sampler(C, 1, a3_n, a3_gamma, a3_ls);
    cudaStream_t s = C->stream;
    double* dp = C->d_tmp[3];
    CK(cudaMemcpyAsync(dp, p, C->n * sizeof(double), cudaMemcpyHostToDevice, s));
    if (C->precision == 64)
        enqueue_sample<double>(C, s, dp, (int)n_words, word_begin, seed, 1, 0, 1, round_id, 1);
    else
        enqueue_sample<float>(C, s, dp, (int)n_words, word_begin, seed, 1, 0, 1, round_id, 1);
    CK(cudaMemcpyAsync(bits, C->d_X, C->n * n_words * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    C->a3.sampler = 0;
    API_END(C)
}

gfors_status gfors_set_relax(gfors_ctx* C, int32_t relax) {
    API_BEGIN(C)
    if (C->stage < 1) throw Err{GFORS_E_STATE, "gfors_set_relax: call gfors_load first"};
    set_relax(C, relax, 0);
    API_END(C)
}

gfors_status gfors_repair(gfors_ctx* C, uint64_t* bits, int64_t n_words) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_repair: call gfors_preprocess first"};
    if (!bits || n_words < 1 || n_words > (1 << 14)) input_error("gfors_repair: bits and 1 <= n_words <= 16384 required");
    const long long keep_m1p = C->m1p;
    set_relax(C, 1, 1);
    C->m1p = keep_m1p;  // the hook does not change the PDHG senses
    ensure_batch(C, (int)n_words);
    cudaStream_t s = C->stream;
    CK(cudaMemcpyAsync(C->d_X, bits, C->n * n_words * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    enqueue_repair(C, s, (int)n_words);
    CK(cudaMemcpyAsync(bits, C->d_X, C->n * n_words * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    C->repair = false;
    API_END(C)
}

gfors_status gfors_cover_complete(gfors_ctx* C, const double* p, uint64_t* bits, int64_t n_words) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_cover_complete: call gfors_preprocess first"};
    if (!p || !bits || n_words < 1 || n_words > (1 << 14)) input_error("gfors_cover_complete: p, bits and 1 <= n_words <= 16384 required");
    ensure_batch(C, (int)n_words);
    set_complete(C, 1, (int)n_words);
    cudaStream_t s = C->stream;
    double* dp = C->d_tmp[3];
    CK(cudaMemcpyAsync(dp, p, C->n * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(C->d_X, bits, C->n * n_words * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    if (C->precision == 64) enqueue_cover<double>(C, s, dp, (int)n_words, 1); else enqueue_cover<float>(C, s, dp, (int)n_words, 1);
    CK(cudaMemcpyAsync(bits, C->d_X, C->n * n_words * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    C->complete = false;
    API_END(C)
}

gfors_status gfors_eval(gfors_ctx* C, const uint64_t* bits, int64_t n_words, uint8_t* feasible, double* z) {
    API_BEGIN(C)
    if (C->stage < 1) throw Err{GFORS_E_STATE, "gfors_eval: call gfors_load first"};
    if (!bits) input_error("gfors_eval: bits required");
    if (n_words < 1 || n_words > (1 << 20)) input_error("gfors_eval: n_words out of range");
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_eval: call gfors_preprocess first"};
    const int W = (int)n_words;
    ensure_batch(C, W);
    cudaStream_t s = C->stream;
    CK(cudaMemcpyAsync(C->d_X, bits, C->n * n_words * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    enqueue_reset(C, s, W, ~0ull);
    enqueue_eval(C, s, W);
    std::vector<unsigned long long> viol(W);
    std::vector<double> zz(64LL * W);
    CK(cudaMemcpyAsync(viol.data(), C->d_viol, W * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(zz.data(), C->d_z, 64LL * W * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (long long l = 0; l < 64LL * W; ++l) {
        if (feasible) feasible[l] = (uint8_t)(((viol[l >> 6] >> (l & 63)) & 1ull) ? 0 : 1);
        if (z) z[l] = zz[l];
    }
    API_END(C)
}

gfors_status gfors_sample_eval_timed(gfors_ctx* C, const double* p, uint64_t seed, int64_t n_words, int32_t rounds,
                                     double* ms_out) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_sample_eval_timed: call gfors_preprocess first"};
    if (!p || !ms_out || rounds < 1) input_error("gfors_sample_eval_timed: p, ms_out and rounds >= 1 required");
    if (n_words < 1 || n_words > (1 << 14)) input_error("gfors_sample_eval_timed: n_words out of range");
    for (long long i = 0; i < C->n; ++i)
        if (!(p[i] >= 0.0 && p[i] <= 1.0)) input_error("gfors_sample_eval_timed: p[%lld] not in [0,1]", i);
    const int W = (int)n_words;
    ensure_batch(C, W);
    set_sampler(C, 0, 0, 0.0, 0);
    cudaStream_t s = C->stream;
    double* dp = C->d_tmp[3];
    CK(cudaMemcpyAsync(dp, p, C->n * sizeof(double), cudaMemcpyHostToDevice, s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    for (int r = 0; r < rounds; ++r) {  // RandSampleStep + EvalBest + argmin (hook mode: no incumbent update)
        if (C->precision == 64) enqueue_sample<double>(C, s, dp, W, 0, seed, 1, 0, 1, (unsigned)r, 1);
        else enqueue_sample<float>(C, s, dp, W, 0, seed, 1, 0, 1, (unsigned)r, 1);
        enqueue_reset(C, s, W, ~0ull);
        enqueue_eval(C, s, W, nullptr, C->a3.sampler != 1);
        LAUNCH(C, s, KC_ARGMIN, (k_argmin<<<1, NT, 0, s>>>(C->d_z, C->d_viol, 64LL * W, 0, C->d_ctrl, 0, 0, 1, 2)));
    }
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = ms;
    API_END(C)
}

gfors_status gfors_set_state(gfors_ctx* C, const double* x, const double* xbar, const double* y) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_set_state: call gfors_preprocess first"};
    if (C->precision == 64) set_state_t<double>(C, x, xbar, y); else set_state_t<float>(C, x, xbar, y);
    API_END(C)
}

gfors_status gfors_get_state(gfors_ctx* C, double* x, double* xbar, double* y) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_get_state: call gfors_preprocess first"};
    if (C->precision == 64) get_state_t<double>(C, x, xbar, y); else get_state_t<float>(C, x, xbar, y);
    API_END(C)
}

gfors_status gfors_step(gfors_ctx* C, int64_t iters, double rho, double tau1, double tau2) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_step: call gfors_preprocess first"};
    if (iters < 0) input_error("gfors_step: iters must be >= 0");
    cudaStream_t s = C->stream;
    Ctrl h{};
    h.rho = rho; h.tau1 = tau1; h.tau2 = tau2;
    CK(cudaMemcpyAsync(C->d_ctrl, &h, sizeof h, cudaMemcpyHostToDevice, s));
    for (long long t = 0; t < iters; ++t) {
        if (C->precision == 64) enqueue_iter<double>(C, s, 0, C->hk); else enqueue_iter<float>(C, s, 0, C->hk);
        C->hk++;
    }
    CK(cudaStreamSynchronize(s));
    API_END(C)
}

gfors_status gfors_indicators(gfors_ctx* C, double rho, double tau1, double tau2, double* out) {
    API_BEGIN(C)
    if (C->stage < 2 || C->hk < 1) throw Err{GFORS_E_STATE, "gfors_indicators: take a gfors_step first"};
    cudaStream_t s = C->stream;
    Ctrl h{};
    h.rho = rho; h.tau1 = tau1; h.tau2 = tau2;
    CK(cudaMemcpyAsync(C->d_ctrl, &h, sizeof h, cudaMemcpyHostToDevice, s));
    if (C->precision == 64) enqueue_trigger<double>(C, s, 0, C->hk - 1); else enqueue_trigger<float>(C, s, 0, C->hk - 1);
    double* o4 = C->d_tmp[3];
    k_indicators_only<<<1, NT, 0, s>>>(C->d_part1, C->nb1, C->d_part2, C->nb2, C->n, o4);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, o4, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    API_END(C)
}

gfors_status gfors_get_trace(gfors_ctx* C, double* rows, int64_t max_rows, int64_t* n_rows) {
    API_BEGIN(C)
    if (!C->have_run) throw Err{GFORS_E_STATE, "gfors_get_trace: call gfors_run first"};
    const long long total = C->last_info.n_trace;
    const long long cap = C->trace_cap;
    const long long avail = std::min(total, cap);
    const long long k = std::min<long long>(avail, max_rows);
    std::vector<double> all(8 * cap);
    CK(cudaMemcpy(all.data(), C->d_trace, 8 * cap * sizeof(double), cudaMemcpyDeviceToHost));
    const long long first = total - avail;  // oldest kept row index
    for (long long r = 0; r < k; ++r) {
        const long long src = (first + r) % cap;
        memcpy(rows + 8 * r, all.data() + 8 * src, 8 * sizeof(double));
    }
    if (n_rows) *n_rows = k;
    API_END(C)
}

const char* gfors_kernel_class_name(int32_t k) { return (k >= 0 && k < KC_N) ? kClassNames[k] : ""; }

gfors_status gfors_profile_active(gfors_ctx* C, double* active_ms, double* active_launches, int32_t max_classes) {
    if (!C) return GFORS_E_STATE;
    if (C->prof_active_ms.empty()) return GFORS_E_STATE;
    for (int k = 0; k < std::min<int>(KC_N, max_classes); ++k) {
        active_ms[k] = C->prof_active_ms[k];
        active_launches[k] = C->prof_active_n[k];
    }
    return GFORS_OK;
}

int64_t gfors_launches_per_block(gfors_ctx* C, const gfors_params* p) {
    if (!C || C->stage < 2) return -1;
    // eager structure of one block, counted by a dry enqueue (LAUNCH counts, launches nothing)
    gfors_params d;
    gfors_params_default(&d);
    if (!p) p = &d;
    const int W = (int)(p->k_b / 64);
    HaltPar hp{{p->tol_primal, p->tol_dual, p->tol_binary}, p->stall_rel, p->stall_window, p->trace_cap,
               p->k_int, p->k_r, p->k_b * (long long)C->world, C->sharded ? 1 : 0};
    const long long before = C->launches;
    C->launches = 0;
    C->dry = true;
    long long n = -1;
    try {
        set_sampler(C, p->sampler, p->a3_n, p->a3_gamma, p->a3_ls);
        set_relax(C, p->relax, p->repair);
        set_complete(C, p->complete, W);
        set_row_shard(C, p->row_shard, C->precision);
        if (C->precision == 64) enqueue_block<double>(C, C->stream, p, W, hp, cudaGraphConditionalHandle{}, 0);
        else enqueue_block<float>(C, C->stream, p, W, hp, cudaGraphConditionalHandle{}, 0);
        n = C->launches;
    } catch (...) {
    }
    C->rs_on = false;
    C->dry = false;
    C->launches = before;
    return n;
}

gfors_status gfors_profile_blocks(gfors_ctx* C, const gfors_params* p, int32_t blocks, double* ms_out,
                                  int32_t max_classes, int32_t* n_classes) {
    API_BEGIN(C)
    if (C->stage < 2) throw Err{GFORS_E_STATE, "gfors_profile_blocks: call gfors_preprocess first"};
    gfors_params d;
    gfors_params_default(&d);
    if (!p) p = &d;
    validate_params(p);
    if (blocks < 1) input_error("gfors_profile_blocks: blocks must be >= 1");
    // a normal run with max_iters = blocks*k_int in eager mode, events around every launch
    gfors_params q = *p;
    q.max_iters = (long long)blocks * p->k_int;
    q.use_graph = 0;
    q.tol_primal = q.tol_dual = q.tol_binary = -1.0;  // never halt on criteria
    q.stall_rel = -1.0;
    C->profiling = true;
    C->prof_ev.clear();
    try {
        if (C->precision == 64) do_run_t<double>(C, &q, nullptr); else do_run_t<float>(C, &q, nullptr);
    } catch (...) {
        C->profiling = false;
        throw;
    }
    C->profiling = false;
    CK(cudaStreamSynchronize(C->stream));
    std::vector<double> sum(KC_N, 0.0);
    C->prof_active_ms.assign(KC_N, 0.0);
    C->prof_active_n.assign(KC_N, 0.0);
    for (auto& e : C->prof_ev) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
        sum[e.first] += ms;
        if (ms > 0.010f) { C->prof_active_ms[e.first] += ms; C->prof_active_n[e.first] += 1.0; }  // > 10 us: did work
        cudaEventDestroy(e.second.first);
        cudaEventDestroy(e.second.second);
    }
    C->prof_ev.clear();
    const int nc = std::min<int>(KC_N, max_classes);
    for (int k = 0; k < nc; ++k) ms_out[k] = sum[k] / blocks;  // per block
    if (n_classes) *n_classes = nc;
    API_END(C)
}

gfors_status gfors_nccl_unique_id(void* out128) {
    if (!out128) return GFORS_E_INPUT;
    NcclApi& api = nccl();
    if (!api.ok) return GFORS_E_NCCL;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != 0) return GFORS_E_NCCL;
    memcpy(out128, &id, sizeof id);
    return GFORS_OK;
}

const char* gfors_graph_note(const gfors_ctx* C) { return C ? C->graph_note.c_str() : ""; }

int32_t gfors_merge_records(const double* z, const int64_t* index, const int32_t* valid, int32_t world) {
    // lowest z among valid records, ties -> lowest global sample index (reading R11)
    int32_t best = -1;
    for (int32_t r = 0; r < world; ++r) {
        if (!valid[r]) continue;
        if (best < 0 || z[r] < z[best] || (z[r] == z[best] && index[r] < index[best])) best = r;
    }
    return best;
}

}  // extern "C"
