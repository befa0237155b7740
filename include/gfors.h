/*
 * gfors.h — C ABI of the B200-native GFORS hot path (arXiv 2510.27117).
 *
 * GFORS solves the binary integer program (eq. bip)
 *
 *     min  x'Qx + c'x + c0   s.t.  K x >= r (GE rows) | K x = r (EQ) | K x <= r (LE),  x in {0,1}^n
 *
 * with Alg. 1: Preprocess, then a device loop of UpdatePenalty ->
 * FirstOrderStep (Alg. 2, PDHG on the rho-penalised saddle form)
 * -> every k_int iterations k_r rounds of RandSampleStep (Alg. 3) + EvalBest
 * -> CheckHalt; finally EvalBest(round(x_k)).
 * Everything after gfors_load runs in this library's sm_100a kernels.  No CPU fallback.
 *
 * Call order: gfors_create -> gfors_load -> gfors_preprocess -> gfors_run* ->
 * gfors_best_incumbent -> gfors_destroy.  Any other order returns GFORS_E_STATE.
 * All functions return a gfors_status; no C++ exception crosses this boundary.  On error
 * gfors_last_error() returns a message naming the offending argument/field/index.
 * Threading: one context per (process, GPU); a context must not be used concurrently.
 * Ownership: the library copies every input at the call and retains no caller pointer; the
 * caller owns every output buffer it passes.  Host pointers are plain host memory (pinned or
 * pageable); device pointers are CUDA device memory of the context's device.
 */
#ifndef GFORS_H
#define GFORS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GFORS_OK = 0,
    GFORS_NO_INCUMBENT = 2, /* SPEC L674 exit 2: run finished, no feasible sample found */
    GFORS_E_INPUT = 3,      /* SPEC L674 exit 3: invalid argument / instance */
    GFORS_E_DIVERGED = 4,   /* SPEC L674 exit 4: non-finite indicator (NaN guard) */
    GFORS_E_CUDA = 5,       /* CUDA runtime error (message has the CUDA error string) */
    GFORS_E_NCCL = 6,       /* NCCL unavailable or failed (world > 1) */
    GFORS_E_STATE = 7,      /* wrong call order */
    GFORS_E_OOM = 8         /* device allocation failed */
} gfors_status;

typedef struct gfors_ctx gfors_ctx;

/* Device/rank options.  stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)
 * or NULL for a library-owned stream.  rank/world: sample-sharded data parallelism
 * (DESIGN.md §7): rank r draws global sample words [r*W, (r+1)*W).  nccl_id: 128-byte
 * ncclUniqueId (identical on all ranks, see gfors_nccl_unique_id) for the in-loop incumbent exchange,
 * or NULL: independent shards whose incumbents the caller merges (gfors_merge_records). */
typedef struct {
    int32_t device;
    void *stream;
    int32_t rank, world;
    const void *nccl_id;
    /* loopback != 0 (test mode, needs rank = 0 and nccl_id = NULL): this one context runs all `world`
     * ranks of the exchange one after another on its stream — rank q's words [q*W, (q+1)*W), its
     * record written straight into the gathered slots — then the same merge, winner regeneration and
     * halt agreement as the NCCL path; the result equals one rank with k_b*world. */
    int32_t loopback;
    /* Optional device allocator, e.g. torch's caching allocator: alloc(bytes, alloc_ctx)
     * returns device memory of `device` usable on `stream` (NULL = out of memory -> GFORS_E_OOM), free(p,
     * alloc_ctx) takes back what alloc returned.  Every device buffer of this context then comes from it,
     * allocated and freed inside this context's API calls (gfors_destroy included).  NULL: the library's
     * private stream-ordered pool. */
    void *(*alloc)(size_t bytes, void *alloc_ctx);
    void (*free)(void *p, void *alloc_ctx);
    void *alloc_ctx;
} gfors_device_opts;

/* Problem in USER form.  CSR K (m x n): k_rowptr[m+1] (nondecreasing, [0]=0),
 * k_col[nnz] (strictly increasing within a row, in [0,n)), k_val[nnz] (finite, nonzero);
 * r[m]; sense[m] in {+1 GE, 0 EQ, -1 LE}.  Q (n x n, symmetric, full storage; q_rowptr NULL
 * means Q = 0); c[n]; c0; maximize != 0 maximises.  mem_space: 0 host pointers, 1 device
 * pointers.  Requirements: 0 < n < 2^31, nnz(K), nnz(Q) < 2^31. */
typedef struct {
    int64_t n, m;
    int32_t mem_space;
    const int64_t *k_rowptr;
    const int32_t *k_col;
    const double *k_val;
    const double *r;
    const int8_t *sense;
    const int64_t *q_rowptr;
    const int32_t *q_col;
    const double *q_val;
    const double *c;
    double c0;
    int32_t maximize;
} gfors_problem;

/* Preprocess options.  precision: 64 -> fp64 iterates,
 * 32 -> fp32 iterates (sums accumulate in fp64 either way; Preprocess is always fp64). */
typedef struct {
    double tol;        /* power-iteration relative-change tolerance, default 1e-7 */
    int32_t max_iter;  /* power-iteration sweeps, default 500 */
    int32_t precision; /* 64 (default) or 32 */
} gfors_prep_opts;

/* Scaling record: obj_scale = ||Q||_2 + ||c||_2 (1 if 0), k_scale = ||D^-1 K||_2
 * (1 if 0), zero_rows = rows of K with no nonzero (kept with row scale 1). */
typedef struct {
    double obj_scale, k_scale;
    int64_t zero_rows;
} gfors_scaling;

/* Alg. 1 parameters (SPEC L293, L632-635, L667 defaults via gfors_params_default). */
typedef struct {
    double sigma;                 /* tau1 = tau2 = sqrt(sigma), 0 < sigma < 1 */
    int32_t k_int, k_r;           /* sampling interval, rounds per trigger */
    int64_t k_b;                  /* samples per round PER RANK, multiple of 64 */
    double rho_min, rho_max, growth_T, growth_p, rho_delta; /* UpdatePenalty */
    double tol_primal, tol_dual, tol_binary, stall_rel;     /* CheckHalt */
    int32_t stall_window;         /* W checks, 1..1024 */
    int64_t max_iters;
    double time_limit_s;
    uint64_t seed;                /* Philox key */
    int32_t use_graph;            /* 1: CUDA graph with a device WHILE node (default); 0: eager */
    int32_t trace_cap;            /* trace ring-buffer rows (default 4096) */
    /* RandSampleStep: 0 = Bernoulli(x_k) (Alg. 3, default); 1 = customised 3D-assignment sampler
     * (Alg. 4; R25): variables must be the a3_n^3
     * triples (i,j,k) at flat index i*a3_n^2 + j*a3_n + k (a3_n <= 4096); every candidate is a
     * feasible 3D assignment built from the ceil(a3_gamma*a3_n) largest x_k, a random completion
     * and a3_ls pairwise interchanges (-1: 2*a3_n; SPEC L381 defaults gamma 4, L 2n). */
    int32_t sampler;
    int32_t a3_ls;
    int64_t a3_n;
    double a3_gamma;
    /* Monotone relaxation (R26): relax = 1 needs Q = 0,
     * canonical c >= 0 and K_u >= 0; the PDHG step and indicators then treat every row as >= (upper
     * closure) while EvalBest keeps the original equalities.  repair = 1 (needs relax, integral
     * data, world == 1) drops each lane's 1-entries in decreasing-cost order (ties: lower index)
     * while all rows stay >= before EvalBest; every lane is repaired, whatever its size. */
    int32_t relax;
    int32_t repair;
    /* complete = 1: cover completion before EvalBest (R27): every covering
     * row (>=, coefficients 1, rhs 1) a lane violates gets its largest-x_k variable (ties: lowest
     * index) switched on in that lane; decisions on the batch as sampled (order-free).  One rank
 * (repair, complete and sampler 1 are rejected with the NCCL-sharded loop: its winner regeneration
 * replays the Bernoulli contract). */
    int32_t complete;
    /* row_shard = 1 (needs world > 1 — NCCL or loopback — and the row-block dual): the PDHG dual is
     * row-sharded (north_star "row-sharded for K"): rank r computes the dual of its
     * nnz-balanced range of row blocks only, then the ranks all-gather y (and, at the trigger
     * iteration, K_u xbar) — m values instead of the n-vector K'y — and every rank recomputes w and
     * runs the rest of the iteration replicated, so iterates and decisions stay bit-identical to the
     * unsharded run. */
    int32_t row_shard;
} gfors_params;

/* halt_reason: 1 criteria met, 2 max_iters, 3 time limit, 4 diverged. */
typedef struct {
    int64_t iters, rounds, candidates;
    int32_t halt_reason;
    double elapsed_s;   /* device time of the loop (CUDA events), Preprocess excluded */
    int64_t n_trace;    /* trace rows written (ring keeps the last trace_cap) */
    int64_t launches;   /* kernels this call launched (graph mode: unconditional nodes per block x blocks
                           + the kernels of the conditional branches taken, counted on the device) */
} gfors_run_info;

typedef struct {
    int64_t found_iter, found_round, found_index; /* round/index -1: final round(x_k) */
    double found_time_s;                          /* %globaltimer since loop start */
    int32_t has_incumbent;
} gfors_incumbent_info;

void gfors_params_default(gfors_params *p);
void gfors_prep_opts_default(gfors_prep_opts *p);

gfors_status gfors_create(gfors_ctx **out, const gfors_device_opts *opts);
/* Validates (CSR invariants, finiteness, Q symmetry, sense) and canonicalises (maximise ->
 * negate; LE -> GE by negation; rows stably permuted GE first), builds the device
 * layouts (CSR K, CSR K', CSR Q) and classifies rows for the evaluator.  Copies inputs. */
gfors_status gfors_load(gfors_ctx *ctx, const gfors_problem *prob);
/* TUReformulate (PAPER §2.4.1, Theorem L823-846; Alg. 1), optional,
 * between gfors_load and gfors_preprocess.  rows_J[count]: INPUT row indices (as passed to
 * gfors_load) of equality rows; cols_I[count]: columns (no pairing between J[t] and I[t] needed);
 * B_J must be TU with B_J, d_J integral and B_JI invertible (any such B_JI: signed permutation,
 * triangular, ...).  S is formed by an exact sparse Gauss-Jordan elimination of the J rows with +-1
 * pivots (the paper applies an LU of B_JI instead, L848-850); a singular B_JI or a non-TU B_J (an
 * entry outside {-1,0,1} appears) returns GFORS_E_INPUT.  Eliminates
 * x_I = s + S x_Ibar (s = B_JI^-1 d_J, S = -B_JI^-1 B_J,Ibar) exactly by substitution into Q, c, c0
 * and the other rows, adds the box rows S x >= -s, -S x >= s - 1 (those every binary x satisfies
 * are dropped) and loads the reduced problem in place (reduced variables = Ibar ascending; rows =
 * the non-J input rows in input order, then the box rows; reading R24).  Afterwards
 * gfors_sample/gfors_eval/state hooks work on the reduced variables (gfors_dims), while
 * gfors_best_incumbent returns z in the original sense and x lifted to the ORIGINAL n variables.
 * Host only; copies; errors name the offending row/column. */
gfors_status gfors_tu_reformulate(gfors_ctx *ctx, const int64_t *rows_J, const int32_t *cols_I, int64_t count);
/* Test hook: one Alg. 4 batch (sampler 1) of n_words*64 candidates from the fixed p (n entries,
 * host), Philox key seed, round id, lanes 64*word_begin ...; bits as gfors_sample. */
gfors_status gfors_sample_assign3d(gfors_ctx *ctx, const double *p, uint64_t seed, uint32_t round_id,
                                   int64_t word_begin, int64_t n_words, int64_t a3_n, double a3_gamma,
                                   int64_t a3_ls, uint64_t *bits);
/* Test hooks of f4: the relaxation for gfors_step / gfors_indicators (0/1), and the repair of a
 * host batch in place (bits as gfors_sample, n_words words per variable; needs relax = 1). */
gfors_status gfors_set_relax(gfors_ctx *ctx, int32_t relax);
/* Test hook: cover completion (complete = 1) of a host batch in place, p host (n entries). */
gfors_status gfors_cover_complete(gfors_ctx *ctx, const double *p, uint64_t *bits, int64_t n_words);
gfors_status gfors_repair(gfors_ctx *ctx, uint64_t *bits, int64_t n_words);
/* Current problem dimensions (reduced after gfors_tu_reformulate) and the original n. */
gfors_status gfors_dims(gfors_ctx *ctx, int64_t *n, int64_t *m, int64_t *n_orig);
/* Preprocess on the device (row norms, power iterations).  out may be NULL. */
gfors_status gfors_preprocess(gfors_ctx *ctx, const gfors_prep_opts *opts, gfors_scaling *out);
/* Alg. 1 from x0 = 0.5*1, y0 = 0 (reading R14).  Blocks until the loop has finished.
 * Collective when world > 1 (all ranks must call with identical params except k_b). */
gfors_status gfors_run(gfors_ctx *ctx, const gfors_params *p, gfors_run_info *out);
/* z: objective in ORIGINAL units and sense (+inf if none); x: n bytes (0/1) or NULL (host); after
 * gfors_tu_reformulate, x has the ORIGINAL n (n_orig of gfors_dims) entries, lifted.
 * Returns GFORS_NO_INCUMBENT if no feasible point was found. */
gfors_status gfors_best_incumbent(gfors_ctx *ctx, double *z, uint8_t *x, gfors_incumbent_info *info);
const char *gfors_last_error(const gfors_ctx *ctx);
/* Test/benchmark options (production defaults otherwise); invalidate the cached loop graph.
 *   "force_deadline_rank" r, "force_deadline_block" b: rank r (a loopback rank, or this rank) reports
 *     its time limit as passed from block b on — the OR over ranks must halt every rank together
 *     (CheckHalt);
 *   "force_capture_fail" 1: a sharded run's graph capture fails, so the eager loop runs instead.
 * Unknown key: GFORS_E_INPUT. */
gfors_status gfors_set_option(gfors_ctx *ctx, const char *key, int64_t value);
void gfors_destroy(gfors_ctx *ctx);
/* Device memory of destroyed contexts stays mapped in the library's private per-device pool, so the
 * next context of the process reuses it without the driver's page mapping.  This
 * returns the pool's memory on `device` to the system; GFORS_E_STATE while a context of the device is
 * alive, GFORS_E_INPUT for a bad device.  Contexts with a caller allocator (gfors_device_opts.alloc)
 * do not use the pool. */
gfors_status gfors_release_memory(int32_t device);

/* ---------------- hooks for parity tests and benchmarks (same library, host buffers) ------- */
/* Preprocess results: row scale divisors s_j (m, canonical row order), and the scaled saddle
 * vectors r (m) and c (n) as fp64.  Any pointer may be NULL. */
gfors_status gfors_get_scaled(gfors_ctx *ctx, double *row_scale, double *r_scaled, double *c_scaled);
/* RandSampleStep of p (n, host fp64 in [0,1]) for global words [word_begin, word_begin+n_words):
 * bits[i*n_words + w] (host).  Same contract as the loop's sampler (DESIGN.md §3 R10). */
gfors_status gfors_sample(gfors_ctx *ctx, const double *p, uint64_t seed, uint32_t round_id,
                          int64_t word_begin, int64_t n_words, uint64_t *bits);
/* EvalBest pieces on a host batch bits[n][n_words]: feasible[64*n_words] (0/1) and z (canonical
 * minimisation objective, original units). */
gfors_status gfors_eval(gfors_ctx *ctx, const uint64_t *bits, int64_t n_words, uint8_t *feasible, double *z);
/* Sampling-only throughput (bench): `rounds` rounds of RandSampleStep of p (host fp64,
 * uploaded once) for k_b = 64*n_words candidates (round ids 0..rounds-1) + EvalBest + argmin, on the
 * device, no PDHG and no incumbent update; *ms_out = CUDA-event time of the rounds. */
gfors_status gfors_sample_eval_timed(gfors_ctx *ctx, const double *p, uint64_t seed, int64_t n_words, int32_t rounds,
                                     double *ms_out);
/* Set/get the PDHG iterate (host fp64; y in canonical row order). */
gfors_status gfors_set_state(gfors_ctx *ctx, const double *x, const double *xbar, const double *y);
gfors_status gfors_get_state(gfors_ctx *ctx, double *x, double *xbar, double *y);
/* iters Alg. 2 steps with fixed rho, tau1, tau2 (no sampling, no halting). */
gfors_status gfors_step(gfors_ctx *ctx, int64_t iters, double rho, double tau1, double tau2);
/* Indicators after the last step: out[0]=primal_gap, [1]=||s^x||, [2]=||s^y||, [3]=binary_gap. */
gfors_status gfors_indicators(gfors_ctx *ctx, double rho, double tau1, double tau2, double *out);
/* Trace rows of the last run (8 doubles: iter, rho, primal_gap, sx, sy, binary_gap,
 * z_best canonical, improved), oldest first; returns rows copied in *n_rows. */
gfors_status gfors_get_trace(gfors_ctx *ctx, double *rows, int64_t max_rows, int64_t *n_rows);
/* Kernel timing of one loop block (bench): runs `blocks` blocks eagerly with CUDA events
 * around every launch; ms_out[k] = mean duration of kernel class k, names via
 * gfors_kernel_class_name(k); n_classes out.  Uses p as in gfors_run; state is reset. */
gfors_status gfors_profile_blocks(gfors_ctx *ctx, const gfors_params *p, int32_t blocks,
                                  double *ms_out, int32_t max_classes, int32_t *n_classes);
const char *gfors_kernel_class_name(int32_t k);
/* After gfors_profile_blocks: per kernel class, total ms and number of launches that did work
 * (duration > 10 us; the mode-switched PDHG kernels exit in ~3 us when their mode is not chosen). */
gfors_status gfors_profile_active(gfors_ctx *ctx, double *active_ms, double *active_launches, int32_t max_classes);
/* Number of kernel launches per loop block for p (bench "gpu_launches" accounting). */
int64_t gfors_launches_per_block(gfors_ctx *ctx, const gfors_params *p);
/* Cross-rank incumbent merge rule (host-only, no GPU needed): given world records
 * (z, global sample index, flags) pick the winner: lowest z among valid, ties -> lowest index.
 * Returns the winning record position or -1. */
int32_t gfors_merge_records(const double *z, const int64_t *index, const int32_t *valid, int32_t world);

#ifdef __cplusplus
}
#endif
#endif
