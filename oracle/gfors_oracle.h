/*
 * gfors_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded fp64 CPU implementation of the GFORS hot path
 * (arXiv 2510.27117), written directly from PAPER.md.  It exists only to check
 * the CUDA library (include/gfors.h).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * source, header, table or helper with paper_2510_27117_b200/.
 *
 * Citations "PAPER Lx" are lines of /root/reference/PAPER.md; "SPEC Lx" lines of
 * /root/reference/SPEC.md; "Rn" are the readings listed in DESIGN.md §3.
 *
 * Conventions:
 *   user form   : min x'Qx + c'x + c0  s.t.  K_u x >= r (GE) / = r (EQ) / <= r (LE)
 *   canonical   : maximize -> (c,Q,c0) negated; LE rows negated to GE; rows
 *                 stably permuted GE first, then EQ
 *   saddle form : K = -K_u (canonical), r unchanged; then Preprocess scaling.
 * Every function returns 0 on success, a negative code on error:
 *   -3 input error (SPEC exit 3), -4 divergence (SPEC exit 4), -7 call order.
 */
#ifndef GFORS_ORACLE_H
#define GFORS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_ctx orc_ctx;

/* Philox4x32-10 (Salmon et al., SC'11). Reading R10: the paper's RNG is unnamed
 * (PAPER L753); the sampling contract of DESIGN.md §3 fixes this generator. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Load + validate + canonicalize.
 * sense[j]: +1 GE, 0 EQ, -1 LE.  q_* may be NULL (Q = 0).  Copies everything. */
int orc_create(orc_ctx **out, int64_t n, int64_t m,
               const int64_t *k_rowptr, const int32_t *k_col, const double *k_val,
               const double *r, const int8_t *sense,
               const int64_t *q_rowptr, const int32_t *q_col, const double *q_val,
               const double *c, double c0, int maximize);
void orc_destroy(orc_ctx *o);
const char *orc_last_error(void);

/* Facts about the canonical problem. */
void orc_info(const orc_ctx *o, int64_t *m1, int64_t *m2, int *integral);
/* canonical row j -> input row index */
void orc_row_perm(const orc_ctx *o, int64_t *perm);

/* Spectral norm of a CSR matrix by power iteration on M'M (
 * readings R5, R6).  Start 1/sqrt(ncols)*ones, stop when
 * |s_t - s_{t-1}| <= tol*s_t or after max_iter sweeps. */
double orc_spectral_norm(int64_t rows, int64_t cols, const int64_t *ptr,
                         const int32_t *idx, const double *val, double tol, int max_iter);

/* Preprocess: row 2-norm scaling of K,r; (Q,c) /= ||Q||_2+||c||_2;
 * (K,r) /= ||K||_2.  Outputs the scaling record. */
int orc_preprocess(orc_ctx *o, double tol, int max_iter,
                   double *obj_scale, double *k_scale, int64_t *zero_rows);
/* Scaled saddle-form data, for inspection: K (m x n) dense row-major, r (m),
 * Qs (n x n) dense, cs (n).  Any pointer may be NULL.  Small problems only. */
int orc_scaled_dense(const orc_ctx *o, double *K, double *r, double *Qs, double *cs);
/* Row scale divisors s_j (zero rows -> 1), length m. */
int orc_row_scales(const orc_ctx *o, double *s);

/* UpdatePenalty: rho_t = clip(rho_min(1+t/T)^p, rho_{t-1}+delta, rho_max),
 * rho_{-1} = rho_min (reading R8).  Writes rho_0..rho_{count-1}. */
void orc_rho_schedule(double rho_min, double rho_max, double T, double p, double delta,
                      int64_t count, double *rho);

/* PDHG state (reading R14: x0 = 0.5*1, y0 = 0, xbar0 = x0). */
int orc_state_init(orc_ctx *o);
int orc_set_state(orc_ctx *o, const double *x, const double *xbar, const double *y);
int orc_get_state(const orc_ctx *o, double *x, double *xbar, double *y);
/* One Alg. 2 step with penalty rho and steps tau1, tau2. */
int orc_step(orc_ctx *o, double rho, double tau1, double tau2);
/* Indicators after the last orc_step:
 * out[0]=primal_gap, out[1]=||s^x||, out[2]=||s^y||, out[3]=binary_gap. */
int orc_indicators(const orc_ctx *o, double rho, double tau1, double tau2, double *out);

/* RandSampleStep under the Philox bit-plane contract:
 * bits[i*n_words + w] holds lanes 64*(word_begin+w) .. +63 of variable i. */
void orc_sample(const double *p, int64_t n, uint64_t seed, uint32_t round_id,
                int64_t word_begin, int64_t n_words, uint64_t *bits);

/* Same contract for a subset of variables: bits[k*n_words + w] for variable idx[k]. */
void orc_sample_subset(const double *p_sub, const int64_t *idx, int64_t count, uint64_t seed,
                       uint32_t round_id, int64_t word_begin, int64_t n_words, uint64_t *bits);

/* Customised RandSampleStep for 3D assignment (PAPER Alg. 4; next row
 * f3; reading R25).  Variables are the n^3 triples (i,j,k) at flat index i*n^2 + j*n + k; p and
 * cost (canonical, minimisation) have n^3 entries.  (1) the K = ceil(gamma*n) largest p (ties:
 * lower flat index); (2) greedy partial assignment in that order (accept a triple iff its i, j and
 * k are all unused); (3) per lane: the unused j's and k's (ascending) are shuffled by Fisher-Yates
 * (t = r-1..1: s = (u*(t+1)) >> 32, u = Philox out0 of ctr (lane, round, t, 0xA3D00001 / 2)) and
 * assigned to the unused i's in ascending order; (4) L pairwise interchanges: step s draws
 * Philox ctr (lane, round, s, 0xA3D00003): a = (o0*n)>>32, b = (o1*(n-1))>>32 (+1 if >= a),
 * coordinate j if o2 is even else k; the two triples swap that coordinate iff the cost sum
 * strictly decreases.  Lane = 64*(word_begin + w) + bit.  Every lane is a feasible assignment. */
void orc_sample_assign3d(const double *p, int64_t n, const double *cost, uint64_t seed, uint32_t round_id,
                         int64_t word_begin, int64_t n_words, double gamma, int64_t L, uint64_t *bits);
/* Monotone relaxation (reading R26): with Q = 0, c >= 0 and K_u >= 0 (canonical),
 * the PDHG step and indicators treat every row as >= (upper closure); EvalBest keeps the original
 * equalities.  relax = 0 restores the original senses. */
int orc_set_relax(orc_ctx *o, int relax);
/* Repair (reading R26): per lane, drop 1-entries in order of decreasing cost (ties: lower index
 * first) while every row keeps sum K_ji x_i >= r_j; needs the relaxation.  Every lane is repaired,
 * whatever its number of 1-entries. */
int orc_repair(const orc_ctx *o, uint64_t *bits, int64_t n_words);
/* Cover completion (R27): each covering row (>=, coefficients 1, rhs 1) violated by a
 * lane gets its variable with the largest p (ties: lowest index) switched on in that lane; the
 * decisions are all taken on the batch as passed in (order-free). */
int orc_cover_complete(const orc_ctx *o, const double *p, uint64_t *bits, int64_t n_words);
/* canonical (minimisation) cost vector c (n entries) of a loaded problem */
void orc_canonical_c(const orc_ctx *o, double *c);

/* Evaluate a bit-sliced batch on the ORIGINAL canonical data (SPEC L147-155,
 * L138-146): feasible[l] in {0,1}, z[l] canonical (minimisation) objective. */
int orc_eval(const orc_ctx *o, const uint64_t *bits, int64_t n_words,
             uint8_t *feasible, double *z);
/* Objective / feasibility of a single 0/1 vector (uint8 per variable). */
int orc_eval_point(const orc_ctx *o, const uint8_t *x, int *feasible, double *z);

/* CheckHalt state machine (reading R9). */
typedef struct {
    double tol[3];          /* primal, dual, binary */
    double stall_rel;       /* relative range threshold */
    int window;             /* W checks */
    int count;              /* checks seen */
    double hist[3][1024];   /* ring buffers, window <= 1024 */
    int64_t since_improve;  /* checks since the last incumbent improvement */
} orc_halt_state;
void orc_halt_init(orc_halt_state *h, double tol_p, double tol_d, double tol_b,
                   double stall_rel, int window);
/* Push one check; returns 1 if halt. */
int orc_halt_push(orc_halt_state *h, double primal_gap, double dual_gap,
                  double binary_gap, int improved);

/* Alg. 1 driver.  Parameters follow SPEC L632-635/L667 defaults. */
typedef struct {
    double sigma; int32_t k_int, k_r; int64_t k_b;
    double rho_min, rho_max, growth_T, growth_p, rho_delta;
    double tol_primal, tol_dual, tol_binary, stall_rel; int32_t stall_window;
    int64_t max_iters; double time_limit_s; uint64_t seed;
    int32_t sampler;        /* 0: Bernoulli (Alg. 3), 1: 3D assignment (Alg. 4) */
    int32_t a3_ls;          /* Alg. 4 L (-1: 2*a3_n) */
    int64_t a3_n;           /* Alg. 4 n (variables = a3_n^3) */
    double a3_gamma;        /* Alg. 4 gamma (default 4) */
    int32_t relax;          /* monotone relaxation: equality rows act as >= in PDHG */
    int32_t repair;         /* per-lane greedy repair before EvalBest (needs relax) */
    int32_t complete;       /* cover completion of the sampled lanes before EvalBest (R27) */
} orc_params;
void orc_params_default(orc_params *p);
typedef struct {
    int64_t iters, rounds, candidates; int halt_reason; /* 1 criteria 2 max_iters 3 time 4 diverged */
    int64_t found_iter, found_round, found_index; int has_incumbent;
    double z_best;          /* ORIGINAL sense (sign restored) */
} orc_run_info;
/* trace: optional, n_trace_max rows of 8 doubles
 * (iter, rho, primal_gap, sx, sy, binary_gap, z_best_canonical, improved). */
int orc_run(orc_ctx *o, const orc_params *p, orc_run_info *info,
            double *trace, int64_t n_trace_max, int64_t *n_trace);
/* Best incumbent as a 0/1 byte vector in the ORIGINAL variable order. */
int orc_best(const orc_ctx *o, double *z_original, uint8_t *x);

#ifdef __cplusplus
}
#endif
#endif
