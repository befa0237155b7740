/*
 * gfors_oracle.c — TEST INFRASTRUCTURE ONLY (see gfors_oracle.h).
 *
 * Plain fp64 CPU oracle of the GFORS hot path, written from PAPER.md in the
 * paper's order and notation.  Single-threaded; every sum runs in ascending
 * index order; compiled with -O2 -ffp-contract=off so each
 * expression rounds in its written order.  No blocking, fusion or reordering.
 * This file must never be linked into, or include anything from, the CUDA
 * library under paper_2510_27117_b200/.
 */
#include "gfors_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------- */
/* small helpers                                                              */
/* ------------------------------------------------------------------------- */
static char g_err[512];
const char *orc_last_error(void) { return g_err; }
static int fail(int code, const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

typedef struct {
    int64_t rows, cols, nnz;
    int64_t *ptr;
    int32_t *idx;
    double *val;
} csr_t;

static void csr_free(csr_t *a) {
    free(a->ptr); free(a->idx); free(a->val);
    memset(a, 0, sizeof *a);
}

static int csr_alloc(csr_t *a, int64_t rows, int64_t cols, int64_t nnz) {
    a->rows = rows; a->cols = cols; a->nnz = nnz;
    a->ptr = (int64_t *)calloc((size_t)rows + 1, sizeof(int64_t));
    a->idx = (int32_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
    a->val = (double *)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
    return (a->ptr && a->idx && a->val) ? 0 : -1;
}

static int is_integer_value(double v) {
    return isfinite(v) && v == floor(v) && fabs(v) < 9007199254740992.0; /* 2^53 */
}

struct orc_ctx {
    int64_t n, m, m1, m2;
    int64_t m1p;            /* rows [0,m1p) are inequalities for the PDHG step: m1, or m under the
                               monotone relaxation (reading R26) */
    int maximize, integral;
    /* canonical user form: rows [0,m1) are  Ku x >= ru,  rows [m1,m) are  Ku x = ru */
    csr_t Ku;
    double *ru;
    int64_t *perm;          /* canonical row -> input row */
    csr_t Q;                /* canonical (sign-flipped if maximize), may have nnz 0 */
    double *c;
    double c0;
    /* Preprocess output: saddle form, explicitly materialised */
    int preprocessed;
    csr_t K;                /* K = -Ku / (s_j * kappa) */
    double *r;              /* r = ru / (s_j * kappa) */
    csr_t Qs;               /* Q / omega */
    double *cs;             /* c / omega */
    double *row_scale;      /* s_j */
    double obj_scale, k_scale;
    int64_t zero_rows;
    /* PDHG state (Alg. 2) and the previous iterate for the indicators */
    int have_state, have_prev;
    double *x, *xbar, *y;
    double *x_prev, *xbar_prev, *y_prev;
    double *work_n, *work_m;
    /* incumbent (Alg. 1 z_best, x_best), canonical objective */
    int has_inc;
    double z_best;
    uint8_t *x_best;
    int64_t found_iter, found_round, found_index;
};

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11; Random123)              */
/* ------------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += W0; k1 += W1; }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------- */
/* Load, validate, canonicalise                                              */
/* ------------------------------------------------------------------------- */
static int validate_csr(int64_t rows, int64_t cols, const int64_t *ptr, const int32_t *idx,
                        const double *val, const char *name) {
    char msg[256];
    if (ptr[0] != 0) { snprintf(msg, sizeof msg, "%s: row_ptr[0] != 0", name); return fail(-3, msg); }
    for (int64_t j = 0; j < rows; ++j) {
        if (ptr[j + 1] < ptr[j]) {
            snprintf(msg, sizeof msg, "%s: row_ptr decreases at row %lld", name, (long long)j);
            return fail(-3, msg);
        }
        for (int64_t p = ptr[j]; p < ptr[j + 1]; ++p) {
            if (idx[p] < 0 || idx[p] >= cols) {
                snprintf(msg, sizeof msg, "%s: column index out of range at nnz %lld", name, (long long)p);
                return fail(-3, msg);
            }
            if (p > ptr[j] && idx[p] <= idx[p - 1]) {
                snprintf(msg, sizeof msg, "%s: columns not strictly increasing in row %lld", name, (long long)j);
                return fail(-3, msg);
            }
            if (!isfinite(val[p])) {
                snprintf(msg, sizeof msg, "%s: non-finite value at nnz %lld", name, (long long)p);
                return fail(-3, msg);
            }
            if (val[p] == 0.0) {
                snprintf(msg, sizeof msg, "%s: explicit zero at nnz %lld", name, (long long)p);
                return fail(-3, msg);
            }
        }
    }
    return 0;
}

static double csr_lookup(const csr_t *a, int64_t i, int64_t j, int *found) {
    int64_t lo = a->ptr[i], hi = a->ptr[i + 1] - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (a->idx[mid] == j) { *found = 1; return a->val[mid]; }
        if (a->idx[mid] < j) lo = mid + 1; else hi = mid - 1;
    }
    *found = 0;
    return 0.0;
}

int orc_create(orc_ctx **out, int64_t n, int64_t m,
               const int64_t *k_rowptr, const int32_t *k_col, const double *k_val,
               const double *r, const int8_t *sense,
               const int64_t *q_rowptr, const int32_t *q_col, const double *q_val,
               const double *c, double c0, int maximize) {
    *out = NULL;
    if (n <= 0 || m < 0) return fail(-3, "dimension: n must be > 0 and m >= 0");
    if (n >= 2147483647) return fail(-3, "dimension: n must fit int32 column indices");
    if (m > 0 && (!k_rowptr || !r || !sense)) return fail(-3, "K, r and sense required when m > 0");
    if (!c) return fail(-3, "c required");
    if (!isfinite(c0)) return fail(-3, "c0 non-finite");
    if (m > 0) {
        int rc = validate_csr(m, n, k_rowptr, k_col, k_val, "K");
        if (rc) return rc;
        for (int64_t j = 0; j < m; ++j) {
            if (!isfinite(r[j])) return fail(-3, "r: non-finite value");
            if (sense[j] != 1 && sense[j] != 0 && sense[j] != -1) return fail(-3, "sense: must be +1, 0 or -1");
        }
    }
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(c[i])) return fail(-3, "c: non-finite value");

    orc_ctx *o = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    o->n = n; o->m = m; o->maximize = maximize ? 1 : 0;

    /* Q: copy, negate if maximise, check symmetry. */
    int64_t qnnz = q_rowptr ? q_rowptr[n] : 0;
    csr_alloc(&o->Q, n, n, qnnz);
    if (q_rowptr) {
        int rc = validate_csr(n, n, q_rowptr, q_col, q_val, "Q");
        if (rc) { orc_destroy(o); return rc; }
        for (int64_t i = 0; i <= n; ++i) o->Q.ptr[i] = q_rowptr[i];
        for (int64_t p = 0; p < qnnz; ++p) {
            o->Q.idx[p] = q_col[p];
            o->Q.val[p] = maximize ? -q_val[p] : q_val[p];
        }
        for (int64_t i = 0; i < n; ++i)
            for (int64_t p = o->Q.ptr[i]; p < o->Q.ptr[i + 1]; ++p) {
                int found = 0;
                double v = csr_lookup(&o->Q, o->Q.idx[p], i, &found);
                if (!found || v != o->Q.val[p]) { orc_destroy(o); return fail(-3, "Q: not symmetric"); }
            }
    }
    o->c = (double *)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) o->c[i] = maximize ? -c[i] : c[i];
    o->c0 = maximize ? -c0 : c0;

    /* K_u rows: LE -> GE by negation; stable order GE rows first, then EQ. */
    int64_t knnz = m > 0 ? k_rowptr[m] : 0;
    csr_alloc(&o->Ku, m, n, knnz);
    o->ru = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
    o->perm = (int64_t *)malloc((size_t)(m ? m : 1) * sizeof(int64_t));
    int64_t cj = 0;
    for (int pass = 0; pass < 2; ++pass) {
        for (int64_t j = 0; j < m; ++j) {
            int is_eq = (sense[j] == 0);
            if (is_eq != pass) continue;
            double s = (sense[j] == -1) ? -1.0 : 1.0;
            o->perm[cj] = j;
            o->ru[cj] = s * r[j];
            int64_t q = o->Ku.ptr[cj];
            for (int64_t p = k_rowptr[j]; p < k_rowptr[j + 1]; ++p, ++q) {
                o->Ku.idx[q] = k_col[p];
                o->Ku.val[q] = s * k_val[p];
            }
            o->Ku.ptr[cj + 1] = q;
            ++cj;
        }
        if (pass == 0) o->m1 = cj;
    }
    o->m2 = m - o->m1;
    o->m1p = o->m1;

    /* Integral data => exact integer evaluation (reading R12, A23). */
    int integral = is_integer_value(o->c0);
    double bound = fabs(o->c0);
    for (int64_t i = 0; i < n && integral; ++i) { integral = is_integer_value(o->c[i]); bound += fabs(o->c[i]); }
    for (int64_t p = 0; p < qnnz && integral; ++p) { integral = is_integer_value(o->Q.val[p]); bound += fabs(o->Q.val[p]); }
    for (int64_t p = 0; p < knnz && integral; ++p) integral = is_integer_value(o->Ku.val[p]);
    for (int64_t j = 0; j < m && integral; ++j) integral = is_integer_value(o->ru[j]);
    if (bound >= 9007199254740992.0) integral = 0;
    o->integral = integral;

    o->x_best = (uint8_t *)calloc((size_t)n, 1);
    o->z_best = INFINITY;
    o->found_iter = o->found_round = o->found_index = -1;
    *out = o;
    return 0;
}

void orc_destroy(orc_ctx *o) {
    if (!o) return;
    csr_free(&o->Ku); csr_free(&o->Q); csr_free(&o->K); csr_free(&o->Qs);
    free(o->ru); free(o->perm); free(o->c); free(o->r); free(o->cs); free(o->row_scale);
    free(o->x); free(o->xbar); free(o->y); free(o->x_prev); free(o->xbar_prev); free(o->y_prev);
    free(o->work_n); free(o->work_m); free(o->x_best);
    free(o);
}

void orc_info(const orc_ctx *o, int64_t *m1, int64_t *m2, int *integral) {
    if (m1) *m1 = o->m1;
    if (m2) *m2 = o->m2;
    if (integral) *integral = o->integral;
}

void orc_row_perm(const orc_ctx *o, int64_t *perm) {
    for (int64_t j = 0; j < o->m; ++j) perm[j] = o->perm[j];
}

/* ------------------------------------------------------------------------- */
/* Spectral norm by power iteration (readings R5, R6)   */
/* ------------------------------------------------------------------------- */
static double norm2(const double *v, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

double orc_spectral_norm(int64_t rows, int64_t cols, const int64_t *ptr,
                         const int32_t *idx, const double *val, double tol, int max_iter) {
    if (rows == 0 || cols == 0) return 0.0;
    double *v = (double *)malloc((size_t)cols * sizeof(double));
    double *u = (double *)malloc((size_t)cols * sizeof(double));
    double *w = (double *)malloc((size_t)rows * sizeof(double));
    for (int64_t i = 0; i < cols; ++i) v[i] = 1.0 / sqrt((double)cols);
    double sigma = 0.0, sigma_prev = 0.0;
    int restarted = 0;
    for (int t = 1; t <= max_iter; ++t) {
        /* w = M v */
        for (int64_t j = 0; j < rows; ++j) {
            double s = 0.0;
            for (int64_t p = ptr[j]; p < ptr[j + 1]; ++p) s += val[p] * v[idx[p]];
            w[j] = s;
        }
        sigma = norm2(w, rows);
        /* u = M' w  (transposed traversal, ascending j per column) */
        for (int64_t i = 0; i < cols; ++i) u[i] = 0.0;
        for (int64_t j = 0; j < rows; ++j)
            for (int64_t p = ptr[j]; p < ptr[j + 1]; ++p) u[idx[p]] += val[p] * w[j];
        double nu = norm2(u, cols);
        if (nu == 0.0) {
            if (t == 1 && !restarted) {
                /* start vector in the null space: restart once from a Philox vector (R5) */
                uint32_t key[2] = {0x9E3779B9u, 0u};
                for (int64_t i = 0; i < cols; ++i) {
                    uint32_t ctr[4] = {(uint32_t)i, 0u, 0u, 0u}, o4[4];
                    orc_philox4x32_10(ctr, key, o4);
                    v[i] = ((double)o4[0] + 0.5) * (1.0 / 4294967296.0);
                }
                double nv = norm2(v, cols);
                for (int64_t i = 0; i < cols; ++i) v[i] /= nv;
                restarted = 1;
                t = 0;
                continue;
            }
            break;  /* zero matrix (or exact null space twice): sigma is exact */
        }
        for (int64_t i = 0; i < cols; ++i) v[i] = u[i] / nu;
        if (t > 1 && fabs(sigma - sigma_prev) <= tol * sigma) break;
        sigma_prev = sigma;
    }
    free(v); free(u); free(w);
    return sigma;
}

/* ------------------------------------------------------------------------- */
/* Preprocess (reading R4)            */
/* ------------------------------------------------------------------------- */
int orc_preprocess(orc_ctx *o, double tol, int max_iter,
                   double *obj_scale, double *k_scale, int64_t *zero_rows) {
    const int64_t n = o->n, m = o->m;
    csr_free(&o->K); csr_free(&o->Qs);
    free(o->r); free(o->cs); free(o->row_scale);
    /* saddle form K = -[A;B], r = (b;d) */
    csr_alloc(&o->K, m, n, o->Ku.nnz);
    o->r = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
    o->row_scale = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
    for (int64_t j = 0; j <= m; ++j) o->K.ptr[j] = o->Ku.ptr[j];
    for (int64_t p = 0; p < o->Ku.nnz; ++p) { o->K.idx[p] = o->Ku.idx[p]; o->K.val[p] = -o->Ku.val[p]; }
    for (int64_t j = 0; j < m; ++j) o->r[j] = o->ru[j];

    /* step 1: normalise each row of K by its 2-norm, update r accordingly */
    o->zero_rows = 0;
    for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int64_t p = o->K.ptr[j]; p < o->K.ptr[j + 1]; ++p) s += o->K.val[p] * o->K.val[p];
        s = sqrt(s);
        if (s == 0.0) { s = 1.0; o->zero_rows++; }
        o->row_scale[j] = s;
        for (int64_t p = o->K.ptr[j]; p < o->K.ptr[j + 1]; ++p) o->K.val[p] = o->K.val[p] / s;
        o->r[j] = o->r[j] / s;
    }

    /* step 2: normalise Q and c by ||Q||_2 + ||c||_2 (skip if zero) */
    csr_alloc(&o->Qs, n, n, o->Q.nnz);
    for (int64_t i = 0; i <= n; ++i) o->Qs.ptr[i] = o->Q.ptr[i];
    for (int64_t p = 0; p < o->Q.nnz; ++p) { o->Qs.idx[p] = o->Q.idx[p]; o->Qs.val[p] = o->Q.val[p]; }
    o->cs = (double *)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) o->cs[i] = o->c[i];
    double qn = o->Q.nnz ? orc_spectral_norm(n, n, o->Q.ptr, o->Q.idx, o->Q.val, tol, max_iter) : 0.0;
    double omega = qn + norm2(o->c, n);
    if (omega > 0.0) {
        for (int64_t p = 0; p < o->Qs.nnz; ++p) o->Qs.val[p] = o->Qs.val[p] / omega;
        for (int64_t i = 0; i < n; ++i) o->cs[i] = o->cs[i] / omega;
        o->obj_scale = omega;
    } else {
        o->obj_scale = 1.0;
    }

    /* step 3: normalise K and r by the spectral norm of K */
    double kappa = m ? orc_spectral_norm(m, n, o->K.ptr, o->K.idx, o->K.val, tol, max_iter) : 0.0;
    if (kappa > 0.0) {
        for (int64_t p = 0; p < o->K.nnz; ++p) o->K.val[p] = o->K.val[p] / kappa;
        for (int64_t j = 0; j < m; ++j) o->r[j] = o->r[j] / kappa;
        o->k_scale = kappa;
    } else {
        o->k_scale = 1.0;
    }
    o->preprocessed = 1;
    o->have_state = o->have_prev = 0;
    if (obj_scale) *obj_scale = o->obj_scale;
    if (k_scale) *k_scale = o->k_scale;
    if (zero_rows) *zero_rows = o->zero_rows;
    return 0;
}

int orc_scaled_dense(const orc_ctx *o, double *K, double *r, double *Qs, double *cs) {
    if (!o->preprocessed) return fail(-7, "preprocess first");
    const int64_t n = o->n, m = o->m;
    if (K) {
        memset(K, 0, (size_t)(m * n) * sizeof(double));
        for (int64_t j = 0; j < m; ++j)
            for (int64_t p = o->K.ptr[j]; p < o->K.ptr[j + 1]; ++p) K[j * n + o->K.idx[p]] = o->K.val[p];
    }
    if (r) for (int64_t j = 0; j < m; ++j) r[j] = o->r[j];
    if (Qs) {
        memset(Qs, 0, (size_t)(n * n) * sizeof(double));
        for (int64_t i = 0; i < n; ++i)
            for (int64_t p = o->Qs.ptr[i]; p < o->Qs.ptr[i + 1]; ++p) Qs[i * n + o->Qs.idx[p]] = o->Qs.val[p];
    }
    if (cs) for (int64_t i = 0; i < n; ++i) cs[i] = o->cs[i];
    return 0;
}

int orc_row_scales(const orc_ctx *o, double *s) {
    if (!o->preprocessed) return fail(-7, "preprocess first");
    for (int64_t j = 0; j < o->m; ++j) s[j] = o->row_scale[j];
    return 0;
}

/* ------------------------------------------------------------------------- */
/* UpdatePenalty (readings R7, R8)                             */
/* ------------------------------------------------------------------------- */
void orc_rho_schedule(double rho_min, double rho_max, double T, double p, double delta,
                      int64_t count, double *rho) {
    double prev = rho_min;
    for (int64_t t = 0; t < count; ++t) {
        double tilde = rho_min * pow(1.0 + (double)t / T, p);
        double lo = prev + delta;
        /* clip(a, lo, hi) = min(max(a, lo), hi) */
        double v = tilde < lo ? lo : tilde;
        v = v > rho_max ? rho_max : v;
        rho[t] = v;
        prev = v;
    }
}

/* ------------------------------------------------------------------------- */
/* PDHG (Alg. 2)                                             */
/* ------------------------------------------------------------------------- */
static void ensure_state(orc_ctx *o) {
    const int64_t n = o->n, m = o->m ? o->m : 1;
    if (!o->x) {
        o->x = (double *)malloc((size_t)n * sizeof(double));
        o->xbar = (double *)malloc((size_t)n * sizeof(double));
        o->x_prev = (double *)malloc((size_t)n * sizeof(double));
        o->xbar_prev = (double *)malloc((size_t)n * sizeof(double));
        o->work_n = (double *)malloc((size_t)n * sizeof(double));
        o->y = (double *)malloc((size_t)m * sizeof(double));
        o->y_prev = (double *)malloc((size_t)m * sizeof(double));
        o->work_m = (double *)malloc((size_t)m * sizeof(double));
    }
}

int orc_state_init(orc_ctx *o) {
    if (!o->preprocessed) return fail(-7, "preprocess first");
    ensure_state(o);
    for (int64_t i = 0; i < o->n; ++i) { o->x[i] = 0.5; o->xbar[i] = 0.5; }
    for (int64_t j = 0; j < o->m; ++j) o->y[j] = 0.0;
    o->have_state = 1; o->have_prev = 0;
    return 0;
}

int orc_set_state(orc_ctx *o, const double *x, const double *xbar, const double *y) {
    if (!o->preprocessed) return fail(-7, "preprocess first");
    ensure_state(o);
    for (int64_t i = 0; i < o->n; ++i) { o->x[i] = x[i]; o->xbar[i] = xbar[i]; }
    for (int64_t j = 0; j < o->m; ++j) o->y[j] = y[j];
    o->have_state = 1; o->have_prev = 0;
    return 0;
}

int orc_get_state(const orc_ctx *o, double *x, double *xbar, double *y) {
    if (!o->have_state) return fail(-7, "no state");
    if (x) for (int64_t i = 0; i < o->n; ++i) x[i] = o->x[i];
    if (xbar) for (int64_t i = 0; i < o->n; ++i) xbar[i] = o->xbar[i];
    if (y) for (int64_t j = 0; j < o->m; ++j) y[j] = o->y[j];
    return 0;
}

int orc_set_relax(orc_ctx *o, int relax) {
    if (relax) {
        for (int64_t i = 0; i < o->n; ++i)
            if (o->c[i] < 0.0) return fail(-3, "monotone relaxation: needs c >= 0 (canonical)");
        if (o->Q.nnz) return fail(-3, "monotone relaxation: needs Q = 0");
        for (int64_t p = 0; p < o->Ku.nnz; ++p)
            if (o->Ku.val[p] < 0.0) return fail(-3, "monotone relaxation: needs K_u >= 0");
    }
    o->m1p = relax ? o->m : o->m1;
    return 0;
}

int orc_step(orc_ctx *o, double rho, double tau1, double tau2) {
    if (!o->have_state) return fail(-7, "state not initialised");
    const int64_t n = o->n, m = o->m, m1 = o->m1p;
    /* keep x_{k-1}, xbar_{k-1}, y_{k-1} for the Thm. 2 residuals */
    for (int64_t i = 0; i < n; ++i) { o->x_prev[i] = o->x[i]; o->xbar_prev[i] = o->xbar[i]; }
    for (int64_t j = 0; j < m; ++j) o->y_prev[j] = o->y[j];

    /* y_k = Pi_{R+^{m1} x R^{m2}}( y_{k-1} + tau2 (K xbar_{k-1} + r) ) */
    for (int64_t j = 0; j < m; ++j) {
        double t = 0.0;
        for (int64_t p = o->K.ptr[j]; p < o->K.ptr[j + 1]; ++p) t += o->K.val[p] * o->xbar_prev[o->K.idx[p]];
        double yj = o->y_prev[j] + tau2 * (t + o->r[j]);
        if (j < m1 && yj < 0.0) yj = 0.0;
        o->y[j] = yj;
    }
    /* a = K' y_k  (CSR traversal scattered in ascending row order) */
    double *a = o->work_n;
    for (int64_t i = 0; i < n; ++i) a[i] = 0.0;
    for (int64_t j = 0; j < m; ++j)
        for (int64_t p = o->K.ptr[j]; p < o->K.ptr[j + 1]; ++p) a[o->K.idx[p]] += o->K.val[p] * o->y[j];
    /* delta = c + rho + K'y_k + 2 Q x_{k-1} - 2 rho x_{k-1}   (reading R1: scalar rho added to every c_i)
     * x_k = Pi_[0,1]( x_{k-1} - tau1 delta );  xbar_k = 2 x_k - x_{k-1} */
    for (int64_t i = 0; i < n; ++i) {
        double b = 0.0;
        for (int64_t p = o->Qs.ptr[i]; p < o->Qs.ptr[i + 1]; ++p) b += o->Qs.val[p] * o->x_prev[o->Qs.idx[p]];
        double delta = o->cs[i] + rho + a[i] + 2.0 * b - 2.0 * rho * o->x_prev[i];
        double xi = o->x_prev[i] - tau1 * delta;
        if (xi < 0.0) xi = 0.0;
        if (xi > 1.0) xi = 1.0;
        o->x[i] = xi;
        o->xbar[i] = 2.0 * xi - o->x_prev[i];
    }
    o->have_prev = 1;
    return 0;
}

/* Indicators ("primal feasibility gap, dual feasibility gap, binary gap";
 * Thm. 2 residuals PAPER L652; reading R9).
 *   s^x = (x_{k-1}-x_k)/tau1 + grad_x L(x_k,y_k) - grad_x L(x_{k-1},y_k)
 *       = (x_{k-1}-x_k)/tau1 + 2Q(x_k-x_{k-1}) - 2 rho (x_k-x_{k-1})     by eq:dy (L428)
 *   s^y = (y_{k-1}-y_k)/tau2 - grad_y L(x_k,y_k) + grad_y L(xbar_{k-1},y_k)
 *       = (y_{k-1}-y_k)/tau2 - K(x_k - xbar_{k-1})                       by eq:dy (L428) */
int orc_indicators(const orc_ctx *o, double rho, double tau1, double tau2, double *out) {
    if (!o->have_prev) return fail(-7, "no step taken");
    const int64_t n = o->n, m = o->m, m1 = o->m1p;
    double pg_ineq = 0.0, pg_eq = 0.0, sy2 = 0.0;
    for (int64_t j = 0; j < m; ++j) {
        double kx = 0.0, kd = 0.0;
        for (int64_t p = o->K.ptr[j]; p < o->K.ptr[j + 1]; ++p) {
            kx += o->K.val[p] * o->x[o->K.idx[p]];
            kd += o->K.val[p] * (o->x[o->K.idx[p]] - o->xbar_prev[o->K.idx[p]]);
        }
        double g = kx + o->r[j];  /* (K x_k + r)_j ; a GE row is satisfied iff g <= 0 */
        if (j < m1) { double v = g > 0.0 ? g : 0.0; if (v > pg_ineq) pg_ineq = v; }
        else { double v = fabs(g); if (v > pg_eq) pg_eq = v; }
        double sy = (o->y_prev[j] - o->y[j]) / tau2 - kd;
        sy2 += sy * sy;
    }
    double sx2 = 0.0, bg = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double qd = 0.0;
        for (int64_t p = o->Qs.ptr[i]; p < o->Qs.ptr[i + 1]; ++p)
            qd += o->Qs.val[p] * (o->x[o->Qs.idx[p]] - o->x_prev[o->Qs.idx[p]]);
        double dx = o->x[i] - o->x_prev[i];
        double sx = (o->x_prev[i] - o->x[i]) / tau1 + 2.0 * qd - 2.0 * rho * dx;
        sx2 += sx * sx;
        bg += o->x[i] * (1.0 - o->x[i]);
    }
    out[0] = pg_ineq + pg_eq;
    out[1] = sqrt(sx2);
    out[2] = sqrt(sy2);
    out[3] = bg / (double)n;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* RandSampleStep (Alg. 3) under the Philox bit-plane contract */
/* (reading R10).  Literal: all 32 planes are drawn for every lane.            */
/* ------------------------------------------------------------------------- */
static uint64_t sample_word(double p, uint32_t i, uint64_t wg, uint32_t round_id, const uint32_t key[2]) {
    /* T_i = ceil(p_i * 2^32), exact in fp64 (p outside [0,1] is clamped) */
    double pi = p < 0.0 ? 0.0 : (p > 1.0 ? 1.0 : p);
    uint64_t T = (uint64_t)ceil(pi * 4294967296.0);
    uint64_t plane[32];
    for (uint32_t q = 0; q < 16; ++q) {
        uint32_t ctr[4] = {i, (uint32_t)wg, q, round_id}, o4[4];
        orc_philox4x32_10(ctr, key, o4);
        plane[2 * q] = (uint64_t)o4[0] | ((uint64_t)o4[1] << 32);
        plane[2 * q + 1] = (uint64_t)o4[2] | ((uint64_t)o4[3] << 32);
    }
    uint64_t word = 0;
    for (int b = 0; b < 64; ++b) {
        uint64_t u = 0;  /* plane 0 is the most significant bit of u */
        for (int t = 0; t < 32; ++t) u |= ((plane[t] >> b) & 1u) << (31 - t);
        uint64_t xb = (u < T) ? 1u : 0u;  /* Bernoulli(p_i) */
        word |= xb << b;
    }
    return word;
}

void orc_sample(const double *p, int64_t n, uint64_t seed, uint32_t round_id,
                int64_t word_begin, int64_t n_words, uint64_t *bits) {
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    for (int64_t i = 0; i < n; ++i)
        for (int64_t w = 0; w < n_words; ++w)
            bits[i * n_words + w] = sample_word(p[i], (uint32_t)i, (uint64_t)(word_begin + w), round_id, key);
}

void orc_sample_subset(const double *p_sub, const int64_t *idx, int64_t count, uint64_t seed,
                       uint32_t round_id, int64_t word_begin, int64_t n_words, uint64_t *bits) {
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    for (int64_t k = 0; k < count; ++k)
        for (int64_t w = 0; w < n_words; ++w)
            bits[k * n_words + w] = sample_word(p_sub[k], (uint32_t)idx[k], (uint64_t)(word_begin + w), round_id, key);
}

/* ------------------------------------------------------------------------- */
/* Customised RandSampleStep for 3D assignment (PAPER Alg. 4)  */
/* ------------------------------------------------------------------------- */
typedef struct { double p; int64_t idx; } a3_entry;
static int a3_cmp(const void *x, const void *y) {
    const a3_entry *a = (const a3_entry *)x, *b = (const a3_entry *)y;
    if (a->p > b->p) return -1;          /* descending p */
    if (a->p < b->p) return 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);  /* ties: lower flat index first */
}

static uint32_t a3_draw(uint32_t lane, uint32_t round_id, uint32_t step, uint32_t tag,
                        const uint32_t key[2], uint32_t out[4]) {
    const uint32_t ctr[4] = {lane, round_id, step, tag};
    orc_philox4x32_10(ctr, key, out);
    return out[0];
}

void orc_sample_assign3d(const double *p, int64_t n, const double *cost, uint64_t seed, uint32_t round_id,
                         int64_t word_begin, int64_t n_words, double gamma, int64_t L, uint64_t *bits) {
    const int64_t N = n * n * n;
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    memset(bits, 0, (size_t)(N * n_words) * sizeof(uint64_t));
    /* (1) the ceil(gamma*n) largest entries of p */
    int64_t K = (int64_t)ceil(gamma * (double)n);
    if (K > N) K = N;
    a3_entry *e = (a3_entry *)malloc((size_t)N * sizeof(a3_entry));
    for (int64_t v = 0; v < N; ++v) { e[v].p = p[v]; e[v].idx = v; }
    qsort(e, (size_t)N, sizeof(a3_entry), a3_cmp);
    /* (2) greedy partial non-conflict assignment in that order */
    int64_t *sj0 = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *sk0 = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    char *uj = (char *)calloc((size_t)n, 1), *uk = (char *)calloc((size_t)n, 1);
    for (int64_t i = 0; i < n; ++i) sj0[i] = sk0[i] = -1;
    for (int64_t t = 0; t < K; ++t) {
        const int64_t v = e[t].idx, i = v / (n * n), j = (v / n) % n, k = v % n;
        if (sj0[i] < 0 && !uj[j] && !uk[k]) { sj0[i] = j; sk0[i] = k; uj[j] = 1; uk[k] = 1; }
    }
    int64_t r = 0;
    int64_t *Ri = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *Rj = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *Rk = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t rj = 0, rk = 0;
    for (int64_t i = 0; i < n; ++i) if (sj0[i] < 0) Ri[r++] = i;
    for (int64_t j = 0; j < n; ++j) if (!uj[j]) Rj[rj++] = j;
    for (int64_t k = 0; k < n; ++k) if (!uk[k]) Rk[rk++] = k;
    int64_t *pj = (int64_t *)malloc((size_t)n * sizeof(int64_t)), *pk = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *sj = (int64_t *)malloc((size_t)n * sizeof(int64_t)), *sk = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    for (int64_t w = 0; w < n_words; ++w) {
        for (int b = 0; b < 64; ++b) {
            const uint32_t lane = (uint32_t)(64 * (word_begin + w) + b);
            uint32_t o4[4];
            /* (3) random completion: Fisher-Yates on the unused j's and k's */
            for (int64_t t = 0; t < r; ++t) { pj[t] = Rj[t]; pk[t] = Rk[t]; }
            for (int64_t t = r - 1; t >= 1; --t) {
                uint64_t u = a3_draw(lane, round_id, (uint32_t)t, 0xA3D00001u, key, o4);
                int64_t q = (int64_t)((u * (uint64_t)(t + 1)) >> 32);
                int64_t tmp = pj[t]; pj[t] = pj[q]; pj[q] = tmp;
                u = a3_draw(lane, round_id, (uint32_t)t, 0xA3D00002u, key, o4);
                q = (int64_t)((u * (uint64_t)(t + 1)) >> 32);
                tmp = pk[t]; pk[t] = pk[q]; pk[q] = tmp;
            }
            for (int64_t i = 0; i < n; ++i) { sj[i] = sj0[i]; sk[i] = sk0[i]; }
            for (int64_t t = 0; t < r; ++t) { sj[Ri[t]] = pj[t]; sk[Ri[t]] = pk[t]; }
            /* (4) L pairwise interchanges (swap a coordinate iff the cost strictly decreases) */
            for (int64_t st = 0; st < L && n >= 2; ++st) {
                a3_draw(lane, round_id, (uint32_t)st, 0xA3D00003u, key, o4);
                const int64_t a = (int64_t)(((uint64_t)o4[0] * (uint64_t)n) >> 32);
                int64_t bb = (int64_t)(((uint64_t)o4[1] * (uint64_t)(n - 1)) >> 32);
                if (bb >= a) bb += 1;
                const double old_c = cost[a * n * n + sj[a] * n + sk[a]] + cost[bb * n * n + sj[bb] * n + sk[bb]];
                if ((o4[2] & 1u) == 0) {
                    const double new_c = cost[a * n * n + sj[bb] * n + sk[a]] + cost[bb * n * n + sj[a] * n + sk[bb]];
                    if (new_c < old_c) { int64_t tmp = sj[a]; sj[a] = sj[bb]; sj[bb] = tmp; }
                } else {
                    const double new_c = cost[a * n * n + sj[a] * n + sk[bb]] + cost[bb * n * n + sj[bb] * n + sk[a]];
                    if (new_c < old_c) { int64_t tmp = sk[a]; sk[a] = sk[bb]; sk[bb] = tmp; }
                }
            }
            for (int64_t i = 0; i < n; ++i) {
                const int64_t v = i * n * n + sj[i] * n + sk[i];
                bits[v * n_words + w] |= (uint64_t)1 << b;
            }
        }
    }
    free(e); free(sj0); free(sk0); free(uj); free(uk); free(Ri); free(Rj); free(Rk);
    free(pj); free(pk); free(sj); free(sk);
}

/* Repair after the monotone relaxation (reading R26): per lane, the lane's 1-entries in
 * order of decreasing canonical cost (ties: lower index first) are dropped one by one while every row
 * keeps sum_i K_ji x_i >= r_j (all rows read as >=).  Requires the relaxation (m1p == m). */
typedef struct { double c; int64_t i; } rp_entry;
static int rp_cmp(const void *x, const void *y) {
    const rp_entry *a = (const rp_entry *)x, *b = (const rp_entry *)y;
    if (a->c > b->c) return -1;
    if (a->c < b->c) return 1;
    return (a->i < b->i) ? -1 : (a->i > b->i);
}

int orc_repair(const orc_ctx *o, uint64_t *bits, int64_t n_words) {
    if (o->m1p != o->m) return fail(-3, "repair needs the monotone relaxation");
    const int64_t n = o->n, m = o->m;
    /* column lists of K_u (plain transpose by scanning the rows in order) */
    int64_t *cptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t p = 0; p < o->Ku.nnz; ++p) cptr[o->Ku.idx[p] + 1]++;
    for (int64_t i = 0; i < n; ++i) cptr[i + 1] += cptr[i];
    int64_t *crow = (int64_t *)malloc((size_t)(o->Ku.nnz ? o->Ku.nnz : 1) * sizeof(int64_t));
    double *cval = (double *)malloc((size_t)(o->Ku.nnz ? o->Ku.nnz : 1) * sizeof(double));
    int64_t *fill = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    for (int64_t j = 0; j < m; ++j)
        for (int64_t p = o->Ku.ptr[j]; p < o->Ku.ptr[j + 1]; ++p) {
            const int64_t i = o->Ku.idx[p];
            crow[cptr[i] + fill[i]] = j; cval[cptr[i] + fill[i]] = o->Ku.val[p]; fill[i]++;
        }
    rp_entry *ones = (rp_entry *)malloc((size_t)n * sizeof(rp_entry));
    double *srow = (double *)malloc((size_t)(m ? m : 1) * sizeof(double));
    for (int64_t l = 0; l < 64 * n_words; ++l) {
        const int64_t w = l / 64;
        const uint64_t bit = (uint64_t)1 << (l % 64);
        int64_t cnt = 0;
        for (int64_t i = 0; i < n; ++i)
            if (bits[i * n_words + w] & bit) { ones[cnt].c = o->c[i]; ones[cnt].i = i; cnt++; }
        qsort(ones, (size_t)cnt, sizeof(rp_entry), rp_cmp);
        for (int64_t j = 0; j < m; ++j) srow[j] = 0.0;
        for (int64_t t = 0; t < cnt; ++t)
            for (int64_t q = cptr[ones[t].i]; q < cptr[ones[t].i + 1]; ++q) srow[crow[q]] += cval[q];
        for (int64_t t = 0; t < cnt; ++t) {
            const int64_t i = ones[t].i;
            int ok = 1;
            for (int64_t q = cptr[i]; q < cptr[i + 1] && ok; ++q) ok = (srow[crow[q]] - cval[q] >= o->ru[crow[q]]);
            if (!ok) continue;
            for (int64_t q = cptr[i]; q < cptr[i + 1]; ++q) srow[crow[q]] -= cval[q];
            bits[i * n_words + w] &= ~bit;
        }
    }
    free(cptr); free(crow); free(cval); free(fill); free(ones); free(srow);
    return 0;
}

/* Cover completion (reading R27): in each lane, every covering row (>= row, all
 * coefficients 1, right-hand side 1) that the lane violates gets its variable with the largest p
 * (ties: lowest index) switched on; all decisions are taken on the batch as passed in. */
int orc_cover_complete(const orc_ctx *o, const double *p, uint64_t *bits, int64_t n_words) {
    const int64_t m1 = o->m1;
    int64_t *best = (int64_t *)malloc((size_t)(m1 ? m1 : 1) * sizeof(int64_t));
    char *elig = (char *)calloc((size_t)(m1 ? m1 : 1), 1);
    for (int64_t j = 0; j < m1; ++j) {
        int ok = o->ru[j] == 1.0 && o->Ku.ptr[j + 1] > o->Ku.ptr[j];
        for (int64_t q = o->Ku.ptr[j]; q < o->Ku.ptr[j + 1] && ok; ++q) ok = o->Ku.val[q] == 1.0;
        elig[j] = (char)ok;
        best[j] = -1;
        if (!ok) continue;
        for (int64_t q = o->Ku.ptr[j]; q < o->Ku.ptr[j + 1]; ++q) {
            const int64_t i = o->Ku.idx[q];
            if (best[j] < 0 || p[i] > p[best[j]] || (p[i] == p[best[j]] && i < best[j])) best[j] = i;
        }
    }
    uint64_t *add = (uint64_t *)calloc((size_t)(o->n * n_words), sizeof(uint64_t));
    for (int64_t j = 0; j < m1; ++j) {
        if (!elig[j]) continue;
        for (int64_t w = 0; w < n_words; ++w) {
            uint64_t covered = 0;
            for (int64_t q = o->Ku.ptr[j]; q < o->Ku.ptr[j + 1]; ++q) covered |= bits[o->Ku.idx[q] * n_words + w];
            add[best[j] * n_words + w] |= ~covered;
        }
    }
    for (int64_t t = 0; t < o->n * n_words; ++t) bits[t] |= add[t];
    free(best); free(elig); free(add);
    return 0;
}

void orc_canonical_c(const orc_ctx *o, double *c) {
    for (int64_t i = 0; i < o->n; ++i) c[i] = o->c[i];
}

/* ------------------------------------------------------------------------- */
/* EvalBest pieces (readings R11, R12) */
/* ------------------------------------------------------------------------- */
static void eval_one(const orc_ctx *o, const uint8_t *xh, int *feasible, double *z) {
    const int64_t n = o->n, m = o->m, m1 = o->m1;
    int feas = 1;
    if (o->integral) {
        for (int64_t j = 0; j < m && feas; ++j) {
            int64_t s = 0;
            for (int64_t p = o->Ku.ptr[j]; p < o->Ku.ptr[j + 1]; ++p)
                if (xh[o->Ku.idx[p]]) s += (int64_t)o->Ku.val[p];
            int64_t rj = (int64_t)o->ru[j];
            feas = (j < m1) ? (s >= rj) : (s == rj);
        }
        int64_t zi = 0;
        for (int64_t i = 0; i < n; ++i) if (xh[i]) zi += (int64_t)o->c[i];
        for (int64_t i = 0; i < n; ++i) {
            if (!xh[i]) continue;
            for (int64_t p = o->Q.ptr[i]; p < o->Q.ptr[i + 1]; ++p)
                if (xh[o->Q.idx[p]]) zi += (int64_t)o->Q.val[p];
        }
        zi += (int64_t)o->c0;
        *z = (double)zi;
    } else {
        for (int64_t j = 0; j < m && feas; ++j) {
            double s = 0.0;
            for (int64_t p = o->Ku.ptr[j]; p < o->Ku.ptr[j + 1]; ++p)
                if (xh[o->Ku.idx[p]]) s += o->Ku.val[p];
            feas = (j < m1) ? (o->ru[j] - s <= 1e-9) : (fabs(s - o->ru[j]) <= 1e-9);
        }
        double zs = 0.0;
        for (int64_t i = 0; i < n; ++i) if (xh[i]) zs += o->c[i];
        for (int64_t i = 0; i < n; ++i) {
            if (!xh[i]) continue;
            for (int64_t p = o->Q.ptr[i]; p < o->Q.ptr[i + 1]; ++p)
                if (xh[o->Q.idx[p]]) zs += o->Q.val[p];
        }
        zs += o->c0;
        *z = zs;
    }
    *feasible = feas;
}

int orc_eval(const orc_ctx *o, const uint64_t *bits, int64_t n_words,
             uint8_t *feasible, double *z) {
    const int64_t n = o->n;
    uint8_t *xh = (uint8_t *)malloc((size_t)n);
    for (int64_t l = 0; l < 64 * n_words; ++l) {
        for (int64_t i = 0; i < n; ++i) xh[i] = (uint8_t)((bits[i * n_words + l / 64] >> (l % 64)) & 1u);
        int f; double zl;
        eval_one(o, xh, &f, &zl);
        feasible[l] = (uint8_t)f;
        z[l] = zl;
    }
    free(xh);
    return 0;
}

int orc_eval_point(const orc_ctx *o, const uint8_t *x, int *feasible, double *z) {
    for (int64_t i = 0; i < o->n; ++i)
        if (x[i] > 1) return fail(-3, "x must be 0/1");
    eval_one(o, x, feasible, z);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* CheckHalt (reading R9)                       */
/* ------------------------------------------------------------------------- */
void orc_halt_init(orc_halt_state *h, double tol_p, double tol_d, double tol_b,
                   double stall_rel, int window) {
    memset(h, 0, sizeof *h);
    h->tol[0] = tol_p; h->tol[1] = tol_d; h->tol[2] = tol_b;
    h->stall_rel = stall_rel;
    h->window = window < 1 ? 1 : (window > 1024 ? 1024 : window);
}

int orc_halt_push(orc_halt_state *h, double primal_gap, double dual_gap,
                  double binary_gap, int improved) {
    const double v[3] = {primal_gap, dual_gap, binary_gap};
    const int W = h->window;
    for (int a = 0; a < 3; ++a) h->hist[a][h->count % W] = v[a];
    h->count++;
    if (improved) h->since_improve = 0; else h->since_improve++;
    int all_ok = 1;
    for (int a = 0; a < 3; ++a) {
        int ok = v[a] <= h->tol[a];
        if (!ok && h->count >= W) {
            double mx = h->hist[a][0], mn = h->hist[a][0];
            for (int s = 1; s < W; ++s) {
                if (h->hist[a][s] > mx) mx = h->hist[a][s];
                if (h->hist[a][s] < mn) mn = h->hist[a][s];
            }
            double den = fabs(mx) > 1e-300 ? fabs(mx) : 1e-300;
            ok = (mx - mn) / den < h->stall_rel;
        }
        all_ok = all_ok && ok;
    }
    return (all_ok && h->since_improve >= W) ? 1 : 0;
}

/* ------------------------------------------------------------------------- */
/* Alg. 1                                                   */
/* ------------------------------------------------------------------------- */
void orc_params_default(orc_params *p) {
    /* SPEC L293, L667 */
    p->sigma = 0.99; p->k_int = 10; p->k_r = 1; p->k_b = 128;
    p->rho_min = 1e-3; p->rho_max = 10.0; p->growth_T = 100.0; p->growth_p = 2.0; p->rho_delta = 1e-6;
    p->tol_primal = 1e-6; p->tol_dual = 1e-6; p->tol_binary = 1e-6;
    p->stall_rel = 1e-8; p->stall_window = 50;
    p->max_iters = 100000; p->time_limit_s = 1800.0; p->seed = 20251030ull;
    p->sampler = 0; p->a3_ls = -1; p->a3_n = 0; p->a3_gamma = 4.0;
    p->relax = 0; p->repair = 0; p->complete = 0;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* EvalBest: best feasible lane (min z, ties -> lowest global index), replace iff strictly better */
static int eval_best(orc_ctx *o, const uint64_t *bits, int64_t n_words, int64_t word_begin,
                     int64_t iter, int64_t round_id, uint8_t *feas, double *z) {
    orc_eval(o, bits, n_words, feas, z);
    int64_t best = -1;
    for (int64_t l = 0; l < 64 * n_words; ++l)
        if (feas[l] && (best < 0 || z[l] < z[best])) best = l;
    if (best >= 0 && z[best] < o->z_best) {
        o->z_best = z[best];
        for (int64_t i = 0; i < o->n; ++i)
            o->x_best[i] = (uint8_t)((bits[i * n_words + best / 64] >> (best % 64)) & 1u);
        o->has_inc = 1;
        o->found_iter = iter;
        o->found_round = round_id;
        o->found_index = 64 * word_begin + best;
        return 1;
    }
    return 0;
}

int orc_run(orc_ctx *o, const orc_params *p, orc_run_info *info,
            double *trace, int64_t n_trace_max, int64_t *n_trace) {
    if (!o->preprocessed) return fail(-7, "preprocess first");
    if (!(p->sigma > 0.0 && p->sigma < 1.0)) return fail(-3, "sigma must be in (0,1)");
    if (p->k_b <= 0 || p->k_b % 64) return fail(-3, "k_b must be a positive multiple of 64");
    if (p->k_int < 1 || p->k_r < 1) return fail(-3, "k_int and k_r must be >= 1");
    if (p->sampler == 1 && (p->a3_n < 1 || p->a3_n * p->a3_n * p->a3_n != o->n || !(p->a3_gamma > 0.0)))
        return fail(-3, "sampler 1 (3D assignment): n must equal a3_n^3 and a3_gamma > 0");
    if (p->repair && !p->relax) return fail(-3, "repair needs relax = 1");
    {
        int rc0 = orc_set_relax(o, p->relax);
        if (rc0) return rc0;
    }
    const int64_t n = o->n;
    const double tau1 = sqrt(p->sigma), tau2 = sqrt(p->sigma);  /* reading R3 */
    const int64_t n_words = p->k_b / 64;
    const int64_t n_blocks = p->max_iters / p->k_int + 2;
    double *rho_tab = (double *)malloc((size_t)n_blocks * sizeof(double));
    orc_rho_schedule(p->rho_min, p->rho_max, p->growth_T, p->growth_p, p->rho_delta, n_blocks, rho_tab);
    uint64_t *bits = (uint64_t *)malloc((size_t)(n * n_words) * sizeof(uint64_t));
    uint8_t *feas = (uint8_t *)malloc((size_t)(64 * n_words));
    double *z = (double *)malloc((size_t)(64 * n_words) * sizeof(double));

    orc_state_init(o);
    o->has_inc = 0; o->z_best = INFINITY;
    o->found_iter = o->found_round = o->found_index = -1;
    orc_halt_state *hs = (orc_halt_state *)malloc(sizeof(orc_halt_state));
    orc_halt_init(hs, p->tol_primal, p->tol_dual, p->tol_binary, p->stall_rel, p->stall_window);

    const double t0 = now_s();
    int64_t k = 0, rounds = 0, nt = 0;
    int halt_reason = 2;
    int rc = 0;
    while (k < p->max_iters) {
        /* UpdatePenalty: the counter advances once per sampling block (reading R7) */
        double rho = rho_tab[k / p->k_int];
        k += 1;
        orc_step(o, rho, tau1, tau2);
        if (k % p->k_int == 0) {
            int improved = 0;
            for (int32_t rr = 0; rr < p->k_r; ++rr) {
                int64_t round_id = (k / p->k_int - 1) * p->k_r + rr;
                if (p->sampler == 1)
                    orc_sample_assign3d(o->x, p->a3_n, o->c, p->seed, (uint32_t)round_id, 0, n_words, p->a3_gamma,
                                        p->a3_ls < 0 ? 2 * p->a3_n : p->a3_ls, bits);
                else
                    orc_sample(o->x, n, p->seed, (uint32_t)round_id, 0, n_words, bits);
                if (p->repair) orc_repair(o, bits, n_words);
                if (p->complete) orc_cover_complete(o, o->x, bits, n_words);
                improved |= eval_best(o, bits, n_words, 0, k, round_id, feas, z);
                rounds++;
            }
            double ind[4];
            orc_indicators(o, rho, tau1, tau2, ind);
            double dual_gap = ind[1] + ind[2];
            if (trace && nt < n_trace_max) {
                double *row = trace + 8 * nt;
                row[0] = (double)k; row[1] = rho; row[2] = ind[0]; row[3] = ind[1];
                row[4] = ind[2]; row[5] = ind[3]; row[6] = o->z_best; row[7] = improved;
            }
            nt++;
            if (!isfinite(ind[0]) || !isfinite(dual_gap) || !isfinite(ind[3])) {
                halt_reason = 4; rc = fail(-4, "diverged: non-finite indicator");
                break;
            }
            if (orc_halt_push(hs, ind[0], dual_gap, ind[3], improved)) { halt_reason = 1; break; }
            if (now_s() - t0 >= p->time_limit_s) { halt_reason = 3; break; }
        }
    }
    /* final EvalBest(round(x_k)), ties x = 0.5 -> 1 (reading R13) */
    if (rc == 0) {
        uint8_t *xr = (uint8_t *)malloc((size_t)n);
        for (int64_t i = 0; i < n; ++i) xr[i] = o->x[i] >= 0.5 ? 1 : 0;
        int f; double zr;
        eval_one(o, xr, &f, &zr);
        if (f && zr < o->z_best) {
            o->z_best = zr;
            memcpy(o->x_best, xr, (size_t)n);
            o->has_inc = 1;
            o->found_iter = k; o->found_round = -1; o->found_index = -1;
        }
        free(xr);
    }
    if (info) {
        info->iters = k; info->rounds = rounds; info->candidates = rounds * p->k_b;
        info->halt_reason = halt_reason;
        info->found_iter = o->found_iter; info->found_round = o->found_round;
        info->found_index = o->found_index; info->has_incumbent = o->has_inc;
        info->z_best = o->has_inc ? (o->maximize ? -o->z_best : o->z_best) : INFINITY;
    }
    if (n_trace) *n_trace = nt;
    free(rho_tab); free(bits); free(feas); free(z); free(hs);
    return rc;
}

int orc_best(const orc_ctx *o, double *z_original, uint8_t *x) {
    if (z_original) *z_original = o->has_inc ? (o->maximize ? -o->z_best : o->z_best) : INFINITY;
    if (x) memcpy(x, o->x_best, (size_t)o->n);
    return o->has_inc ? 0 : 2;
}
