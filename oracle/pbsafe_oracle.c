/*
 * pbsafe_oracle.c -- CPU restatement of the reference's p-BiCGSafe hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle: it may be loaded
 * by tests/, by __graft_entry__.smoke() and by bench.py's cpu_baseline /
 * `--impl reference` legs, and nowhere else.  The product path
 * (paper_2108_10591_b200/) never links, imports or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/pipesafe, read-only):
 *   - the numba kernels, kernels.py:95-137: strictly sequential ascending
 *     accumulation, no FMA contraction (built with -ffp-contract=off),
 *     left-associative evaluation exactly as written;
 *   - PartitionPlan.balanced, reduction.py:80-87 (np.linspace(0,n,W+1) floor);
 *   - ReductionEngine._range_partials/_combine, reduction.py:282-294: one
 *     sequential chain per plan range, then a fixed left-to-right combine;
 *   - guard_denominator / compute_alpha_beta_safe / compute_zeta_eta_safe,
 *     coefficients.py:35-106;
 *   - the solver loops _solve_pipelined (solvers.py:595-739, p-BiCGSafe and
 *     p-BiCGSafe-rr) and solve_ssbicgsafe2 (solvers.py:485-592), including
 *     the _Run bookkeeping (solvers.py:154-197) and the termination order;
 *   - the product-type comparators solve_bicgstab (solvers.py:210-327) and
 *     solve_gpbicg (solvers.py:330-460) with compute_zeta_eta_gpbicg
 *     (coefficients.py:109-135);
 *   - p-BiCGStab (Cools & Vanroose), which the reference does NOT ship: its
 *     restatement here (solve_pstab) follows the published algorithm with the
 *     reference BiCGStab's conventions and is pinned only through BiCGStab
 *     equivalence in exact arithmetic (tests/test_oracle.py) — parity for it
 *     is unpinned against reference outputs.
 *
 * Threads: rows of SpMV / vector updates are split across OpenMP threads
 * (element-wise, so bitwise neutral); the dot batch runs one thread per plan
 * range (each range a sequential chain) and combines left to right, so a run
 * with `workers = W` is bitwise identical to the reference driven by
 * ReductionEngine(PartitionPlan.balanced(n, W)) in either engine mode.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ kernels */

/* kernels.py:95-100 _spmv_range_nb */
OR_API void or_spmv_range(const int64_t* rp, const int64_t* ci, const double* v,
                          const double* x, double* out, int64_t lo, int64_t hi) {
#pragma omp parallel for schedule(static)
  for (int64_t i = lo; i < hi; ++i) {
    double acc = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc += v[k] * x[ci[k]];
    out[i] = acc;
  }
}

/* kernels.py:103-107 _dot_range_nb */
OR_API double or_dot_range(const double* x, const double* y, int64_t lo, int64_t hi) {
  double acc = 0.0;
  for (int64_t k = lo; k < hi; ++k) acc += x[k] * y[k];
  return acc;
}

/* kernels.py:110-112 */
OR_API void or_lincomb2(int64_t n, double* out, double sa, const double* a, double sb,
                        const double* b) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = sa * a[i] + sb * b[i];
}

/* kernels.py:115-117 */
OR_API void or_lincomb3(int64_t n, double* out, double sa, const double* a, double sb,
                        const double* b, double sc, const double* c) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = sa * a[i] + sb * b[i] + sc * c[i];
}

/* kernels.py:120-122 */
OR_API void or_lincomb4(int64_t n, double* out, double sa, const double* a, double sb,
                        const double* b, double sc, const double* c, double sd,
                        const double* d) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = sa * a[i] + sb * b[i] + sc * c[i] + sd * d[i];
}

/* kernels.py:125-127 */
OR_API void or_lincomb_nested(int64_t n, double* out, double sa, const double* a, double sb,
                              const double* b, double sc, const double* c) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = sa * a[i] + sb * (b[i] + sc * c[i]);
}

/* kernels.py:130-132 */
OR_API void or_add_scaled_diff(int64_t n, double* out, const double* base, double s,
                               const double* a, const double* b) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = base[i] + s * (a[i] - b[i]);
}

/* kernels.py:135-137 */
OR_API void or_add_scaled_damped_diff(int64_t n, double* out, const double* base, double s,
                                      const double* a, double w, const double* b) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = base[i] + s * (a[i] - w * b[i]);
}

/* --------------------------------------------------------------- the plan */

/* reduction.py:80-87 PartitionPlan.balanced: workers = min(W, max(n,1));
 * bounds = np.linspace(0, n, workers+1).astype(int64).  numpy computes
 * linspace as arange(num) * (delta/div) + start with the last point forced
 * to `stop`; astype(int64) truncates toward zero. */
OR_API int64_t or_plan_balanced(int64_t n, int64_t workers, int64_t* bounds) {
  if (workers < 1) return -1;
  int64_t cap = n > 1 ? n : 1;
  if (workers > cap) workers = cap;
  double step = (double)n / (double)workers;
  for (int64_t k = 0; k < workers; ++k) {
    double y = (step == 0.0) ? ((double)k / (double)workers) * (double)n : (double)k * step;
    bounds[k] = (int64_t)(y + 0.0);
  }
  bounds[workers] = n;
  return workers;
}

typedef struct {
  int64_t workers;
  int64_t* bounds;
  int compensated; /* near-exact dots instead of the plan's chains */
} or_plan;

/* Near-exact dot over [lo, hi): double-double accumulation with exact
 * products (Dekker TwoProduct, no FMA needed), rounded once at the end — in
 * all but pathological cases the correctly rounded dot, hence independent of
 * summation order.  The reference has no such mode; it is the order-free
 * yardstick for the GPU's double-double tree batch (iteration-count
 * parity). */
typedef struct {
  double hi, lo;
} dd_t;

static dd_t dd_add(dd_t a, dd_t b) {
  double s = a.hi + b.hi;
  double bb = s - a.hi;
  double e = (a.hi - (s - bb)) + (b.hi - bb);
  e = e + (a.lo + b.lo);
  double hi = s + e;
  dd_t r = {hi, e - (hi - s)};
  return r;
}

static dd_t two_prod(double a, double b) {
  const double sp = 134217729.0; /* 2^27 + 1 */
  double p = a * b;
  double ca = sp * a, cb = sp * b;
  double ah = ca - (ca - a), al = a - ah;
  double bh = cb - (cb - b), bl = b - bh;
  double err = ((ah * bh - p) + ah * bl + al * bh) + al * bl;
  dd_t r = {p, err};
  return r;
}

static double dot_compensated(const double* x, const double* y, int64_t lo, int64_t hi) {
  dd_t acc = {0.0, 0.0};
  for (int64_t k = lo; k < hi; ++k) acc = dd_add(acc, two_prod(x[k], y[k]));
  return acc.hi + acc.lo;
}


/* reduction.py:282-294: per range sequential partials, left-to-right combine */
static void plan_batch(const or_plan* P, int npairs, const double* const* xs,
                       const double* const* ys, double* out) {
  if (P->compensated) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int p = 0; p < npairs; ++p) out[p] = dot_compensated(xs[p], ys[p], 0, P->bounds[P->workers]);
    return;
  }
  int64_t W = P->workers;
  double* part = (double*)malloc(sizeof(double) * (size_t)(W * npairs));
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t w = 0; w < W; ++w)
    for (int p = 0; p < npairs; ++p)
      part[w * npairs + p] = or_dot_range(xs[p], ys[p], P->bounds[w], P->bounds[w + 1]);
  for (int p = 0; p < npairs; ++p) {
    double acc = part[p];
    for (int64_t w = 1; w < W; ++w) acc = acc + part[w * npairs + p];
    out[p] = acc;
  }
  free(part);
}

/* reduction.py:455-464 plan_dot */
static double plan_dot(const or_plan* P, const double* x, const double* y) {
  const double* xs[1] = {x};
  const double* ys[1] = {y};
  double out;
  plan_batch(P, 1, xs, ys, &out);
  return out;
}

OR_API double or_plan_dot(int64_t workers, int64_t n, const double* x, const double* y) {
  or_plan P;
  P.bounds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(workers + 2));
  P.workers = or_plan_balanced(n, workers, P.bounds);
  P.compensated = 0;
  double d = plan_dot(&P, x, y);
  free(P.bounds);
  return d;
}

/* ------------------------------------------------------------ coefficients */

#define BREAKDOWN_RTOL 1e-14 /* coefficients.py:19 */

/* Breakdown quantities, numbered in the order the reference names them
 * (coefficients.py:77, 80, 83, 102, 105). */
enum {
  Q_NONE = 0,
  Q_INITIAL_ALPHA = 1, /* "initial alpha denominator (r0*, s)" */
  Q_BETA = 2,          /* "beta denominator zeta_prev * f_prev" */
  Q_ALPHA = 3,         /* "alpha denominator g + beta*h" */
  Q_ZETA = 4,          /* "zeta denominator (s, s)" */
  Q_ZETA_ETA = 5,      /* "zeta/eta denominator a*b - c^2" */
  /* the product-type comparators (solvers.py:270-309, 390-450; coefficients.py:130-135) */
  Q_STAB_ALPHA = 6,    /* "alpha denominator (r0*, Ap)" */
  Q_STAB_OMEGA = 7,    /* "omega denominator (At, At)" */
  Q_STAB_BETA_OMEGA = 8, /* "beta denominator omega" */
  Q_BETA_F = 9,        /* "beta denominator (r0*, r)" */
  Q_GP_ZETA = 10,      /* "zeta denominator (At, At)" */
  Q_GP_ZETA_ETA = 11,  /* "zeta/eta denominator e*a - d^2" */
  Q_GP_BETA_ZETA = 12, /* "beta denominator zeta" */
  /* p-BiCGStab (not in the reference; see solve_pstab) */
  Q_PSTAB_ALPHA = 13,  /* "alpha denominator (r0*, w) + beta*((r0*, s) - omega*(r0*, z))" */
  Q_PSTAB_OMEGA = 14   /* "omega denominator (y, y)" */
};

/* coefficients.py:35-39 guard_denominator: returns nonzero on breakdown */
static int guard(double q, double scale) { return !isfinite(q) || fabs(q) <= BREAKDOWN_RTOL * scale; }

/* coefficients.py:60-84 */
static int alpha_beta_safe(double f, double f_prev, double g, double h, double alpha_prev,
                           double zeta_prev, int first, double* alpha, double* beta) {
  if (first) {
    if (guard(g, fabs(g))) return Q_INITIAL_ALPHA;
    *alpha = f / g;
    *beta = 0.0;
    return Q_NONE;
  }
  double denom_beta = zeta_prev * f_prev;
  if (guard(denom_beta, fabs(denom_beta))) return Q_BETA;
  double bt = (alpha_prev * f) / denom_beta;
  double denom_alpha = g + bt * h;
  if (guard(denom_alpha, fabs(g) + fabs(bt * h))) return Q_ALPHA;
  *alpha = f / denom_alpha;
  *beta = bt;
  return Q_NONE;
}

/* coefficients.py:87-106 */
static int zeta_eta_safe(double a, double b, double c, double d, double e, int first,
                         double* zeta, double* eta) {
  if (first || (b == 0.0 && c == 0.0 && e == 0.0)) {
    if (guard(a, fabs(a))) return Q_ZETA;
    *zeta = d / a;
    *eta = 0.0;
    return Q_NONE;
  }
  double det = a * b - c * c;
  if (guard(det, fabs(a * b) + c * c)) return Q_ZETA_ETA;
  *zeta = (b * d - c * e) / det;
  *eta = (a * e - c * d) / det;
  return Q_NONE;
}

OR_API int or_alpha_beta_safe(double f, double f_prev, double g, double h, double alpha_prev,
                              double zeta_prev, int first, double* out2) {
  return alpha_beta_safe(f, f_prev, g, h, alpha_prev, zeta_prev, first, &out2[0], &out2[1]);
}

OR_API int or_zeta_eta_safe(double a, double b, double c, double d, double e, int first,
                            double* out2) {
  return zeta_eta_safe(a, b, c, d, e, first, &out2[0], &out2[1]);
}

/* coefficients.py:109-135 compute_zeta_eta_gpbicg */
static int zeta_eta_gpbicg(double a, double b, double c, double d, double e, int first,
                           double* zeta, double* eta) {
  if (first || (a == 0.0 && c == 0.0 && d == 0.0)) {
    if (e == 0.0) {
      *zeta = 0.0;
      *eta = 0.0;
      return Q_NONE;
    }
    if (guard(e, fabs(e))) return Q_GP_ZETA;
    *zeta = b / e;
    *eta = 0.0;
    return Q_NONE;
  }
  double det = e * a - d * d;
  if (guard(det, fabs(e * a) + d * d)) return Q_GP_ZETA_ETA;
  *zeta = (a * b - c * d) / det;
  *eta = (e * c - d * b) / det;
  return Q_NONE;
}

OR_API int or_zeta_eta_gpbicg(double a, double b, double c, double d, double e, int first,
                              double* out2) {
  return zeta_eta_gpbicg(a, b, c, d, e, first, &out2[0], &out2[1]);
}

/* ------------------------------------------------------------------ solver */

enum { ST_CONVERGED = 0, ST_MAX_ITERS = 1, ST_BREAKDOWN = 2, ST_NON_FINITE = 3 };
enum { M_PBICGSAFE = 0, M_PBICGSAFE_RR = 1, M_SSBICGSAFE2 = 2, M_BICGSTAB = 3, M_GPBICG = 4, M_PBICGSTAB = 5 };

/* SpMV tags for the NonFiniteVectorError message (reduction.py:330, 451) */
enum { T_NONE = 0, T_AX = 1, T_AR = 2, T_AS = 3, T_AW = 4, T_AO = 5, T_AU = 6, T_AT = 7, T_AY = 8, T_AP = 9, T_AZ = 10 };

typedef struct {
  double tol;
  int64_t max_iters;
  int64_t rr_epoch;
  int64_t rr_cutoff; /* < 0: defaults to max_iters (solvers.py:634) */
  int32_t method;
  int32_t workers; /* PartitionPlan.balanced(n, workers) */
  int32_t threads; /* OpenMP threads; <= 0 keeps the runtime default */
  int32_t pad;
} or_config;

typedef struct {
  int32_t status;
  int32_t breakdown; /* Q_* */
  int64_t iterations;
  int64_t failure_iter; /* -1 = None */
  int64_t n_records;
  double r0_norm;
  int32_t nonfinite_tag; /* nonzero: NonFiniteVectorError raised from this SpMV */
  int32_t pad;
  int64_t nonfinite_index;
  int64_t n_spmv;
} or_result;

/* trace(i, vecs, scalars, user): vecs = x r p u o t w y z s q g l r0s
 * (14 arrays, live; copy them), scalars = alpha beta zeta eta f_prev + 9 dots */
typedef void (*or_trace_fn)(int64_t, double**, const double*, void*);

typedef struct {
  int64_t n;
  const int64_t *rp, *ci;
  const double* v;
  or_result* res;
} mat_t;

/* ReductionEngine.spmv + check_finite (reduction.py:418-453, linalg.py:142-146) */
static int spmv_checked(mat_t* A, const double* x, double* y, int tag) {
  or_spmv_range(A->rp, A->ci, A->v, x, y, 0, A->n);
  A->res->n_spmv++;
  for (int64_t i = 0; i < A->n; ++i)
    if (!isfinite(y[i])) {
      A->res->nonfinite_tag = tag;
      A->res->nonfinite_index = i;
      return 1;
    }
  return 0;
}

/* _Run.rel_of, solvers.py:176-179 */
static double rel_of(double r0_norm, double rr) {
  if (r0_norm == 0.0) return 0.0;
  double m = (0.0 > rr) ? 0.0 : rr; /* Python max(rr, 0.0) keeps rr unless 0.0 > rr */
  return sqrt(m) / r0_norm;
}

typedef struct {
  double* rel;        /* [max_iters+1] */
  uint8_t* replaced;  /* [max_iters+1] */
  double* coef;       /* [4*(max_iters+1)] alpha beta zeta eta */
  uint8_t* has_coef;  /* [max_iters+1] */
  int64_t count;
} hist_t;

static void record(hist_t* H, int64_t i, double rel, int replaced) {
  (void)i;
  H->rel[H->count] = rel;
  H->replaced[H->count] = (uint8_t)replaced;
  H->has_coef[H->count] = 0;
  H->count++;
}

static void set_coef(hist_t* H, double a, double b, double z, double e) {
  int64_t k = H->count - 1;
  H->coef[4 * k + 0] = a;
  H->coef[4 * k + 1] = b;
  H->coef[4 * k + 2] = z;
  H->coef[4 * k + 3] = e;
  H->has_coef[k] = 1;
}

#define VEC(name) double* name = buf + (size_t)(idx++) * (size_t)n

/* _safe_batch order (solvers.py:467-482) packed as BATCH_LABELS a..h, r */
static void safe_batch(const or_plan* P, const double* s, const double* y, const double* r,
                       const double* r0s, const double* t, double* d9) {
  const double* xs[9] = {s, y, s, s, y, r0s, r0s, r0s, r};
  const double* ys[9] = {s, y, y, r, r, r, s, t, r};
  plan_batch(P, 9, xs, ys, d9);
}

/* The two product-type comparators with their reduction phases:
 *   BiCGStab  solvers.py:210-327 (2 phases: g after A p; b e c d after A t)
 *   GPBi-CG   solvers.py:330-460 (3 phases: g; a b c d e after A t; f r)
 * The coefficient record holds alpha beta zeta eta, with BiCGStab's omega
 * in the zeta slot.  trace vecs: x r p t Ap At (BiCGStab) or
 * x r p u t w y z (GPBi-CG); scalars alpha beta omega|zeta eta f rr. */
static int solve_product(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                         const double* b, const double* x0, const or_config* cfg, double* x_out,
                         double* hist_rel, uint8_t* hist_replaced, double* hist_coef,
                         uint8_t* hist_has_coef, or_result* res, or_trace_fn trace, void* user) {
  mat_t A = {n, rp, ci, v, res};
  or_plan P;
  int32_t wk = cfg->workers < 0 ? 1 : cfg->workers;
  P.bounds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(wk + 2));
  P.workers = or_plan_balanced(n, wk, P.bounds);
  P.compensated = cfg->workers < 0;
  hist_t H = {hist_rel, hist_replaced, hist_coef, hist_has_coef, 0};
  const int gp = cfg->method == M_GPBICG;
  double* buf = (double*)calloc((size_t)12 * (size_t)(n > 0 ? n : 1), sizeof(double));
  int idx = 0;
  VEC(x); VEC(r); VEC(r0s); VEC(p); VEC(u); VEC(t); VEC(w); VEC(y); VEC(z);
  VEC(ap); VEC(at); VEC(tmp);
  if (x0) memcpy(x, x0, sizeof(double) * (size_t)n);
  int rc = 0;
  int64_t iterations = 0;
  double r0_norm = 0.0;
  /* r0 = b - A x0 ; r0s = r0 ; rr = (r, r) ; f = rr (solvers.py:238-248, 359-369) */
  if (spmv_checked(&A, x, tmp, T_AX)) { rc = 1; goto done; }
  or_lincomb2(n, r, 1.0, b, -1.0, tmp);
  memcpy(r0s, r, sizeof(double) * (size_t)n);
  double rr = plan_dot(&P, r, r);
  double f = rr;
  r0_norm = sqrt(rr);
  double alpha = 0.0, beta = 0.0, omega = 0.0, zeta = 0.0, eta = 0.0;
  for (int64_t i = 0; i < cfg->max_iters; ++i) {
    double rel = rel_of(r0_norm, rr);
    record(&H, i, rel, 0);
    if (!isfinite(rel)) { res->status = ST_NON_FINITE; res->failure_iter = i; iterations = i; goto finish; }
    if (rel <= cfg->tol) { res->status = ST_CONVERGED; iterations = i; goto finish; }
    int q = Q_NONE;
    if (gp)
      or_add_scaled_diff(n, p, r, beta, p, u);               /* p = r + beta*(p - u) */
    else
      or_add_scaled_damped_diff(n, p, r, beta, p, omega, ap); /* p = r + beta*(p - omega*Ap) */
    if (spmv_checked(&A, p, ap, T_AP)) { rc = 1; goto done; }
    double gdot = plan_dot(&P, r0s, ap);
    if (guard(gdot, fabs(gdot))) { q = Q_STAB_ALPHA; goto broke; }
    alpha = f / gdot;
    if (gp) {
      or_lincomb4(n, y, 1.0, t, -1.0, r, -alpha, w, alpha, ap); /* y = t - r - alpha w + alpha Ap */
      or_lincomb3(n, u, 1.0, t, -1.0, r, beta, u);              /* u = t - r + beta u (stash) */
    }
    or_lincomb2(n, t, 1.0, r, -alpha, ap);                      /* t = r - alpha*Ap */
    if (spmv_checked(&A, t, at, T_AT)) { rc = 1; goto done; }
    if (!gp) {
      const double* xs[4] = {at, at, r0s, t};
      const double* ys[4] = {t, at, at, t};
      double d4[4]; /* b e c d */
      plan_batch(&P, 4, xs, ys, d4);
      if (d4[1] == 0.0 && d4[3] == 0.0) {
        omega = 0.0;
      } else {
        if (guard(d4[1], fabs(d4[1]))) { q = Q_STAB_OMEGA; goto broke; }
        omega = d4[0] / d4[1];
      }
      or_lincomb3(n, x, 1.0, x, alpha, p, omega, t); /* x = x + alpha*p + omega*t */
      or_lincomb2(n, r, 1.0, t, -omega, at);         /* r = t - omega*At */
      double f_next = (f - alpha * gdot) - omega * d4[2];
      double v2 = d4[3] - 2.0 * omega * d4[0] + omega * omega * d4[1];
      rr = (0.0 > v2) ? 0.0 : v2; /* Python max(v, 0.0) */
      if (rr == 0.0) {
        beta = 0.0;
      } else {
        if (guard(omega, fabs(omega))) { q = Q_STAB_BETA_OMEGA; goto broke; }
        if (guard(f, fabs(f))) { q = Q_BETA_F; goto broke; }
        beta = (alpha / omega) * (f_next / f);
      }
      f = f_next;
      set_coef(&H, alpha, beta, omega, NAN);
      if (!(isfinite(alpha) && isfinite(beta) && isfinite(omega))) {
        res->status = ST_NON_FINITE; res->failure_iter = i; iterations = i; goto finish;
      }
      if (trace) {
        double* vecs[6] = {x, r, p, t, ap, at};
        double sc[14] = {alpha, beta, omega, 0.0, f, rr};
        trace(i, vecs, sc, user);
      }
    } else {
      const double* xs[5] = {y, at, y, at, at};
      const double* ys[5] = {y, t, t, y, at};
      double d5[5]; /* a b c d e */
      plan_batch(&P, 5, xs, ys, d5);
      q = zeta_eta_gpbicg(d5[0], d5[1], d5[2], d5[3], d5[4], i == 0, &zeta, &eta);
      if (q) goto broke;
      or_lincomb2(n, u, zeta, ap, eta, u);             /* u = zeta*Ap + eta*(stash) */
      or_lincomb3(n, z, zeta, r, eta, z, -alpha, u);   /* z = zeta*r + eta*z - alpha*u */
      or_lincomb3(n, x, 1.0, x, alpha, p, 1.0, z);     /* x = x + alpha*p + z */
      or_lincomb3(n, r, 1.0, t, -eta, y, -zeta, at);   /* r = t - eta*y - zeta*At */
      const double* xs3[2] = {r0s, r};
      const double* ys3[2] = {r, r};
      double d2[2]; /* f r */
      plan_batch(&P, 2, xs3, ys3, d2);
      rr = d2[1];
      if (rr == 0.0) {
        beta = 0.0;
      } else {
        if (guard(zeta, fabs(zeta))) { q = Q_GP_BETA_ZETA; goto broke; }
        if (guard(f, fabs(f))) { q = Q_BETA_F; goto broke; }
        beta = (alpha / zeta) * (d2[0] / f);
      }
      f = d2[0];
      or_lincomb2(n, w, 1.0, at, beta, ap);            /* w = At + beta*Ap */
      set_coef(&H, alpha, beta, zeta, eta);
      if (!(isfinite(alpha) && isfinite(beta) && isfinite(zeta) && isfinite(eta))) {
        res->status = ST_NON_FINITE; res->failure_iter = i; iterations = i; goto finish;
      }
      if (trace) {
        double* vecs[8] = {x, r, p, u, t, w, y, z};
        double sc[14] = {alpha, beta, zeta, eta, f, rr};
        trace(i, vecs, sc, user);
      }
    }
    iterations = i + 1;
    continue;
  broke:
    res->status = ST_BREAKDOWN;
    res->breakdown = q;
    res->failure_iter = i;
    iterations = i;
    goto finish;
  }
  {
    double rel = rel_of(r0_norm, rr); /* solvers.py:324-327, 457-460 */
    record(&H, cfg->max_iters, rel, 0);
    res->status = rel <= cfg->tol ? ST_CONVERGED : ST_MAX_ITERS;
    iterations = cfg->max_iters;
  }
finish:
  res->iterations = iterations;
  res->r0_norm = r0_norm;
  res->n_records = H.count;
  memcpy(x_out, x, sizeof(double) * (size_t)n);
done:
  free(buf);
  free(P.bounds);
  return rc;
}

/* p-BiCGStab: the pipelined BiCGStab of Cools & Vanroose (2017), the
 * comparator the paper cites for Table 3 (its algorithm
 * is NOT in the reference).  It maintains w = A r, s = A p,
 * z = A s, t = A w, v = A z, q = r - alpha s, y = w - alpha z (= A q) by
 * recurrences, so each of its two reduction phases is followed by an
 * independent product it can overlap: (q,y) (y,y) with v = A z, and the
 * five dots of the next alpha / beta / convergence check with t = A w.
 * Conventions follow the reference's solve_bicgstab (solvers.py:210-327):
 * shadow residual r0* = r0, f = (r0*, r), check order (record, non-finite,
 * converged, then guards), the t = 0 omega rule, the rr == 0 beta rule, the
 * BiCGStab breakdown guards (coefficients.py:35-39) and the coefficient
 * record (alpha, beta, omega).  The alpha denominator is (r0*, A p) by its
 * recurrence: (r0*, w) + beta*((r0*, s) - omega*(r0*, z)).
 *
 *   setup   r = b - A x0; r0* = r; w = A r; rr = (r, r), gw = (r0*, w)
 *   loop i  check i; alpha = f / (gw + beta*(sd - omega*zd)); t = A w
 *           p = r + beta*(p - omega s); s = w + beta*(s - omega z)
 *           z = t + beta*(z - omega v); q = r - alpha s; y = w - alpha z
 *           [b = (q, y), e = (y, y), d = (q, q)]  v = A z
 *           omega = b / e (0 when e = d = 0)
 *           x = x + alpha p + omega q; r = q - omega y; w = y - omega (t - alpha v)
 *           [f' = (r0*, r), rr = (r, r), gw = (r0*, w), sd = (r0*, s), zd = (r0*, z)]
 *           beta = (alpha / omega) (f' / f) (0 when rr = 0); record (alpha, beta, omega)
 *
 * trace vecs: x r p s z q y w t v; scalars alpha beta omega 0 f rr. */
static int solve_pstab(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                       const double* b, const double* x0, const or_config* cfg, double* x_out,
                       double* hist_rel, uint8_t* hist_replaced, double* hist_coef,
                       uint8_t* hist_has_coef, or_result* res, or_trace_fn trace, void* user) {
  mat_t A = {n, rp, ci, v, res};
  or_plan P;
  int32_t wk = cfg->workers < 0 ? 1 : cfg->workers;
  P.bounds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(wk + 2));
  P.workers = or_plan_balanced(n, wk, P.bounds);
  P.compensated = cfg->workers < 0;
  hist_t H = {hist_rel, hist_replaced, hist_coef, hist_has_coef, 0};
  double* buf = (double*)calloc((size_t)12 * (size_t)(n > 0 ? n : 1), sizeof(double));
  int idx = 0;
  VEC(x); VEC(r); VEC(r0s); VEC(p); VEC(s); VEC(z); VEC(q); VEC(y); VEC(w); VEC(t); VEC(av);
  VEC(tmp);
  if (x0) memcpy(x, x0, sizeof(double) * (size_t)n);
  int rc = 0;
  int64_t iterations = 0;
  double r0_norm = 0.0;
  if (spmv_checked(&A, x, tmp, T_AX)) { rc = 1; goto done; }
  or_lincomb2(n, r, 1.0, b, -1.0, tmp); /* r0 = b - A x0 */
  memcpy(r0s, r, sizeof(double) * (size_t)n);
  if (spmv_checked(&A, r, w, T_AR)) { rc = 1; goto done; } /* w0 = A r0 */
  double rr, gw;
  {
    const double* xs[2] = {r, r0s};
    const double* ys[2] = {r, w};
    double d2[2];
    plan_batch(&P, 2, xs, ys, d2);
    rr = d2[0];
    gw = d2[1];
  }
  double f = rr; /* (r0*, r0) = ||r0||^2 */
  r0_norm = sqrt(rr);
  double alpha = 0.0, beta = 0.0, omega = 0.0, sd = 0.0, zd = 0.0;
  for (int64_t i = 0; i < cfg->max_iters; ++i) {
    double rel = rel_of(r0_norm, rr);
    record(&H, i, rel, 0);
    if (!isfinite(rel)) { res->status = ST_NON_FINITE; res->failure_iter = i; iterations = i; goto finish; }
    if (rel <= cfg->tol) { res->status = ST_CONVERGED; iterations = i; goto finish; }
    int q_bd = Q_NONE;
    {
      const double bt = beta * (sd - omega * zd);
      const double den = gw + bt;
      if (guard(den, fabs(gw) + fabs(bt))) { q_bd = Q_PSTAB_ALPHA; goto broke; }
      alpha = f / den;
    }
    if (spmv_checked(&A, w, t, T_AW)) { rc = 1; goto done; } /* t = A w */
    or_add_scaled_damped_diff(n, p, r, beta, p, omega, s);   /* p = r + beta*(p - omega*s) */
    or_add_scaled_damped_diff(n, s, w, beta, s, omega, z);   /* s = w + beta*(s - omega*z) */
    or_add_scaled_damped_diff(n, z, t, beta, z, omega, av);  /* z = t + beta*(z - omega*v) */
    or_lincomb2(n, q, 1.0, r, -alpha, s);                    /* q = r - alpha*s */
    or_lincomb2(n, y, 1.0, w, -alpha, z);                    /* y = w - alpha*z */
    double d3[3]; /* b e d */
    {
      const double* xs[3] = {q, y, q};
      const double* ys[3] = {y, y, q};
      plan_batch(&P, 3, xs, ys, d3);
    }
    if (spmv_checked(&A, z, av, T_AZ)) { rc = 1; goto done; } /* v = A z */
    if (d3[1] == 0.0 && d3[2] == 0.0) {
      omega = 0.0; /* q = 0: the alpha half-step already landed */
    } else {
      if (guard(d3[1], fabs(d3[1]))) { q_bd = Q_PSTAB_OMEGA; goto broke; }
      omega = d3[0] / d3[1];
    }
    or_lincomb3(n, x, 1.0, x, alpha, p, omega, q);           /* x = x + alpha*p + omega*q */
    or_lincomb2(n, r, 1.0, q, -omega, y);                    /* r = q - omega*y */
    or_add_scaled_damped_diff(n, w, y, -omega, t, alpha, av); /* w = y - omega*(t - alpha*v) */
    double d5[5]; /* f' rr gw sd zd */
    {
      const double* xs[5] = {r0s, r, r0s, r0s, r0s};
      const double* ys[5] = {r, r, w, s, z};
      plan_batch(&P, 5, xs, ys, d5);
    }
    rr = d5[1];
    if (rr == 0.0) {
      beta = 0.0;
    } else {
      if (guard(omega, fabs(omega))) { q_bd = Q_STAB_BETA_OMEGA; goto broke; }
      if (guard(f, fabs(f))) { q_bd = Q_BETA_F; goto broke; }
      beta = (alpha / omega) * (d5[0] / f);
    }
    f = d5[0];
    gw = d5[2];
    sd = d5[3];
    zd = d5[4];
    set_coef(&H, alpha, beta, omega, NAN);
    if (!(isfinite(alpha) && isfinite(beta) && isfinite(omega))) {
      res->status = ST_NON_FINITE; res->failure_iter = i; iterations = i; goto finish;
    }
    if (trace) {
      double* vecs[10] = {x, r, p, s, z, q, y, w, t, av};
      double sc[14] = {alpha, beta, omega, 0.0, f, rr};
      trace(i, vecs, sc, user);
    }
    iterations = i + 1;
    continue;
  broke:
    res->status = ST_BREAKDOWN;
    res->breakdown = q_bd;
    res->failure_iter = i;
    iterations = i;
    goto finish;
  }
  {
    double rel = rel_of(r0_norm, rr);
    record(&H, cfg->max_iters, rel, 0);
    res->status = rel <= cfg->tol ? ST_CONVERGED : ST_MAX_ITERS;
    iterations = cfg->max_iters;
  }
finish:
  res->iterations = iterations;
  res->r0_norm = r0_norm;
  res->n_records = H.count;
  memcpy(x_out, x, sizeof(double) * (size_t)n);
done:
  free(buf);
  free(P.bounds);
  return rc;
}

/* solvers.py:595-739 (_solve_pipelined) and solvers.py:485-592 (ssBiCGSafe2).
 * Returns 0, or 1 when a NonFiniteVectorError would have been raised. */
OR_API int or_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    const double* b, const double* x0, const or_config* cfg, double* x_out,
                    double* hist_rel, uint8_t* hist_replaced, double* hist_coef,
                    uint8_t* hist_has_coef, or_result* res, or_trace_fn trace, void* user) {
#ifdef _OPENMP
  if (cfg->threads > 0) omp_set_num_threads(cfg->threads);
#endif
  memset(res, 0, sizeof(*res));
  res->failure_iter = -1;
  res->nonfinite_index = -1;
  if (cfg->method == M_BICGSTAB || cfg->method == M_GPBICG)
    return solve_product(n, rp, ci, v, b, x0, cfg, x_out, hist_rel, hist_replaced, hist_coef,
                         hist_has_coef, res, trace, user);
  if (cfg->method == M_PBICGSTAB)
    return solve_pstab(n, rp, ci, v, b, x0, cfg, x_out, hist_rel, hist_replaced, hist_coef,
                       hist_has_coef, res, trace, user);
  mat_t A = {n, rp, ci, v, res};
  or_plan P;
  int32_t wk = cfg->workers < 0 ? 1 : cfg->workers;
  P.bounds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(wk + 2));
  P.workers = or_plan_balanced(n, wk, P.bounds);
  P.compensated = cfg->workers < 0; /* workers < 0: near-exact dots (order-free yardstick) */
  hist_t H = {hist_rel, hist_replaced, hist_coef, hist_has_coef, 0};
  const int pipelined = cfg->method != M_SSBICGSAFE2;
  const int replace_residuals = cfg->method == M_PBICGSAFE_RR;

  double* buf = (double*)calloc((size_t)17 * (size_t)(n > 0 ? n : 1), sizeof(double));
  int idx = 0;
  VEC(x); VEC(r); VEC(r0s); VEC(p); VEC(u); VEC(t); VEC(y); VEC(z);
  VEC(g); VEC(l); VEC(w); VEC(o); VEC(q); VEC(s); VEC(as); VEC(aw); VEC(tmp);
  if (x0) memcpy(x, x0, sizeof(double) * (size_t)n); /* _prepare copies x0 */

  int rc = 0;
  double d9[9];
  double alpha = 0.0, beta = 0.0, zeta = 0.0, eta = 0.0, f_prev = 0.0;
  double r0_norm = 0.0;
  int pending_replaced = 0;
  int64_t epoch = cfg->rr_epoch;
  int64_t cutoff = cfg->rr_cutoff >= 0 ? cfg->rr_cutoff : cfg->max_iters;
  int64_t iterations = 0;

  /* setup: r0 = b - A x0 ; r0s = r0 ; [pipelined] s0 = A r0 */
  if (spmv_checked(&A, x, tmp, T_AX)) { rc = 1; goto done; }
  or_lincomb2(n, r, 1.0, b, -1.0, tmp);
  memcpy(r0s, r, sizeof(double) * (size_t)n);
  if (pipelined && spmv_checked(&A, r, s, T_AR)) { rc = 1; goto done; }

  for (int64_t i = 0; i < cfg->max_iters; ++i) {
    int first = i == 0;
    if (pipelined) {
      /* engine.overlap: batch (reduce) then As (solvers.py:641) */
      safe_batch(&P, s, y, r, r0s, t, d9);
      if (spmv_checked(&A, s, as, T_AS)) { rc = 1; goto done; }
    } else {
      if (spmv_checked(&A, r, s, T_AR)) { rc = 1; goto done; } /* solvers.py:530 */
      safe_batch(&P, s, y, r, r0s, t, d9);
    }
    if (first) {
      /* the first batch only holds a, d, f, g, r (solvers.py:469) */
      d9[1] = d9[2] = d9[4] = d9[7] = 0.0;
      r0_norm = sqrt(d9[8]);
    }
    double rel = rel_of(r0_norm, d9[8]);
    record(&H, i, rel, pending_replaced);
    pending_replaced = 0;
    if (!isfinite(rel)) { res->status = ST_NON_FINITE; res->failure_iter = i; iterations = i; goto finish; }
    if (rel <= cfg->tol) { res->status = ST_CONVERGED; iterations = i; goto finish; }
    {
      int q = alpha_beta_safe(d9[5], f_prev, d9[6], d9[7], alpha, zeta, first, &alpha, &beta);
      if (!q) q = zeta_eta_safe(d9[0], d9[1], d9[2], d9[3], d9[4], first, &zeta, &eta);
      if (q) { res->status = ST_BREAKDOWN; res->breakdown = q; res->failure_iter = i; iterations = i; goto finish; }
    }
    f_prev = d9[5];
    set_coef(&H, alpha, beta, zeta, eta);
    if (!(isfinite(alpha) && isfinite(beta) && isfinite(zeta) && isfinite(eta))) {
      res->status = ST_NON_FINITE; res->failure_iter = i; iterations = i; goto finish;
    }

    if (pipelined) {
      int replace = replace_residuals && (i % epoch == 0) && 0 < i && i < cutoff;
      or_add_scaled_diff(n, p, r, beta, p, u);         /* p = r + beta*(p - u) */
      or_lincomb2(n, o, 1.0, s, beta, t);              /* o = s + beta*t */
      or_lincomb_nested(n, u, zeta, o, eta, y, beta, u); /* u = zeta*o + eta*(y + beta*u) */
      if (replace) {
        if (spmv_checked(&A, o, q, T_AO)) { rc = 1; goto done; }
        if (spmv_checked(&A, u, w, T_AU)) { rc = 1; goto done; }
      } else {
        or_lincomb2(n, q, 1.0, as, beta, l);             /* q = As + beta*l */
        or_lincomb_nested(n, w, zeta, q, eta, g, beta, w); /* w = zeta*q + eta*(g + beta*w) */
      }
      or_lincomb2(n, t, 1.0, o, -1.0, w);                /* t = o - w */
      or_lincomb3(n, z, zeta, r, eta, z, -alpha, u);     /* z = zeta*r + eta*z - alpha*u */
      or_lincomb3(n, y, zeta, s, eta, y, -alpha, w);     /* y = zeta*s + eta*y - alpha*w */
      or_lincomb3(n, x, 1.0, x, alpha, p, 1.0, z);       /* x = x + alpha*p + z */
      if (replace) {
        if (spmv_checked(&A, x, tmp, T_AX)) { rc = 1; goto done; }
        or_lincomb2(n, r, 1.0, b, -1.0, tmp);            /* r = b - A x */
        if (spmv_checked(&A, t, l, T_AT)) { rc = 1; goto done; }
        if (spmv_checked(&A, y, g, T_AY)) { rc = 1; goto done; }
        if (spmv_checked(&A, r, s, T_AR)) { rc = 1; goto done; }
        pending_replaced = 1;
      } else {
        or_lincomb3(n, r, 1.0, r, -alpha, o, -1.0, y);   /* r = r - alpha*o - y */
        if (spmv_checked(&A, w, aw, T_AW)) { rc = 1; goto done; }
        or_lincomb2(n, l, 1.0, q, -1.0, aw);             /* l = q - A w */
        or_lincomb3(n, g, zeta, as, eta, g, -alpha, aw); /* g = zeta*As + eta*g - alpha*Aw */
        or_lincomb3(n, s, 1.0, s, -alpha, q, -1.0, g);   /* s = s - alpha*q - g */
      }
    } else {
      /* solvers.py:563-580 */
      or_add_scaled_diff(n, p, r, beta, p, u);
      or_lincomb2(n, o, 1.0, s, beta, t);
      or_lincomb_nested(n, u, zeta, o, eta, y, beta, u);
      if (spmv_checked(&A, u, w, T_AU)) { rc = 1; goto done; }
      or_lincomb2(n, t, 1.0, o, -1.0, w);
      or_lincomb3(n, z, zeta, r, eta, z, -alpha, u);
      or_lincomb3(n, y, zeta, s, eta, y, -alpha, w);
      or_lincomb3(n, x, 1.0, x, alpha, p, 1.0, z);
      or_lincomb3(n, r, 1.0, r, -alpha, o, -1.0, y);
    }
    if (trace) {
      double* vecs[14] = {x, r, p, u, o, t, w, y, z, s, q, g, l, r0s};
      double sc[14] = {alpha, beta, zeta, eta, f_prev};
      memcpy(sc + 5, d9, sizeof(d9));
      trace(i, vecs, sc, user);
    }
    iterations = i + 1;
  }
  {
    /* solvers.py:736-739 / 589-592 */
    double rel = rel_of(r0_norm, plan_dot(&P, r, r));
    record(&H, cfg->max_iters, rel, pending_replaced);
    res->status = rel <= cfg->tol ? ST_CONVERGED : ST_MAX_ITERS;
    iterations = cfg->max_iters;
  }
finish:
  res->iterations = iterations;
  res->r0_norm = r0_norm;
  res->n_records = H.count;
  memcpy(x_out, x, sizeof(double) * (size_t)n);
done:
  free(buf);
  free(P.bounds);
  return rc;
}
