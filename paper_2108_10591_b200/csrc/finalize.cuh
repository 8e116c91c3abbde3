// finalize.cuh — the coefficient step and _Run bookkeeping of one check
// (solvers.py:645-674, 736-739; coefficients.py:35-106), the deterministic
// reduction of the dot-batch partials, and two ways to run them: fused into
// the tail of the kernel that produced the partials (the last CTA to finish,
// by ticket) or as a separate 1-CTA kernel (plan order, multi-GPU, step seam).
#pragma once
#include "common.cuh"

namespace pbs {

__device__ __forceinline__ bool guard(double q, double scale) {
  return !isfinite(q) || fabs(q) <= mul(1e-14, scale);
}

// The check's three independent computations, one thread each so their
// division / square-root chains run side by side: the relative residual
// (_Run.rel_of), compute_alpha_beta_safe, compute_zeta_eta_safe.  The commit
// then applies the reference's control flow to them (a breakdown in
// alpha/beta wins over one in zeta/eta, as the reference raises it first).
struct CheckVals {
  double r0_norm, rel;
  double alpha, beta;
  int q_ab;
  double zeta, eta;
  int q_ze;
  double f;  // this check's f, the next check's f_prev
};

__device__ __forceinline__ void check_rel(const SolverState* st, bool first, const double* d, CheckVals* cv) {
  const double r0n = first ? sqrt(d[DR]) : st->r0_norm;
  // _Run.rel_of (solvers.py:176-179): Python max(rr, 0.0) keeps rr unless 0.0 > rr
  double rel;
  if (r0n == 0.0) {
    rel = 0.0;
  } else {
    const double m = (0.0 > d[DR]) ? 0.0 : d[DR];
    rel = sqrt(m) / r0n;
  }
  cv->r0_norm = r0n;
  cv->rel = rel;
}

// compute_alpha_beta_safe (coefficients.py:60-84)
__device__ __forceinline__ void check_ab(const SolverState* st, bool first, const double* d, CheckVals* cv) {
  const double f = d[DF], g = d[DG], h = first ? 0.0 : d[DH];
  double alpha = 0.0, beta = 0.0;
  int q = PBS_BD_NONE;
  if (first) {
    if (guard(g, fabs(g))) q = PBS_BD_INITIAL_ALPHA;
    alpha = f / g;
    beta = 0.0;
  } else {
    const double denom_beta = mul(st->zeta, st->f_prev);
    if (guard(denom_beta, fabs(denom_beta))) {
      q = PBS_BD_BETA;
    } else {
      beta = mul(st->alpha, f) / denom_beta;
      const double bh = mul(beta, h);
      const double denom_alpha = add(g, bh);
      if (guard(denom_alpha, add(fabs(g), fabs(bh)))) q = PBS_BD_ALPHA;
      alpha = f / denom_alpha;
    }
  }
  cv->alpha = alpha;
  cv->beta = beta;
  cv->q_ab = q;
  cv->f = f;
}

// compute_zeta_eta_safe (coefficients.py:87-106)
__device__ __forceinline__ void check_ze(bool first, const double* d, CheckVals* cv) {
  double zeta = 0.0, eta = 0.0;
  int q = PBS_BD_NONE;
  const double a = d[DA], b = first ? 0.0 : d[DB], c = first ? 0.0 : d[DC], dd = d[DD], e = first ? 0.0 : d[DE];
  if (first || (b == 0.0 && c == 0.0 && e == 0.0)) {
    if (guard(a, fabs(a))) q = PBS_BD_ZETA;
    zeta = dd / a;
    eta = 0.0;
  } else {
    const double ab = mul(a, b), cc = mul(c, c);
    const double det = sub(ab, cc);
    if (guard(det, add(fabs(ab), cc))) {
      q = PBS_BD_ZETA_ETA;
    } else {
      zeta = sub(mul(b, dd), mul(c, e)) / det;
      eta = sub(mul(a, e), mul(c, dd)) / det;
    }
  }
  cv->zeta = zeta;
  cv->eta = eta;
  cv->q_ze = q;
}

// Bookkeeping of check j (solvers.py:645-674, 736-739) on precomputed values.
// One thread.
static __device__ void check_commit(SolverState* st, long long j, const CheckVals& cv, int replaced) {
  const bool first = j == 0;
  if (first) st->r0_norm = cv.r0_norm;
  const double rel = cv.rel;
  long long slot = st->n_records;
  if (st->record_history) {
    st->hist_rel[slot] = rel;
    st->hist_flags[slot] = replaced ? PBS_HIST_REPLACED : 0;
    st->n_records = slot + 1;
  }
  auto stop = [&](int status, long long iters, bool failure) {
    st->status = status;
    st->iterations = iters;
    if (failure) st->failure_iter = j;
    st->stop_check = j;
    st->run_all = 0;
    if (st->spine_done) st->run_spine = 0;
  };
  if (j == st->max_iters) {  // final record after the loop
    stop(rel <= st->tol ? PBS_CONVERGED : PBS_MAX_ITERS, st->max_iters, false);
    st->run_spine = 0;
    return;
  }
  if (!isfinite(rel)) return stop(PBS_NON_FINITE, j, true);
  if (rel <= st->tol) return stop(PBS_CONVERGED, j, false);
  const int q = cv.q_ab != PBS_BD_NONE ? cv.q_ab : cv.q_ze;
  if (q != PBS_BD_NONE) {
    st->breakdown = q;
    return stop(PBS_BREAKDOWN, j, true);
  }
  st->alpha = cv.alpha;
  st->beta = cv.beta;
  st->zeta = cv.zeta;
  st->eta = cv.eta;
  st->f_prev = cv.f;
  if (st->record_history) {
    st->hist_coef[4 * slot + 0] = cv.alpha;
    st->hist_coef[4 * slot + 1] = cv.beta;
    st->hist_coef[4 * slot + 2] = cv.zeta;
    st->hist_coef[4 * slot + 3] = cv.eta;
    st->hist_flags[slot] |= PBS_HIST_HAS_COEF;
  }
  if (!(isfinite(cv.alpha) && isfinite(cv.beta) && isfinite(cv.zeta) && isfinite(cv.eta)))
    return stop(PBS_NON_FINITE, j, true);
}

// The check's working copy of the state.  The check is one thread's chain of
// dependent reads and writes; run against global memory every read after a
// write is another L2 round trip.  Instead the CTA loads the state into
// shared memory in one round (overlapping the partials' reduction), thread 0
// edits the copy, and the block the check owns (carried scalars .. n_records)
// is written back.
constexpr int kStateWords = (int)(sizeof(SolverState) / 8);

template <int NT>
__device__ __forceinline__ void state_load(const SolverState* st, SolverState* ss) {
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(st);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(ss);
  for (int k = threadIdx.x; k < kStateWords; k += NT) dst[k] = __ldcg(src + k);
}

__device__ __forceinline__ void state_store(SolverState* st, const SolverState* ss) {
  constexpr int w0 = (int)(offsetof(SolverState, alpha) / 8), w1 = (int)(offsetof(SolverState, nf_row) / 8);
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(ss);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(st);
#pragma unroll
  for (int k = w0; k < w1; ++k) dst[k] = src[k];
}

// check j on the shared copy (its three computations in threads 0, 32, 64),
// write back, mirror to the host.  Called by all NT threads after the copy
// and dots are visible.
template <int NT, bool NAMED>
__device__ __forceinline__ void check_and_publish(SolverState* st, SolverState* ss, const double* dots,
                                                  int replaced) {
  __shared__ CheckVals cv;
  const long long j = ss->iter;
  const bool first = j == 0;
  const bool work = !dev_err(ss) && ss->run_all;
  if (work) {
    if (threadIdx.x == 0) check_rel(ss, first, dots, &cv);
    else if (threadIdx.x == 32) check_ab(ss, first, dots, &cv);
    else if (threadIdx.x == 64) check_ze(first, dots, &cv);
  }
  block_bar<NT, NAMED>();
  if (threadIdx.x != 0) return;
  if (work) {
    for (int k = 0; k < kNumDots; ++k) ss->dots[k] = dots[k];
    check_commit(ss, j, cv, replaced);
  } else if (!dev_err(ss)) {
    ss->run_spine = 0;  // the stop iteration's spine product has run
  }
  ss->iter = j + 1;
  state_store(st, ss);
  // host mirror: posted stores, no fence (a stale field only delays the host's
  // stop by one poll; every launch is gated on the device state anyway)
  if (ss->mirror) {
    ss->mirror->iter = j + 1;
    ss->mirror->run_all = ss->run_all;
    ss->mirror->err = dev_err(ss) ? 1 : 0;
  }
}

// ---- the product-type comparators: BiCGStab (solvers.py:210-327) and
// GPBi-CG (solvers.py:330-460).  Their coefficient steps are split across
// the iteration's reduction phases; each phase runs in the tail of the kernel
// that produced its dots (or a 1-CTA finalize in plan order):
//   setup      (r, r)                 -> r0_norm, f, check 0          (solvers.py:244-266)
//   alpha      g = (r0*, Ap)          -> alpha                        (269-276, 385-392)
//   stab omega b e c d after A t      -> omega, x/r go-ahead, f, rr,  (283-317)
//                                        beta, record, check i+1
//   gp zeta    a b c d e after A t    -> zeta, eta                    (401-413)
//   gp beta    f, r after x/r update  -> beta, f, record, check i+1   (421-450)
// ("no check" variants leave check i+1 to kPhProdCheck so a trace hook can
// run between them, as in the reference.)
enum Phase {
  kPhSafe = 0,
  kPhProdSetup,
  kPhProdAlpha,
  kPhStabOmega,
  kPhStabOmegaNC,
  kPhGpZeta,
  kPhGpBeta,
  kPhGpBetaNC,
  kPhProdCheck,
  // p-BiCGStab (oracle solve_pstab)
  kPhPsSetup,   // rr, g -> r0_norm, f, check 0, alpha 0
  kPhPsOmega,   // b e d after t = A w and the p s z q y update -> omega
  kPhPsBeta,    // f r g a h after v = A z and the x r w update -> beta, record,
  kPhPsBetaNC,  //   check i+1, alpha i+1 ("NC": leave the check to kPhPsCheck)
  kPhPsCheck,
};

__device__ __forceinline__ void prod_stop(SolverState* ss, int status, long long iters, long long fail, int stage) {
  ss->status = status;
  ss->iterations = iters;
  if (fail >= 0) ss->failure_iter = fail;
  ss->run_all = 0;
  ss->run_spine = 0;
  ss->stop_stage = stage;
}

__device__ __forceinline__ double prod_rel(const SolverState* ss, double rr) {  // _Run.rel_of
  if (ss->r0_norm == 0.0) return 0.0;
  return sqrt((0.0 > rr) ? 0.0 : rr) / ss->r0_norm;
}

// the loop-top record and tests of check j (solvers.py:258-263, 324-327)
static __device__ void prod_check(SolverState* ss, long long j) {
  const double rel = prod_rel(ss, ss->rr);
  if (ss->record_history) {
    const long long slot = ss->n_records;
    ss->hist_rel[slot] = rel;
    ss->hist_flags[slot] = 0;
    ss->n_records = slot + 1;
  }
  ss->iter = j + 1;
  if (j == ss->max_iters) return prod_stop(ss, rel <= ss->tol ? PBS_CONVERGED : PBS_MAX_ITERS, j, -1, 0);
  if (!isfinite(rel)) return prod_stop(ss, PBS_NON_FINITE, j, j, 0);
  if (rel <= ss->tol) return prod_stop(ss, PBS_CONVERGED, j, -1, 0);
}

// rec.coefficients of iteration i, then the non-finite test (solvers.py:310-313, 443-446)
static __device__ bool prod_record_coef(SolverState* ss, long long i, double a, double b, double z, double e,
                                 bool has_eta) {
  if (ss->record_history) {
    const long long slot = ss->n_records - 1;
    ss->hist_coef[4 * slot + 0] = a;
    ss->hist_coef[4 * slot + 1] = b;
    ss->hist_coef[4 * slot + 2] = z;
    ss->hist_coef[4 * slot + 3] = e;
    ss->hist_flags[slot] |= PBS_HIST_HAS_COEF;
  }
  if (isfinite(a) && isfinite(b) && isfinite(z) && (!has_eta || isfinite(e))) return true;
  prod_stop(ss, PBS_NON_FINITE, i, i, 4);
  return false;
}

// compute_zeta_eta_gpbicg (coefficients.py:109-135); returns a PBS_BD_* or 0
static __device__ int zeta_eta_gpbicg(double a, double b, double c, double d, double e, bool first, double* zeta,
                               double* eta) {
  if (first || (a == 0.0 && c == 0.0 && d == 0.0)) {
    if (e == 0.0) {
      *zeta = 0.0;
      *eta = 0.0;
      return PBS_BD_NONE;
    }
    if (guard(e, fabs(e))) return PBS_BD_GP_ZETA;
    *zeta = b / e;
    *eta = 0.0;
    return PBS_BD_NONE;
  }
  const double ea = mul(e, a), dd = mul(d, d);
  const double det = sub(ea, dd);
  if (guard(det, add(fabs(ea), dd))) return PBS_BD_GP_ZETA_ETA;
  *zeta = sub(mul(a, b), mul(c, d)) / det;
  *eta = sub(mul(e, c), mul(d, b)) / det;
  return PBS_BD_NONE;
}

// p-BiCGStab's alpha for the iteration whose loop-top check just passed
// (ss->iter == i + 1): f / ((r0*, w) + beta*((r0*, s) - omega*(r0*, z))),
// the recurrence for (r0*, A p), with beta and omega of iteration i - 1
static __device__ void ps_alpha(SolverState* ss) {
  if (!ss->run_all) return;
  const long long i = ss->iter - 1;
  const double gw = ss->dots[DG], sd = ss->dots[DA], zd = ss->dots[DH];
  const double bt = mul(ss->beta, sub(sd, mul(ss->omega, zd)));
  const double den = add(gw, bt);
  if (guard(den, add(fabs(gw), fabs(bt)))) {
    ss->breakdown = PBS_BD_PSTAB_ALPHA;
    prod_stop(ss, PBS_BREAKDOWN, i, i, 1);
    return;
  }
  ss->alpha = ss->f_prev / den;
}

// One phase on the shared state copy (thread 0).  i = the iteration whose
// body is running: its loop-top check was check i, so ss->iter == i + 1.
static __device__ void prod_phase(SolverState* ss, int phase, const double* d) {
  const long long i = ss->iter - 1;
  auto brk = [&](int q, int stage) {
    ss->breakdown = q;
    prod_stop(ss, PBS_BREAKDOWN, i, i, stage);
  };
  switch (phase) {
    case kPhProdSetup: {  // rr = (r, r); f = rr; r0_norm = sqrt(rr)
      const double rr = d[DR];
      ss->r0_norm = sqrt(rr);
      ss->f_prev = rr;
      ss->rr = rr;
      ss->upd = 0;
      prod_check(ss, 0);
      return;
    }
    case kPhProdAlpha: {  // guard (r0*, Ap); alpha = f / g
      ss->upd = 0;
      const double g = d[DG];
      ss->dots[DG] = g;
      if (guard(g, fabs(g))) return brk(PBS_BD_PROD_ALPHA, 1);
      ss->alpha = ss->f_prev / g;
      return;
    }
    case kPhStabOmega:
    case kPhStabOmegaNC: {
      const double b = d[DB], e = d[DE], c = d[DC], dd = d[DD];
      double omega;
      if (e == 0.0 && dd == 0.0) {
        omega = 0.0;  // t = 0: the alpha half-step already landed
      } else {
        if (guard(e, fabs(e))) return brk(PBS_BD_STAB_OMEGA, 2);
        omega = b / e;
      }
      ss->upd = 1;  // x = x + alpha p + omega t ; r = t - omega At run from here on
      ss->omega = omega;
      for (int k = 0; k < kNumDots; ++k)
        if ((kDotsStabB >> k) & 1u) ss->dots[k] = d[k];
      const double f = ss->f_prev, alpha = ss->alpha, g = ss->dots[DG];
      const double f_next = sub(sub(f, mul(alpha, g)), mul(omega, c));
      const double v = add(sub(dd, mul(mul(2.0, omega), b)), mul(mul(omega, omega), e));
      const double rr = (0.0 > v) ? 0.0 : v;  // Python max(v, 0.0)
      double beta;
      if (rr == 0.0) {
        beta = 0.0;
      } else {
        if (guard(omega, fabs(omega))) return brk(PBS_BD_STAB_BETA, 3);
        if (guard(f, fabs(f))) return brk(PBS_BD_BETA_F, 3);
        beta = mul(alpha / omega, f_next / f);
      }
      ss->f_prev = f_next;
      ss->beta = beta;
      ss->rr = rr;
      if (!prod_record_coef(ss, i, alpha, beta, omega, __longlong_as_double(0x7ff8000000000000LL), false)) return;
      if (phase == kPhStabOmega) prod_check(ss, i + 1);
      return;
    }
    case kPhGpZeta: {
      double zeta = 0.0, eta = 0.0;
      const int q = zeta_eta_gpbicg(d[DA], d[DB], d[DC], d[DD], d[DE], i == 0, &zeta, &eta);
      for (int k = 0; k < kNumDots; ++k)
        if ((kDotsGpB >> k) & 1u) ss->dots[k] = d[k];
      if (q) return brk(q, 2);
      ss->zeta = zeta;
      ss->eta = eta;
      return;
    }
    case kPhGpBeta:
    case kPhGpBetaNC: {
      const double fn = d[DF], rr = d[DR], f = ss->f_prev, alpha = ss->alpha, zeta = ss->zeta;
      ss->dots[DF] = fn;
      ss->dots[DR] = rr;
      ss->rr = rr;
      double beta;
      if (rr == 0.0) {
        beta = 0.0;
      } else {
        if (guard(zeta, fabs(zeta))) return brk(PBS_BD_GP_BETA, 3);
        if (guard(f, fabs(f))) return brk(PBS_BD_BETA_F, 3);
        beta = mul(alpha / zeta, fn / f);
      }
      ss->f_prev = fn;
      ss->beta = beta;
      if (!prod_record_coef(ss, i, alpha, beta, zeta, ss->eta, true)) return;
      if (phase == kPhGpBeta) prod_check(ss, i + 1);
      return;
    }
    case kPhProdCheck:
      prod_check(ss, i + 1);
      return;
    case kPhPsSetup: {
      const double rr = d[DR];
      ss->r0_norm = sqrt(rr);
      ss->f_prev = rr;
      ss->rr = rr;
      ss->dots[DG] = d[DG];
      ss->dots[DA] = 0.0;
      ss->dots[DH] = 0.0;
      ss->alpha = ss->beta = ss->omega = 0.0;
      prod_check(ss, 0);
      ps_alpha(ss);
      return;
    }
    case kPhPsOmega: {
      const double b = d[DB], e = d[DE], dd = d[DD];
      ss->dots[DB] = b;
      ss->dots[DE] = e;
      ss->dots[DD] = dd;
      if (e == 0.0 && dd == 0.0) {
        ss->omega = 0.0;  // q = 0: the alpha half-step already landed
      } else {
        if (guard(e, fabs(e))) return brk(PBS_BD_PSTAB_OMEGA, 2);
        ss->omega = b / e;
      }
      return;
    }
    case kPhPsBeta:
    case kPhPsBetaNC: {
      const double fn = d[DF], rr = d[DR], f = ss->f_prev, alpha = ss->alpha, omega = ss->omega;
      ss->rr = rr;
      double beta;
      if (rr == 0.0) {
        beta = 0.0;
      } else {
        if (guard(omega, fabs(omega))) return brk(PBS_BD_STAB_BETA, 3);
        if (guard(f, fabs(f))) return brk(PBS_BD_BETA_F, 3);
        beta = mul(alpha / omega, fn / f);
      }
      ss->f_prev = fn;
      ss->beta = beta;
      ss->dots[DF] = fn;
      ss->dots[DR] = rr;
      ss->dots[DG] = d[DG];
      ss->dots[DA] = d[DA];
      ss->dots[DH] = d[DH];
      if (!prod_record_coef(ss, i, alpha, beta, omega, __longlong_as_double(0x7ff8000000000000LL), false)) return;
      if (phase == kPhPsBeta) {
        prod_check(ss, i + 1);
        ps_alpha(ss);
      }
      return;
    }
    case kPhPsCheck:
      prod_check(ss, i + 1);
      ps_alpha(ss);
      return;
  }
}

// state_store + host mirror (the tail of check_and_publish)
template <int NT, bool NAMED>
__device__ __forceinline__ void prod_and_publish(SolverState* st, SolverState* ss, const double* dots, int phase) {
  block_bar<NT, NAMED>();
  if (threadIdx.x != 0) return;
  if (!dev_err(ss) && ss->run_all) prod_phase(ss, phase, dots);
  state_store(st, ss);
  if (ss->mirror) {
    ss->mirror->iter = ss->iter;
    ss->mirror->run_all = ss->run_all;
    ss->mirror->err = dev_err(ss) ? 1 : 0;
  }
}

// Reduce partial records (kPartStride doubles each: hi/lo per dot) -> dots[9]
// with NT threads, fixed shape: one warp per dot, each lane summing a strided
// subset of the records in double-double (pairwise, 16 records per pass),
// then the warp's xor butterfly, rounded once.  Dots in
// mask2 come from a second record set (partials2, nparts2): the
// s-independent dots K12 produced.  chain: the reference's left-to-right
// combine of plain per-range values (reduction.py:285-294 _combine), one
// thread per dot.
template <int NT, bool NAMED>
__device__ void reduce_parts(const double* partials, int nparts, int chain, double* dots,
                             const double* partials2 = nullptr, int nparts2 = 0, unsigned mask2 = 0,
                             int rs = 1, int fs = kMaxParts) {
  const int t = threadIdx.x;
  if (chain) {
    if (t < kNumDots) {
      double acc = __ldcg(partials + (size_t)(2 * t) * fs);
      const double* p = partials + (size_t)(2 * t) * fs;
      for (int b = 1; b < nparts; ++b) acc = add(acc, __ldcg(p + (size_t)b * rs));
      dots[t] = acc;
    }
    block_bar<NT, NAMED>();
    return;
  }
  // warp w sums dots w, w + NW, ...: lane l takes records l, l + 32, ... in
  // order (eight records' loads in flight per round), then the xor butterfly
  constexpr int NW = NT / 32;
  const int lane = t & 31, warp = t >> 5;
#ifdef PBS_TAIL_CLOCKS
  const long long q0 = clock64();
  long long q1 = 0, q2 = 0, q3 = 0;
#endif
  for (int j = warp; j < kNumDots; j += NW) {
    const bool second = (mask2 >> j) & 1u;
    const double* src = (second ? partials2 : partials) + (size_t)(2 * j) * fs;
    const int np = second ? nparts2 : nparts;
    Ddbl acc{0.0, 0.0};
    constexpr int U = 16;  // records per lane per pass: all loads in flight, then a pairwise tree
    for (int b0 = lane; b0 < np; b0 += 32 * U) {
      Ddbl v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + 32 * u;
        v[u] = b < np ? Ddbl{__ldcg(src + (size_t)b * rs), __ldcg(src + (size_t)b * rs + fs)}
                      : Ddbl{0.0, 0.0};
      }
#ifdef PBS_TAIL_CLOCKS
      if (v[U - 1].hi == 12345.0) acc.lo += 1.0;  // force the loads to land
      q1 = clock64();
#endif
#pragma unroll
      for (int w = 1; w < U; w *= 2)
#pragma unroll
        for (int u = 0; u < U; u += 2 * w) v[u] = dd_add(v[u], v[u + w]);
      acc = dd_add(acc, v[0]);
    }
#ifdef PBS_TAIL_CLOCKS
    q2 = clock64();
#endif
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = dd_add(acc, dd_shfl_xor(acc, o));
    if (lane == 0) dots[j] = add(acc.hi, acc.lo);
#ifdef PBS_TAIL_CLOCKS
    q3 = clock64();
#endif
  }
  block_bar<NT, NAMED>();
#ifdef PBS_TAIL_CLOCKS
  if (t == 0) printf("reduce parts: loads %lld tree %lld butterfly %lld\n", q1 - q0, q2 - q1, q3 - q2);
#endif
}

// Multi-GPU local step: reduce this rank's CTA partial records to ONE record
// of 9 compensated pairs (not rounded), the payload of the all-gather.
static __global__ void __launch_bounds__(288) reduce_pairs_kernel(const double* partials, int nparts, double* out) {
  constexpr int T = 288 / kNumDots;
  __shared__ Ddbl team[kNumDots][T];
  const int t = threadIdx.x, j = t / T, l = t % T;
  if (j < kNumDots) {
    Ddbl acc{0.0, 0.0};
    for (int b = l; b < nparts; b += T) {
      const double* p = partials + (size_t)(2 * j) * kMaxParts + b;
      acc = dd_add(acc, Ddbl{__ldcg(p), __ldcg(p + kMaxParts)});
    }
    team[j][l] = acc;
  }
  __syncthreads();
  if (t < kNumDots) {
    Ddbl acc = team[t][0];
    for (int k = 1; k < T; ++k) acc = dd_add(acc, team[t][k]);
    out[2 * t] = acc.hi;
    out[2 * t + 1] = acc.lo;
  }
}

// Run by every participating thread of each CTA after its block_reduce9:
// the last CTA to arrive reduces all partials and performs the check.
template <int NT, bool NAMED>
__device__ void finalize_tail(SolverState* st, const double* partials, int nparts, int replaced,
                              const double* partials2 = nullptr, int nparts2 = 0, unsigned mask2 = 0,
                              int phase = kPhSafe) {
  __shared__ int last;
  __shared__ double dots[kNumDots];
  block_bar<NT, NAMED>();
  if (threadIdx.x == 0) {
    fence_gpu();
    const unsigned int ticket = atomicAdd(&st->done_ctas, 1u);
    last = ticket == (unsigned int)nparts - 1;
  }
  block_bar<NT, NAMED>();
  if (!last) return;
  fence_gpu();
  __shared__ SolverState ss;
  state_load<NT>(st, &ss);
  reduce_parts<NT, NAMED>(partials, nparts, 0, dots, partials2, nparts2, mask2);  // ends with a barrier
  if (threadIdx.x == 0) st->done_ctas = 0;
  if (phase == kPhSafe)
    check_and_publish<NT, NAMED>(st, &ss, dots, replaced);
  else
    prod_and_publish<NT, NAMED>(st, &ss, dots, phase);
}

// Standalone finalize (1 CTA, 288 threads): reduce (tree or plan chain), then
// the check for j = st->iter, then advance st->iter.
static __global__ void __launch_bounds__(288) finalize_kernel(SolverState* st, const double* partials, int nparts,
                                                       int chain, int replaced, const double* partials2 = nullptr,
                                                       int nparts2 = 0, unsigned mask2 = 0, int rs = 1,
                                                       int fs = kMaxParts, int phase = kPhSafe) {
  __shared__ double dots[kNumDots];
  __shared__ SolverState ss;
#ifdef PBS_TAIL_CLOCKS
  long long c0 = clock64();
#endif
  state_load<288>(st, &ss);
  reduce_parts<288, false>(partials, nparts, chain, dots, partials2, nparts2, mask2, rs, fs);  // ends with a barrier
#ifdef PBS_TAIL_CLOCKS
  long long c1 = clock64();
#endif
  if (phase == kPhSafe)
    check_and_publish<288, false>(st, &ss, dots, replaced);
  else
    prod_and_publish<288, false>(st, &ss, dots, phase);
#ifdef PBS_TAIL_CLOCKS
  if (threadIdx.x == 0) {
    long long c2 = clock64();
    printf("tail clocks: reduce %lld check+publish %lld\n", c1 - c0, c2 - c1);
  }
#endif
}

}  // namespace pbs
