// finalize.cuh — the coefficient step and _Run bookkeeping of one check
// (solvers.py:645-674, 736-739; coefficients.py:35-106), the deterministic
// reduction of the dot-batch partials, and two ways to run them: fused into
// the tail of the kernel that produced the partials (the last CTA to finish,
// by ticket) or as a separate 1-CTA kernel (plan order, multi-GPU, step seam).
#pragma once
#include "common.cuh"

namespace pbs {

// Coefficient step + bookkeeping for check j.  One thread.
__device__ __forceinline__ bool guard(double q, double scale) {
  return !isfinite(q) || fabs(q) <= mul(1e-14, scale);
}

__device__ void check_iteration(SolverState* st, long long j, const double* d, int replaced) {
  const bool first = j == 0;
  if (first) st->r0_norm = sqrt(d[DR]);
  // _Run.rel_of (solvers.py:176-179): Python max(rr, 0.0) keeps rr unless 0.0 > rr
  double rel;
  if (st->r0_norm == 0.0) {
    rel = 0.0;
  } else {
    const double m = (0.0 > d[DR]) ? 0.0 : d[DR];
    rel = sqrt(m) / st->r0_norm;
  }
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
  // compute_alpha_beta_safe (coefficients.py:60-84)
  const double f = d[DF], g = d[DG], h = first ? 0.0 : d[DH];
  double alpha, beta;
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
  // compute_zeta_eta_safe (coefficients.py:87-106)
  double zeta = 0.0, eta = 0.0;
  if (q == PBS_BD_NONE) {
    const double a = d[DA], b = first ? 0.0 : d[DB], c = first ? 0.0 : d[DC], dd = d[DD],
                 e = first ? 0.0 : d[DE];
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
  }
  if (q != PBS_BD_NONE) {
    st->breakdown = q;
    return stop(PBS_BREAKDOWN, j, true);
  }
  st->alpha = alpha;
  st->beta = beta;
  st->zeta = zeta;
  st->eta = eta;
  st->f_prev = f;
  if (st->record_history) {
    st->hist_coef[4 * slot + 0] = alpha;
    st->hist_coef[4 * slot + 1] = beta;
    st->hist_coef[4 * slot + 2] = zeta;
    st->hist_coef[4 * slot + 3] = eta;
    st->hist_flags[slot] |= PBS_HIST_HAS_COEF;
  }
  if (!(isfinite(alpha) && isfinite(beta) && isfinite(zeta) && isfinite(eta)))
    return stop(PBS_NON_FINITE, j, true);
}


__device__ __forceinline__ void publish(SolverState* st, long long next_iter) {
  st->iter = next_iter;
  if (st->mirror) {
    st->mirror->iter = next_iter;
    st->mirror->run_all = st->run_all;
    st->mirror->err = dev_err(st) ? 1 : 0;
    __threadfence_system();
  }
}

// Reduce partial records (kPartStride doubles each: hi/lo per dot) -> dots[9]
// with NT threads, fixed shape: dot j is summed in double-double by a team of
// T = NT/9 threads (strided, sequential per thread), then the team's values
// in order, then rounded once.  chain: the reference's left-to-right combine
// of plain per-range values (reduction.py:285-294 _combine), one thread per dot.
template <int NT, bool NAMED>
__device__ void reduce_parts(const double* partials, int nparts, int chain, double* dots) {
  constexpr int T = NT / kNumDots;
  __shared__ Ddbl team[kNumDots][T];
  const int t = threadIdx.x;
  if (chain) {
    if (t < kNumDots) {
      double acc = __ldcg(partials + 2 * t);
      for (int b = 1; b < nparts; ++b) acc = add(acc, __ldcg(partials + (size_t)b * kPartStride + 2 * t));
      dots[t] = acc;
    }
  } else {
    const int j = t / T, l = t % T;
    if (j < kNumDots) {
      Ddbl acc{0.0, 0.0};
      for (int b = l; b < nparts; b += T) {
        const double* p = partials + (size_t)b * kPartStride + 2 * j;
        acc = dd_add(acc, Ddbl{__ldcg(p), __ldcg(p + 1)});
      }
      team[j][l] = acc;
    }
    block_bar<NT, NAMED>();
    if (t < kNumDots) {
      Ddbl acc = team[t][0];
      for (int k = 1; k < T; ++k) acc = dd_add(acc, team[t][k]);
      dots[t] = add(acc.hi, acc.lo);
    }
  }
  block_bar<NT, NAMED>();
}

// Multi-GPU local step: reduce this rank's CTA partial records to ONE record
// of 9 compensated pairs (not rounded), the payload of the all-gather.
__global__ void __launch_bounds__(288) reduce_pairs_kernel(const double* partials, int nparts, double* out) {
  constexpr int T = 288 / kNumDots;
  __shared__ Ddbl team[kNumDots][T];
  const int t = threadIdx.x, j = t / T, l = t % T;
  if (j < kNumDots) {
    Ddbl acc{0.0, 0.0};
    for (int b = l; b < nparts; b += T) {
      const double* p = partials + (size_t)b * kPartStride + 2 * j;
      acc = dd_add(acc, Ddbl{__ldcg(p), __ldcg(p + 1)});
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
__device__ void finalize_tail(SolverState* st, const double* partials, int nparts, int replaced) {
  __shared__ int last;
  __shared__ double dots[kNumDots];
  block_bar<NT, NAMED>();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int ticket = atomicAdd(&st->done_ctas, 1u);
    last = ticket == (unsigned int)nparts - 1;
  }
  block_bar<NT, NAMED>();
  if (!last) return;
  __threadfence();
  reduce_parts<NT, NAMED>(partials, nparts, 0, dots);
  if (threadIdx.x == 0) {
    st->done_ctas = 0;
    const long long j = st->iter;
    if (!dev_err(st) && st->run_all) {
      for (int k = 0; k < kNumDots; ++k) st->dots[k] = dots[k];
      check_iteration(st, j, dots, replaced);
    }
    publish(st, j + 1);
  }
}

// Standalone finalize (1 CTA, 288 threads): reduce (tree or plan chain), then
// the check for j = st->iter, then advance st->iter.
__global__ void __launch_bounds__(288) finalize_kernel(SolverState* st, const double* partials, int nparts,
                                                       int chain, int replaced) {
  __shared__ double dots[kNumDots];
  __shared__ int work;
  if (threadIdx.x == 0) work = !dev_err(st) && st->run_all;
  __syncthreads();
  const long long j = st->iter;
  if (work) {
    reduce_parts<288, false>(partials, nparts, chain, dots);
    if (threadIdx.x == 0) {
      for (int k = 0; k < kNumDots; ++k) st->dots[k] = dots[k];
      check_iteration(st, j, dots, replaced);
    }
  } else if (threadIdx.x == 0 && !dev_err(st)) {
    st->run_spine = 0;  // the stop iteration's spine product has run
  }
  if (threadIdx.x == 0) publish(st, j + 1);
}

}  // namespace pbs
