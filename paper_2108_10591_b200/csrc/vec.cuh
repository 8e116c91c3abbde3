// vec.cuh — fused vector-update kernels, dot-batch reductions and the
// single-CTA coefficient/bookkeeping kernel (sm_100a).
#pragma once
#include "common.cuh"

namespace pbs {

// Workspace vector slots (one padded HBM allocation each).
enum Vec {
  VX = 0, VR, VR0S, VP, VU, VO, VT, VW, VY, VZ, VS, VQ, VG, VL, VAS, VAW, VTMP, VB, kNumVecs
};

struct VecPtrs {
  double* v[kNumVecs];
};

// ---------------------------------------------------------------------------
// K2: block 1 of the pipelined iteration (solvers.py:678-701, 715) in one
// pass.  Reads r p u s t y As l g w z x (12 vectors), writes p u w t z y x r
// (8); o and q stay in registers unless the single-step seam asks for them.
__global__ void __launch_bounds__(kThreads) k2_update_kernel(VecPtrs V, long long n, SolverState* st,
                                                             int store_temps) {
  if (!gate_all(st)) return;
  const double alpha = st->alpha, beta = st->beta, zeta = st->zeta, eta = st->eta;
  double *__restrict__ x = V.v[VX], *__restrict__ r = V.v[VR], *__restrict__ p = V.v[VP],
         *__restrict__ u = V.v[VU], *__restrict__ t = V.v[VT], *__restrict__ w = V.v[VW],
         *__restrict__ y = V.v[VY], *__restrict__ z = V.v[VZ];
  const double *__restrict__ s = V.v[VS], *__restrict__ as = V.v[VAS], *__restrict__ l = V.v[VL],
               *__restrict__ g = V.v[VG];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double rv = r[i], pv = p[i], uv = u[i], sv = s[i], tv = t[i], yv = y[i];
    const double asv = __ldcs(as + i), lv = l[i], gv = g[i], wv = w[i], zv = z[i], xv = x[i];
    const double pn = asd(rv, beta, pv, uv);                 // p = r + beta*(p - u)
    const double o = lc2(1.0, sv, beta, tv);                 // o = s + beta*t
    const double un = lcn(zeta, o, eta, yv, beta, uv);       // u = zeta*o + eta*(y + beta*u)
    const double q = lc2(1.0, asv, beta, lv);                // q = As + beta*l
    const double wn = lcn(zeta, q, eta, gv, beta, wv);       // w = zeta*q + eta*(g + beta*w)
    const double tn = lc2(1.0, o, -1.0, wn);                 // t = o - w
    const double zn = lc3(zeta, rv, eta, zv, -alpha, un);    // z = zeta*r + eta*z - alpha*u
    const double yn = lc3(zeta, sv, eta, yv, -alpha, wn);    // y = zeta*s + eta*y - alpha*w
    const double xn = lc3(1.0, xv, alpha, pn, 1.0, zn);      // x = x + alpha*p + z
    const double rn = lc3(1.0, rv, -alpha, o, -1.0, yn);     // r = r - alpha*o - y
    p[i] = pn;
    u[i] = un;
    w[i] = wn;
    t[i] = tn;
    z[i] = zn;
    y[i] = yn;
    x[i] = xn;
    r[i] = rn;
    if (store_temps) {
      V.v[VO][i] = o;
      V.v[VQ][i] = q;
    }
  }
}

// p, o, u (solvers.py:678-683; also ssBiCGSafe2 solvers.py:563-568)
__global__ void __launch_bounds__(kThreads) pou_kernel(VecPtrs V, long long n, SolverState* st) {
  if (!gate_all(st)) return;
  const double beta = st->beta, zeta = st->zeta, eta = st->eta;
  double *__restrict__ p = V.v[VP], *__restrict__ u = V.v[VU], *__restrict__ o = V.v[VO];
  const double *__restrict__ r = V.v[VR], *__restrict__ s = V.v[VS], *__restrict__ t = V.v[VT],
               *__restrict__ y = V.v[VY];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double ov = lc2(1.0, s[i], beta, t[i]);
    p[i] = asd(r[i], beta, p[i], u[i]);
    o[i] = ov;
    u[i] = lcn(zeta, ov, eta, y[i], beta, u[i]);
  }
}

// t, z, y, x after q = A o, w = A u were recomputed (solvers.py:694-701)
__global__ void __launch_bounds__(kThreads) tzyx_kernel(VecPtrs V, long long n, SolverState* st) {
  if (!gate_all(st)) return;
  const double alpha = st->alpha, zeta = st->zeta, eta = st->eta;
  double *__restrict__ t = V.v[VT], *__restrict__ z = V.v[VZ], *__restrict__ y = V.v[VY],
         *__restrict__ x = V.v[VX];
  const double *__restrict__ o = V.v[VO], *__restrict__ w = V.v[VW], *__restrict__ r = V.v[VR],
               *__restrict__ u = V.v[VU], *__restrict__ s = V.v[VS], *__restrict__ p = V.v[VP];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double wv = w[i];
    const double zn = lc3(zeta, r[i], eta, z[i], -alpha, u[i]);
    t[i] = lc2(1.0, o[i], -1.0, wv);
    z[i] = zn;
    y[i] = lc3(zeta, s[i], eta, y[i], -alpha, wv);
    x[i] = lc3(1.0, x[i], alpha, p[i], 1.0, zn);
  }
}

// ---------------------------------------------------------------------------
// kernel-table entry points (kernels.py:110-137), kinds as in pbsafe.h
__global__ void __launch_bounds__(kThreads) lincomb_kernel(int kind, long long n, double* out, double s0,
                                                           double s1, double s2, double s3,
                                                           const double* a, const double* b,
                                                           const double* c, const double* d) {
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    double v;
    switch (kind) {
      case 2: v = lc2(s0, a[i], s1, b[i]); break;
      case 3: v = lc3(s0, a[i], s1, b[i], s2, c[i]); break;
      case 4: v = lc4(s0, a[i], s1, b[i], s2, c[i], s3, d[i]); break;
      case 5: v = lcn(s0, a[i], s1, b[i], s2, c[i]); break;
      case 6: v = asd(a[i], s0, b[i], c[i]); break;
      default: v = asdd(a[i], s0, b[i], s1, c[i]); break;
    }
    out[i] = v;
  }
}

// ---------------------------------------------------------------------------
// dot reductions

// tree dot over [lo, hi): per-thread strided partial, block tree, written to
// partials[blockIdx]; finished by dot_final_kernel (deterministic shape)
__global__ void __launch_bounds__(kThreads) dot_partial_kernel(const double* x, const double* y, long long lo,
                                                               long long hi, double* partials) {
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = lo + (long long)blockIdx.x * kThreads + threadIdx.x; i < hi; i += stride)
    acc = add(acc, mul(x[i], y[i]));
  __shared__ double red[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) acc = add(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = red[0];
    for (int w = 1; w < kThreads / 32; ++w) v = add(v, red[w]);
    partials[blockIdx.x] = v;
  }
}

__global__ void dot_final_kernel(const double* partials, int nparts, double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 32) acc = add(acc, partials[i]);
  for (int o = 16; o > 0; o >>= 1) acc = add(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if (threadIdx.x == 0) *out = acc;
}

// batch of the 9 safe dots, tree order, into partials[blk*9 + j]
__global__ void __launch_bounds__(kThreads) dots9_tree_kernel(long long n, const double* s, const double* y,
                                                              const double* r, const double* r0s,
                                                              const double* t, double* partials,
                                                              const SolverState* st) {
  if (st && !gate_all(st)) return;
  double acc[kNumDots];
#pragma unroll
  for (int j = 0; j < kNumDots; ++j) acc[j] = 0.0;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double sv = s[i], yv = y[i], rv = r[i], r0 = r0s[i], tv = t[i];
    acc[DA] = add(acc[DA], mul(sv, sv));
    acc[DB] = add(acc[DB], mul(yv, yv));
    acc[DC] = add(acc[DC], mul(sv, yv));
    acc[DD] = add(acc[DD], mul(sv, rv));
    acc[DE] = add(acc[DE], mul(yv, rv));
    acc[DF] = add(acc[DF], mul(r0, rv));
    acc[DG] = add(acc[DG], mul(r0, sv));
    acc[DH] = add(acc[DH], mul(r0, tv));
    acc[DR] = add(acc[DR], mul(rv, rv));
  }
  block_reduce9(acc, partials + (size_t)blockIdx.x * kNumDots);
}

// PartitionPlan chains (reduction.py:282-283 with kernels.py:103-107): block w
// handles range [bounds[w], bounds[w+1]); thread j < 9 sums pair j
// sequentially in ascending index order -> partials[w*9 + j].
__global__ void dots9_plan_kernel(const long long* bounds, const double* s, const double* y,
                                  const double* r, const double* r0s, const double* t,
                                  double* partials, const SolverState* st) {
  if (st && !gate_all(st)) return;
  const int j = threadIdx.x;
  if (j >= kNumDots) return;
  const double* xs[kNumDots] = {s, y, s, s, y, r0s, r0s, r0s, r};
  const double* ys[kNumDots] = {s, y, y, r, r, r, s, t, r};
  const double* xa = xs[j];
  const double* ya = ys[j];
  const long long lo = bounds[blockIdx.x], hi = bounds[blockIdx.x + 1];
  double acc = 0.0;
  for (long long k = lo; k < hi; ++k) acc = add(acc, mul(xa[k], ya[k]));
  partials[(size_t)blockIdx.x * kNumDots + j] = acc;
}

// ---------------------------------------------------------------------------
// Coefficient step + _Run bookkeeping for check j (solvers.py:645-674,
// 736-739; coefficients.py:35-106).  One thread.

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

// Finalize: reduce the batch partials (tree: xor-butterfly per dot across
// nparts blocks; plan: left-to-right chain, reduction.py:285-294), then run
// the check for j = st->iter and advance st->iter.  9 warps, 1 CTA.
__global__ void __launch_bounds__(288) finalize_kernel(SolverState* st, const double* partials, int nparts,
                                                       int chain, int replaced) {
  __shared__ double dots[kNumDots];
  __shared__ int work;
  if (threadIdx.x == 0) work = !dev_err(st) && st->run_all;
  __syncthreads();
  const long long j = st->iter;
  if (work) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc;
    if (chain) {
      if (lane == 0) {
        acc = partials[warp];
        for (int b = 1; b < nparts; ++b) acc = add(acc, partials[(size_t)b * kNumDots + warp]);
        dots[warp] = acc;
      }
    } else {
      acc = 0.0;
      for (int b = lane; b < nparts; b += 32) acc = add(acc, partials[(size_t)b * kNumDots + warp]);
      for (int o = 16; o > 0; o >>= 1) acc = add(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (lane == 0) dots[warp] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 0; k < kNumDots; ++k) st->dots[k] = dots[k];
      check_iteration(st, j, dots, replaced);
    }
  } else if (threadIdx.x == 0 && !dev_err(st)) {
    st->run_spine = 0;  // the stop iteration's spine product has run
  }
  if (threadIdx.x == 0) {
    st->iter = j + 1;
    if (st->mirror) {
      st->mirror->iter = j + 1;
      st->mirror->run_all = st->run_all;
      st->mirror->err = dev_err(st) ? 1 : 0;
      __threadfence_system();
    }
  }
}

}  // namespace pbs
