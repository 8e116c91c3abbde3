// vec.cuh — fused vector-update kernels, dot-batch reductions and the
// single-CTA coefficient/bookkeeping kernel (sm_100a).
#pragma once
#include "common.cuh"
#include "finalize.cuh"

namespace pbs {

// Workspace vector slots (one padded HBM allocation each).
enum Vec {
  VX = 0, VR, VR0S, VP, VU, VO, VT, VW, VY, VZ, VS, VQ, VG, VL, VAS, VAW, VTMP, VB, kNumVecs
};
// the product-type comparators keep A p and A t in the As / Aw slots
constexpr int VAP = VAS, VAT = VAW;

struct VecPtrs {
  double* v[kNumVecs];
};

// Gate of the first kernel after the spine SpMV: once a check has stopped the
// solve, the stop iteration's spine product has now run, so close the spine
// gate for any iterations the host launched ahead.
__device__ __forceinline__ bool gate_after_spine(SolverState* st) {
  if (gate_all(st)) return true;
  if (st && blockIdx.x == 0 && threadIdx.x == 0 && !dev_err(st) && !st->run_all) st->run_spine = 0;
  return false;
}

// ---------------------------------------------------------------------------
// K2: block 1 of the pipelined iteration (solvers.py:678-701, 715) in one
// pass.  Reads r p u s t y As l g w z x (12 vectors), writes p u w t z y x r
// (8); o and q stay in registers unless the single-step seam asks for them.
static __global__ void __launch_bounds__(kThreads) k2_update_kernel(VecPtrs V, long long n, SolverState* st,
                                                             int store_temps) {
  if (!gate_after_spine(st)) return;
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
static __global__ void __launch_bounds__(kThreads) pou_kernel(VecPtrs V, long long n, SolverState* st) {
  if (!gate_after_spine(st)) return;
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
static __global__ void __launch_bounds__(kThreads) tzyx_kernel(VecPtrs V, long long n, SolverState* st) {
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
// product-type comparators (BiCGStab solvers.py:210-327, GPBi-CG 330-460).
// Grid-stride loops; kernels that carry a reduction phase accumulate its
// compensated dots and the last CTA runs that phase (finalize_tail).

// after r0 = b - A x0: p0 = r + 0*(p - ...) on the zeroed workspace (the
// first iteration's p update, solvers.py:265 / 381) and the partials of
// (r, r) (solvers.py:244 / 365) -> r0_norm, f, check 0
static __global__ void __launch_bounds__(kThreads) prod_setup_kernel(VecPtrs V, long long n, SolverState* st, int gp,
                                                              double* partials, int fuse) {
  __shared__ int go;
  if (threadIdx.x == 0) go = gate_all(st);
  __syncthreads();
  if (!go) return;
  Ddbl acc[kNumDots];
#pragma unroll
  for (int j = 0; j < kNumDots; ++j) acc[j] = Ddbl{0.0, 0.0};
  double *__restrict__ p = V.v[VP];
  const double *__restrict__ r = V.v[VR], *__restrict__ u = V.v[VU], *__restrict__ ap = V.v[VAP];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double rv = r[i];
    p[i] = gp ? asd(rv, 0.0, p[i], u[i]) : asdd(rv, 0.0, p[i], 0.0, ap[i]);
    acc[DR] = dot2_step(acc[DR], rv, rv);
  }
  if (!partials) return;
  block_reduce9<kThreads, false, kDotsRR>(acc, partials + blockIdx.x);
  if (fuse) finalize_tail<kThreads, false>(st, partials, gridDim.x, 0, nullptr, 0, 0u, kPhProdSetup);
}

// BiCGStab t = r - alpha*Ap (solvers.py:279)
static __global__ void __launch_bounds__(kThreads) stab_t_kernel(VecPtrs V, long long n, SolverState* st) {
  if (!gate_all(st)) return;
  const double alpha = st->alpha;
  double *__restrict__ t = V.v[VT];
  const double *__restrict__ r = V.v[VR], *__restrict__ ap = V.v[VAP];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
    t[i] = lc2(1.0, r[i], -alpha, ap[i]);
}

// BiCGStab x = x + alpha*p + omega*t; r = t - omega*At (solvers.py:295-298),
// then (with_p) the next iteration's p = r + beta*(p - omega*Ap)
// (solvers.py:265).  Gated on the omega phase's go-ahead: the update runs
// even when the beta guard or check i+1 stops the solve.
static __global__ void __launch_bounds__(kThreads) stab_xrp_kernel(VecPtrs V, long long n, SolverState* st, int with_p) {
  if (dev_err(st) || !st->upd) return;
  const double alpha = st->alpha, omega = st->omega, beta = st->beta;
  double *__restrict__ x = V.v[VX], *__restrict__ r = V.v[VR], *__restrict__ p = V.v[VP];
  const double *__restrict__ t = V.v[VT], *__restrict__ at = V.v[VAT], *__restrict__ ap = V.v[VAP];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double tv = t[i], pv = p[i];
    x[i] = lc3(1.0, x[i], alpha, pv, omega, tv);
    const double rn = lc2(1.0, tv, -omega, at[i]);
    r[i] = rn;
    if (with_p) p[i] = asdd(rn, beta, pv, omega, ap[i]);
  }
}

// the p update at the top of the next iteration, when a trace hook had to
// see the old p: BiCGStab p = r + beta*(p - omega*Ap), GPBi-CG
// p = r + beta*(p - u) (solvers.py:265, 381)
static __global__ void __launch_bounds__(kThreads) prod_p_kernel(VecPtrs V, long long n, SolverState* st, int gp) {
  if (!gate_all(st)) return;
  const double beta = st->beta, omega = st->omega;
  double *__restrict__ p = V.v[VP];
  const double *__restrict__ r = V.v[VR], *__restrict__ u = V.v[VU], *__restrict__ ap = V.v[VAP];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
    p[i] = gp ? asd(r[i], beta, p[i], u[i]) : asdd(r[i], beta, p[i], omega, ap[i]);
}

// GPBi-CG y = t - r - alpha*w + alpha*Ap; u = t - r + beta*u (stash);
// t = r - alpha*Ap (solvers.py:394-399) in one pass
static __global__ void __launch_bounds__(kThreads) gp_yut_kernel(VecPtrs V, long long n, SolverState* st) {
  if (!gate_all(st)) return;
  const double alpha = st->alpha, beta = st->beta;
  double *__restrict__ y = V.v[VY], *__restrict__ u = V.v[VU], *__restrict__ t = V.v[VT];
  const double *__restrict__ r = V.v[VR], *__restrict__ w = V.v[VW], *__restrict__ ap = V.v[VAP];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double tv = t[i], rv = r[i], apv = ap[i];
    y[i] = lc4(1.0, tv, -1.0, rv, -alpha, w[i], alpha, apv);
    u[i] = lc3(1.0, tv, -1.0, rv, beta, u[i]);
    t[i] = lc2(1.0, rv, -alpha, apv);
  }
}

// GPBi-CG u = zeta*Ap + eta*u; z = zeta*r + eta*z - alpha*u; x = x + alpha*p
// + z; r = t - eta*y - zeta*At (solvers.py:416-419), with the partials of
// the third phase f = (r0*, r), rr = (r, r) (solvers.py:421-423)
static __global__ void __launch_bounds__(kThreads) gp_uzxr_kernel(VecPtrs V, long long n, SolverState* st,
                                                           double* partials, int fuse, int phase) {
  __shared__ int go;
  if (threadIdx.x == 0) go = gate_all(st);
  __syncthreads();
  if (!go) return;
  const double alpha = st->alpha, zeta = st->zeta, eta = st->eta;
  double *__restrict__ u = V.v[VU], *__restrict__ z = V.v[VZ], *__restrict__ x = V.v[VX], *__restrict__ r = V.v[VR];
  const double *__restrict__ ap = V.v[VAP], *__restrict__ p = V.v[VP], *__restrict__ t = V.v[VT],
               *__restrict__ y = V.v[VY], *__restrict__ at = V.v[VAT], *__restrict__ r0s = V.v[VR0S];
  Ddbl acc[kNumDots];
#pragma unroll
  for (int j = 0; j < kNumDots; ++j) acc[j] = Ddbl{0.0, 0.0};
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double rv = r[i];
    const double un = lc2(zeta, ap[i], eta, u[i]);
    const double zn = lc3(zeta, rv, eta, z[i], -alpha, un);
    u[i] = un;
    z[i] = zn;
    x[i] = lc3(1.0, x[i], alpha, p[i], 1.0, zn);
    const double rn = lc3(1.0, t[i], -eta, y[i], -zeta, at[i]);
    r[i] = rn;
    acc[DF] = dot2_step(acc[DF], r0s[i], rn);
    acc[DR] = dot2_step(acc[DR], rn, rn);
  }
  if (!partials) return;
  block_reduce9<kThreads, false, kDotsGpC>(acc, partials + blockIdx.x);
  if (fuse) finalize_tail<kThreads, false>(st, partials, gridDim.x, 0, nullptr, 0, 0u, phase);
}

// GPBi-CG w = At + beta*Ap (solvers.py:440), then (with_p) the next
// iteration's p = r + beta*(p - u) (solvers.py:381)
static __global__ void __launch_bounds__(kThreads) gp_wp_kernel(VecPtrs V, long long n, SolverState* st, int with_p) {
  if (!gate_all(st)) return;
  const double beta = st->beta;
  double *__restrict__ w = V.v[VW], *__restrict__ p = V.v[VP];
  const double *__restrict__ at = V.v[VAT], *__restrict__ ap = V.v[VAP], *__restrict__ r = V.v[VR],
               *__restrict__ u = V.v[VU];
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    w[i] = lc2(1.0, at[i], beta, ap[i]);
    if (with_p) p[i] = asd(r[i], beta, p[i], u[i]);
  }
}

// PartitionPlan chains over up to 9 arbitrary pairs (reduction.py:282-283):
// block w sums range w of pair j (mask bit j) sequentially into field 2j
struct DotPairs {
  const double* x[kNumDots];
  const double* y[kNumDots];
  unsigned mask;
};
static __global__ void dots_pairs_plan_kernel(const long long* bounds, DotPairs P, double* partials,
                                       const SolverState* st) {
  if (st && !gate_all(st)) return;
  const int j = threadIdx.x;
  if (j >= kNumDots || !((P.mask >> j) & 1u)) return;
  const double* xa = P.x[j];
  const double* ya = P.y[j];
  const long long lo = bounds[blockIdx.x], hi = bounds[blockIdx.x + 1];
  double acc = 0.0;
  for (long long k = lo; k < hi; ++k) acc = add(acc, mul(xa[k], ya[k]));
  partials[(size_t)(2 * j) * kMaxParts + blockIdx.x] = acc;
  partials[(size_t)(2 * j + 1) * kMaxParts + blockIdx.x] = 0.0;
}

// ---------------------------------------------------------------------------
// kernel-table entry points (kernels.py:110-137), kinds as in pbsafe.h
static __global__ void __launch_bounds__(kThreads) lincomb_kernel(int kind, long long n, double* out, double s0,
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
static __global__ void __launch_bounds__(kThreads) dot_partial_kernel(const double* x, const double* y, long long lo,
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

static __global__ void dot_final_kernel(const double* partials, int nparts, double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 32) acc = add(acc, partials[i]);
  for (int o = 16; o > 0; o >>= 1) acc = add(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if (threadIdx.x == 0) *out = acc;
}

// batch of the 9 safe dots, compensated tree, into record blk of partials
static __global__ void __launch_bounds__(kThreads) dots9_tree_kernel(long long n, const double* s, const double* y,
                                                              const double* r, const double* r0s,
                                                              const double* t, double* partials,
                                                              const SolverState* st) {
  if (st && !gate_all(st)) return;
  Ddbl acc[kNumDots];
#pragma unroll
  for (int j = 0; j < kNumDots; ++j) acc[j] = Ddbl{0.0, 0.0};
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double sv = s[i], yv = y[i], rv = r[i], r0 = r0s[i], tv = t[i];
    acc[DA] = dot2_step(acc[DA], sv, sv);
    acc[DB] = dot2_step(acc[DB], yv, yv);
    acc[DC] = dot2_step(acc[DC], sv, yv);
    acc[DD] = dot2_step(acc[DD], sv, rv);
    acc[DE] = dot2_step(acc[DE], yv, rv);
    acc[DF] = dot2_step(acc[DF], r0, rv);
    acc[DG] = dot2_step(acc[DG], r0, sv);
    acc[DH] = dot2_step(acc[DH], r0, tv);
    acc[DR] = dot2_step(acc[DR], rv, rv);
  }
  block_reduce9<kThreads, false>(acc, partials + blockIdx.x);
}

// The batch of the next check as its own streaming kernel (s y r r0s t ->
// 9 compensated dots), with the check fused into the last CTA's tail.
static __global__ void __launch_bounds__(kThreads) dots9_check_kernel(long long n, const double* __restrict__ s,
                                                               const double* __restrict__ y,
                                                               const double* __restrict__ r,
                                                               const double* __restrict__ r0s,
                                                               const double* __restrict__ t, double* partials,
                                                               SolverState* st, int fuse, int replaced) {
  __shared__ int go;
  if (threadIdx.x == 0) go = gate_all(st);
  __syncthreads();
  if (!go) return;
  Ddbl acc[kNumDots];
#pragma unroll
  for (int j = 0; j < kNumDots; ++j) acc[j] = Ddbl{0.0, 0.0};
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double sv = __ldcs(s + i), yv = __ldcs(y + i), rv = __ldcs(r + i), r0 = __ldcs(r0s + i),
                 tv = __ldcs(t + i);
    acc[DA] = dot2_step(acc[DA], sv, sv);
    acc[DB] = dot2_step(acc[DB], yv, yv);
    acc[DC] = dot2_step(acc[DC], sv, yv);
    acc[DD] = dot2_step(acc[DD], sv, rv);
    acc[DE] = dot2_step(acc[DE], yv, rv);
    acc[DF] = dot2_step(acc[DF], r0, rv);
    acc[DG] = dot2_step(acc[DG], r0, sv);
    acc[DH] = dot2_step(acc[DH], r0, tv);
    acc[DR] = dot2_step(acc[DR], rv, rv);
  }
  block_reduce9<kThreads, false>(acc, partials + blockIdx.x);
  if (fuse) finalize_tail<kThreads, false>(st, partials, gridDim.x, replaced);
}

// PartitionPlan chains (reduction.py:282-283 with kernels.py:103-107): block w
// handles range [bounds[w], bounds[w+1]); thread j < 9 sums pair j
// sequentially in ascending index order -> field 2j of record w.
static __global__ void dots9_plan_kernel(const long long* bounds, const double* s, const double* y,
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
  partials[(size_t)(2 * j) * kMaxParts + blockIdx.x] = acc;
  partials[(size_t)(2 * j + 1) * kMaxParts + blockIdx.x] = 0.0;
}

}  // namespace pbs
