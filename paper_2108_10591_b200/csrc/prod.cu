// prod.cu — schedules of the product-type comparators BiCGStab and
// GPBi-CG (solvers.py:210-460), each reduction phase in the tail of the
// kernel that produced its dots.
#include "host.h"

// ---- product-type comparators: BiCGStab (solvers.py:210-327) and GPBi-CG
// (solvers.py:330-460).  Per iteration (p materialised by the previous one):
//   BiCGStab: Ap = A p + g [alpha] -> t -> At = A t + b e c d [omega, beta,
//             check i+1] -> x, r and the next p
//   GPBi-CG:  Ap = A p + g [alpha] -> y u t -> At = A t + a..e [zeta, eta]
//             -> u z x r + f rr [beta, check i+1] -> w and the next p
// Tree mode runs each phase in the tail of the kernel that produced its
// dots; plan mode computes the reference's PartitionPlan chains and runs a
// 1-CTA finalize.  With a trace hook the next p waits until after the hook.


void setup_prod(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  spmv_launch(L, ws->X.v[VX], epi_resid(ws, true), 0, ws->n, KS);  // r0 = b - A x0 ; r0s = r0
  const int gp = md.method == PBS_METHOD_GPBICG;
  long long nblk = (ws->n + kThreads - 1) / kThreads;
  int np = grid_for(L.ctx, (const void*)prod_setup_kernel, nblk);
  prod_setup_kernel<<<np, kThreads, 0, L.s>>>(ws->V, ws->n, ws->st, gp, md.plan ? nullptr : ws->partials, 1);
  L.done(KS);
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DR] = V[VR];
    y[DR] = V[VR];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsRR, x, y)), 1, 0, 0, kPhProdSetup);
  }
}

static EpiPA epi_pa(Workspace* ws, const Mode& md) {
  EpiPA e{};
  e.ap = ws->V.v[VAP];
  e.st = ws->st;
  e.sink = sink_for(ws, md, 1, 0);
  e.sink.phase = kPhProdAlpha;
  e.in[0] = ws->V.v[VR0S];
  return e;
}

template <class E>
static E epi_prod_b(Workspace* ws, const Mode& md, int second, int phase) {
  E e{};
  e.at = ws->V.v[VAT];
  e.st = ws->st;
  e.sink = sink_for(ws, md, 1, 0);
  e.sink.phase = phase;
  e.in[0] = ws->V.v[VT];
  e.in[1] = ws->V.v[second];
  return e;
}

// Ap = A p + g, then alpha
static void prod_alpha(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  spmv_launch(L, ws->X.v[VP], epi_pa(ws, md), 0, ws->n, KK1);
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DG] = V[VR0S];
    y[DG] = V[VAP];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsProdA, x, y)), 1, 0, 0, kPhProdAlpha);
  }
}

void iter_stab(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  const bool tracing = L.trace_cfg != nullptr;
  prod_alpha(L, ws, md);
  vec_launch(L, stab_t_kernel, ws->n, KK2, ws->V, ws->n, ws->st);
  const int ph = tracing ? kPhStabOmegaNC : kPhStabOmega;
  spmv_launch(L, ws->X.v[VT], epi_prod_b<EpiStabB>(ws, md, VR0S, ph), 0, ws->n, KK3);
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DB] = V[VAT], y[DB] = V[VT];
    x[DE] = V[VAT], y[DE] = V[VAT];
    x[DC] = V[VR0S], y[DC] = V[VAT];
    x[DD] = V[VT], y[DD] = V[VT];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsStabB, x, y)), 1, 0, 0, ph);
  }
  vec_launch(L, stab_xrp_kernel, ws->n, KK2, ws->V, ws->n, ws->st, tracing ? 0 : 1);
  if (tracing) {
    L.trace_point();
    finalize(L, ws, 0, 1, 0, 0, kPhProdCheck);
    vec_launch(L, prod_p_kernel, ws->n, KK2, ws->V, ws->n, ws->st, 0);
  }
}

void iter_gp(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  const bool tracing = L.trace_cfg != nullptr;
  prod_alpha(L, ws, md);
  vec_launch(L, gp_yut_kernel, ws->n, KK2, ws->V, ws->n, ws->st);
  spmv_launch(L, ws->X.v[VT], epi_prod_b<EpiGpB>(ws, md, VY, kPhGpZeta), 0, ws->n, KK3);
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DA] = V[VY], y[DA] = V[VY];
    x[DB] = V[VAT], y[DB] = V[VT];
    x[DC] = V[VY], y[DC] = V[VT];
    x[DD] = V[VAT], y[DD] = V[VY];
    x[DE] = V[VAT], y[DE] = V[VAT];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsGpB, x, y)), 1, 0, 0, kPhGpZeta);
  }
  const int ph = tracing ? kPhGpBetaNC : kPhGpBeta;
  {
    long long nblk = (ws->n + kThreads - 1) / kThreads;
    int np = grid_for(L.ctx, (const void*)gp_uzxr_kernel, nblk);
    gp_uzxr_kernel<<<np, kThreads, 0, L.s>>>(ws->V, ws->n, ws->st, md.plan ? nullptr : ws->partials, 1, ph);
    L.done(KK2);
  }
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DF] = V[VR0S], y[DF] = V[VR];
    x[DR] = V[VR], y[DR] = V[VR];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsGpC, x, y)), 1, 0, 0, ph);
  }
  vec_launch(L, gp_wp_kernel, ws->n, KK2, ws->V, ws->n, ws->st, tracing ? 0 : 1);
  if (tracing) {
    L.trace_point();
    finalize(L, ws, 0, 1, 0, 0, kPhProdCheck);
    vec_launch(L, prod_p_kernel, ws->n, KK2, ws->V, ws->n, ws->st, 1);
  }
}

void iter_stab_batch(Launcher& L, Workspace* ws, const Mode& md) {
  for (int k = 0; k < graph_iters(); ++k) iter_stab(L, ws, md);
}
void iter_gp_batch(Launcher& L, Workspace* ws, const Mode& md) {
  for (int k = 0; k < graph_iters(); ++k) iter_gp(L, ws, md);
}
