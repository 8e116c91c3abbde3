// pstab.cu — the paper's p-BiCGStab comparator (Cools & Vanroose; oracle
// solve_pstab): two SpMV kernels per iteration, each carrying one reduction
// phase in its last CTA's tail.
#include "host.h"

// ---- p-BiCGStab (oracle solve_pstab).  Two SpMV kernels per iteration,
// each carrying one reduction phase in its tail:
//   t = A w  + p s z q y + b e d   [omega]
//   v = A z  + x r w + f r g a h   [beta, record, check i+1, alpha i+1]
// v (A z) lives in the o slot.  On several GPUs each phase's reduction would
// overlap the next SpMV, which is the method's point; on one GPU the two
// kernels simply stream.

static EpiPsW epi_ps_w(Workspace* ws, const Mode& md) {
  EpiPsW e{};
  auto& V = ws->V.v;
  e.w = V[VW];
  e.st = ws->st;
  e.sink = sink_for(ws, md, 1, 0);
  e.sink.phase = kPhPsSetup;
  e.in[0] = V[VR];
  e.in[1] = V[VR0S];
  return e;
}

static EpiPsA epi_ps_a(Workspace* ws, const Mode& md) {
  EpiPsA e{};
  auto& V = ws->V.v;
  e.t = V[VT];
  e.p = V[VP];
  e.s = V[VS];
  e.z = V[VZ];
  e.q = V[VQ];
  e.y = V[VY];
  e.st = ws->st;
  e.sink = sink_for(ws, md, 1, 0);
  e.sink.phase = kPhPsOmega;
  const int in[6] = {VR, VP, VS, VW, VZ, VO};
  for (int k = 0; k < 6; ++k) e.in[k] = V[in[k]];
  return e;
}

static EpiPsB epi_ps_b(Workspace* ws, const Mode& md, int phase) {
  EpiPsB e{};
  auto& V = ws->V.v;
  e.v = V[VO];
  e.x = V[VX];
  e.r = V[VR];
  e.w = V[VW];
  e.st = ws->st;
  e.sink = sink_for(ws, md, 1, 0);
  e.sink.phase = phase;
  const int in[8] = {VX, VP, VQ, VY, VT, VR0S, VS, VZ};
  for (int k = 0; k < 8; ++k) e.in[k] = V[in[k]];
  return e;
}

void setup_pstab(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  spmv_launch(L, ws->X.v[VX], epi_resid(ws, true), 0, ws->n, KS);  // r0 = b - A x0 ; r0* = r0
  spmv_launch(L, ws->X.v[VR], epi_ps_w(ws, md), 0, ws->n, KS);      // w0 = A r0 + rr, g
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DR] = V[VR], y[DR] = V[VR];
    x[DG] = V[VR0S], y[DG] = V[VW];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsPsW, x, y)), 1, 0, 0, kPhPsSetup);
  }
}

void iter_pstab(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  const bool tracing = L.trace_cfg != nullptr;
  spmv_launch(L, ws->X.v[VW], epi_ps_a(ws, md), 0, ws->n, KK1);
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DB] = V[VQ], y[DB] = V[VY];
    x[DE] = V[VY], y[DE] = V[VY];
    x[DD] = V[VQ], y[DD] = V[VQ];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsPsA, x, y)), 1, 0, 0, kPhPsOmega);
  }
  const int ph = tracing ? kPhPsBetaNC : kPhPsBeta;
  spmv_launch(L, ws->X.v[VZ], epi_ps_b(ws, md, ph), 0, ws->n, KK3);
  if (md.plan) {
    const double* x[kNumDots] = {};
    const double* y[kNumDots] = {};
    x[DF] = V[VR0S], y[DF] = V[VR];
    x[DR] = V[VR], y[DR] = V[VR];
    x[DG] = V[VR0S], y[DG] = V[VW];
    x[DA] = V[VR0S], y[DA] = V[VS];
    x[DH] = V[VR0S], y[DH] = V[VZ];
    finalize(L, ws, plan_pairs(L, ws, pairs_of(kDotsPsB, x, y)), 1, 0, 0, ph);
  }
  if (tracing) {
    L.trace_point();
    finalize(L, ws, 0, 1, 0, 0, kPhPsCheck);
  }
}

void iter_pstab_batch(Launcher& L, Workspace* ws, const Mode& md) {
  for (int k = 0; k < graph_iters(); ++k) iter_pstab(L, ws, md);
}
