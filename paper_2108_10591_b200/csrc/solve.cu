// solve.cu — the single-GPU schedules of the Safe methods (p-BiCGSafe,
// p-BiCGSafe-rr, ssBiCGSafe2) and the solve loop shared with the
// product-type comparators (CUDA graphs, device-side stop, a bounded number
// of iterations in flight, no per-iteration host sync).
//
// Per steady p-BiCGSafe iteration j (solvers.py:639-734) the device runs
//   K12 As = A s fused with the row-local block 1 (p o u q w t z y x r) and
//       the five s-independent dots of check j+1 (b e f h r)
//   K3  Aw = A w -> l g s + the four dots that need the new s (a c d g); the
//       last CTA reduces both record sets and runs check j+1
// captured four iterations to a graph; residual-replacement iterations
// (solvers.py:676-713) use a second graph.
#include "host.h"

// setup of the pipelined methods (solvers.py:612-631) + check 0
static void setup_pipelined(Launcher& L, Workspace* ws, const Mode& md) {
  spmv_launch(L, ws->X.v[VX], epi_resid(ws, true), 0, ws->n, KS);
  spmv_s_check(L, ws, md, KS, 0, 0);
}

// one steady p-BiCGSafe iteration: K12 (As = A s + row-local updates), K3
// (Aw + l g s + the fused check of j+1)
static void iter_steady(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  // the batch split between K12 and K3: CSR, and stencils on the z-marching
  // engine (register room for the five accumulators)
  const bool split = !L.m->stencil || k12_dots() == 2 || stencil_zm_ok(L.m, 0, ws->n);
  if (!md.plan && !k3_dots_split() && k12_dots() && split) {
    const int fuse = L.trace_cfg || !fuse_check() ? 0 : 1;
    const int np12 = spmv_launch(L, ws->X.v[VS], epi_k12d(ws, md), 0, ws->n, KK1);
    const int grid = spmv_launch(L, ws->X.v[VW], epi_k3s(ws, md, fuse, np12), 0, ws->n, KK3);
    if (!fuse) {
      L.trace_point();
      finalize(L, ws, grid, 0, 0, np12);
    }
    return;
  }
  spmv_launch(L, ws->X.v[VS], epi_k12(ws, md), 0, ws->n, KK1);
  if (!md.plan && k3_dots_split()) {
    spmv_launch(L, ws->X.v[VW], epi_k3n(ws, md), 0, ws->n, KK3);
    const int np = dots_check(L, ws, L.trace_cfg ? 0 : 1, 0);
    if (L.trace_cfg) {
      L.trace_point();
      finalize(L, ws, np, 0, 0);
    }
    return;
  }
  const int grid = spmv_launch(L, ws->X.v[VW], epi_k3(ws, md, L.trace_cfg ? 0 : 1), 0, ws->n, KK3);
  if (md.plan) {
    int np = plan_dots(L, ws, KD);
    L.trace_point();
    finalize(L, ws, np, 1, 0);
  } else if (L.trace_cfg) {
    L.trace_point();  // tracing: the check runs after the hook, as in the reference
    finalize(L, ws, grid, 0, 0);
  }
}

// residual-replacement iteration (solvers.py:676-713)
static void iter_replace(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  spmv_launch(L, ws->X.v[VS], epi_store(ws, VAS, PBS_TAG_AS, 1), 0, ws->n, KK1);
  vec_launch(L, pou_kernel, ws->n, KR, ws->V, ws->n, ws->st);
  spmv_launch(L, ws->X.v[VO], epi_store(ws, VQ, PBS_TAG_AO, 0), 0, ws->n, KRS);
  spmv_launch(L, ws->X.v[VU], epi_store(ws, VW, PBS_TAG_AU, 0), 0, ws->n, KRS);
  vec_launch(L, tzyx_kernel, ws->n, KR, ws->V, ws->n, ws->st);
  spmv_launch(L, ws->X.v[VX], epi_resid(ws, false), 0, ws->n, KRS);
  spmv_launch(L, ws->X.v[VT], epi_store(ws, VL, PBS_TAG_AT, 0), 0, ws->n, KRS);
  spmv_launch(L, ws->X.v[VY], epi_store(ws, VG, PBS_TAG_AY, 0), 0, ws->n, KRS);
  if (L.trace_cfg) {
    int np = spmv_launch(L, ws->X.v[VR], epi_dots(ws, md, 0, 0, 1), 0, ws->n, KRS);
    if (md.plan) np = plan_dots(L, ws, KD);
    L.trace_point();
    finalize(L, ws, np, md.plan, 1);
  } else {
    spmv_s_check(L, ws, md, KRS, 0, 1);
  }
}

// one ssBiCGSafe2 iteration (solvers.py:528-587): s = A r + batch + check,
// p o u, w = A u + t z y x r
static void iter_ss(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  spmv_s_check(L, ws, md, KK1, 1, 0);
  vec_launch(L, pou_kernel, ws->n, KK2, ws->V, ws->n, ws->st);
  spmv_launch(L, ws->X.v[VU], epi_ss3(ws), 0, ws->n, KK3);
  L.trace_point();
}

// final record of ssBiCGSafe2 after max_iters: plan_dot(r, r) (solvers.py:589)
static void final_ss(Launcher& L, Workspace* ws, const Mode& md) {
  auto& V = ws->V.v;
  int np;
  if (md.plan) {
    np = plan_dots(L, ws, KD);
  } else {
    long long nblk = (ws->n + kThreads - 1) / kThreads;
    np = grid_for(L.ctx, (const void*)dots9_tree_kernel, nblk);
    dots9_tree_kernel<<<np, kThreads, 0, L.s>>>(ws->n, V[VS], V[VY], V[VR], V[VR0S], V[VT],
                                                ws->partials, ws->st);
    L.done(KD);
  }
  finalize(L, ws, np, md.plan, 0);
}

static void iter_steady_batch(Launcher& L, Workspace* ws, const Mode& md) {
  for (int k = 0; k < graph_iters(); ++k) iter_steady(L, ws, md);
}


int run_solve(pbs_mat* m, int method, const pbs_config* cfg, pbs_result* res) {
  if (m->part.dist) return run_solve_dist(m, method, cfg, res);
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  const long long n = ws->n;
  Mode md;
  md.plan = cfg->reduce_mode == PBS_REDUCE_PLAN;
  const bool tracing = cfg->trace_fn != nullptr;
  md.store_temps = tracing ? 1 : 0;
  md.method = method;
  const bool product = method == PBS_METHOD_BICGSTAB || method == PBS_METHOD_GPBICG ||
                       method == PBS_METHOD_PBICGSTAB;
  if (md.plan) {
    int rc = ensure_plan(m, cfg->plan_workers);
    if (rc) return rc;
  }
  cudaStream_t s = ctx->stream;
  // device state
  SolverState h{};
  h.tol = cfg->tol;
  h.max_iters = cfg->max_iters;
  h.record_history = cfg->record_history ? 1 : 0;
  h.spine_done = method == PBS_METHOD_SSBICGSAFE2 ? 1 : 0;
  h.upd = 0;
  h.stop_stage = 0;
  h.iter = 0;
  h.run_all = 1;
  h.run_spine = 1;
  h.status = -1;
  h.failure_iter = -1;
  h.nf_row = (unsigned long long)kNoError;
  h.hist_rel = ws->hist_rel;
  h.hist_flags = ws->hist_flags;
  h.hist_coef = ws->hist_coef;
  h.mirror = ws->mirror_d;
  ws->mirror_h->iter = 0;
  ws->mirror_h->run_all = 1;
  ws->mirror_h->err = 0;
  CK(cudaMemcpyAsync(ws->st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  // zero-initialised workspace (solvers.py:621-628; 251-253, 371-376)
  const int zero_slots[] = {VP, VU, VT, VY, VZ, VG, VL, VW, VAP, VAT};
  for (int k : zero_slots) CK(cudaMemsetAsync(ws->V.v[k], 0, sizeof(double) * n, s));
  if (method == PBS_METHOD_PBICGSTAB) {  // s and v (o slot) start at zero too
    CK(cudaMemsetAsync(ws->V.v[VS], 0, sizeof(double) * n, s));
    CK(cudaMemsetAsync(ws->V.v[VO], 0, sizeof(double) * n, s));
  }

  std::vector<std::pair<int, cudaEvent_t>> marks;
  ctx->events.reset();
  Launcher L{ctx, m, s};
  L.timing = cfg->timing != 0 && !tracing;
  L.marks = &marks;
  if (tracing) {
    L.trace_cfg = cfg;
    L.trace_ws = ws;
    L.trace_method = method;
  }
  const bool graphs = cfg->use_graphs && !L.timing && !tracing;
  const bool pipelined = method == PBS_METHOD_PBICGSAFE || method == PBS_METHOD_PBICGSAFE_RR;
  const bool rr = method == PBS_METHOD_PBICGSAFE_RR;
  const long long cutoff = cfg->rr_cutoff >= 0 ? cfg->rr_cutoff : cfg->max_iters;
  const long long key_base = (long long)md.plan * 4;

  CK(cudaEventRecord(ws->ev0, s));
  if (L.timing) marks.push_back({-1, ws->ev0});
  if (pipelined) {
    setup_pipelined(L, ws, md);
    if (L.err) return L.err;
  } else if (method == PBS_METHOD_PBICGSTAB) {
    setup_pstab(L, ws, md);
    if (L.err) return L.err;
  } else if (product) {
    setup_prod(L, ws, md);
    if (L.err) return L.err;
  } else {
    spmv_launch(L, ws->X.v[VX], epi_resid(ws, true), 0, n, KS);
  }
  const long long lookahead = 6;
  long long launched_graph_kernels = 0;
  long long j = 0;
  for (; j < cfg->max_iters; ++j) {
    // stop once the device has stopped (the stop iteration's spine SpMV is
    // part of iteration j = stop, so keep launching through it)
    for (;;) {
      const long long dev_iter = ws->mirror_h->iter;
      if (ws->mirror_h->err) goto loop_end;
      if (!ws->mirror_h->run_all && j >= dev_iter) goto loop_end;
      if (j <= dev_iter + lookahead) break;
      if (cudaStreamQuery(s) == cudaSuccess) {
        // idle device but the mirror did not advance far enough: every
        // launched iteration was gated off (stopped or failed) -> read the
        // authoritative state and stop if nothing is left to run
        SolverState chk;
        CK(cudaMemcpy(&chk, ws->st, sizeof(chk), cudaMemcpyDeviceToHost));
        if (chk.nf_row != (unsigned long long)kNoError || !chk.run_all) goto loop_end;
        if (ws->mirror_h->iter == dev_iter) goto loop_end;  // no progress possible
        continue;
      }
      std::this_thread::yield();
    }
    {
      auto is_replace = [&](long long i) { return rr && (i % cfg->rr_epoch == 0) && 0 < i && i < cutoff; };
      const bool replace = is_replace(j);
      IterFn fn = method == PBS_METHOD_BICGSTAB ? iter_stab
                  : method == PBS_METHOD_GPBICG ? iter_gp
                  : method == PBS_METHOD_PBICGSTAB ? iter_pstab
                  : !pipelined ? iter_ss
                  : (replace ? iter_replace : iter_steady);
      IterFn bfn = method == PBS_METHOD_BICGSTAB ? iter_stab_batch
                   : method == PBS_METHOD_GPBICG ? iter_gp_batch
                   : method == PBS_METHOD_PBICGSTAB ? iter_pstab_batch
                   : iter_steady_batch;
      const int gu = graph_iters();
      bool batch = graphs && (pipelined || product) && gu > 1 && j + gu <= cfg->max_iters;
      for (long long i = j; batch && i < j + gu; ++i) batch = !is_replace(i);
      if (batch) {
        cudaGraphExec_t ge;
        long long nk = 0;
        int rc = get_graph(ctx, m, key_base + 8 + 16 * method, bfn, md, &ge, &nk);
        if (rc) return rc;
        CK(cudaGraphLaunch(ge, s));
        launched_graph_kernels += nk;
        j += gu - 1;
      } else if (graphs) {
        long long key = key_base + (product ? 16 * method : (!pipelined ? 2 : (replace ? 1 : 0)));
        cudaGraphExec_t ge;
        long long nk = 0;
        int rc = get_graph(ctx, m, key, fn, md, &ge, &nk);
        if (rc) return rc;
        CK(cudaGraphLaunch(ge, s));
        launched_graph_kernels += nk;
      } else {
        L.iter = j;
        fn(L, ws, md);
        if (L.trace_rc) return L.trace_rc;
        if (L.err) return L.err;
      }
    }
  }
  if (method == PBS_METHOD_SSBICGSAFE2) final_ss(L, ws, md);
loop_end:
  CK(cudaEventRecord(ws->ev1, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  return collect_result(m, method, cfg, res, L, marks, launched_graph_kernels);
}
