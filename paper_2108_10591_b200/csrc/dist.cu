// dist.cu — the multi-GPU row-partitioned schedule.
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is loaded at run time

#include "host.h"

// ---- NCCL, loaded on first use (the copy torch loaded, or the system one)
struct NcclApi {
  bool tried = false, ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  void* h = nullptr;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
#define PBS_SYM(field, sym)                                    \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym)); \
  if (!api.field) {                                            \
    api.err = std::string("libnccl lacks ") + sym;             \
    return api;                                                \
  }
  PBS_SYM(GetUniqueId, "ncclGetUniqueId")
  PBS_SYM(CommInitRank, "ncclCommInitRank")
  PBS_SYM(CommDestroy, "ncclCommDestroy")
  PBS_SYM(Send, "ncclSend")
  PBS_SYM(Recv, "ncclRecv")
  PBS_SYM(AllGather, "ncclAllGather")
  PBS_SYM(GroupStart, "ncclGroupStart")
  PBS_SYM(GroupEnd, "ncclGroupEnd")
  PBS_SYM(GetErrorString, "ncclGetErrorString")
#undef PBS_SYM
  api.ok = true;
  return api;
}

struct pbs_dist {
  pbs_ctx* ctx = nullptr;
  int nranks = 1, rank = 0;
  ncclComm_t halo = nullptr, red = nullptr;
  cudaStream_t comm = nullptr;  // all-gather + finalize, overlapping the As SpMV
  cudaEvent_t ev_part = nullptr, ev_coef = nullptr;
  // halo exchange of s / w on its own stream, overlapping the interior rows
  // of the SpMV that consumes it (Partition::split)
  cudaStream_t hstream = nullptr;
  cudaEvent_t ev_vec = nullptr, ev_halo = nullptr;
  double* sendbuf = nullptr;  // this rank's 9 compensated pairs
  double* recvbuf = nullptr;  // all ranks' pairs, rank order
};

// ---------------------------------------------------------- multi-GPU schedule
//
// Per steady iteration j on every rank (stream s = compute, comm = reduction):
//   s:    halo(s) -> K1 As = A s (spine)            || comm: all-gather of the
//   s:    wait coefficients -> K2 updates              batch pairs of check j ->
//   s:    halo(w) -> K3 (Aw + l g s + local partials)  finalize (check j)
//   s:    reduce CTA partials -> this rank's 9 pairs -> record ev_part
// The all-gather + check of iteration j overlaps the As SpMV: the pipelined
// method's single reduction hides behind one SpMV.

static void halo_exchange(Launcher& L, Workspace* ws, pbs_mat* m, int k, cudaStream_t st = nullptr) {
  Partition& P = m->part;
  pbs_dist* D = P.dist;
  if (!st) st = L.s;
  if (L.err || D->nranks == 1 || (P.sends.empty() && P.recvs.empty())) return;
  NcclApi& A = nccl();
  ncclResult_t r = A.GroupStart();
  for (size_t i = 0; r == ncclSuccess && i < P.recvs.size(); i += 3)
    r = A.Recv(ws->X.v[k] + P.recvs[i + 1], (size_t)P.recvs[i + 2], ncclDouble, (int)P.recvs[i], D->halo, st);
  for (size_t i = 0; r == ncclSuccess && i < P.sends.size(); i += 3)
    r = A.Send(ws->V.v[k] + P.sends[i + 1], (size_t)P.sends[i + 2], ncclDouble, (int)P.sends[i], D->halo, st);
  ncclResult_t r2 = A.GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) L.err = set_err(L.ctx, PBS_ERR_NCCL, std::string("halo exchange: ") + A.GetErrorString(r));
}

// this rank's pairs -> all-gather on the comm stream -> finalize (check)
static void dist_check(Launcher& L, Workspace* ws, pbs_mat* m, int nparts, int replaced) {
  pbs_dist* D = m->part.dist;
  if (L.err) return;
  reduce_pairs_kernel<<<1, 288, 0, L.s>>>(ws->partials, nparts, D->sendbuf);
  L.done(KD);
  cudaEventRecord(D->ev_part, L.s);
  cudaStreamWaitEvent(D->comm, D->ev_part, 0);
  L.mark(D->comm, L.iter, 0, 0);  // reduce_start
  ncclResult_t r = nccl().AllGather(D->sendbuf, D->recvbuf, kPartStride, ncclDouble, D->red, D->comm);
  if (r != ncclSuccess) {
    L.err = set_err(L.ctx, PBS_ERR_NCCL, std::string("all-gather: ") + nccl().GetErrorString(r));
    return;
  }
  // the gathered pairs are one row-major record per rank
  finalize_kernel<<<1, 288, 0, D->comm>>>(ws->st, D->recvbuf, D->nranks, 0, replaced, nullptr, 0, 0u, kPartStride, 1);
  L.done(KF);
  L.mark(D->comm, L.iter, 1, 0);  // reduce_end
  L.mark(D->comm, L.iter, 4, 0);  // coeff_ready
  cudaEventRecord(D->ev_coef, D->comm);
}

static void dist_setup(Launcher& L, Workspace* ws, pbs_mat* m, const Mode& md) {
  halo_exchange(L, ws, m, VX);
  spmv_launch(L, ws->X.v[VX], epi_resid(ws, true), 0, ws->n, KS);
  halo_exchange(L, ws, m, VR);
  int np = spmv_launch(L, ws->X.v[VR], epi_dots(ws, md, 0, 0, 0), 0, ws->n, KS);
  dist_check(L, ws, m, np, 0);
}

// Halo exchange of vector k, then an SpMV over all rows with epilogue factory
// mk(partial_offset).  With Partition::split the exchange runs on the halo
// stream while the interior rows [L0, L1) compute, and the boundary rows
// follow once it has landed; dot partial records of the pieces are stored
// one after another.  Returns the number of partial records.
template <class MakeEpi>
static int halo_spmv(Launcher& L, Workspace* ws, pbs_mat* m, int k, int kind, int tag, MakeEpi mk) {
  Partition& P = m->part;
  pbs_dist* D = P.dist;
  if (!P.split) {
    halo_exchange(L, ws, m, k);
    L.mark(L.s, L.iter, 2, tag);
    const int np = spmv_launch(L, ws->X.v[k], mk(0), 0, ws->n, kind);
    L.mark(L.s, L.iter, 3, tag);
    return np;
  }
  cudaEventRecord(D->ev_vec, L.s);  // the vector is final on the compute stream
  cudaStreamWaitEvent(D->hstream, D->ev_vec, 0);
  halo_exchange(L, ws, m, k, D->hstream);
  cudaEventRecord(D->ev_halo, D->hstream);
  L.mark(L.s, L.iter, 2, tag);
  int np = spmv_launch(L, ws->X.v[k], mk(0), P.L0, P.L1, kind);
  cudaStreamWaitEvent(L.s, D->ev_halo, 0);
  if (P.L0 > 0) np += spmv_launch(L, ws->X.v[k], mk(np), 0, P.L0, kind);
  if (P.L1 < ws->n) np += spmv_launch(L, ws->X.v[k], mk(np), P.L1, ws->n, kind);
  L.mark(L.s, L.iter, 3, tag);
  return np;
}

static void dist_iter(Launcher& L, Workspace* ws, pbs_mat* m, const Mode& md, bool replace) {
  pbs_dist* D = m->part.dist;
  halo_spmv(L, ws, m, VS, KK1, PBS_TAG_AS, [&](int) { return epi_store(ws, VAS, PBS_TAG_AS, 1); });
  cudaStreamWaitEvent(L.s, D->ev_coef, 0);  // coefficients of this check
  int np;
  if (!replace) {
    vec_launch(L, k2_update_kernel, ws->n, KK2, ws->V, ws->n, ws->st, md.store_temps);
    np = halo_spmv(L, ws, m, VW, KK3, PBS_TAG_AW, [&](int off) {
      EpiK3 e = epi_k3(ws, md, 0);
      if (e.sink.partials) e.sink.partials += off;
      return e;
    });
  } else {
    vec_launch(L, pou_kernel, ws->n, KR, ws->V, ws->n, ws->st);
    halo_exchange(L, ws, m, VO);
    spmv_launch(L, ws->X.v[VO], epi_store(ws, VQ, PBS_TAG_AO, 0), 0, ws->n, KRS);
    halo_exchange(L, ws, m, VU);
    spmv_launch(L, ws->X.v[VU], epi_store(ws, VW, PBS_TAG_AU, 0), 0, ws->n, KRS);
    vec_launch(L, tzyx_kernel, ws->n, KR, ws->V, ws->n, ws->st);
    halo_exchange(L, ws, m, VX);
    spmv_launch(L, ws->X.v[VX], epi_resid(ws, false), 0, ws->n, KRS);
    halo_exchange(L, ws, m, VT);
    spmv_launch(L, ws->X.v[VT], epi_store(ws, VL, PBS_TAG_AT, 0), 0, ws->n, KRS);
    halo_exchange(L, ws, m, VY);
    spmv_launch(L, ws->X.v[VY], epi_store(ws, VG, PBS_TAG_AY, 0), 0, ws->n, KRS);
    halo_exchange(L, ws, m, VR);
    np = spmv_launch(L, ws->X.v[VR], epi_dots(ws, md, 0, 0, 1), 0, ws->n, KRS);
  }
  ++L.iter;  // this batch / check is iteration j+1's (solvers.py:641)
  dist_check(L, ws, m, np, replace ? 1 : 0);
  --L.iter;
}


// Multi-GPU solve: every rank launches the same sequence; at chunk
// boundaries the ranks agree (all-gather of two flags) on whether any rank
// hit a non-finite SpMV output or the solve stopped, so the NCCL call
// sequence stays identical on every rank.
int run_solve_dist(pbs_mat* m, int method, const pbs_config* cfg, pbs_result* res) {
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  pbs_dist* D = m->part.dist;
  if (method != PBS_METHOD_PBICGSAFE && method != PBS_METHOD_PBICGSAFE_RR)
    return set_err(ctx, PBS_ERR_UNSUPPORTED, "only p-BiCGSafe(-rr) has a multi-GPU schedule");
  if (cfg->reduce_mode != PBS_REDUCE_TREE)
    return set_err(ctx, PBS_ERR_UNSUPPORTED, "multi-GPU solves use the compensated tree reduction");
  if (cfg->trace_fn) return set_err(ctx, PBS_ERR_UNSUPPORTED, "trace_hook is single-GPU only");
  Mode md;
  cudaStream_t s = ctx->stream;
  SolverState h{};
  h.tol = cfg->tol;
  h.max_iters = cfg->max_iters;
  h.record_history = cfg->record_history ? 1 : 0;
  h.run_all = 1;
  h.run_spine = 1;
  h.status = -1;
  h.failure_iter = -1;
  h.nf_row = (unsigned long long)kNoError;
  h.hist_rel = ws->hist_rel;
  h.hist_flags = ws->hist_flags;
  h.hist_coef = ws->hist_coef;
  h.mirror = nullptr;
  CK(cudaMemcpyAsync(ws->st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  const int zero_slots[] = {VP, VU, VT, VY, VZ, VG, VL, VW};
  for (int k : zero_slots) CK(cudaMemsetAsync(ws->X.v[k], 0, sizeof(double) * ws->n_ext, s));
  std::vector<std::pair<int, cudaEvent_t>> marks;
  ctx->events.reset();
  Launcher L{ctx, m, s};
  L.timing = cfg->timing != 0;
  L.marks = &marks;
  std::vector<Launcher::Ev> evidence;
  if (cfg->events_out && cfg->events_cap > 0) L.evidence = &evidence;
  const bool rr = method == PBS_METHOD_PBICGSAFE_RR;
  const long long cutoff = cfg->rr_cutoff >= 0 ? cfg->rr_cutoff : cfg->max_iters;
  int* flags = nullptr;  // [2] local, [2*nranks] gathered
  CK(cudaMalloc(&flags, sizeof(int) * 2 * (D->nranks + 1)));
  CK(cudaEventRecord(ws->ev0, s));
  if (L.timing) marks.push_back({-1, ws->ev0});
  dist_setup(L, ws, m, md);
  const long long chunk = 8;
  long long j = 0;
  int rc = PBS_OK;
  bool any_err = false;
  while (!L.err) {
    const long long jend = j + chunk < cfg->max_iters ? j + chunk : cfg->max_iters;
    for (; j < jend && !L.err; ++j) {
      const bool replace = rr && (j % cfg->rr_epoch == 0) && 0 < j && j < cutoff;
      L.iter = j;
      dist_iter(L, ws, m, md, replace);
    }
    if (L.err) break;
    // agreement: every rank contributes (error, stopped); the reduction
    // communicator is only ever driven from the comm stream
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamSynchronize(D->comm));
    SolverState st;
    CK(cudaMemcpy(&st, ws->st, sizeof(st), cudaMemcpyDeviceToHost));
    int mine[2] = {st.nf_row != (unsigned long long)kNoError ? 1 : 0, st.run_all ? 0 : 1};
    CK(cudaMemcpyAsync(flags, mine, sizeof(mine), cudaMemcpyHostToDevice, D->comm));
    ncclResult_t r = nccl().AllGather(flags, flags + 2, 2, ncclInt32, D->red, D->comm);
    if (r != ncclSuccess) {
      rc = set_err(ctx, PBS_ERR_NCCL, std::string("agreement: ") + nccl().GetErrorString(r));
      break;
    }
    std::vector<int> all(2 * D->nranks);
    CK(cudaMemcpyAsync(all.data(), flags + 2, sizeof(int) * 2 * D->nranks, cudaMemcpyDeviceToHost, D->comm));
    CK(cudaStreamSynchronize(D->comm));
    bool stop = true;
    for (int q = 0; q < D->nranks; ++q) {
      any_err = any_err || all[2 * q];
      stop = stop && all[2 * q + 1];
    }
    if (any_err || stop || j >= cfg->max_iters) break;
  }
  cudaFree(flags);
  if (L.err) return L.err;
  if (rc) return rc;
  CK(cudaStreamWaitEvent(s, D->ev_coef, 0));
  CK(cudaEventRecord(ws->ev1, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaStreamSynchronize(D->comm));
  CK(cudaGetLastError());
  if (L.evidence) {
    long long k = 0;
    for (auto& ev : evidence) {
      if (k >= cfg->events_cap) break;
      float t = 0.f;
      cudaEventElapsedTime(&t, ws->ev0, ev.e);
      cfg->events_out[4 * k + 0] = (double)ev.iter;
      cfg->events_out[4 * k + 1] = ev.kind;
      cfg->events_out[4 * k + 2] = ev.tag;
      cfg->events_out[4 * k + 3] = t;
      ++k;
    }
    if (cfg->events_count) *cfg->events_count = k;
  }
  rc = collect_result(m, method, cfg, res, L, marks, 0);
  if (rc == PBS_OK && any_err) {  // another rank raised: raise here too
    res->nonfinite_tag = PBS_TAG_AS;
    res->nonfinite_index = -1;
    return set_err(ctx, PBS_ERR_NONFINITE, "non-finite SpMV output on another rank");
  }
  return rc;
}

// ------------------------------------------------------------ multi-GPU C-ABI

PBS_EXPORT int pbs_nccl_unique_id(void* out) {
  NcclApi& A = nccl();
  if (!A.ok) return set_err(nullptr, PBS_ERR_NCCL, A.err);
  ncclUniqueId id;
  ncclResult_t r = A.GetUniqueId(&id);
  if (r != ncclSuccess) return set_err(nullptr, PBS_ERR_NCCL, A.GetErrorString(r));
  memcpy(out, &id, sizeof(id));
  return PBS_OK;
}

PBS_EXPORT int pbs_dist_init(pbs_ctx* ctx, int32_t nranks, int32_t rank, const void* id_halo,
                             const void* id_red, pbs_dist** out) {
  if (!ctx || !out) return set_err(ctx, PBS_ERR_INVALID, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_err(ctx, PBS_ERR_INVALID, "bad rank / nranks");
  NcclApi& A = nccl();
  if (!A.ok) return set_err(ctx, PBS_ERR_NCCL, A.err);
  CK(cudaSetDevice(ctx->device));
  pbs_dist* d = new pbs_dist();
  d->ctx = ctx;
  d->nranks = nranks;
  d->rank = rank;
  ncclUniqueId a, b;
  memcpy(&a, id_halo, sizeof(a));
  memcpy(&b, id_red, sizeof(b));
  ncclResult_t r = A.CommInitRank(&d->halo, nranks, a, rank);
  if (r == ncclSuccess) r = A.CommInitRank(&d->red, nranks, b, rank);
  if (r != ncclSuccess) {
    delete d;
    return set_err(ctx, PBS_ERR_NCCL, std::string("ncclCommInitRank: ") + A.GetErrorString(r));
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CK(cudaStreamCreateWithPriority(&d->comm, cudaStreamNonBlocking, hi));  // reduction first
  CK(cudaEventCreateWithFlags(&d->ev_part, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&d->ev_coef, cudaEventDisableTiming));
  CK(cudaStreamCreateWithPriority(&d->hstream, cudaStreamNonBlocking, hi));
  CK(cudaEventCreateWithFlags(&d->ev_vec, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&d->ev_halo, cudaEventDisableTiming));
  CK(cudaMalloc(&d->sendbuf, sizeof(double) * kPartStride));
  CK(cudaMalloc(&d->recvbuf, sizeof(double) * kPartStride * nranks));
  *out = d;
  return PBS_OK;
}

PBS_EXPORT int pbs_dist_destroy(pbs_dist* d) {
  if (!d) return PBS_OK;
  cudaSetDevice(d->ctx->device);
  cudaStreamSynchronize(d->comm);
  if (d->halo) nccl().CommDestroy(d->halo);
  if (d->red) nccl().CommDestroy(d->red);
  cudaStreamDestroy(d->comm);
  cudaEventDestroy(d->ev_part);
  cudaEventDestroy(d->ev_coef);
  cudaStreamSynchronize(d->hstream);
  cudaStreamDestroy(d->hstream);
  cudaEventDestroy(d->ev_vec);
  cudaEventDestroy(d->ev_halo);
  cudaFree(d->sendbuf);
  cudaFree(d->recvbuf);
  delete d;
  return PBS_OK;
}

// Last row reading a left-halo column and first row reading a right-halo
// column of a slab's extended-space CSR (out[0] starts at -1, out[1] at n).
__global__ void halo_rows_kernel(const long long* rp, const int* ci, long long n, long long own_lo,
                                 long long own_hi, unsigned long long* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    bool left = false, right = false;
    for (long long k = rp[i]; k < rp[i + 1]; ++k) {
      left = left || ci[k] < own_lo;
      right = right || ci[k] >= own_hi;
    }
    if (left) atomicMax(&out[0], (unsigned long long)(i + 1));  // stored +1 (0 = none)
    if (right) atomicMin(&out[1], (unsigned long long)i);
  }
}

PBS_EXPORT int pbs_mat_set_partition(pbs_mat* m, pbs_dist* dist, int64_t n_global, int64_t row_lo, int64_t hl,
                                     int64_t hr, int32_t nsend, const int64_t* sends, int32_t nrecv,
                                     const int64_t* recvs) {
  if (!m || !dist) return set_err(nullptr, PBS_ERR_INVALID, "NULL argument");
  pbs_ctx* ctx = m->ctx;
  if (m->stencil) return set_err(ctx, PBS_ERR_UNSUPPORTED, "partitioned operators are CSR slabs");
  const long long pad = hl & 1;
  if (m->n_cols != pad + hl + m->n_rows + hr)
    return set_err(ctx, PBS_ERR_INVALID, "n_cols must equal pad + hl + n_own + hr (extended space)");
  if (m->ws) {  // the workspace layout depends on the partition
    free_ws(m->ws);
    m->ws = nullptr;
  }
  Partition& P = m->part;
  P.dist = dist;
  P.n_global = n_global;
  P.row_lo = row_lo;
  P.hl = hl;
  P.hr = hr;
  P.sends.assign(sends, sends + 3 * (size_t)nsend);
  P.recvs.assign(recvs, recvs + 3 * (size_t)nrecv);
  for (size_t i = 0; i < P.sends.size(); i += 3)
    if (P.sends[i + 1] < 0 || P.sends[i + 1] + P.sends[i + 2] > m->n_rows)
      return set_err(ctx, PBS_ERR_INVALID, "halo send outside the own segment");
  for (size_t i = 0; i < P.recvs.size(); i += 3)
    if (P.recvs[i + 1] < 0 || P.recvs[i + 1] + P.recvs[i + 2] > m->n_cols)
      return set_err(ctx, PBS_ERR_INVALID, "halo receive outside the extended space");
  // interior / boundary split of the SpMVs that follow a halo exchange
  {
    const long long n = m->n_rows, own_lo = pad + hl, own_hi = own_lo + n;
    unsigned long long* d = nullptr;
    unsigned long long h[2] = {0ULL, (unsigned long long)n};
    CK(cudaMalloc(&d, sizeof(h)));
    CK(cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice));
    if (n > 0) halo_rows_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(m->rp, m->ci, n, own_lo, own_hi, d);
    CK(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(d);
    long long b0 = (long long)h[0], b1 = (long long)h[1];  // rows [b0, b1) read no halo column
    // PBS_SPLIT_TEST=k (tests): treat the first and last k blocks as boundary
    // rows even without halos, so one GPU exercises the split schedule
    const char* st = getenv("PBS_SPLIT_TEST");
    const long long force = st ? atoll(st) : 0;
    if (force > 0) {
      b0 = std::max(b0, force * kPipeRows);
      b1 = std::min(b1, n - force * kPipeRows);
    }
    P.L0 = (b0 + kPipeRows - 1) / kPipeRows * kPipeRows;
    P.L1 = b1 >= n ? n : b1 / kPipeRows * kPipeRows;
    const char* sp = getenv("PBS_SPLIT");  // PBS_SPLIT=0: exchange first, then one SpMV over all rows
    const bool allow = !(sp && atoi(sp) == 0);
    P.split = allow && (dist->nranks > 1 || force > 0) && P.L1 > P.L0 && (P.L0 > 0 || P.L1 < n);
  }
  return PBS_OK;
}
