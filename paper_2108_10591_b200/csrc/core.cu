// core.cu — libpbsafe contexts, HBM operators (CSR upload, x windows,
// matrix-free stencils, stencil -> CSR on the device), workspaces, the
// kernel-table entry points and the single-GPU C-ABI declared in
// include/pbsafe.h.
#include <array>
#include <cub/device/device_scan.cuh>

#include "host.h"

// PBS_UPLOAD_TIMING=<ms>: print the host-side phase times of an upload that
// takes longer than <ms> (stall hunting; off by default)
#include <chrono>
struct UploadTimer {
  std::chrono::steady_clock::time_point t0, last;
  std::string log;
  double limit = -1;
  void start() {
    static const char* e = getenv("PBS_UPLOAD_TIMING");
    limit = e ? atof(e) : -1;
    if (limit < 0) return;
    t0 = last = std::chrono::steady_clock::now();
    log.clear();
  }
  void mark(const char* what) {
    if (limit < 0) return;
    auto now = std::chrono::steady_clock::now();
    char buf[96];
    snprintf(buf, sizeof(buf), " %s %.2f", what, std::chrono::duration<double, std::milli>(now - last).count());
    log += buf;
    last = now;
  }
  void stop() {
    if (limit < 0) return;
    const double tot = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (tot > limit) fprintf(stderr, "[pbs upload %.1f ms]%s\n", tot, log.c_str());
  }
};
static UploadTimer g_upt;

std::string g_last_error;

void free_graphs(Workspace* ws) {
  for (auto& kv : ws->graphs) cudaGraphExecDestroy(kv.second.first);
  ws->graphs.clear();
}

void free_ws(Workspace* ws) {
  if (!ws) return;
  free_graphs(ws);
  pbs_ctx* ctx = ws->ctx;
  if (ws->base_ipc)
    cudaFree(ws->base);
  else
    pool_free(ctx, ws->base);
  pool_free(ctx, ws->partials);
  pool_free(ctx, ws->partials12);
  pool_free(ctx, ws->plan_bounds);
  pool_free(ctx, ws->st);
  if (ws->mirror_h) cudaFreeHost(ws->mirror_h);
  pool_free(ctx, ws->hist_rel);
  pool_free(ctx, ws->hist_flags);
  pool_free(ctx, ws->hist_coef);
  if (ws->ev0) cudaEventDestroy(ws->ev0);
  if (ws->ev1) cudaEventDestroy(ws->ev1);
  if (ws->trace_host) cudaFreeHost(ws->trace_host);
  delete ws;
}

MatSig mat_sig(const pbs_mat* m) {
  MatSig g;
  memset(&g, 0, sizeof(g));  // padding too: signatures compare with memcmp
  g.n_rows = m->n_rows;
  g.n_cols = m->n_cols;
  g.nnz = m->nnz;
  g.blk_nnz_max = m->blk_nnz_max;
  g.stencil = m->stencil;
  g.rp = m->rp;
  g.ci = m->ci;
  g.v = m->v;
  g.wc = m->wc;
  g.sell_v = m->sell_v;
  g.sell_c = m->sell_c;
  g.sell_off = m->sell_off;
  g.sell_len = m->sell_len;
  g.sell_vi = m->sell_vi;
  g.sell_dict = m->sell_dict;
  g.sell_mode = m->sell_mode;
  g.sell_lmax = m->sell_lmax;
  memcpy(&g.xwin, &m->xwin, sizeof(XWin));
  memcpy(&g.sv, &m->sv, sizeof(StencilView));
  memcpy(&g.swin, &m->swin, sizeof(StencilWin));
  return g;
}

void drop_ws_cache(pbs_ctx* ctx) {
  if (!ctx || !ctx->ws_cache) return;
  free_ws(ctx->ws_cache);
  ctx->ws_cache = nullptr;
}

int ensure_ws(pbs_mat* m, long long hist_slots) {
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  if (!ws && ctx->ws_cache && !m->part.dist) {
    const MatSig g = mat_sig(m);
    if (ctx->ws_cache->n == m->n_rows) {
      // The vectors, state block, host mirror and events only depend on n:
      // adopt them.  The graphs bake the operator's pointers and layout in,
      // so they survive only an identical signature (the pool usually hands
      // a same-shape upload the same addresses, but not always — and
      // rebuilding the whole workspace, with its page-locked mirror, costs
      // 50-700 ms where re-capturing the graphs costs a few).
      ws = m->ws = ctx->ws_cache;
      ctx->ws_cache = nullptr;
      if (memcmp(&g, &ctx->ws_sig, sizeof(MatSig)) != 0) free_graphs(ws);
    } else {
      drop_ws_cache(ctx);
    }
  }
  if (!ws) {
    ws = new Workspace();
    ws->ctx = ctx;
    m->ws = ws;
    ws->n = m->n_rows;
    ws->n_ext = m->part.dist ? m->n_cols : m->n_rows;
    ws->own_off = m->part.dist ? m->part.hl + (m->part.hl & 1) : 0;  // even: 16-byte aligned
    // +2: aligned bulk-copy over-read; even own offset keeps 16-byte alignment
    ws->stride = ((size_t)ws->n_ext + 4 + 31) / 32 * 32;
    if (m->part.dist) {  // peers copy halos straight into it (CUDA IPC)
      CK(cudaMalloc(&ws->base, sizeof(double) * ws->stride * kNumVecs));
      ws->base_ipc = true;
    } else {
      CK(pool_alloc(ctx, &ws->base, sizeof(double) * ws->stride * kNumVecs));
    }
    CK(cudaMemsetAsync(ws->base, 0, sizeof(double) * ws->stride * kNumVecs, ctx->stream));
    for (int k = 0; k < kNumVecs; ++k) {
      ws->X.v[k] = ws->base + ws->stride * k;
      ws->V.v[k] = ws->X.v[k] + ws->own_off;
    }
    CK(pool_alloc(ctx, &ws->partials, sizeof(double) * kMaxParts * kPartStride));
    CK(pool_alloc(ctx, &ws->partials12, sizeof(double) * kMaxParts * kPartStride));
    CK(pool_alloc(ctx, &ws->st, sizeof(SolverState)));
    CK(cudaHostAlloc(&ws->mirror_h, sizeof(HostMirror), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&ws->mirror_d, ws->mirror_h, 0));
    CK(cudaEventCreate(&ws->ev0));
    CK(cudaEventCreate(&ws->ev1));
  }
  if (hist_slots > ws->hist_cap) {
    pool_free(ctx, ws->hist_rel);
    pool_free(ctx, ws->hist_flags);
    pool_free(ctx, ws->hist_coef);
    long long cap = hist_slots < 1024 ? 1024 : hist_slots;
    CK(pool_alloc(ctx, &ws->hist_rel, sizeof(double) * cap));
    CK(pool_alloc(ctx, &ws->hist_flags, cap));
    CK(pool_alloc(ctx, &ws->hist_coef, sizeof(double) * 4 * cap));
    ws->hist_cap = cap;
    free_graphs(ws);  // graphs capture the state pointer only, but keep it simple
  }
  return PBS_OK;
}

// PartitionPlan.balanced (reduction.py:80-87) bounds, numpy linspace semantics
int plan_balanced(long long n, long long workers, std::vector<long long>& b) {
  long long cap = n > 1 ? n : 1;
  if (workers > cap) workers = cap;
  b.resize(workers + 1);
  double step = (double)n / (double)workers;
  for (long long k = 0; k < workers; ++k) {
    double y = (step == 0.0) ? ((double)k / (double)workers) * (double)n : (double)k * step;
    b[k] = (long long)y;
  }
  b[workers] = n;
  return (int)workers;
}

int ensure_plan(pbs_mat* m, int workers) {
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  if (workers < 1) return set_err(ctx, PBS_ERR_INVALID, "plan_workers must be >= 1");
  if (ws->plan_workers == workers && ws->plan_bounds) return PBS_OK;
  std::vector<long long> b;
  int w = plan_balanced(ws->n, workers, b);
  if (w > kMaxParts) return set_err(ctx, PBS_ERR_INVALID, "plan_workers too large for the device plan");
  pool_free(ctx, ws->plan_bounds);
  CK(pool_alloc(ctx, &ws->plan_bounds, sizeof(long long) * (w + 1)));
  CK(cudaMemcpyAsync(ws->plan_bounds, b.data(), sizeof(long long) * (w + 1), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ws->plan_workers = workers;
  ws->plan_w_actual = w;
  free_graphs(ws);
  return PBS_OK;
}

void Launcher::trace_point() {
  if (!trace_cfg || !trace_cfg->trace_fn || trace_rc) return;
  Workspace* ws = trace_ws;
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    trace_rc = set_err(ctx, PBS_ERR_CUDA, "sync failed while tracing");
    return;
  }
  SolverState st;
  cudaMemcpy(&st, ws->st, sizeof(st), cudaMemcpyDeviceToHost);
  if (!st.run_all || st.nf_row != (unsigned long long)kNoError) return;  // iteration did not run
  const size_t n = (size_t)ws->n;
  if (!ws->trace_host &&
      cudaHostAlloc(&ws->trace_host, sizeof(double) * 13 * (n > 0 ? n : 1), cudaHostAllocDefault) != cudaSuccess) {
    trace_rc = set_err(ctx, PBS_ERR_NOMEM, "cannot allocate trace staging");
    return;
  }
  // the reference's trace_hook dicts: Safe methods (solvers.py:725-732),
  // BiCGStab (315), GPBi-CG (448)
  static const int safe_order[13] = {VX, VR, VP, VU, VO, VT, VW, VY, VZ, VS, VQ, VG, VL};
  static const int stab_order[6] = {VX, VR, VP, VT, VAP, VAT};
  static const int gp_order[8] = {VX, VR, VP, VU, VT, VW, VY, VZ};
  static const int ps_order[10] = {VX, VR, VP, VS, VZ, VQ, VY, VW, VT, VO};
  const int* order = safe_order;
  int nv = 13;
  if (trace_method == PBS_METHOD_BICGSTAB) {
    order = stab_order;
    nv = 6;
  } else if (trace_method == PBS_METHOD_GPBICG) {
    order = gp_order;
    nv = 8;
  } else if (trace_method == PBS_METHOD_PBICGSTAB) {
    order = ps_order;
    nv = 10;
  }
  double* ptrs[13];
  for (int k = 0; k < nv; ++k) {
    ptrs[k] = ws->trace_host + k * n;
    cudaMemcpy(ptrs[k], ws->V.v[order[k]], sizeof(double) * n, cudaMemcpyDeviceToHost);
  }
  trace_cfg->trace_fn(iter, ptrs, trace_cfg->trace_user);
}

int get_graph(pbs_ctx* ctx, pbs_mat* m, long long key, IterFn fn, const Mode& md,
                     cudaGraphExec_t* out, long long* nkernels) {
  Workspace* ws = m->ws;
  auto it = ws->graphs.find(key);
  if (it != ws->graphs.end()) {
    *out = it->second.first;
    *nkernels = it->second.second;
    return PBS_OK;
  }
  cudaGraph_t g;
  Launcher L{ctx, m, ctx->stream};
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  fn(L, ws, md);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  if (L.err) {
    if (e == cudaSuccess) cudaGraphDestroy(g);
    return L.err;
  }
  if (e != cudaSuccess) return set_err(ctx, PBS_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  cudaGraphExec_t ge;
  e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return set_err(ctx, PBS_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  ws->graphs[key] = {ge, L.launches};
  *out = ge;
  *nkernels = L.launches;
  return PBS_OK;
}

// ------------------------------------------------------------------- solving

int validate_cfg(pbs_ctx* ctx, const pbs_config* cfg) {
  if (!cfg) return set_err(ctx, PBS_ERR_INVALID, "config is NULL");
  if (!(cfg->tol > 0.0)) return set_err(ctx, PBS_ERR_INVALID, "tol must be positive");
  if (cfg->max_iters < 1) return set_err(ctx, PBS_ERR_INVALID, "max_iters must be >= 1");
  if (cfg->rr_epoch < 1) return set_err(ctx, PBS_ERR_INVALID, "rr_epoch must be >= 1");
  if (cfg->rr_cutoff > cfg->max_iters) return set_err(ctx, PBS_ERR_INVALID, "rr_cutoff must lie in [0, max_iters]");
  if (cfg->reduce_mode != PBS_REDUCE_TREE && cfg->reduce_mode != PBS_REDUCE_PLAN)
    return set_err(ctx, PBS_ERR_INVALID, "unknown reduce_mode");
  return PBS_OK;
}

// Device state -> pbs_result (+ the reference's SpMV tally)
int collect_result(pbs_mat* m, int method, const pbs_config* cfg, pbs_result* res, Launcher& L,
                          std::vector<std::pair<int, cudaEvent_t>>& marks, long long launched_graph_kernels) {
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  const bool pipelined = method == PBS_METHOD_PBICGSAFE || method == PBS_METHOD_PBICGSAFE_RR;
  const bool rr = method == PBS_METHOD_PBICGSAFE_RR;
  const long long cutoff = cfg->rr_cutoff >= 0 ? cfg->rr_cutoff : cfg->max_iters;
  SolverState out;
  CK(cudaMemcpy(&out, ws->st, sizeof(out), cudaMemcpyDeviceToHost));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ws->ev0, ws->ev1);
  memset(res, 0, sizeof(*res));
  res->device_ms = ms;
  res->kernel_launches = L.launches + launched_graph_kernels;
  if (L.timing) {
    for (size_t k = 1; k < marks.size(); ++k) {
      float d = 0.f;
      cudaEventElapsedTime(&d, marks[k - 1].second, marks[k].second);
      int kind = marks[k].first;
      if (kind >= 0 && kind < PBS_NUM_KERNEL_KINDS) {
        res->kernel_ms[kind] += d;
        res->kernel_count[kind] += 1;
      }
    }
  }
  res->status = out.status;
  res->breakdown = out.breakdown;
  res->iterations = out.iterations;
  res->failure_iter = out.failure_iter;
  res->n_records = out.n_records;
  res->r0_norm = out.r0_norm;
  res->nonfinite_index = -1;
  if (out.nf_row != (unsigned long long)kNoError) {
    res->nonfinite_tag = out.nf_tag & 0xff;  // the multi-GPU schedule adds the launch sequence above
    res->nonfinite_index = (long long)out.nf_row + (m->part.dist ? m->part.row_lo : 0);
    return set_err(ctx, PBS_ERR_NONFINITE, "non-finite SpMV output");
  }
  if (out.status < 0) return set_err(ctx, PBS_ERR_CUDA, "solver ended without a status");
  // SpMV count as the reference tallies it (solvers.py:613-723, 530-569)
  const long long reached = out.status == PBS_MAX_ITERS || out.iterations == cfg->max_iters
                                ? cfg->max_iters
                                : out.iterations + 1;
  const long long completed = out.iterations;
  long long nrep = 0;
  if (rr)
    for (long long i = 1; i < completed && i < cutoff; ++i)
      if (i % cfg->rr_epoch == 0) ++nrep;
  res->n_replacements = nrep;
  res->stop_stage = out.stop_stage;
  if (method == PBS_METHOD_BICGSTAB || method == PBS_METHOD_GPBICG)
    // r0 = b - A x0, then Ap and At per completed iteration; a stopping
    // iteration that got past its loop-top check ran Ap (alpha stage) or both
    res->n_spmv = 1 + 2 * completed + (out.stop_stage == 0 ? 0 : (out.stop_stage == 1 ? 1 : 2));
  else if (method == PBS_METHOD_PBICGSTAB)
    // r0 = b - A x0 and w0 = A r0, then t = A w and v = A z per completed
    // iteration; a stopping iteration past its alpha ran both
    res->n_spmv = 2 + 2 * completed + (out.stop_stage >= 2 ? 2 : 0);
  else if (pipelined)
    res->n_spmv = 2 + reached + completed + 5 * nrep;
  else
    res->n_spmv = 1 + reached + completed;
  return PBS_OK;
}

int copy_history(pbs_mat* m, const pbs_result* res, double* hist_rel, uint8_t* hist_flags,
                        double* hist_coef) {
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  long long k = res->n_records;
  if (k <= 0) return PBS_OK;
  if (hist_rel) CK(cudaMemcpy(hist_rel, ws->hist_rel, sizeof(double) * k, cudaMemcpyDeviceToHost));
  if (hist_flags) CK(cudaMemcpy(hist_flags, ws->hist_flags, k, cudaMemcpyDeviceToHost));
  if (hist_coef) CK(cudaMemcpy(hist_coef, ws->hist_coef, sizeof(double) * 4 * k, cudaMemcpyDeviceToHost));
  return PBS_OK;
}

// ============================================================== C-ABI

PBS_EXPORT const char* pbs_last_error(pbs_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

PBS_EXPORT int pbs_init(int device, pbs_ctx** out) {
  pbs_ctx* ctx = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return set_err(nullptr, PBS_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= count) return set_err(nullptr, PBS_ERR_INVALID, "device index out of range");
  ctx = new pbs_ctx();
  ctx->device = device;
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  ctx->sms = prop.multiProcessorCount;
  ctx->cc_major = prop.major;
  ctx->cc_minor = prop.minor;
  if (prop.major != 10) {
    std::string msg = std::string("libpbsafe is built for sm_100a; device is sm_") +
                      std::to_string(prop.major) + std::to_string(prop.minor);
    delete ctx;
    return set_err(nullptr, PBS_ERR_UNSUPPORTED, msg);
  }
  CK(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
  ctx->stream = ctx->own;
  {
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;  // keep freed blocks cached for the next upload
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  CK(cudaMalloc(&ctx->partials, sizeof(double) * kMaxParts * kPartStride));
  CK(cudaMalloc(&ctx->tmp_state, sizeof(SolverState)));
  *out = ctx;
  return PBS_OK;
}

PBS_EXPORT int pbs_destroy(pbs_ctx* ctx) {
  if (!ctx) return PBS_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  drop_ws_cache(ctx);
  buf_flush(ctx);
  cudaFree(ctx->scratch);
  cudaFree(ctx->partials);
  cudaFree(ctx->tmp_state);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
  return PBS_OK;
}

PBS_EXPORT int pbs_device_info(pbs_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor) {
  if (!ctx) return set_err(nullptr, PBS_ERR_INVALID, "ctx is NULL");
  if (sm_count) *sm_count = ctx->sms;
  if (cc_major) *cc_major = ctx->cc_major;
  if (cc_minor) *cc_minor = ctx->cc_minor;
  return PBS_OK;
}

PBS_EXPORT int pbs_set_stream(pbs_ctx* ctx, uintptr_t stream) {
  if (!ctx) return set_err(nullptr, PBS_ERR_INVALID, "ctx is NULL");
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own;
  return PBS_OK;
}

__global__ void cvt_i64_i32_kernel(const long long* in, int* out, long long n, int* bad, long long ncols) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    long long c = in[i];
    if (c < 0 || c >= ncols) *bad = 1;
    out[i] = (int)c;
  }
}

constexpr int kBinsOut = 1024;  // occupied offset bins read back, at most

__global__ void bins_init_kernel(int* bmin, int* bmax, int* occ, int* wide);
__global__ void bins_compact_kernel(const int* bmin, const int* bmax, int* occ);

// Offset histogram for the x windows: bin = floor((col - row) / 256); per bin
// the min / max offset seen (warp-aggregated atomics); |bin| >= kBins -> wide.
constexpr int kBins = 65536;
__global__ void offset_bins_kernel(const long long* rp, const int* ci, long long n_rows, int* bmin, int* bmax,
                                   int* wide) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long r_first = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long rb = (long long)blockIdx.x * blockDim.x; rb < n_rows; rb += stride) {
    const long long row = rb + threadIdx.x;
    const bool live = row < n_rows;
    long long s = 0, e = 0;
    if (live) {
      s = rp[row];
      e = rp[row + 1];
    }
    int len = (int)(e - s), maxlen = len;
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    for (int k = 0; k < maxlen; ++k) {
      const bool act = k < len;
      long long off = act ? (long long)ci[s + k] - row : 0;
      const long long bin = off >= 0 ? off / 256 : -((-off + 255) / 256);
      const bool in = act && bin > -kBins && bin < kBins;
      if (act && !in) *wide = 1;
      const int key = in ? (int)bin : 0x7fffffff;
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      const int o32 = (int)off;
      const int gmin = __reduce_min_sync(grp, in ? o32 : 0x7fffffff);
      const int gmax = __reduce_max_sync(grp, in ? o32 : (int)0x80000000);
      if (in && (threadIdx.x & 31) == __ffs(grp) - 1) {
        atomicMin(bmin + bin + kBins, gmin);
        atomicMax(bmax + bin + kBins, gmax);
      }
    }
  }
  (void)r_first;
}

__global__ void bins_init_kernel(int* bmin, int* bmax, int* occ, int* wide) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < 2 * kBins) {
    bmin[b] = 0x7fffffff;
    bmax[b] = (int)0x80000000;
  }
  if (b == 0) {
    occ[0] = 0;
    *wide = 0;
  }
}

// occupied bins -> (bin, min, max) triples in occ[1..] (any order; occ[0] counts them all)
__global__ void bins_compact_kernel(const int* bmin, const int* bmax, int* occ) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= 2 * kBins || bmin[b] > bmax[b]) return;
  const int k = atomicAdd(occ, 1);
  if (k < kBinsOut) {
    occ[1 + 3 * k] = b;
    occ[2 + 3 * k] = bmin[b];
    occ[3 + 3 * k] = bmax[b];
  }
}

// Window-local column of every nonzero: the staged offset of x[col] in its
// row block's x windows, by the rule the staged engine's producer and
// consumers use (csr_pipe_kernel: window c spans [r0 + wmin[c], r0 + nr - 1 +
// wmax[c]] clamped to x and aligned down to even, staged at the sum of the
// earlier caps; a column belongs to the last window starting at or before it).
// *bad = 1 when a column falls outside its window (the engine then keeps
// col_idx).
__global__ void window_cols_kernel(const long long* rp, const int* ci, long long n_rows, long long n_cols, XWin W,
                                   unsigned short* wc, int* bad) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (W.band_s) {  // band mode: the column's slot in the circular buffer
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += stride)
      for (long long k = rp[i]; k < rp[i + 1]; ++k) wc[k] = (unsigned short)(ci[k] % W.band_s);
    return;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += stride) {
    const long long r0 = i / kPipeRows * kPipeRows;
    const long long nr = min((long long)kPipeRows, n_rows - r0);
    long long wlo[kMaxWin], whi[kMaxWin];
    int soff[kMaxWin];
    int acc = 0;
#pragma unroll
    for (int c = 0; c < kMaxWin; ++c) {
      wlo[c] = 0x7fffffff;
      whi[c] = 0;
      soff[c] = acc;
      if (c < W.nwin) {
        long long lo = r0 + W.wmin[c], hi = r0 + nr - 1 + W.wmax[c] + 1;
        if (lo < 0) lo = 0;
        if (hi > n_cols) hi = n_cols;
        wlo[c] = lo & ~1LL;
        whi[c] = hi > lo ? ((hi + 1) & ~1LL) : wlo[c];
        acc += W.cap[c];
      }
    }
    for (long long k = rp[i]; k < rp[i + 1]; ++k) {
      const long long col = ci[k];
      int c = 0;
#pragma unroll
      for (int cc = 1; cc < kMaxWin; ++cc)
        if (col >= wlo[cc]) c = cc;
      const long long off = col - wlo[c];
      if (off < 0 || col >= whi[c] || off + soff[c] >= W.total) {
        *bad = 1;
        wc[k] = 0;
      } else {
        wc[k] = (unsigned short)(off + soff[c]);
      }
    }
  }
}

// ---- sliced-ELL copy of a window-mode operator (sell.cuh)

// levels (longest row) of each 256-row block, as entries: out[b + 1] = 256 * L_b
__global__ void sell_levels_kernel(const long long* rp, long long n_rows, long long nblk, long long* out, int* lmax) {
  __shared__ int wmax[8];
  for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
    const long long r = b * kPipeRows + threadIdx.x;
    int len = r < n_rows ? (int)(rp[r + 1] - rp[r]) : 0;
    len = __reduce_max_sync(0xffffffffu, len);
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = len;
    __syncthreads();
    if (threadIdx.x == 0) {
      int L = 0;
      for (int w = 0; w < 8; ++w) L = max(L, wmax[w]);
      out[b + 1] = (long long)L * kPipeRows;
      atomicMax(lmax, L);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

// ---- value dictionary: the distinct f64 bit patterns of the operator, when
// there are at most kSellDict.  An open-addressing table of kDictSlots keys;
// kDictEmpty (a NaN payload) marks a free slot and is itself refused as a value.
constexpr int kDictSlots = 1024;
constexpr unsigned long long kDictEmpty = 0x7ff8dead00000001ULL;

__device__ __forceinline__ unsigned dict_hash(unsigned long long b) {
  b ^= b >> 33;
  b *= 0xff51afd7ed558ccdULL;
  b ^= b >> 33;
  return (unsigned)b & (kDictSlots - 1);
}

// ctl[0]: distinct values seen, ctl[1]: gave up (too many, or the reserved pattern)
__global__ void dict_insert_kernel(const double* v, long long nnz, unsigned long long* table, int* ctl) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  // the thread's last eight distinct patterns: an operator with a handful of
  // values never goes back to the table after its first few nonzeros
  unsigned long long seen[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) seen[k] = kDictEmpty;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[i]);
    if (b == kDictEmpty) {  // the free-slot marker itself: no dictionary for this operator
      ctl[1] = 1;
      return;
    }
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) hit |= b == seen[k];
    if (hit) continue;
#pragma unroll
    for (int k = 7; k > 0; --k) seen[k] = seen[k - 1];
    seen[0] = b;
    if (*(volatile int*)(ctl + 1)) return;
    unsigned h = dict_hash(b);
    for (int probe = 0; probe < kDictSlots; ++probe, h = (h + 1) & (kDictSlots - 1)) {
      unsigned long long cur = *(volatile unsigned long long*)(table + h);
      if (cur == b) break;
      if (cur == kDictEmpty) {
        cur = atomicCAS(table + h, kDictEmpty, b);
        if (cur == kDictEmpty) {
          if (atomicAdd(ctl, 1) >= kSellDict) ctl[1] = 1;
          break;
        }
        if (cur == b) break;
      }
    }
  }
}

// occupied slots -> dictionary entries, in slot order (one thread: 1024 slots)
__global__ void dict_compact_kernel(const unsigned long long* table, double* dict, unsigned char* slot_idx) {
  int n = 0;
  for (int h = 0; h < kDictSlots; ++h) {
    const unsigned long long b = table[h];
    if (b != kDictEmpty && n < kSellDict) {
      dict[n] = __longlong_as_double((long long)b);
      slot_idx[h] = (unsigned char)n++;
    }
  }
  for (; n < kSellDict; ++n) dict[n] = 0.0;
}

__device__ __forceinline__ unsigned char dict_lookup(const unsigned long long* table, const unsigned char* slot_idx,
                                                     double val) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(val);
  unsigned h = dict_hash(b);
  for (int probe = 0; probe < kDictSlots; ++probe, h = (h + 1) & (kDictSlots - 1))
    if (__ldg(table + h) == b) return __ldg(slot_idx + h);
  return 0;  // unreachable: every value was inserted
}

// entry (k, t) of block b: the k-th nonzero of row 256 b + t, or padding.
// table != null: the value's dictionary index goes to svi instead of sv.
__global__ void sell_fill_kernel(const long long* rp, const double* v, const unsigned short* wc, long long n_rows,
                                 long long nblk, const long long* soff, double* sv, unsigned short* sc,
                                 unsigned char* slen, const unsigned long long* table,
                                 const unsigned char* slot_idx, unsigned char* svi) {
  for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
    const long long r = b * kPipeRows + threadIdx.x;
    long long s = 0;
    int len = 0;
    if (r < n_rows) {
      s = rp[r];
      len = (int)(rp[r + 1] - s);
    }
    const long long off = soff[b];
    const int L = (int)((soff[b + 1] - off) / kPipeRows);
    for (int k = 0; k < L; ++k) {
      const long long e = off + (long long)k * kPipeRows + threadIdx.x;
      if (table)
        svi[e] = k < len ? dict_lookup(table, slot_idx, v[s + k]) : (unsigned char)0;
      else
        sv[e] = k < len ? v[s + k] : 0.0;
      sc[e] = k < len ? wc[s + k] : (unsigned short)0;
    }
    slen[b * kPipeRows + threadIdx.x] = (unsigned char)len;
  }
}

// ---- pair dictionary: the distinct (value, staged column - row slot) pairs,
// keyed (value-dictionary index << 32 | relative column) in a second hash set;
// kPairPadKey is the padding entry's pair (value 0, relative column 0).
constexpr unsigned long long kPairPadKey = 0xffffffff00000000ULL;

__device__ __forceinline__ void pair_insert(unsigned long long key, unsigned long long* table, int* ctl) {
  unsigned h = dict_hash(key);
  for (int probe = 0; probe < kDictSlots; ++probe, h = (h + 1) & (kDictSlots - 1)) {
    unsigned long long cur = *(volatile unsigned long long*)(table + h);
    if (cur == key) return;
    if (cur == kDictEmpty) {
      cur = atomicCAS(table + h, kDictEmpty, key);
      if (cur == kDictEmpty) {
        if (atomicAdd(ctl, 1) >= kSellDict) ctl[1] = 1;
        return;
      }
      if (cur == key) return;
    }
  }
}

__global__ void pair_insert_kernel(const long long* rp, const double* v, const unsigned short* wc, long long n_rows,
                                   long long nblk, const long long* soff, const unsigned long long* vtable,
                                   const unsigned char* vslot_idx, unsigned long long* table, int* ctl) {
  unsigned long long seen[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) seen[q] = kDictEmpty;  // no key has this pattern (value index < 256 or the pad key)
  for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
    if (*(volatile int*)(ctl + 1)) return;
    const long long r = b * kPipeRows + threadIdx.x;
    long long s = 0;
    int len = 0;
    if (r < n_rows) {
      s = rp[r];
      len = (int)(rp[r + 1] - s);
    }
    const int L = (int)((soff[b + 1] - soff[b]) / kPipeRows);
    for (int k = 0; k < len; ++k) {
      const unsigned vi = dict_lookup(vtable, vslot_idx, v[s + k]);
      const int rel = (int)wc[s + k] - (int)threadIdx.x;
      const unsigned long long key = ((unsigned long long)vi << 32) | (unsigned)rel;
      bool hit = false;  // the thread's last eight distinct pairs (a stencil row repeats the previous row's)
#pragma unroll
      for (int q = 0; q < 8; ++q) hit |= key == seen[q];
      if (hit) continue;
#pragma unroll
      for (int q = 7; q > 0; --q) seen[q] = seen[q - 1];
      seen[0] = key;
      pair_insert(key, table, ctl);
    }
    if (len < L) pair_insert(kPairPadKey, table, ctl);
  }
}

__global__ void pair_compact_kernel(const unsigned long long* table, const double* vdict, SellPair* pairs,
                                    unsigned char* slot_idx) {
  int n = 0;
  for (int h = 0; h < kDictSlots; ++h) {
    const unsigned long long key = table[h];
    if (key != kDictEmpty && n < kSellDict) {
      SellPair p;
      p.v = key == kPairPadKey ? 0.0 : vdict[(unsigned)(key >> 32)];
      p.rel = key == kPairPadKey ? 0 : (int)(unsigned)key;
      p.pad = 0;
      pairs[n] = p;
      slot_idx[h] = (unsigned char)n++;
    }
  }
  for (; n < kSellDict; ++n) pairs[n] = SellPair{0.0, 0, 0};
}

__global__ void sell_fill_pair_kernel(const long long* rp, const double* v, const unsigned short* wc, long long n_rows,
                                      long long nblk, const long long* soff, const unsigned long long* vtable,
                                      const unsigned char* vslot_idx, const unsigned long long* table,
                                      const unsigned char* slot_idx, unsigned char* spi, unsigned char* slen) {
  for (long long b = blockIdx.x; b < nblk; b += gridDim.x) {
    const long long r = b * kPipeRows + threadIdx.x;
    long long s = 0;
    int len = 0;
    if (r < n_rows) {
      s = rp[r];
      len = (int)(rp[r + 1] - s);
    }
    const long long off = soff[b];
    const int L = (int)((soff[b + 1] - off) / kPipeRows);
    for (int k = 0; k < L; ++k) {
      unsigned long long key = kPairPadKey;
      if (k < len) {
        const unsigned vi = dict_lookup(vtable, vslot_idx, v[s + k]);
        key = ((unsigned long long)vi << 32) | (unsigned)((int)wc[s + k] - (int)threadIdx.x);
      }
      unsigned h = dict_hash(key);
      unsigned char idx = 0;
      for (int probe = 0; probe < kDictSlots; ++probe, h = (h + 1) & (kDictSlots - 1))
        if (__ldg(table + h) == key) {
          idx = __ldg(slot_idx + h);
          break;
        }
      spi[off + (long long)k * kPipeRows + threadIdx.x] = idx;
    }
    slen[b * kPipeRows + threadIdx.x] = (unsigned char)len;
  }
}

static void free_sell(pbs_ctx* ctx, pbs_mat* m) {
  buf_free(ctx, m->sell_v);
  buf_free(ctx, m->sell_c);
  buf_free(ctx, m->sell_off);
  buf_free(ctx, m->sell_len);
  buf_free(ctx, m->sell_vi);
  buf_free(ctx, m->sell_dict);
  m->sell_len = nullptr;
  m->sell_vi = nullptr;
  m->sell_dict = nullptr;
  m->sell_ndict = 0;
  m->sell_mode = 0;
  m->sell_v = nullptr;
  m->sell_c = nullptr;
  m->sell_off = nullptr;
  m->sell_lmax = 0;
  m->sell_entries = 0;
}

// Built when the padding stays small (PBS_SELL_PAD percent over nnz, default
// 12; PBS_SELL=0 keeps CSR order only): stencil-like row lengths.
static int build_sell(pbs_ctx* ctx, pbs_mat* m) {
  free_sell(ctx, m);
  if (!m->wc || !m->xwin.nwin || m->xwin.band_s || !env_int("PBS_SELL", 1, 0, 1)) return PBS_OK;
  if (m->n_rows > 0x7fff0000LL || m->n_cols > 0x7fff0000LL) return PBS_OK;  // the engine keeps row indices in 32 bits
  cudaStream_t s = ctx->stream;
  const long long nblk = (m->n_rows + kPipeRows - 1) / kPipeRows;
  int* lmax = nullptr;
  CK(buf_alloc(ctx, &m->sell_off, sizeof(long long) * (nblk + 1)));
  CK(buf_alloc(ctx, &lmax, sizeof(int)));
  CK(cudaMemsetAsync(lmax, 0, sizeof(int), s));
  sell_levels_kernel<<<(int)std::min<long long>(nblk, ctx->sms * 8), kPipeRows, 0, s>>>(m->rp, m->n_rows, nblk, m->sell_off,
                                                                                       lmax);
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, m->sell_off, m->sell_off, nblk + 1, s);
  void* tmp = nullptr;
  CK(buf_alloc(ctx, &tmp, tmp_bytes));
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, m->sell_off, m->sell_off, nblk + 1, s);
  buf_free(ctx, tmp);
  long long entries = 0;
  int hl = 0;
  CK(cudaMemcpyAsync(&entries, m->sell_off + nblk, sizeof(entries), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&hl, lmax, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  g_upt.mark("levels");
  buf_free(ctx, lmax);
  const long long pad_pct = env_int("PBS_SELL_PAD", 12, 0, 1000);
  if (entries <= 0 || hl > kSellMaxLen || entries > m->nnz + m->nnz * pad_pct / 100 + 64 * kPipeRows) {
    free_sell(ctx, m);
    return PBS_OK;
  }
  // value dictionary (PBS_SELL_DICT=0: keep the f64 value stream)
  unsigned long long* table = nullptr;
  unsigned char* slot_idx = nullptr;
  int hctl[2] = {0, 1};
  if (env_int("PBS_SELL_DICT", 1, 0, 1)) {
    int* ctl = nullptr;
    CK(buf_alloc(ctx, &table, sizeof(unsigned long long) * kDictSlots));
    CK(buf_alloc(ctx, &slot_idx, kDictSlots));
    CK(buf_alloc(ctx, &ctl, sizeof(int) * 2));
    std::vector<unsigned long long> empty(kDictSlots, kDictEmpty);
    CK(cudaMemcpyAsync(table, empty.data(), sizeof(unsigned long long) * kDictSlots, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(slot_idx, 0, kDictSlots, s));
    CK(cudaMemsetAsync(ctl, 0, sizeof(int) * 2, s));
    dict_insert_kernel<<<ctx->sms * 8, 256, 0, s>>>(m->v, m->nnz, table, ctl);
    CK(cudaMemcpyAsync(hctl, ctl, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));  // (also keeps `empty` alive until its copy has run)
    g_upt.mark("dict");
    buf_free(ctx, ctl);
  }
  const bool dict = hctl[1] == 0 && hctl[0] <= kSellDict;
  const int grid = (int)std::min<long long>(nblk, ctx->sms * 8);
  CK(buf_alloc(ctx, &m->sell_len, (size_t)nblk * kPipeRows));
  bool pairs = false;
  if (dict) {
    CK(buf_alloc(ctx, &m->sell_dict, sizeof(double) * kSellDict));
    CK(buf_alloc(ctx, &m->sell_vi, (size_t)entries));
    dict_compact_kernel<<<1, 1, 0, s>>>(table, m->sell_dict, slot_idx);
    m->sell_ndict = hctl[0];
    // pair dictionary (PBS_SELL_PAIR=0: keep the u16 column stream)
    if (env_int("PBS_SELL_PAIR", 1, 0, 1)) {
      unsigned long long* ptable = nullptr;
      unsigned char* pslot = nullptr;
      SellPair* pdict = nullptr;
      int* ctl = nullptr;
      int pctl[2] = {0, 1};
      CK(buf_alloc(ctx, &ptable, sizeof(unsigned long long) * kDictSlots));
      CK(buf_alloc(ctx, &pslot, kDictSlots));
      CK(buf_alloc(ctx, &pdict, sizeof(SellPair) * kSellDict));
      CK(buf_alloc(ctx, &ctl, sizeof(int) * 2));
      std::vector<unsigned long long> empty(kDictSlots, kDictEmpty);
      CK(cudaMemcpyAsync(ptable, empty.data(), sizeof(unsigned long long) * kDictSlots, cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(pslot, 0, kDictSlots, s));
      CK(cudaMemsetAsync(ctl, 0, sizeof(int) * 2, s));
      pair_insert_kernel<<<grid, kPipeRows, 0, s>>>(m->rp, m->v, m->wc, m->n_rows, nblk, m->sell_off, table, slot_idx,
                                                    ptable, ctl);
      CK(cudaMemcpyAsync(pctl, ctl, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      g_upt.mark("pairs");
      buf_free(ctx, ctl);
      pairs = pctl[1] == 0 && pctl[0] <= kSellDict;
      if (pairs) {
        pair_compact_kernel<<<1, 1, 0, s>>>(ptable, m->sell_dict, pdict, pslot);
        sell_fill_pair_kernel<<<grid, kPipeRows, 0, s>>>(m->rp, m->v, m->wc, m->n_rows, nblk, m->sell_off, table,
                                                         slot_idx, ptable, pslot, m->sell_vi, m->sell_len);
        buf_free(ctx, m->sell_dict);
        m->sell_dict = reinterpret_cast<double*>(pdict);
        m->sell_ndict = pctl[0];
        m->sell_mode = kSellPairs;
      } else {
        buf_free(ctx, pdict);
      }
      buf_free(ctx, ptable);
      buf_free(ctx, pslot);
    }
    if (!pairs) m->sell_mode = kSellDictV;
  } else {
    CK(buf_alloc(ctx, &m->sell_v, sizeof(double) * entries));
    m->sell_mode = kSellF64;
  }
  if (!pairs) {
    CK(buf_alloc(ctx, &m->sell_c, sizeof(unsigned short) * entries));
    sell_fill_kernel<<<grid, kPipeRows, 0, s>>>(m->rp, m->v, m->wc, m->n_rows, nblk, m->sell_off, m->sell_v, m->sell_c,
                                                m->sell_len, dict ? table : nullptr, slot_idx, m->sell_vi);
  }
  CK(cudaGetLastError());
  g_upt.mark("fill-launch");
  buf_free(ctx, table);
  buf_free(ctx, slot_idx);
  m->sell_lmax = hl;
  m->sell_entries = entries;
  return PBS_OK;
}

static int build_window_cols_only(pbs_ctx* ctx, pbs_mat* m);
static int build_window_cols(pbs_ctx* ctx, pbs_mat* m) {
  int rc = build_window_cols_only(ctx, m);
  if (rc) return rc;
  return build_sell(ctx, m);
}

static int build_window_cols_only(pbs_ctx* ctx, pbs_mat* m) {
  if (m->wc) {
    buf_free(ctx, m->wc);
    m->wc = nullptr;
  }
  if ((!m->xwin.nwin && !m->xwin.band_s) || m->nnz == 0 || m->xwin.total > 65535) return PBS_OK;
  cudaStream_t s = ctx->stream;
  int* bad = nullptr;
  CK(buf_alloc(ctx, &m->wc, sizeof(unsigned short) * (m->nnz + 16)));
  CK(buf_alloc(ctx, &bad, sizeof(int)));
  CK(cudaMemsetAsync(m->wc + m->nnz, 0, sizeof(unsigned short) * 16, s));
  CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
  window_cols_kernel<<<ctx->sms * 8, 256, 0, s>>>(m->rp, m->ci, m->n_rows, m->n_cols, m->xwin, m->wc, bad);
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  g_upt.mark("wcols");
  buf_free(ctx, bad);
  if (hbad || env_int("PBS_NO_WINDOW_COLS", 0, 0, 1)) {  // 1: keep col_idx (A/B sweeps)
    buf_free(ctx, m->wc);
    m->wc = nullptr;
  }
  return PBS_OK;
}

// clusters of row offsets -> x windows (<= kMaxWin, <= kMaxWinElems staged)
int compute_xwin(pbs_ctx* ctx, pbs_mat* m) {
  m->xwin = XWin{};
  if (!m->stencil) {  // rebuilt below when the new pattern windows
    buf_free(ctx, m->wc);
    m->wc = nullptr;
    free_sell(ctx, m);
  }
  if (m->n_rows == 0 || m->nnz == 0 || m->n_cols > 0x7fffffffLL) return PBS_OK;
  cudaStream_t s = ctx->stream;
  int *bmin = nullptr, *bmax = nullptr, *wide = nullptr;
  CK(buf_alloc(ctx, &bmin, sizeof(int) * 2 * kBins));
  CK(buf_alloc(ctx, &bmax, sizeof(int) * 2 * kBins));
  CK(buf_alloc(ctx, &wide, sizeof(int)));
  // The two 512 KB bin arrays stay on the device: they are initialised there,
  // and only the occupied bins (a handful for any matrix that windows) come
  // back, as (bin, min, max) triples.
  int* occ = nullptr;  // [0] count, then kBinsOut triples
  CK(buf_alloc(ctx, &occ, sizeof(int) * (1 + 3 * kBinsOut)));
  bins_init_kernel<<<(2 * kBins + 255) / 256, 256, 0, s>>>(bmin, bmax, occ, wide);
  offset_bins_kernel<<<ctx->sms * 8, 256, 0, s>>>(m->rp, m->ci, m->n_rows, bmin, bmax, wide);
  bins_compact_kernel<<<(2 * kBins + 255) / 256, 256, 0, s>>>(bmin, bmax, occ);
  int hwide = 0;
  std::vector<int> hocc(1 + 3 * kBinsOut);
  CK(cudaMemcpyAsync(hocc.data(), occ, sizeof(int) * (1 + 3 * kBinsOut), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&hwide, wide, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  g_upt.mark("bins");
  buf_free(ctx, bmin);
  buf_free(ctx, bmax);
  buf_free(ctx, wide);
  buf_free(ctx, occ);
  if (hwide || hocc[0] > kBinsOut) return PBS_OK;  // offsets in more bins than any window set covers: gather x
  std::vector<std::array<int, 3>> bins(hocc[0]);
  for (int k = 0; k < hocc[0]; ++k) bins[k] = {hocc[1 + 3 * k], hocc[2 + 3 * k], hocc[3 + 3 * k]};
  std::sort(bins.begin(), bins.end());  // ascending bin
  std::vector<std::pair<int, int>> cl;  // [min, max] offsets
  for (const auto& b : bins) {
    if (!cl.empty() && (long long)b[1] - cl.back().second <= kPipeRows + 4)
      cl.back().second = b[2] > cl.back().second ? b[2] : cl.back().second;
    else
      cl.push_back({b[1], b[2]});
  }
  while (cl.size() > (size_t)kMaxWin) {  // merge across the smallest gap
    size_t best = 0;
    long long gap = -1;
    for (size_t i = 0; i + 1 < cl.size(); ++i) {
      long long g = (long long)cl[i + 1].first - cl[i].second;
      if (gap < 0 || g < gap) {
        gap = g;
        best = i;
      }
    }
    cl[best].second = cl[best + 1].second;
    cl.erase(cl.begin() + best + 1);
  }
  XWin W{};
  long long total = 0;
  for (size_t c = 0; c < cl.size(); ++c) {
    W.wmin[c] = cl[c].first;
    W.wmax[c] = cl[c].second;
    long long cap = (long long)kPipeRows + cl[c].second - cl[c].first + 4;
    cap = (cap + 1) & ~1LL;
    W.cap[c] = (int)cap;
    total += cap;
  }
  if (cl.empty()) return PBS_OK;
  if (total > kMaxWinElems) {
    // too spread for per-block windows: a band (one circular x buffer per
    // CTA over a contiguous run of blocks) when the whole offset range is
    // narrow enough, else gather x
    const long long lo = cl.front().first, hi = cl.back().second;
    // even size: the pieces stay 16-byte aligned in the circular buffer
    const long long bs = (hi - lo + 2LL * kPipeRows + 8 + 255) / 256 * 256;
    if (bs > kBandMaxElems || env_int("PBS_NO_BAND", 0, 0, 1)) return PBS_OK;
    XWin B{};
    B.band_s = (int)bs;
    B.band_lo = (int)lo;
    B.band_hi = (int)hi;
    m->xwin = B;
    return m->stencil ? PBS_OK : build_window_cols(ctx, m);
  }
  W.nwin = (int)cl.size();
  W.total = (int)total;
  m->xwin = W;
  return m->stencil ? PBS_OK : build_window_cols(ctx, m);
}

// copy a host CSR into m's device buffers (int64 indices narrowed on the
// device, with a range check), then the x windows / window-local columns
static int upload_arrays(pbs_ctx* ctx, pbs_mat* m, const int64_t* row_ptr, const void* col_idx, int32_t col_bytes,
                         const double* values) {
  const long long n_rows = m->n_rows, n_cols = m->n_cols, nnz = m->nnz;
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(m->rp, row_ptr, sizeof(long long) * (n_rows + 1), cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    CK(cudaMemcpyAsync(m->v, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    if (col_bytes == 4) {
      CK(cudaMemcpyAsync(m->ci, col_idx, sizeof(int) * nnz, cudaMemcpyHostToDevice, s));
    } else {
      // stage int64 indices in chunks and narrow on the device
      const long long chunk = 1LL << 24;
      long long* tmp = nullptr;
      int* bad = nullptr;
      CK(buf_alloc(ctx, &tmp, sizeof(long long) * (nnz < chunk ? nnz : chunk)));
      CK(buf_alloc(ctx, &bad, sizeof(int)));
      CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
      for (long long off = 0; off < nnz; off += chunk) {
        long long len = nnz - off < chunk ? nnz - off : chunk;
        CK(cudaMemcpyAsync(tmp, (const long long*)col_idx + off, sizeof(long long) * len,
                           cudaMemcpyHostToDevice, s));
        cvt_i64_i32_kernel<<<ctx->sms * 4, 256, 0, s>>>(tmp, m->ci + off, len, bad, n_cols);
      }
      int hbad = 0;
      CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      buf_free(ctx, tmp);
      buf_free(ctx, bad);
      if (hbad) return set_err(ctx, PBS_ERR_INVALID, "column index out of range");
    }
  }
  CK(cudaStreamSynchronize(s));
  g_upt.mark("h2d+narrow");
  m->blk_nnz_max = 0;
  for (long long r0 = 0; r0 < n_rows; r0 += kPipeRows) {
    const long long r1 = r0 + kPipeRows < n_rows ? r0 + kPipeRows : n_rows;
    const long long bn = row_ptr[r1] - row_ptr[r0];
    if (bn > m->blk_nnz_max) m->blk_nnz_max = bn;
  }
  return compute_xwin(ctx, m);
}

PBS_EXPORT int pbs_csr_upload(pbs_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                              const int64_t* row_ptr, const void* col_idx, int32_t col_bytes,
                              const double* values, pbs_mat** out) {
  if (!ctx || !out) return set_err(ctx, PBS_ERR_INVALID, "NULL argument");
  if (n_rows < 0 || n_cols < 0 || nnz < 0) return set_err(ctx, PBS_ERR_INVALID, "negative matrix dimension");
  if (n_cols > 0x7fffffffLL) return set_err(ctx, PBS_ERR_INVALID, "n_cols exceeds the int32 column index range");
  if (col_bytes != 4 && col_bytes != 8) return set_err(ctx, PBS_ERR_INVALID, "col_bytes must be 4 or 8");
  if (row_ptr[0] != 0 || row_ptr[n_rows] != nnz)
    return set_err(ctx, PBS_ERR_INVALID, "row_ptr endpoints inconsistent with nnz arrays");
  CK(cudaSetDevice(ctx->device));
  g_upt.start();
  if (ctx->ws_cache && ctx->ws_cache->n != n_rows) drop_ws_cache(ctx);  // cannot match: release it now
  if (ctx->spare_rows != n_rows || ctx->spare_nnz != nnz) {  // another shape: its buffers are of no use
    buf_flush(ctx);
    ctx->spare_rows = n_rows;
    ctx->spare_nnz = nnz;
  }
  pbs_mat* m = new pbs_mat();
  m->ctx = ctx;
  m->n_rows = n_rows;
  m->n_cols = n_cols;
  m->nnz = nnz;
  cudaStream_t s = ctx->stream;
  // padding: the pipelined SpMV bulk-copies 16-byte-aligned windows
  CK(buf_alloc(ctx, &m->rp, sizeof(long long) * (n_rows + 4)));
  CK(buf_alloc(ctx, &m->ci, sizeof(int) * (nnz + 8)));
  CK(buf_alloc(ctx, &m->v, sizeof(double) * (nnz + 4)));
  CK(cudaMemsetAsync(m->rp + n_rows + 1, 0, sizeof(long long) * 3, s));
  CK(cudaMemsetAsync(m->ci + nnz, 0, sizeof(int) * 8, s));
  CK(cudaMemsetAsync(m->v + nnz, 0, sizeof(double) * 4, s));
  g_upt.mark("alloc");
  int rc = upload_arrays(ctx, m, row_ptr, col_idx, col_bytes, values);
  g_upt.stop();
  if (rc) {
    pbs_mat_free(m);
    return rc;
  }
  *out = m;
  return PBS_OK;
}

// Upload new CSR arrays of the same shape (n_rows, nnz) into an existing
// operator: the end-to-end step of a resident, partitioned operator (its
// workspace, halo plan and peer mappings stay; the window-local columns are
// rebuilt).
PBS_EXPORT int pbs_csr_update(pbs_mat* m, const int64_t* row_ptr, const void* col_idx, int32_t col_bytes,
                              const double* values) {
  if (!m || m->stencil) return set_err(m ? m->ctx : nullptr, PBS_ERR_INVALID, "need a CSR operator");
  pbs_ctx* ctx = m->ctx;
  if (col_bytes != 4 && col_bytes != 8) return set_err(ctx, PBS_ERR_INVALID, "col_bytes must be 4 or 8");
  if (row_ptr[0] != 0 || row_ptr[m->n_rows] != m->nnz)
    return set_err(ctx, PBS_ERR_INVALID, "row_ptr endpoints inconsistent with the operator's nnz");
  CK(cudaSetDevice(ctx->device));
  const XWin old = m->xwin;
  int rc = upload_arrays(ctx, m, row_ptr, col_idx, col_bytes, values);
  if (rc) return rc;
  if (m->ws && memcmp(&old, &m->xwin, sizeof(XWin)) != 0) free_graphs(m->ws);  // graphs bake the windows in
  return PBS_OK;
}

PBS_EXPORT int pbs_stencil_create(pbs_ctx* ctx, int32_t dim, int64_t k, int32_t npts,
                                  const int32_t* offsets, const double* coeffs, pbs_mat** out) {
  if (!ctx || !out) return set_err(ctx, PBS_ERR_INVALID, "NULL argument");
  if (dim < 1 || dim > 3) return set_err(ctx, PBS_ERR_INVALID, "dim must be 1, 2, or 3");
  if (k < 1) return set_err(ctx, PBS_ERR_INVALID, "k must be >= 1");
  if (npts < 1 || npts > kMaxStencil) return set_err(ctx, PBS_ERR_INVALID, "npts must be in [1, 27]");
  long long n = 1;
  for (int a = 0; a < dim; ++a) n *= k;
  if (n > 0x7fffffffLL) return set_err(ctx, PBS_ERR_INVALID, "grid exceeds the supported size");
  pbs_mat* m = new pbs_mat();
  m->ctx = ctx;
  m->stencil = 1;
  m->n_rows = m->n_cols = n;
  StencilView& S = m->sv;
  S.n = n;
  S.g0 = 0;
  S.xlo = 0;
  S.xhi = n;
  S.k = k;
  S.k2 = k * k;
  S.dk = make_fastdiv(S.k);
  S.dk2 = make_fastdiv(S.k2);
  S.dim = dim;
  S.npts = npts;
  for (int a = 0; a < 3; ++a) S.nlo[a] = S.nhi[a] = 0xffffffffu;
  for (int p = 0; p < npts; ++p)
    for (int a = 0; a < dim; ++a) {
      const int d = offsets[p * dim + a];
      if (d == -1) S.nlo[3 - dim + a] &= ~(1u << p);
      if (d == 1) S.nhi[3 - dim + a] &= ~(1u << p);
    }
  long long nnz = 0;
  long long prev = -(1LL << 62);
  for (int p = 0; p < npts; ++p) {
    long long f = 0;
    for (int a = 0; a < 3; ++a) S.off[p][a] = 0;
    for (int a = 0; a < dim; ++a) {
      int d = offsets[p * dim + a];
      if (d < -1 || d > 1) {
        delete m;
        return set_err(ctx, PBS_ERR_INVALID, "stencil offsets must lie in {-1, 0, 1}");
      }
      S.off[p][3 - dim + a] = d;
      long long w = 1;
      for (int b = a + 1; b < dim; ++b) w *= k;
      f += d * w;
    }
    if (f <= prev) {
      delete m;
      return set_err(ctx, PBS_ERR_INVALID, "stencil offsets must be sorted by flattened offset");
    }
    prev = f;
    S.foff[p] = f;
    S.coef[p] = coeffs[p];
    long long cnt = 1;
    for (int a = 0; a < dim; ++a) cnt *= (k - (offsets[p * dim + a] != 0 ? 1 : 0));
    nnz += cnt;
  }
  m->nnz = nnz;
  // x windows: cluster the flattened offsets like compute_xwin does for CSR
  {
    std::vector<std::pair<long long, int>> offs;
    for (int q = 0; q < npts; ++q) offs.push_back({S.foff[q], q});
    std::sort(offs.begin(), offs.end());
    std::vector<std::pair<long long, long long>> cl;
    std::vector<int> owner(npts);
    for (auto& o : offs) {
      if (!cl.empty() && o.first - cl.back().second <= kPipeRows + 4)
        cl.back().second = o.first;
      else
        cl.push_back({o.first, o.first});
      owner[o.second] = (int)cl.size() - 1;
    }
    while (cl.size() > (size_t)kMaxWin) {  // merge across the smallest gap (plane rows -> planes)
      size_t best = 0;
      long long gap = -1;
      for (size_t q = 0; q + 1 < cl.size(); ++q) {
        long long g = cl[q + 1].first - cl[q].second;
        if (gap < 0 || g < gap) {
          gap = g;
          best = q;
        }
      }
      cl[best].second = cl[best + 1].second;
      cl.erase(cl.begin() + best + 1);
      for (auto& o : owner)
        if (o > (int)best) --o;
    }
    XWin W{};
    long long total = 0;
    if (cl.size() <= (size_t)kMaxWin) {
      for (size_t c = 0; c < cl.size(); ++c) {
        W.wmin[c] = (int)cl[c].first;
        W.wmax[c] = (int)cl[c].second;
        long long cap = ((long long)kPipeRows + cl[c].second - cl[c].first + 4 + 1) & ~1LL;
        W.cap[c] = (int)cap;
        total += cap;
      }
      if (total <= kMaxWinElems) {
        W.nwin = (int)cl.size();
        W.total = (int)total;
        m->xwin = W;
        for (int q = 0; q < npts; ++q) m->swin.pw[q] = owner[q];
        // constant staged offsets of interior blocks (see StencilWin)
        long long soff[kMaxWin] = {0, 0, 0, 0}, clamp = 0;
        for (int c = 1; c < W.nwin; ++c) soff[c] = soff[c - 1] + W.cap[c - 1];
        for (int c = 0; c < W.nwin; ++c)
          if (-(long long)W.wmin[c] > clamp) clamp = -(long long)W.wmin[c];
        for (int q = 0; q < npts; ++q) {
          const int c = owner[q];
          const long long wmin_even = (long long)W.wmin[c] & ~1LL;  // (r0 + wmin) & ~1 == r0 + (wmin & ~1), r0 even
          m->swin.kfix[q] = (int)(S.foff[q] - wmin_even + soff[c]);
        }
        m->swin.clamp_r0 = clamp;
      }
    }
  }
  *out = m;
  return PBS_OK;
}


// ---- stencil -> CSR on the device
__device__ __forceinline__ bool stencil_in(const StencilView& S, long long li, int p) {
  const long long i = li + S.g0;  // grid row of slab-local row li
  int c[3] = {0, 0, 0};
  if (S.dim == 3) {
    const long long z = S.dk2.div(i), rem = i - z * S.k2, yy = S.dk.div(rem);
    c[0] = (int)z;
    c[1] = (int)yy;
    c[2] = (int)(rem - yy * S.k);
  } else if (S.dim == 2) {
    const long long yy = S.dk.div(i);
    c[1] = (int)yy;
    c[2] = (int)(i - yy * S.k);
  } else {
    c[2] = (int)i;
  }
  bool ok = true;
  for (int a = 3 - S.dim; a < 3; ++a) {
    const int cc = c[a] + S.off[p][a];
    ok = ok && cc >= 0 && cc < S.k;
  }
  return ok;
}

__global__ void stencil_count_kernel(const __grid_constant__ StencilView S, long long* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S.n; i += stride) {
    long long c = 0;
    for (int p = 0; p < S.npts; ++p) c += stencil_in(S, i, p);
    counts[i + 1] = c;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = 0;
}

// col_off: a slab's columns are extended-space indices, own segment at col_off
__global__ void stencil_fill_kernel(const __grid_constant__ StencilView S, const long long* rp, int* ci,
                                    double* v, long long col_off) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S.n; i += stride) {
    long long k = rp[i];
    for (int p = 0; p < S.npts; ++p)
      if (stencil_in(S, i, p)) {
        ci[k] = (int)(col_off + i + S.foff[p]);
        v[k] = S.coef[p];
        ++k;
      }
  }
}

// most nonzeros in one kPipeRows-row block (chunk sizing of the CSR engine)
__global__ void block_nnz_max_kernel(const long long* rp, long long n, unsigned long long* out) {
  const long long nb = (n + kPipeRows - 1) / kPipeRows;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
    const long long r0 = b * kPipeRows, r1 = r0 + kPipeRows < n ? r0 + kPipeRows : n;
    atomicMax(out, (unsigned long long)(rp[r1] - rp[r0]));
  }
}


PBS_EXPORT int pbs_stencil_to_csr(pbs_mat* st, pbs_mat** out) {
  if (!st || !out || !st->stencil) return set_err(st ? st->ctx : nullptr, PBS_ERR_INVALID, "need a stencil operator");
  pbs_ctx* ctx = st->ctx;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const long long n = st->n_rows, nnz = st->nnz;
  if (nnz > 0x7fffffffffffLL) return set_err(ctx, PBS_ERR_INVALID, "too many nonzeros");
  buf_flush(ctx);  // spares of an uploaded shape are of no use here
  ctx->spare_rows = ctx->spare_nnz = -1;
  pbs_mat* m = new pbs_mat();
  m->ctx = ctx;
  m->n_rows = n;
  m->n_cols = st->n_cols;  // a slab's extended space (pbs_stencil_slab)
  m->nnz = nnz;
  const long long hl = -st->sv.xlo, col_off = hl + (hl & 1);
  CK(pool_alloc(ctx, &m->rp, sizeof(long long) * (n + 4)));
  CK(pool_alloc(ctx, &m->ci, sizeof(int) * (nnz + 8)));
  CK(pool_alloc(ctx, &m->v, sizeof(double) * (nnz + 4)));
  CK(cudaMemsetAsync(m->rp + n + 1, 0, sizeof(long long) * 3, s));
  CK(cudaMemsetAsync(m->ci + nnz, 0, sizeof(int) * 8, s));
  CK(cudaMemsetAsync(m->v + nnz, 0, sizeof(double) * 4, s));
  StencilView S = st->sv;
  stencil_count_kernel<<<ctx->sms * 8, 256, 0, s>>>(S, m->rp);
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, m->rp, m->rp, n + 1, s);
  void* tmp = nullptr;
  CK(pool_alloc(ctx, &tmp, tmp_bytes));
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, m->rp, m->rp, n + 1, s);
  pool_free(ctx, tmp);
  stencil_fill_kernel<<<ctx->sms * 8, 256, 0, s>>>(S, m->rp, m->ci, m->v, col_off);
  unsigned long long* bmax = nullptr;
  CK(pool_alloc(ctx, &bmax, sizeof(unsigned long long)));
  CK(cudaMemsetAsync(bmax, 0, sizeof(unsigned long long), s));
  block_nnz_max_kernel<<<ctx->sms * 4, 256, 0, s>>>(m->rp, n, bmax);
  unsigned long long hb = 0;
  long long last = 0;
  CK(cudaMemcpyAsync(&hb, bmax, sizeof(hb), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&last, m->rp + n, sizeof(last), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  pool_free(ctx, bmax);
  CK(cudaGetLastError());
  if (last != nnz) {
    pbs_mat_free(m);
    return set_err(ctx, PBS_ERR_CUDA, "stencil CSR nonzero count mismatch");
  }
  m->blk_nnz_max = (long long)hb;
  int rc = compute_xwin(ctx, m);
  if (rc) {
    pbs_mat_free(m);
    return rc;
  }
  *out = m;
  return PBS_OK;
}

// nonzeros of a stencil operator's rows (a slab's share of the grid's)
__global__ void stencil_nnz_kernel(const __grid_constant__ StencilView S, unsigned long long* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S.n; i += stride)
    for (int p = 0; p < S.npts; ++p) c += stencil_in(S, i, p);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Rows [row_lo, row_hi) of a whole-grid stencil operator as a slab of a
// row-partitioned system (reduction.py:55-87, linalg.py:164-172):
// local row i is grid row row_lo + i, and SpMV inputs live in the slab's
// extended space [pad | hl | own | hr] like a CSR slab's (distributed.py).
// hl / hr must cover every column the rows reach outside [row_lo, row_hi).
PBS_EXPORT int pbs_stencil_slab(pbs_mat* st, int64_t row_lo, int64_t row_hi, int64_t hl, int64_t hr,
                                pbs_mat** out) {
  if (!st || !out || !st->stencil || st->sv.g0 != 0 || st->sv.xlo != 0)
    return set_err(st ? st->ctx : nullptr, PBS_ERR_INVALID, "need a whole-grid stencil operator");
  pbs_ctx* ctx = st->ctx;
  const long long n = st->n_rows;
  if (row_lo < 0 || row_hi > n || row_lo >= row_hi) return set_err(ctx, PBS_ERR_INVALID, "slab rows out of range");
  if (hl < 0 || hr < 0 || hl > row_lo || hr > n - row_hi) return set_err(ctx, PBS_ERR_INVALID, "halo out of range");
  CK(cudaSetDevice(ctx->device));
  pbs_mat* m = new pbs_mat();
  *m = *st;
  m->ws = nullptr;
  m->zm_maps.clear();  // tensor maps describe the whole grid's vectors
  m->part = Partition{};
  const long long n_own = row_hi - row_lo;
  m->n_rows = n_own;
  m->n_cols = (hl & 1) + hl + n_own + hr;
  StencilView& S = m->sv;
  S.n = n_own;
  S.g0 = row_lo;
  S.xlo = -hl;
  S.xhi = n_own + hr;
  // blocks whose windows all start inside [xlo, xhi) use the constant staged
  // offsets (StencilWin::kfix); the clamp moves left by the halo
  if (m->xwin.nwin) m->swin.clamp_r0 = st->swin.clamp_r0 - hl;
  unsigned long long* d = nullptr;
  CK(pool_alloc(ctx, &d, sizeof(unsigned long long)));
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), ctx->stream));
  stencil_nnz_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(S, d);
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  pool_free(ctx, d);
  m->nnz = (long long)h;
  *out = m;
  return PBS_OK;
}

PBS_EXPORT int pbs_mat_free(pbs_mat* m) {
  if (!m) return PBS_OK;
  cudaSetDevice(m->ctx->device);
  cudaStreamSynchronize(m->ctx->stream);
  if (m->ws && !m->part.dist) {
    drop_ws_cache(m->ctx);
    m->ctx->ws_cache = m->ws;
    m->ctx->ws_sig = mat_sig(m);
  } else {
    free_ws(m->ws);
  }
  buf_free(m->ctx, m->rp);
  buf_free(m->ctx, m->ci);
  buf_free(m->ctx, m->v);
  buf_free(m->ctx, m->wc);
  buf_free(m->ctx, m->sell_v);
  buf_free(m->ctx, m->sell_c);
  buf_free(m->ctx, m->sell_off);
  buf_free(m->ctx, m->sell_len);
  buf_free(m->ctx, m->sell_vi);
  buf_free(m->ctx, m->sell_dict);
  delete m;
  return PBS_OK;
}

PBS_EXPORT int pbs_mat_layout(pbs_mat* m, int64_t out[8]) {
  if (!m || !out) return set_err(m ? m->ctx : nullptr, PBS_ERR_INVALID, "NULL argument");
  for (int i = 0; i < 8; ++i) out[i] = 0;
  out[6] = m->xwin.nwin;
  out[7] = m->xwin.nwin ? m->xwin.total : m->xwin.band_s;
  if (m->stencil) {
    out[0] = 10;
  } else if (m->sell_vi || m->sell_v) {
    out[0] = m->sell_mode == kSellPairs ? 5 : (m->sell_vi ? 4 : 3);
    out[1] = m->sell_entries;
    out[2] = m->sell_mode == kSellPairs ? 1 : (m->sell_vi ? 3 : 10);
    out[3] = 1;
    out[4] = m->sell_ndict;
    out[5] = m->sell_lmax;
  } else {
    out[0] = m->wc ? (m->xwin.band_s ? 2 : 1) : 0;
    out[1] = m->nnz;
    out[2] = m->wc ? 10 : 12;
    out[3] = 8;
  }
  return PBS_OK;
}

PBS_EXPORT int pbs_mat_info(pbs_mat* m, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, int32_t* is_stencil) {
  if (!m) return set_err(nullptr, PBS_ERR_INVALID, "mat is NULL");
  if (n_rows) *n_rows = m->n_rows;
  if (n_cols) *n_cols = m->n_cols;
  if (nnz) *nnz = m->nnz;
  if (is_stencil) *is_stencil = m->stencil;
  return PBS_OK;
}

static int reset_tmp_state(pbs_ctx* ctx) {
  SolverState h{};
  h.run_all = 1;
  h.run_spine = 1;
  h.nf_row = (unsigned long long)kNoError;
  CK(cudaMemcpyAsync(ctx->tmp_state, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  return PBS_OK;
}

PBS_EXPORT int pbs_spmv_dev(pbs_mat* m, const double* d_x, double* d_y, int64_t* nonfinite_index) {
  if (!m) return set_err(nullptr, PBS_ERR_INVALID, "mat is NULL");
  pbs_ctx* ctx = m->ctx;
  CK(cudaSetDevice(ctx->device));
  int rc = reset_tmp_state(ctx);
  if (rc) return rc;
  Launcher L{ctx, m, ctx->stream};
  EpiStore e{};
  e.y = d_y;
  e.st = ctx->tmp_state;
  e.tag = PBS_TAG_AX;
  const double* xin = d_x;
  if (m->xwin.nwin || m->xwin.band_s) {
    // staged x windows are copied in 16-byte units and may read one element
    // past the end of x: stage a caller's x into a padded buffer
    double* xs = nullptr;
    CK(pool_alloc(ctx, &xs, sizeof(double) * (m->n_cols + 4)));
    CK(cudaMemcpyAsync(xs, d_x, sizeof(double) * m->n_cols, cudaMemcpyDeviceToDevice, ctx->stream));
    xin = xs;
  }
  spmv_launch(L, xin, e, 0, m->n_rows, KS);
  if (xin != d_x) pool_free(ctx, const_cast<double*>(xin));
  if (L.err) return L.err;
  unsigned long long row = 0;
  CK(cudaMemcpyAsync(&row, &ctx->tmp_state->nf_row, sizeof(row), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (nonfinite_index) *nonfinite_index = row == (unsigned long long)kNoError ? -1 : (int64_t)row;
  return PBS_OK;
}

static int solve_common(pbs_mat* m, int32_t method, const pbs_config* cfg) {
  pbs_ctx* ctx = m ? m->ctx : nullptr;
  if (!m) return set_err(nullptr, PBS_ERR_INVALID, "mat is NULL");
  if (!m->part.dist && m->n_rows != m->n_cols) return set_err(ctx, PBS_ERR_INVALID, "solver needs a square operator");
  if (method < 0 || method > PBS_METHOD_PBICGSTAB) return set_err(ctx, PBS_ERR_INVALID, "unknown method");
  int rc = validate_cfg(ctx, cfg);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  return ensure_ws(m, cfg->max_iters + 1);
}

PBS_EXPORT int pbs_solve(pbs_mat* m, int32_t method, const double* b, const double* x0,
                         const pbs_config* cfg, double* x_out, double* hist_rel, uint8_t* hist_flags,
                         double* hist_coef, pbs_result* res) {
  int rc = solve_common(m, method, cfg);
  if (rc) return rc;
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  cudaStream_t s = ctx->stream;
  const size_t bytes = sizeof(double) * ws->n;
  CK(cudaMemcpyAsync(ws->V.v[VB], b, bytes, cudaMemcpyHostToDevice, s));
  if (x0)
    CK(cudaMemcpyAsync(ws->V.v[VX], x0, bytes, cudaMemcpyHostToDevice, s));
  else
    CK(cudaMemsetAsync(ws->V.v[VX], 0, bytes, s));
  rc = run_solve(m, method, cfg, res);
  if (rc) return rc;
  if (x_out) CK(cudaMemcpy(x_out, ws->V.v[VX], bytes, cudaMemcpyDeviceToHost));
  return copy_history(m, res, hist_rel, hist_flags, hist_coef);
}

PBS_EXPORT int pbs_solve_dev(pbs_mat* m, int32_t method, const double* d_b, const double* d_x0,
                             const pbs_config* cfg, double* d_x_out, double* hist_rel,
                             uint8_t* hist_flags, double* hist_coef, pbs_result* res) {
  int rc = solve_common(m, method, cfg);
  if (rc) return rc;
  pbs_ctx* ctx = m->ctx;
  Workspace* ws = m->ws;
  cudaStream_t s = ctx->stream;
  const size_t bytes = sizeof(double) * ws->n;
  CK(cudaMemcpyAsync(ws->V.v[VB], d_b, bytes, cudaMemcpyDeviceToDevice, s));
  if (d_x0)
    CK(cudaMemcpyAsync(ws->V.v[VX], d_x0, bytes, cudaMemcpyDeviceToDevice, s));
  else
    CK(cudaMemsetAsync(ws->V.v[VX], 0, bytes, s));
  rc = run_solve(m, method, cfg, res);
  if (rc) return rc;
  if (d_x_out) CK(cudaMemcpyAsync(d_x_out, ws->V.v[VX], bytes, cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  return copy_history(m, res, hist_rel, hist_flags, hist_coef);
}

// single-iteration parity seam
PBS_EXPORT int pbs_step_dev(pbs_mat* m, double* const* d_state, const double* in, int32_t reduce_mode,
                            int32_t plan_workers, double* outv) {
  if (!m) return set_err(nullptr, PBS_ERR_INVALID, "mat is NULL");
  pbs_ctx* ctx = m->ctx;
  CK(cudaSetDevice(ctx->device));
  int rc = ensure_ws(m, 4);
  if (rc) return rc;
  Workspace* ws = m->ws;
  cudaStream_t s = ctx->stream;
  Mode md;
  md.plan = reduce_mode == PBS_REDUCE_PLAN;
  md.store_temps = 1;
  if (md.plan && (rc = ensure_plan(m, plan_workers))) return rc;
  const int order[16] = {VX, VR, VP, VU, VO, VT, VW, VY, VZ, VS, VQ, VG, VL, VR0S, VB, VAS};
  const size_t bytes = sizeof(double) * ws->n;
  for (int k = 0; k < 16; ++k)
    CK(cudaMemcpyAsync(ws->V.v[order[k]], d_state[k], bytes, cudaMemcpyDeviceToDevice, s));
  const long long j = (long long)in[0];
  SolverState h{};
  h.tol = -1.0;  // never converge inside a single step
  h.max_iters = j + 2;
  h.record_history = 1;
  h.alpha = in[1];
  h.zeta = in[2];
  h.f_prev = in[3];
  h.r0_norm = in[4];
  h.iter = j;
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
  Launcher L{ctx, m, s};
  // the batch of iteration j over the given state, then the check
  int np;
  if (md.plan) {
    np = plan_dots(L, ws, KD);
  } else {
    long long nblk = (ws->n + kThreads - 1) / kThreads;
    np = grid_for(ctx, (const void*)dots9_tree_kernel, nblk);
    dots9_tree_kernel<<<np, kThreads, 0, s>>>(ws->n, ws->V.v[VS], ws->V.v[VY], ws->V.v[VR],
                                              ws->V.v[VR0S], ws->V.v[VT], ws->partials, ws->st);
  }
  finalize_kernel<<<1, 288, 0, s>>>(ws->st, ws->partials, np, md.plan, 0);
  // iteration body without its trailing check
  {
    auto& V = ws->V.v;
    Mode nm = md;  // the step's batch comes first; the body's partials are not needed
    if (in[5] != 0.0) {
      spmv_launch(L, ws->X.v[VS], epi_store(ws, VAS, PBS_TAG_AS, 1), 0, ws->n, KK1);
      vec_launch(L, pou_kernel, ws->n, KR, ws->V, ws->n, ws->st);
      spmv_launch(L, ws->X.v[VO], epi_store(ws, VQ, PBS_TAG_AO, 0), 0, ws->n, KRS);
      spmv_launch(L, ws->X.v[VU], epi_store(ws, VW, PBS_TAG_AU, 0), 0, ws->n, KRS);
      vec_launch(L, tzyx_kernel, ws->n, KR, ws->V, ws->n, ws->st);
      spmv_launch(L, ws->X.v[VX], epi_resid(ws, false), 0, ws->n, KRS);
      spmv_launch(L, ws->X.v[VT], epi_store(ws, VL, PBS_TAG_AT, 0), 0, ws->n, KRS);
      spmv_launch(L, ws->X.v[VY], epi_store(ws, VG, PBS_TAG_AY, 0), 0, ws->n, KRS);
      nm.plan = 1;  // no partials
      spmv_launch(L, ws->X.v[VR], epi_dots(ws, nm, 0, 0, 0), 0, ws->n, KRS);
    } else {
      nm.plan = 1;
      nm.store_temps = 1;
      spmv_launch(L, ws->X.v[VS], epi_k12(ws, nm), 0, ws->n, KK1);
      spmv_launch(L, ws->X.v[VW], epi_k3(ws, nm, 0), 0, ws->n, KK3);
    }
  }
  if (L.err) return L.err;
  for (int k = 0; k < 16; ++k)
    CK(cudaMemcpyAsync(d_state[k], ws->V.v[order[k]], bytes, cudaMemcpyDeviceToDevice, s));
  SolverState out;
  CK(cudaMemcpyAsync(&out, ws->st, sizeof(out), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  outv[0] = out.alpha;
  outv[1] = out.beta;
  outv[2] = out.zeta;
  outv[3] = out.eta;
  for (int k = 0; k < kNumDots; ++k) outv[4 + k] = out.dots[k];
  outv[13] = out.status;
  if (out.nf_row != (unsigned long long)kNoError) return set_err(ctx, PBS_ERR_NONFINITE, "non-finite SpMV output");
  return PBS_OK;
}

// ------------------------------------------------------- kernel backend table

static int scratch(pbs_ctx* ctx, size_t bytes, void** p) {
  if (bytes > ctx->scratch_bytes) {
    cudaFree(ctx->scratch);
    ctx->scratch = nullptr;
    size_t cap = bytes < (1 << 20) ? (1 << 20) : bytes;
    CK(cudaMalloc(&ctx->scratch, cap));
    ctx->scratch_bytes = cap;
  }
  *p = ctx->scratch;
  return PBS_OK;
}

static size_t al(size_t b) { return (b + 255) / 256 * 256; }

PBS_EXPORT int pbs_k_spmv_range(pbs_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                                const int64_t* col_idx, const double* values, const double* x,
                                double* out, int64_t lo, int64_t hi) {
  if (!ctx) return set_err(nullptr, PBS_ERR_INVALID, "ctx is NULL");
  if (lo < 0 || hi > n_rows || lo > hi) return set_err(ctx, PBS_ERR_INVALID, "row range out of bounds");
  if (hi == lo) return PBS_OK;
  CK(cudaSetDevice(ctx->device));
  const long long nnz = row_ptr[n_rows];
  size_t b_rp = al(sizeof(long long) * (n_rows + 4)), b_ci = al(sizeof(long long) * (nnz + 1)),
         b_ci32 = al(sizeof(int) * (nnz + 8)), b_v = al(sizeof(double) * (nnz + 4)),
         b_x = al(sizeof(double) * (n_cols + 1)), b_y = al(sizeof(double) * (n_rows + 1));
  char* base;
  int rc = scratch(ctx, b_rp + b_ci + b_ci32 + b_v + b_x + b_y + 256, (void**)&base);
  if (rc) return rc;
  long long* d_rp = (long long*)base;
  long long* d_ci64 = (long long*)(base + b_rp);
  int* d_ci = (int*)(base + b_rp + b_ci);
  double* d_v = (double*)(base + b_rp + b_ci + b_ci32);
  double* d_x = (double*)(base + b_rp + b_ci + b_ci32 + b_v);
  double* d_y = (double*)(base + b_rp + b_ci + b_ci32 + b_v + b_x);
  int* d_bad = (int*)(base + b_rp + b_ci + b_ci32 + b_v + b_x + b_y);
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(d_rp, row_ptr, sizeof(long long) * (n_rows + 1), cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    CK(cudaMemcpyAsync(d_ci64, col_idx, sizeof(long long) * nnz, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_v, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
    cvt_i64_i32_kernel<<<ctx->sms, 256, 0, s>>>(d_ci64, d_ci, nnz, d_bad, n_cols > 0 ? n_cols : 1);
  }
  if (n_cols > 0) CK(cudaMemcpyAsync(d_x, x, sizeof(double) * n_cols, cudaMemcpyHostToDevice, s));
  pbs_mat tmp;
  tmp.ctx = ctx;
  tmp.rp = d_rp;
  tmp.ci = d_ci;
  tmp.v = d_v;
  tmp.n_rows = n_rows;
  tmp.n_cols = n_cols;
  tmp.nnz = nnz;
  Launcher L{ctx, &tmp, s};
  EpiStore e{};
  e.y = d_y;
  spmv_launch(L, d_x, e, lo, hi, KS);
  if (L.err) return L.err;
  CK(cudaMemcpyAsync(out + lo, d_y + lo, sizeof(double) * (hi - lo), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  tmp.rp = nullptr;
  tmp.ci = nullptr;
  tmp.v = nullptr;
  return PBS_OK;
}

PBS_EXPORT int pbs_k_dot_range(pbs_ctx* ctx, const double* x, const double* y, int64_t lo, int64_t hi,
                               double* result) {
  if (!ctx) return set_err(nullptr, PBS_ERR_INVALID, "ctx is NULL");
  if (hi <= lo) {
    *result = 0.0;
    return PBS_OK;
  }
  CK(cudaSetDevice(ctx->device));
  const long long n = hi - lo;
  size_t b = al(sizeof(double) * n);
  char* base;
  int rc = scratch(ctx, 2 * b + 256, (void**)&base);
  if (rc) return rc;
  double* dx = (double*)base;
  double* dy = (double*)(base + b);
  double* dout = (double*)(base + 2 * b);
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(dx, x + lo, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dy, y + lo, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  long long nblk = (n + kThreads - 1) / kThreads;
  int grid = grid_for(ctx, (const void*)dot_partial_kernel, nblk);
  dot_partial_kernel<<<grid, kThreads, 0, s>>>(dx, dy, 0, n, ctx->partials);
  dot_final_kernel<<<1, 32, 0, s>>>(ctx->partials, grid, dout);
  CK(cudaMemcpyAsync(result, dout, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  return PBS_OK;
}

PBS_EXPORT int pbs_k_lincomb(pbs_ctx* ctx, int32_t kind, int64_t n, double* out, const double* sc,
                             const double* a, const double* b, const double* c, const double* d) {
  if (!ctx) return set_err(nullptr, PBS_ERR_INVALID, "ctx is NULL");
  if (kind < 2 || kind > 7) return set_err(ctx, PBS_ERR_INVALID, "unknown lincomb kind");
  if (n <= 0) return PBS_OK;
  CK(cudaSetDevice(ctx->device));
  size_t bb = al(sizeof(double) * n);
  char* base;
  int rc = scratch(ctx, 5 * bb, (void**)&base);
  if (rc) return rc;
  double* dv[5];
  for (int k = 0; k < 5; ++k) dv[k] = (double*)(base + k * bb);
  const double* in[4] = {a, b, c, d};
  int nin = kind == 2 ? 2 : (kind == 4 ? 4 : 3);
  cudaStream_t s = ctx->stream;
  for (int k = 0; k < nin; ++k)
    CK(cudaMemcpyAsync(dv[k], in[k], sizeof(double) * n, cudaMemcpyHostToDevice, s));
  long long nblk = (n + kThreads - 1) / kThreads;
  int grid = grid_for(ctx, (const void*)lincomb_kernel, nblk);
  lincomb_kernel<<<grid, kThreads, 0, s>>>(kind, n, dv[4], sc[0], sc[1], sc[2], sc[3], dv[0], dv[1],
                                           dv[2], dv[3]);
  CK(cudaMemcpyAsync(out, dv[4], sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  return PBS_OK;
}

PBS_EXPORT int pbs_dot_batch_dev(pbs_ctx* ctx, int64_t n, const double* d_s, const double* d_y,
                                 const double* d_r, const double* d_r0s, const double* d_t,
                                 int32_t reduce_mode, int32_t plan_workers, double* out9) {
  if (!ctx) return set_err(nullptr, PBS_ERR_INVALID, "ctx is NULL");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  int rc = reset_tmp_state(ctx);
  if (rc) return rc;
  int np;
  int chain = reduce_mode == PBS_REDUCE_PLAN;
  long long* d_bounds = nullptr;
  if (chain) {
    std::vector<long long> b;
    np = plan_balanced(n, plan_workers < 1 ? 1 : plan_workers, b);
    if (np > kMaxParts) return set_err(ctx, PBS_ERR_INVALID, "plan_workers too large");
    CK(cudaMalloc(&d_bounds, sizeof(long long) * (np + 1)));
    CK(cudaMemcpyAsync(d_bounds, b.data(), sizeof(long long) * (np + 1), cudaMemcpyHostToDevice, s));
    dots9_plan_kernel<<<np, 32, 0, s>>>(d_bounds, d_s, d_y, d_r, d_r0s, d_t, ctx->partials, nullptr);
  } else {
    long long nblk = (n + kThreads - 1) / kThreads;
    np = grid_for(ctx, (const void*)dots9_tree_kernel, nblk);
    dots9_tree_kernel<<<np, kThreads, 0, s>>>(n, d_s, d_y, d_r, d_r0s, d_t, ctx->partials, nullptr);
  }
  // reuse the finalize reduction with a state whose run_all makes it reduce;
  // tol < 0 and max_iters > 0 keep the check from stopping anything
  SolverState h{};
  h.tol = -1.0;
  h.max_iters = 1LL << 60;
  h.iter = 1;
  h.run_all = 1;
  h.run_spine = 1;
  h.alpha = 1.0;
  h.zeta = 1.0;
  h.f_prev = 1.0;
  h.r0_norm = 1.0;
  h.nf_row = (unsigned long long)kNoError;
  CK(cudaMemcpyAsync(ctx->tmp_state, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  finalize_kernel<<<1, 288, 0, s>>>(ctx->tmp_state, ctx->partials, np, chain, 0);
  CK(cudaMemcpyAsync(out9, ctx->tmp_state->dots, sizeof(double) * kNumDots, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaFree(d_bounds);
  CK(cudaGetLastError());
  return PBS_OK;
}
