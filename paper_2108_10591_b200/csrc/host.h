// host.h — host-side core of libpbsafe shared by its translation units
// (core.cu: contexts, operators, workspaces, the C-ABI; solve.cu: the
// single-GPU schedules of the Safe methods; prod.cu: the product-type
// comparators; dist.cu: the multi-GPU row-partitioned schedule).
#pragma once
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <map>
#include <algorithm>
#include <thread>

#include "common.cuh"
#include "spmv.cuh"
#include "vec.cuh"
#include "zmarch.cuh"
#include "sell.cuh"

using namespace pbs;

#define PBS_EXPORT extern "C" __attribute__((visibility("default")))

extern std::string g_last_error;

struct EventPool {
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    return ev[used++];
  }
  void reset() { used = 0; }
  ~EventPool() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

struct pbs_dist;  // dist.cu

struct ZmMap {  // a CUtensorMap that std::map can hold (64-byte aligned)
  CUtensorMap map;
};

// Multi-GPU row partition of an operator (dist.cu, include/pbsafe.h).  The
// partition's SpMV inputs live in an extended space [pad | left halo | own |
// right halo]; sends are (peer, own offset, length, peer extended offset)
// quadruples, recvs (peer, extended offset, length) triples.
struct Partition {
  pbs_dist* dist = nullptr;
  long long n_global = 0, row_lo = 0, hl = 0, hr = 0;
  std::vector<long long> sends, recvs;
  // interior rows [L0, L1) read no halo column; both bounds are multiples of
  // the 256-row block, so all three launches keep the staged engine's
  // window-local columns.  split: the SpMVs after a halo exchange run the
  // interior while the exchange is in flight, then the boundary rows.
  bool split = false;
  long long L0 = 0, L1 = 0;
};

struct Workspace;

// What a captured solver graph bakes in about its operator: pointers and the
// staged-engine metadata.  A workspace (with its graphs) freed together with
// an operator is kept by the context and adopted by the next operator whose
// signature is identical — the stream-ordered pool hands an upload of the
// same shape the same addresses, so a solve(CsrMatrix) per step re-uses the
// graphs instead of capturing and instantiating them again.
struct MatSig {
  long long n_rows, n_cols, nnz, blk_nnz_max;
  long long stencil;
  const void *rp, *ci, *v, *wc;
  const void *sell_v, *sell_c, *sell_off, *sell_len, *sell_vi, *sell_dict;
  long long sell_mode;
  long long sell_lmax;
  XWin xwin;
  StencilView sv;
  StencilWin swin;
};

struct pbs_ctx {
  int device = 0;
  int sms = 148;
  int cc_major = 0, cc_minor = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  // kernel-table scratch (grow-only)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  double* partials = nullptr;  // dot partials for ad-hoc reductions
  SolverState* tmp_state = nullptr;
  std::map<const void*, int> occ;  // kernel -> resident CTAs per SM
  EventPool events;
  Workspace* ws_cache = nullptr;  // workspace of the last freed single-GPU operator
  MatSig ws_sig{};
  // Buffers of the last uploaded CSR shape (operator arrays and upload
  // temporaries), kept by exact size when freed and handed to the next upload
  // of the same shape: a solve(CsrMatrix) per step then makes no allocation
  // at all.  (Going back to the stream-ordered pool each time stalled an
  // upload for 20-700 ms every few dozen calls, whenever the pool had split
  // a cached block and had to map new memory.)
  std::multimap<size_t, void*> spare;
  std::map<void*, size_t> spare_sizes;  // live buffers that came from buf_alloc
  size_t spare_bytes = 0;
  long long spare_rows = -1, spare_nnz = -1;
};

struct pbs_mat {
  pbs_ctx* ctx = nullptr;
  int stencil = 0;
  long long n_rows = 0, n_cols = 0, nnz = 0;
  long long* rp = nullptr;
  int* ci = nullptr;
  double* v = nullptr;
  unsigned short* wc = nullptr;  // window-local column per nonzero (staged engine; null: col_idx)
  // sliced-ELL copy of the nonzeros for sell_pipe_kernel (sell.cuh; null: CSR order only)
  double* sell_v = nullptr;
  unsigned short* sell_c = nullptr;
  long long* sell_off = nullptr;
  unsigned char* sell_len = nullptr;  // nonzeros per row, 256 per block
  // value dictionary (<= 256 distinct values): u8 index per entry instead of sell_v
  unsigned char* sell_vi = nullptr;
  double* sell_dict = nullptr;
  int sell_ndict = 0;
  int sell_mode = 0;  // kSellF64 / kSellDictV / kSellPairs (sell_dict then holds SellPairs, sell_c is null)
  int sell_lmax = 0;          // most levels (longest row) in one block
  long long sell_entries = 0;
  StencilView sv{};
  XWin xwin{};  // x windows of the pipelined engines (nwin = 0: gather x)
  StencilWin swin{};  // stencil point -> window
  long long blk_nnz_max = 0;  // most nonzeros in one 256-row block (chunk sizing)
  Partition part;  // multi-GPU row partition (part.dist == nullptr: single GPU)
  Workspace* ws = nullptr;
  std::map<std::pair<const double*, int>, ZmMap> zm_maps;  // z-marching engine: tensor map per input vector, rows per thread
};

static inline int set_err(pbs_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  g_last_error = msg;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_err(ctx, PBS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Large buffers come from the device's stream-ordered memory pool, which keeps
// freed memory cached (release threshold = max): a solve on a host CsrMatrix
// uploads and frees its operator and workspace every call, and plain
// cudaFree of hundreds of MB can stall for hundreds of ms.
template <class T>
static cudaError_t pool_alloc(pbs_ctx* ctx, T** p, size_t bytes) {
  return cudaMallocAsync((void**)p, bytes, ctx->stream);
}
static inline void pool_free(pbs_ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

constexpr size_t kSpareCapBytes = 6ULL << 30;  // buffers kept for the next same-shape upload, at most

template <class T>
static cudaError_t buf_alloc(pbs_ctx* ctx, T** p, size_t bytes) {
  auto it = ctx->spare.lower_bound(bytes);  // the oldest spare of exactly this size
  if (it != ctx->spare.end() && it->first == bytes) {
    *p = (T*)it->second;
    ctx->spare.erase(it);
    ctx->spare_bytes -= bytes;
    ctx->spare_sizes[(void*)*p] = bytes;
    return cudaSuccess;
  }
  cudaError_t e = cudaMallocAsync((void**)p, bytes, ctx->stream);
  if (e == cudaSuccess) ctx->spare_sizes[(void*)*p] = bytes;
  return e;
}
static inline void buf_free(pbs_ctx* ctx, void* p) {
  if (!p) return;
  auto it = ctx->spare_sizes.find(p);
  if (it == ctx->spare_sizes.end()) {  // not from buf_alloc
    cudaFreeAsync(p, ctx->stream);
    return;
  }
  const size_t bytes = it->second;
  ctx->spare_sizes.erase(it);
  if (ctx->spare_bytes + bytes > kSpareCapBytes) {
    cudaFreeAsync(p, ctx->stream);
    return;
  }
  ctx->spare.emplace(bytes, p);  // after the older spares of this size
  ctx->spare_bytes += bytes;
}
static inline void buf_flush(pbs_ctx* ctx) {
  for (auto& kv : ctx->spare) cudaFreeAsync(kv.second, ctx->stream);
  ctx->spare.clear();
  ctx->spare_bytes = 0;
}

static inline int grid_for(pbs_ctx* ctx, const void* kernel, long long work_blocks, int cap_per_sm = 8,
                           int sms = 0) {
  auto it = ctx->occ.find(kernel);
  int per_sm;
  if (it == ctx->occ.end()) {
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    ctx->occ[kernel] = per_sm;
  } else {
    per_sm = it->second;
  }
  if (per_sm > cap_per_sm) per_sm = cap_per_sm;
  long long g = (long long)(sms > 0 ? sms : ctx->sms) * per_sm;
  if (work_blocks < g) g = work_blocks;
  if (g < 1) g = 1;
  return (int)g;
}


// ------------------------------------------------------------------ workspace

struct Workspace {
  pbs_ctx* ctx = nullptr;
  long long n = 0;
  size_t stride = 0;  // padded elements per vector
  double* base = nullptr;
  bool base_ipc = false;  // cudaMalloc'd (IPC-exportable: peers map it), not from the pool
  VecPtrs V{};  // own segments (elementwise kernels, SpMV outputs, epilogue inputs)
  VecPtrs X{};  // extended-space bases (SpMV inputs: [left halo | own | right halo])
  long long n_ext = 0, own_off = 0;
  double* partials = nullptr;
  double* partials12 = nullptr;  // K12's records of the s-independent dots
  long long* plan_bounds = nullptr;
  int plan_workers = 0;
  int plan_w_actual = 0;
  SolverState* st = nullptr;
  HostMirror* mirror_h = nullptr;
  HostMirror* mirror_d = nullptr;
  double* hist_rel = nullptr;
  unsigned char* hist_flags = nullptr;
  double* hist_coef = nullptr;
  long long hist_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double* trace_host = nullptr;  // pinned staging for trace_hook (13 vectors)
  // graph cache: key -> exec
  std::map<long long, std::pair<cudaGraphExec_t, long long>> graphs;  // exec, kernels per launch
};

// ---- workspace / plan management (core.cu)
void free_graphs(Workspace* ws);
void free_ws(Workspace* ws);
MatSig mat_sig(const pbs_mat* m);
void drop_ws_cache(pbs_ctx* ctx);
int ensure_ws(pbs_mat* m, long long hist_slots);
int plan_balanced(long long n, long long workers, std::vector<long long>& b);
int ensure_plan(pbs_mat* m, int workers);
int compute_xwin(pbs_ctx* ctx, pbs_mat* m);

// ------------------------------------------------------------------ launching

enum Kind { KK1 = 0, KK2, KK3, KF, KR, KRS, KS, KD };

struct Launcher {
  pbs_ctx* ctx;
  pbs_mat* m;
  cudaStream_t s;
  bool timing = false;
  std::vector<std::pair<int, cudaEvent_t>>* marks = nullptr;
  long long launches = 0;
  // trace_hook support: called by the iteration bodies where the reference
  // calls trace_hook (after the updates, before the next check)
  const pbs_config* trace_cfg = nullptr;
  Workspace* trace_ws = nullptr;
  int trace_method = 0;
  long long iter = 0;
  int trace_rc = 0;
  int err = 0;  // first launch-configuration failure (sticky)
  // multi-GPU schedule: SMs the launches may fill (0: all; the reduction's
  // kernels need one left free beside a persistent SpMV grid, and a loopback
  // partition emulating one GPU of N gets sms / N), and a cap on one launch's
  // grid (its partial records must fit the buffer after earlier pieces')
  int sm_limit = 0;
  long long grid_cap = 0;
  bool leave_room = false;  // many-CTAs-per-SM engines keep one CTA slot per SM free
  int sms() const { return sm_limit > 0 ? sm_limit : ctx->sms; }
  int cap_grid(long long g) const {
    if (grid_cap > 0 && g > grid_cap) g = grid_cap;
    return (int)(g > 0 ? g : 1);
  }
  // schedule evidence: (iter, kind, tag, event) — resolved to times at the end
  struct Ev {
    long long iter;
    int kind, tag;
    cudaEvent_t e;
  };
  std::vector<Ev>* evidence = nullptr;
  void mark(cudaStream_t st, long long it, int kind, int tag) {
    if (!evidence) return;
    cudaEvent_t e = ctx->events.get();
    cudaEventRecord(e, st);
    evidence->push_back({it, kind, tag, e});
  }
  void trace_point();
  void done(int kind) {
    ++launches;
    if (timing && marks) {
      cudaEvent_t e = ctx->events.get();
      cudaEventRecord(e, s);
      marks->push_back({kind, e});
    }
  }
};

// pipelined CSR engine knobs (env overrides for tuning sweeps):
//   PBS_PIPE_CTAS    CTAs per SM tried first (falls back while slots do not fit)
//   PBS_PIPE_CHUNK   nonzeros per chunk stage
//   PBS_PIPE_SLOTS   block slots = chunk stages (cap)
static inline int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = getenv(name);
  int v = e ? atoi(e) : dflt;
  return v < lo ? lo : (v > hi ? hi : v);
}
static inline int pipe_ctas_per_sm() {
  static int v = env_int("PBS_PIPE_CTAS", 2, 1, 4);
  return v;
}
static inline int pipe_chunk_cap() {
  static int v = env_int("PBS_PIPE_CHUNK", 2048, 256, kPipeChunkMax) & ~3;
  return v;
}
// band mode runs one CTA per SM (the circular x buffer takes 84+ KiB), where
// larger chunks stream better (profiles/sweeps/r1_band.log: config 3, 2048 ->
// 3072 nonzeros per chunk, 705 -> 667 us per iteration)
static inline int band_chunk_cap() {
  static int v = env_int("PBS_BAND_CHUNK", 3072, 256, kPipeChunkMax) & ~3;
  return v;
}
static inline int csr_engine_tpr() {  // PBS_CSR_ENGINE=tpr: thread-per-row CSR engine for every product
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PBS_CSR_ENGINE");
    v = (e && std::string(e) == "tpr") ? 1 : 0;
  }
  return v;
}
// Programmatic dependent launch per engine, PBS_PDL bitmask (A/B sweeps):
// 1 staged CSR, 2 staged stencil, 4 direct stencil.  Default 1: the staged
// CSR engine gains (its producer streams matrix chunks before the wait);
// the direct stencil engine loses (profiles/sweeps/r1_pdl.log).
enum { kPdlCsrPipe = 1, kPdlStencilPipe = 2, kPdlStencilDirect = 4, kPdlStencilZm = 8 };
static inline bool use_pdl(int engine) {
  static int v = env_int("PBS_PDL", kPdlCsrPipe | kPdlStencilZm, 0, 15);
  return (v & engine) != 0;
}
static inline int pipe_slots_cap() {
  static int v = env_int("PBS_PIPE_SLOTS", 2, 2, kMaxStages);
  return v;
}
static inline int sell_slots_cap() {  // block slots of the sliced-ELL engine
  static int v = env_int("PBS_SELL_SLOTS", 3, 2, kMaxStages);
  return v;
}
// L2 prefetch distance of the block slots' streams, in blocks.  Off: asking L2
// for the next blocks' lines ahead of their copies loses on configs 2 and 4
// (9726 -> 9470 / 9210 / 8746 it/s at distance 1 / 2 / 4; the copies already
// keep HBM busy and the prefetches only add requests, profiles/r2/sweeps_sell.md)
static inline int sell_prefetch() {
  static int v = env_int("PBS_SELL_PF", 0, 0, 8);
  return v;
}
static inline int pipe_extra_chunks() {  // chunk stages beyond the block slots
  static int v = env_int("PBS_PIPE_XCHUNK", 0, 0, 4);
  return v;
}

// The epilogue inputs are always staged by the producer: the build that let
// the consumers load them instead lost everywhere measured
// (profiles/sweeps/r1_c4_pipe.log) and is no longer compiled.

// Ring sizing.  The engine is bound by the bytes each SM keeps in flight
// (Little's law: ~45 KB/us per SM at full HBM rate times ~1-2 us of loaded
// latency), so among CTAs-per-SM choices take the one whose rings hold the
// most shared memory: block slots (row_ptr, x windows, epilogue inputs) plus
// chunk stages, with every chunk stage the budget allows beyond the slots
// (PBS_PIPE_XCHUNK caps them) when blocks span several chunks.  Ties
// (within 5%) go to more CTAs per SM.
// Config 2 keeps 2 CTAs/SM; config 4's 27-point rows (7k nonzeros and 25 KB
// of x windows per block) get 1 CTA/SM with 4 extra chunk stages
// (13.8 -> 10.6 ms per iteration).
template <class Epi>
static int pipe_config(pbs_ctx* ctx, const XWin& W, int colb, long long blk_nnz_max, int* bslots, int* cstages,
                       size_t* smem, int* ctas, int* chunk, int* stage_in) {
  // one chunk per row block when the densest block fits the cap (stencils:
  // ~7 or ~27 nonzeros per row), else cap-sized chunks
  int ch = W.band_s ? band_chunk_cap() : pipe_chunk_cap();
  if (blk_nnz_max > 0 && blk_nnz_max < ch) ch = (int)((blk_nnz_max + 3) & ~3LL);
  const ChunkLayout CL(ch, colb);
  int per_sm = 0, optin = 0;
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  const int si = 1;
  const BlockLayout BL(W.total, si ? Epi::kInStaged : 0);
  // extra chunk stages pay when a block spans several chunks (the consumers
  // walk them in turn); with one chunk per block (7-point stencils, config 2:
  // 162 -> 166 us per iteration with them) the slots already double-buffer
  const char* xenv = getenv("PBS_PIPE_XCHUNK");
  const int xcap = xenv ? pipe_extra_chunks() : (blk_nnz_max > ch ? kMaxStages : 0);
  int n = 0, c = 0, xc = 0;
  size_t best = 0;
  for (int cc = pipe_ctas_per_sm(); cc >= 1; --cc) {
    // per-CTA budget: the SM's shared memory split between the resident CTAs,
    // less the 1 KiB the runtime reserves per CTA and the kernel's static smem
    size_t budget = (size_t)per_sm / cc - 1024 - 2048;
    if (budget > (size_t)optin - 2048) budget = (size_t)optin - 2048;
    const size_t fixed = kPipeBarrierBytes + (size_t)W.band_s * sizeof(double);
    if (budget <= fixed) continue;
    budget -= fixed;
    int nn = (int)(budget / (BL.bytes + CL.bytes));
    if (nn > pipe_slots_cap()) nn = pipe_slots_cap();
    if (nn < 2) continue;
    int xx = (int)((budget - (size_t)nn * (BL.bytes + CL.bytes)) / CL.bytes);
    if (xx > xcap) xx = xcap;
    if (nn + xx > kMaxStages) xx = kMaxStages - nn;
    const size_t bytes = (size_t)cc * ((size_t)nn * BL.bytes + (size_t)(nn + xx) * CL.bytes);
    if (bytes * 20 > best * 21) {  // > 5% more in flight than the larger-CTA choice
      best = bytes;
      n = nn;
      c = cc;
      xc = xx;
    }
  }
  if (n < 2) return set_err(ctx, PBS_ERR_UNSUPPORTED, "not enough shared memory for the SpMV pipeline");
  *ctas = c;
  *bslots = n;
  *cstages = n + xc;
  *chunk = ch;
  *stage_in = si;
  *smem = kPipeBarrierBytes + (size_t)W.band_s * sizeof(double) + (size_t)n * BL.bytes + (size_t)(n + xc) * CL.bytes;
  const void* k = c == 1 ? (const void*)csr_pipe_kernel<Epi, true, 1> : (const void*)csr_pipe_kernel<Epi, true>;
  auto it = ctx->occ.find(k);
  if (it == ctx->occ.end() || (size_t)it->second < *smem) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
    if (e != cudaSuccess) return set_err(ctx, PBS_ERR_CUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    ctx->occ[k] = (int)*smem;
  }
  return PBS_OK;
}

// Ring sizing of the sliced-ELL engine (sell.cuh), by the same rule: block
// slots hold the x windows and epilogue inputs (no row_ptr slice), chunk
// stages klev levels of the block (one chunk per block when its longest row
// has at most kSellLevMax nonzeros: 7-point stencils).
template <class Epi>
static int sell_config(pbs_ctx* ctx, const XWin& W, int lmax, int mode, int* bslots, int* cstages, size_t* smem,
                       int* ctas, int* klev) {
  static int lev_cap = env_int("PBS_SELL_LEV", kSellLevMax, 1, kSellLevMax);
  static int lev_cap_pair = env_int("PBS_SELL_LEV_PAIR", kSellLevMaxPair, 1, kSellLevMaxPair);
  const int cap = mode == kSellPairs ? lev_cap_pair : lev_cap;
  int kl = lmax < cap ? lmax : cap;
  if (kl < 1) kl = 1;
  const SellChunkLayout CL(kl, mode);
  const SellBlockLayout BL(W.total, Epi::kInStaged);
  int per_sm = 0, optin = 0;
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  const char* xenv = getenv("PBS_PIPE_XCHUNK");
  const int xcap = xenv ? pipe_extra_chunks() : (lmax > kl ? kMaxStages : 0);
  int n = 0, c = 0, xc = 0;
  size_t best = 0;
  for (int cc = pipe_ctas_per_sm(); cc >= 1; --cc) {
    // less the 1 KiB the runtime reserves per CTA and the kernel's static smem (the dictionary)
    const size_t fixed = 1024 + 512 + (mode == kSellPairs ? 4096 : 2048);
    size_t budget = (size_t)per_sm / cc - fixed;
    if (budget > (size_t)optin - fixed) budget = (size_t)optin - fixed;
    if (budget <= kPipeBarrierBytes) continue;
    budget -= kPipeBarrierBytes;
    int nn = (int)(budget / (BL.bytes + CL.bytes));
    if (nn > sell_slots_cap()) nn = sell_slots_cap();
    if (nn < 2) continue;
    int xx = (int)((budget - (size_t)nn * (BL.bytes + CL.bytes)) / CL.bytes);
    if (xx > xcap) xx = xcap;
    if (nn + xx > kMaxStages) xx = kMaxStages - nn;
    const size_t bytes = (size_t)cc * ((size_t)nn * BL.bytes + (size_t)(nn + xx) * CL.bytes);
    if (bytes * 20 > best * 21) {
      best = bytes;
      n = nn;
      c = cc;
      xc = xx;
    }
  }
  if (n < 2) return set_err(ctx, PBS_ERR_UNSUPPORTED, "not enough shared memory for the SpMV pipeline");
  *ctas = c;
  *bslots = n;
  *cstages = n + xc;
  *klev = kl;
  *smem = kPipeBarrierBytes + (size_t)n * BL.bytes + (size_t)(n + xc) * CL.bytes;
  const void* k;
  if (mode == kSellPairs)
    k = c == 1 ? (const void*)sell_pipe_kernel<Epi, 1, kSellPairs> : (const void*)sell_pipe_kernel<Epi, 2, kSellPairs>;
  else if (mode == kSellDictV)
    k = c == 1 ? (const void*)sell_pipe_kernel<Epi, 1, kSellDictV> : (const void*)sell_pipe_kernel<Epi, 2, kSellDictV>;
  else
    k = c == 1 ? (const void*)sell_pipe_kernel<Epi, 1, kSellF64> : (const void*)sell_pipe_kernel<Epi, 2, kSellF64>;
  auto it = ctx->occ.find(k);
  if (it == ctx->occ.end() || (size_t)it->second < *smem) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
    if (e != cudaSuccess) return set_err(ctx, PBS_ERR_CUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    ctx->occ[k] = (int)*smem;
  }
  return PBS_OK;
}

// PBS_STENCIL_ENGINE=direct|pipe forces one stencil engine; default: per
// epilogue (Epi::kStencilPipe — the staged engine for the dot-carrying K3,
// the L1-cached direct engine for the streaming K12), except that stencils
// wider than 7 points stage everything: 27 L1 neighbour loads per row cost
// the direct engine more than the staging (config 4 K12: 1883 -> 1758 us,
// profiles/sweeps/r1_stencil_engines.log)
template <class Epi>
static bool stencil_engine_pipe(int npts) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PBS_STENCIL_ENGINE");
    v = (e && std::string(e) == "direct") ? 0 : ((e && std::string(e) == "pipe") ? 1 : 2);
  }
  return v == 2 ? (Epi::kStencilPipe || npts > 7) : v == 1;
}

// The z-marching engine (zmarch.cuh) takes every 3D 7- and 27-point stencil
// product whose rows are whole planes of a grid with an even edge
// (PBS_STENCIL_ENGINE=pipe|direct forces the older engines for A/B runs).
// PBS_ZM_RING: plane stages per CTA; PBS_ZM_WAVES: work items per CTA
// (the z-chunk length follows).
static inline bool stencil_zm_ok(const pbs_mat* m, long long lo, long long hi) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("PBS_STENCIL_ENGINE");
    forced = (e && (std::string(e) == "pipe" || std::string(e) == "direct")) ? 1 : 0;
  }
  // 7-point stencils stay on the direct / staged engines by default: their
  // rows read 3 planes of only 7 points, which the L1-cached direct engine
  // (K12, K1) and the staged engine (K3) already stream near the copy peak
  // (config 2 matrix-free: 8861 vs 8785 it/s); PBS_ZM7=1 moves them too
  static int zm7 = env_int("PBS_ZM7", 0, 0, 1);
  if (!m->stencil) return false;
  const StencilView& S = m->sv;
  if (forced || S.dim != 3 || (S.npts != 27 && !(S.npts == 7 && zm7)) || (S.k & 1) || S.k < 4) return false;
  for (int p = 0; p < S.npts; ++p)  // the engine's compile-time neighbour table
    for (int a = 0; a < 3; ++a)
      if (S.off[p][a] != (S.npts == 27 ? zm_off<27>(p, a) : zm_off<7>(p, a))) return false;
  const long long k2 = S.k2;
  return !(lo % k2 || hi % k2 || S.g0 % k2 || (-S.xlo) % k2 || S.xhi % k2 || hi <= lo);
}

template <class Epi>
static bool stencil_zm_geom(pbs_ctx* ctx, int sms, const pbs_mat* m, long long lo, long long hi,
                            const void* kernel, size_t* smem, int* grid, ZmGeom* G) {
  using Sh = ZmShape<zm_rpt<Epi>()>;
  if (!stencil_zm_ok(m, lo, hi)) return false;
  const StencilView& S = m->sv;
  const long long k2 = S.k2;
  static int ring_env = env_int("PBS_ZM_RING", 8, 4, kZmMaxRing);
  static int waves_env = env_int("PBS_ZM_WAVES", 8, 1, 64);
  G->tiles_y = (int)((S.k + kZmTY - 1) / kZmTY);
  G->tiles_x = (int)((S.k + Sh::TX - 1) / Sh::TX);
  G->z_lo = (int)(lo / k2);
  G->z_hi = (int)(hi / k2);
  G->zx_lo = (int)(S.xlo / k2);
  G->zx_hi = (int)(S.xhi / k2);
  G->gz0 = S.g0 / k2;
  G->ring = ring_env;
  *smem = 256 + sizeof(double) * (size_t)Sh::Stage * G->ring;
  auto it = ctx->occ.find(kernel);
  if (it == ctx->occ.end() || (size_t)it->second < *smem) {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem) != cudaSuccess)
      return false;
    ctx->occ[kernel] = (int)*smem;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kZmCTA, *smem);
  if (per_sm < 1) per_sm = 1;
  const long long ntiles = (long long)G->tiles_y * G->tiles_x, nz = G->z_hi - G->z_lo;
  const long long cap = (long long)sms * per_sm;
  // about waves_env work items per CTA, each a run of >= 2 planes
  long long zc = (nz * ntiles + cap * waves_env - 1) / (cap * waves_env);
  if (zc < 2) zc = 2;
  if (zc > nz) zc = nz;
  G->zchunk = (int)zc;
  const long long items = ntiles * ((nz + zc - 1) / zc);
  *grid = (int)(items < cap ? items : cap);
  return true;
}

// The 3-D tensor map of a stencil operator's input vector x for the
// z-marching engine: dims (k, k, planes present), box (TX+4, TY+2, 1), zeros
// out of range.  Encoded once per (operator, x) and kept in the operator.
typedef CUresult (*PfnTensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                            CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                            CUtensorMapFloatOOBfill);
template <int RPT>
static const CUtensorMap* stencil_zm_map(pbs_mat* m, const double* x, const ZmGeom& G) {
  auto it = m->zm_maps.find({x, RPT});
  if (it != m->zm_maps.end()) return &it->second.map;
  if (m->zm_maps.size() >= 64) m->zm_maps.clear();  // callers' temporary x buffers
  static PfnTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", (void**)&encode, 12000, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      encode = nullptr;
      return nullptr;
    }
  }
  const StencilView& S = m->sv;
  const cuuint64_t dims[3] = {(cuuint64_t)S.k, (cuuint64_t)S.k, (cuuint64_t)(G.zx_hi - G.zx_lo)};
  const cuuint64_t strides[2] = {(cuuint64_t)S.k * sizeof(double), (cuuint64_t)S.k2 * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)ZmShape<RPT>::RowW, kZmTY + 2, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  ZmMap zm;
  void* base = (void*)(x + (long long)G.zx_lo * S.k2);
  if (encode(&zm.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return nullptr;
  return &m->zm_maps.emplace(std::make_pair(x, RPT), zm).first->second.map;
}

template <class Epi, int DIM, int NP>
static int stencil_pipe_set_smem(pbs_ctx* ctx, size_t smem) {
  const void* k = (const void*)stencil_pipe_kernel<Epi, DIM, NP>;
  auto it = ctx->occ.find(k);
  if (it == ctx->occ.end() || (size_t)it->second < smem) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_err(ctx, PBS_ERR_CUDA, std::string("smem attribute: ") + cudaGetErrorString(e));
    ctx->occ[k] = (int)smem;
  }
  return PBS_OK;
}

template <class Epi>
static int stencil_pipe_config(pbs_ctx* ctx, const XWin& W, int* bslots, size_t* smem, int* ctas) {
  const BlockLayout BL(W.total, Epi::kInStaged);
  int per_sm = 0, optin = 0;
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  int n = 0, c = pipe_ctas_per_sm();
  for (; c >= 1; --c) {
    size_t budget = (size_t)per_sm / c - 1024 - 2048;
    if (budget > (size_t)optin - 2048) budget = (size_t)optin - 2048;
    budget -= kPipeBarrierBytes;
    n = (int)(budget / BL.bytes);
    if (n > 4) n = 4;
    if (n >= 2) break;
  }
  if (n < 2) return set_err(ctx, PBS_ERR_UNSUPPORTED, "not enough shared memory for the stencil pipeline");
  *ctas = c;
  *bslots = n;
  *smem = kPipeBarrierBytes + (size_t)n * BL.bytes;
  int rc = stencil_pipe_set_smem<Epi, 3, 7>(ctx, *smem);
  if (!rc) rc = stencil_pipe_set_smem<Epi, 3, 27>(ctx, *smem);
  if (!rc) rc = stencil_pipe_set_smem<Epi, 3, 0>(ctx, *smem);
  if (!rc) rc = stencil_pipe_set_smem<Epi, 2, 5>(ctx, *smem);
  if (!rc) rc = stencil_pipe_set_smem<Epi, 2, 0>(ctx, *smem);
  if (!rc) rc = stencil_pipe_set_smem<Epi, 1, 3>(ctx, *smem);
  if (!rc) rc = stencil_pipe_set_smem<Epi, 1, 0>(ctx, *smem);
  return rc;
}

// Launch with the programmatic-dependent-launch attribute when PBS_PDL is on
// (kernels launched this way call griddep_wait before reading anything the
// previous kernel wrote).
template <class... KArgs, class... Args>
static void launch_pdl(Launcher& L, int engine, void (*kernel)(KArgs...), int grid, int block, size_t smem,
                       Args... args) {
  if (!use_pdl(engine)) {
    kernel<<<grid, block, smem, L.s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = L.s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) L.err = set_err(L.ctx, PBS_ERR_CUDA, std::string("PDL launch: ") + cudaGetErrorString(e));
}

// The plain products (no or one epilogue input: setup and replacement
// SpMVs) of short-row CSR matrices run on the thread-per-row engine: with ~7
// nonzeros per row the staged engine's consumers wait on their block
// barriers (56% of warp samples) while each thread pays a block's
// bookkeeping for one row; at full occupancy with x from L1/L2 the plain
// SpMV of config 2 takes 41 instead of 50 us (0.84 vs 0.68 of the HBM peak).
// Not for the multi-GPU schedule's K1 (leave_room): filling every SM it keeps
// the reduction's 1-CTA kernels from running beside it, and the iteration
// loses more than K1 gains (5195 vs 5465 it/s, partitioned config 2).  Rows
// of 27 nonzeros stream better staged (config 4: 4.1 vs 8.7 ms).
// PBS_PLAIN_TPR=0 keeps the staged engine.
template <class Epi>
static bool csr_plain_tpr(const pbs_mat* m) {
  static int on = env_int("PBS_PLAIN_TPR", 1, 0, 2);  // 2: even when the sliced-ELL form exists (A/B)
  if (on == 1 && (m->sell_v || m->sell_vi)) return false;  // 3 or 10 B per entry, no row_ptr: streams less
  return on && (std::is_same<Epi, EpiStore>::value || std::is_same<Epi, EpiResid>::value) &&
         m->nnz <= 8 * m->n_rows;
}

template <class Epi>
static int spmv_launch(Launcher& L, const double* x, Epi epi, long long lo, long long hi, int kind) {
  pbs_mat* m = L.m;
  long long nblk = (hi - lo + kThreads - 1) / kThreads;
  int grid;
  ZmGeom zm;
  size_t zm_smem = 0;
  const CUtensorMap* zm_map = nullptr;
  if (!m->stencil && (csr_engine_tpr() || (csr_plain_tpr<Epi>(m) && !L.leave_room))) {
    CsrView A{m->rp, m->ci, m->v, lo, hi, m->n_cols, nullptr};
    // leave_room: one CTA slot per SM stays free for the reduction's 1-CTA
    // kernels (the multi-GPU K1 overlaps them)
    auto tpr_grid = [&](const void* k) {
      const int full = grid_for(L.ctx, k, 1LL << 40, 8, L.sms()) / L.sms();
      const int per_sm = L.leave_room && full > 1 ? full - 1 : full;
      return L.cap_grid(grid_for(L.ctx, k, nblk, per_sm, L.sms()));
    };
    grid = tpr_grid((const void*)csr_tpr_kernel<Epi, false>);
    csr_tpr_kernel<Epi, false><<<grid, kThreads, 0, L.s>>>(A, x, epi);
  } else if (!m->stencil && (m->sell_v || m->sell_vi) && (lo % kPipeRows) == 0) {
    // sliced-ELL form (sell.cuh): row blocks counted from row 0, like the
    // window-local columns
    SellView A{m->sell_v, m->sell_vi, (const void*)m->sell_dict, m->sell_c, m->sell_len, m->sell_off, lo, hi, m->n_cols};
    const int mode = m->sell_mode;
    int bslots, cstages, ctas, klev;
    size_t smem;
    int rc = sell_config<Epi>(L.ctx, m->xwin, m->sell_lmax, mode, &bslots, &cstages, &smem, &ctas, &klev);
    if (rc) {
      L.err = rc;
      return 0;
    }
    const long long nb = (hi - lo + kPipeRows - 1) / kPipeRows;
    const long long cap = (long long)L.sms() * ctas;
    grid = L.cap_grid(nb < cap ? nb : cap);
#define PBS_SELL(MB, D)                                                                                      \
  launch_pdl(L, kPdlCsrPipe, sell_pipe_kernel<Epi, MB, D>, grid, kSellThreads, smem, A, x, epi, m->xwin, bslots, \
             cstages, klev, sell_prefetch())
    if (mode == kSellPairs && ctas == 1) PBS_SELL(1, kSellPairs);
    else if (mode == kSellPairs) PBS_SELL(2, kSellPairs);
    else if (mode == kSellDictV && ctas == 1) PBS_SELL(1, kSellDictV);
    else if (mode == kSellDictV) PBS_SELL(2, kSellDictV);
    else if (ctas == 1) PBS_SELL(1, kSellF64);
    else PBS_SELL(2, kSellF64);
#undef PBS_SELL
    if (L.err) return 0;
  } else if (!m->stencil) {
    // window-local columns describe the 256-row blocks counted from row 0, so
    // any launch starting on a block boundary can use them
    CsrView A{m->rp, m->ci, m->v, lo, hi, m->n_cols, (lo % kPipeRows) == 0 ? m->wc : nullptr};
    // staged x windows need the window-local columns; otherwise gather x
    const XWin W = A.wc ? m->xwin : XWin{};
    int bslots, cstages, ctas, chunk, stage_in;
    size_t smem;
    int rc = pipe_config<Epi>(L.ctx, W, A.wc ? 2 : 4, m->blk_nnz_max, &bslots, &cstages, &smem, &ctas, &chunk,
                              &stage_in);
    if (rc) {
      L.err = rc;
      return 0;
    }
    const long long cap = (long long)L.sms() * ctas;
    grid = L.cap_grid(nblk < cap ? nblk : cap);
    // programmatic dependent launch: overlaps this CTA's prologue and first
    // matrix chunks with the previous kernel's drain
    (void)stage_in;
    if (ctas == 1)  // 1-CTA layout: the instantiation with more products in flight
      launch_pdl(L, kPdlCsrPipe, csr_pipe_kernel<Epi, true, 1>, grid, kPipeThreads, smem, A, x, epi, W, bslots,
                 cstages, chunk);
    else
      launch_pdl(L, kPdlCsrPipe, csr_pipe_kernel<Epi, true>, grid, kPipeThreads, smem, A, x, epi, W, bslots, cstages,
                 chunk);
    if (L.err) return 0;
  } else if (m->stencil &&
             stencil_zm_geom<Epi>(L.ctx, L.sms(), m, lo, hi,
                                  m->sv.npts == 27 ? (const void*)stencil_zm_kernel<Epi, 27>
                                                   : (const void*)stencil_zm_kernel<Epi, 7>,
                                  &zm_smem, &grid, &zm) &&
             (zm_map = stencil_zm_map<zm_rpt<Epi>()>(m, x, zm)) != nullptr) {
    grid = L.cap_grid(grid);
    StencilView S = m->sv;
    S.row_lo = lo;
    S.row_hi = hi;
    if (S.npts == 27)
      launch_pdl(L, kPdlStencilZm, stencil_zm_kernel<Epi, 27>, grid, kZmCTA, zm_smem, S, *zm_map, epi, zm);
    else
      launch_pdl(L, kPdlStencilZm, stencil_zm_kernel<Epi, 7>, grid, kZmCTA, zm_smem, S, *zm_map, epi, zm);
  } else if (m->stencil && m->xwin.nwin && stencil_engine_pipe<Epi>(m->sv.npts)) {
    StencilView S = m->sv;
    S.row_lo = lo;
    S.row_hi = hi;
    int bslots, ctas;
    size_t smem;
    int rc = stencil_pipe_config<Epi>(L.ctx, m->xwin, &bslots, &smem, &ctas);
    if (rc) {
      L.err = rc;
      return 0;
    }
    const long long cap = (long long)L.sms() * ctas;
    grid = L.cap_grid(nblk < cap ? nblk : cap);
#define PBS_SPIPE(D, NP)                                                                                   \
  launch_pdl(L, kPdlStencilPipe, stencil_pipe_kernel<Epi, D, NP>, grid, kPipeThreads, smem, S, x, epi, m->xwin, \
             m->swin, bslots);
    if (S.dim == 3 && S.npts == 7) PBS_SPIPE(3, 7)
    else if (S.dim == 3 && S.npts == 27) PBS_SPIPE(3, 27)
    else if (S.dim == 3) PBS_SPIPE(3, 0)
    else if (S.dim == 2 && S.npts == 5) PBS_SPIPE(2, 5)
    else if (S.dim == 2) PBS_SPIPE(2, 0)
    else if (S.dim == 1 && S.npts == 3) PBS_SPIPE(1, 3)
    else PBS_SPIPE(1, 0)
#undef PBS_SPIPE
  } else {
    StencilView S = m->sv;
    S.row_lo = lo;
    S.row_hi = hi;
#define PBS_STENCIL(D, NP)                                                                 \
  {                                                                                        \
    grid = L.cap_grid(grid_for(L.ctx, (const void*)stencil_spmv_kernel<Epi, D, NP>, nblk, 8, L.sms())); \
    launch_pdl(L, kPdlStencilDirect, stencil_spmv_kernel<Epi, D, NP>, grid, kThreads, 0, S, x, epi); \
  }
    if (S.dim == 3 && S.npts == 7) PBS_STENCIL(3, 7)
    else if (S.dim == 3 && S.npts == 27) PBS_STENCIL(3, 27)
    else if (S.dim == 3) PBS_STENCIL(3, 0)
    else if (S.dim == 2 && S.npts == 5) PBS_STENCIL(2, 5)
    else if (S.dim == 2) PBS_STENCIL(2, 0)
    else if (S.dim == 1 && S.npts == 3) PBS_STENCIL(1, 3)
    else PBS_STENCIL(1, 0)
#undef PBS_STENCIL
  }
  L.done(kind);
  return grid;
}

template <class K, class... Args>
static void vec_launch(Launcher& L, K kernel, long long n, int kind, Args... args) {
  long long nblk = (n + kThreads - 1) / kThreads;
  int grid = L.cap_grid(grid_for(L.ctx, (const void*)kernel, nblk, 8, L.sms()));
  kernel<<<grid, kThreads, 0, L.s>>>(args...);
  L.done(kind);
}

struct Mode {
  int plan = 0;  // PBS_REDUCE_PLAN
  int store_temps = 0;
  int method = PBS_METHOD_PBICGSAFE;
};

// ---- epilogue constructors (pointers into the workspace)

static inline EpiStore epi_store(Workspace* ws, int out, int tag, int spine) {
  EpiStore e{};
  e.y = ws->V.v[out];
  e.st = ws->st;
  e.tag = tag;
  e.spine = spine;
  return e;
}

static inline EpiResid epi_resid(Workspace* ws, bool with_r0s) {
  EpiResid e{};
  e.r = ws->V.v[VR];
  e.r0s = with_r0s ? ws->V.v[VR0S] : nullptr;
  e.st = ws->st;
  e.tag = PBS_TAG_AX;
  e.in[0] = ws->V.v[VB];
  return e;
}

static inline DotSink sink_for(Workspace* ws, const Mode& md, int fuse, int replaced) {
  DotSink k{};
  k.partials = md.plan ? nullptr : ws->partials;
  k.fuse = md.plan ? 0 : fuse;
  k.replaced = replaced;
  return k;
}

static inline EpiDots epi_dots(Workspace* ws, const Mode& md, int spine, int fuse, int replaced) {
  EpiDots e{};
  auto& V = ws->V.v;
  e.s = V[VS];
  e.st = ws->st;
  e.tag = PBS_TAG_AR;
  e.spine = spine;
  e.sink = sink_for(ws, md, fuse, replaced);
  e.in[0] = V[VY];
  e.in[1] = V[VR];
  e.in[2] = V[VR0S];
  e.in[3] = V[VT];
  return e;
}

template <class E>
static E epi_k12_fill(Workspace* ws, const Mode& md) {
  E e{};
  auto& V = ws->V.v;
  e.as = V[VAS];
  e.p = V[VP];
  e.u = V[VU];
  e.w = V[VW];
  e.t = V[VT];
  e.z = V[VZ];
  e.y = V[VY];
  e.x = V[VX];
  e.r = V[VR];
  e.o_out = md.store_temps ? V[VO] : nullptr;
  e.q_out = md.store_temps ? V[VQ] : nullptr;
  e.st = ws->st;
  const int in[12] = {VR, VP, VU, VS, VT, VY, VL, VG, VW, VZ, VX, VR0S};
  for (int k = 0; k < E::kIn; ++k) e.in[k] = V[in[k]];
  return e;
}

static inline EpiK12 epi_k12(Workspace* ws, const Mode& md) { return epi_k12_fill<EpiK12>(ws, md); }

static inline EpiK12d epi_k12d(Workspace* ws, const Mode& md) {
  EpiK12d e = epi_k12_fill<EpiK12d>(ws, md);
  e.parts = ws->partials12;
  return e;
}

static inline EpiK3n epi_k3n(Workspace* ws, const Mode& md) {
  EpiK3n e{};
  auto& V = ws->V.v;
  e.l = V[VL];
  e.g = V[VG];
  e.s = V[VS];
  e.q_out = md.store_temps ? V[VQ] : nullptr;
  e.st = ws->st;
  e.tag = PBS_TAG_AW;
  const int in[4] = {VAS, VL, VG, VS};
  for (int k = 0; k < 4; ++k) e.in[k] = V[in[k]];
  return e;
}

// K3's batch fused into K3's epilogue (default) or as a separate streaming
// kernel (PBS_K3_DOTS=split; slower on B200: the compensated FP64 batch hides
// better under K3's memory traffic, profiles/r1_engine_sweep.log)
static inline bool k3_dots_split() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PBS_K3_DOTS");
    v = (e && std::string(e) == "split") ? 1 : 0;
  }
  return v;
}

// the next check's batch as a streaming kernel; returns nparts
static inline int dots_check(Launcher& L, Workspace* ws, int fuse, int replaced) {
  auto& V = ws->V.v;
  long long nblk = (ws->n + kThreads - 1) / kThreads;
  int np = grid_for(L.ctx, (const void*)dots9_check_kernel, nblk);
  dots9_check_kernel<<<np, kThreads, 0, L.s>>>(ws->n, V[VS], V[VY], V[VR], V[VR0S], V[VT], ws->partials,
                                               ws->st, fuse, replaced);
  L.done(KD);
  return np;
}

static inline EpiK3 epi_k3(Workspace* ws, const Mode& md, int fuse) {
  EpiK3 e{};
  auto& V = ws->V.v;
  e.l = V[VL];
  e.g = V[VG];
  e.s = V[VS];
  e.q_out = md.store_temps ? V[VQ] : nullptr;
  e.st = ws->st;
  e.tag = PBS_TAG_AW;
  e.sink = sink_for(ws, md, fuse, 0);
  const int in[8] = {VAS, VL, VG, VS, VY, VR, VR0S, VT};
  for (int k = 0; k < 8; ++k) e.in[k] = V[in[k]];
  return e;
}

// K3 carrying only the dots that need the new s; the check also reduces
// K12's records (np12 of them) for the other five
static inline EpiK3s epi_k3s(Workspace* ws, const Mode& md, int fuse, int np12) {
  EpiK3s e{};
  auto& V = ws->V.v;
  e.l = V[VL];
  e.g = V[VG];
  e.s = V[VS];
  e.q_out = md.store_temps ? V[VQ] : nullptr;
  e.st = ws->st;
  e.tag = PBS_TAG_AW;
  e.sink = sink_for(ws, md, fuse, 0);
  e.sink.partials2 = ws->partials12;
  e.sink.nparts2 = np12;
  e.sink.mask2 = kDotsK12;
  const int in[7] = {VAS, VL, VG, VS, VY, VR, VR0S};
  for (int k = 0; k < 7; ++k) e.in[k] = V[in[k]];
  return e;
}

// the batch split between K12 (b e f h r) and K3 (a c d g): default on for
// CSR (the staged K12 has the registers to spare); the direct stencil K12
// loses occupancy to the accumulators, so stencils keep all nine in K3.
// PBS_K12_DOTS=0 keeps all nine in K3 for CSR too.
// PBS_FUSE_CHECK=0: the check as its own 1-CTA kernel instead of the last
// K3 CTA's tail (A/B of the tail's cost)
static inline bool fuse_check() {
  static int v = env_int("PBS_FUSE_CHECK", 1, 0, 1);
  return v;
}

static inline int k12_dots() {
  static int v = env_int("PBS_K12_DOTS", 1, 0, 2);
  return v;
}

static inline EpiSS3 epi_ss3(Workspace* ws) {
  EpiSS3 e{};
  auto& V = ws->V.v;
  e.w = V[VW];
  e.t = V[VT];
  e.z = V[VZ];
  e.y = V[VY];
  e.x = V[VX];
  e.r = V[VR];
  e.st = ws->st;
  e.tag = PBS_TAG_AU;
  const int in[8] = {VO, VS, VU, VP, VY, VZ, VX, VR};
  for (int k = 0; k < 8; ++k) e.in[k] = V[in[k]];
  return e;
}

// batch partials over (s, y, r, r0s, t) for PLAN mode (tree mode fuses them
// into the producing SpMV); returns nparts
static inline int plan_dots(Launcher& L, Workspace* ws, int kind) {
  dots9_plan_kernel<<<ws->plan_w_actual, 32, 0, L.s>>>(ws->plan_bounds, ws->V.v[VS], ws->V.v[VY],
                                                      ws->V.v[VR], ws->V.v[VR0S], ws->V.v[VT],
                                                      ws->partials, ws->st);
  L.done(kind);
  return ws->plan_w_actual;
}

static inline void finalize(Launcher& L, Workspace* ws, int nparts, int chain, int replaced, int np12 = 0,
                     int phase = kPhSafe) {
  finalize_kernel<<<1, 288, 0, L.s>>>(ws->st, ws->partials, nparts, chain, replaced, ws->partials12, np12,
                                      np12 ? kDotsK12 : 0u, 1, kMaxParts, phase);
  L.done(KF);
}

// s = A r (+ the batch of the next check); tree mode fuses the check into the
// SpMV's last CTA, plan mode runs the plan chains + a separate finalize
static inline void spmv_s_check(Launcher& L, Workspace* ws, const Mode& md, int kind, int spine, int replaced) {
  spmv_launch(L, ws->X.v[VR], epi_dots(ws, md, spine, 1, replaced), 0, ws->n, kind);
  if (md.plan) finalize(L, ws, plan_dots(L, ws, KD), 1, replaced);
}

// ---- PartitionPlan chains over arbitrary pairs (plan mode of the comparators)
static inline int plan_pairs(Launcher& L, Workspace* ws, const DotPairs& P) {
  dots_pairs_plan_kernel<<<ws->plan_w_actual, 32, 0, L.s>>>(ws->plan_bounds, P, ws->partials, ws->st);
  L.done(KD);
  return ws->plan_w_actual;
}

static inline DotPairs pairs_of(unsigned mask, const double* const* x, const double* const* y) {
  DotPairs P{};
  P.mask = mask;
  for (int k = 0; k < kNumDots; ++k) {
    P.x[k] = x[k];
    P.y[k] = y[k];
  }
  return P;
}

typedef void (*IterFn)(Launcher&, Workspace*, const Mode&);

// steady iterations per graph (PBS_GRAPH_ITERS, default 4): inside one graph
// K3 -> next K12 is a programmatic edge too, so the next iteration's matrix
// stream starts while the check tail runs
static inline int graph_iters() {
  static int v = env_int("PBS_GRAPH_ITERS", 4, 1, 16);
  return v;
}

// ---- core.cu
int get_graph(pbs_ctx* ctx, pbs_mat* m, long long key, IterFn fn, const Mode& md, cudaGraphExec_t* out,
              long long* nkernels);
int validate_cfg(pbs_ctx* ctx, const pbs_config* cfg);
int collect_result(pbs_mat* m, int method, const pbs_config* cfg, pbs_result* res, Launcher& L,
                   std::vector<std::pair<int, cudaEvent_t>>& marks, long long launched_graph_kernels);
int copy_history(pbs_mat* m, const pbs_result* res, double* hist_rel, uint8_t* hist_flags, double* hist_coef);

// ---- solve.cu: runs a solve with b / x0 already in the workspace (VB, VX)
int run_solve(pbs_mat* m, int method, const pbs_config* cfg, pbs_result* res);

// ---- prod.cu: the product-type comparators' schedules
void setup_prod(Launcher& L, Workspace* ws, const Mode& md);
void iter_stab(Launcher& L, Workspace* ws, const Mode& md);
void iter_gp(Launcher& L, Workspace* ws, const Mode& md);
void setup_pstab(Launcher& L, Workspace* ws, const Mode& md);
void iter_pstab(Launcher& L, Workspace* ws, const Mode& md);
void iter_stab_batch(Launcher& L, Workspace* ws, const Mode& md);
void iter_gp_batch(Launcher& L, Workspace* ws, const Mode& md);
void iter_pstab_batch(Launcher& L, Workspace* ws, const Mode& md);

// ---- dist.cu: the multi-GPU schedule of a partitioned operator
int run_solve_dist(pbs_mat* m, int method, const pbs_config* cfg, pbs_result* res);
