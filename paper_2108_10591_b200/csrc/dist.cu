// dist.cu — the multi-GPU row-partitioned schedule.
//
// The reference's only parallelism is a row partition: PartitionPlan ranges
// (reduction.py:55-87), row-range SpMV (linalg.py:164-172) and one combine of
// per-range dot partials per batch (reduction.py:282-294).  Here each range
// is a partition of the system on its own GPU (one process per GPU), or — the
// loopback group — N partitions of one system in one process on one GPU,
// which runs the identical schedule, kernels and transport so the N-partition
// path is exercised (and held to the oracle) on a single device.
//
// Transport (PBS_TRANSPORT_P2P, the default): no SM does communication.
//  * halo: the owner of a boundary slice pushes it straight into the
//    neighbour's extended-space vector (CUDA-IPC-mapped peer memory) with one
//    cudaMemcpyAsync per face on a halo stream — the copy engines move it over
//    NVLink — and raises the neighbour's arrival flag with a stream memory op;
//    the neighbour's compute stream waits on that flag (front-end wait, no
//    SM) before its boundary rows, and hands the halo back with a "freed"
//    flag once the SpMV that reads it is issued;
//  * the one reduction per iteration: a 1-CTA publish kernel reduces the
//    partition's CTA records to 9 compensated pairs and stores them into a
//    slot of every peer's mailbox (peer stores over NVLink), then raises the
//    peer's flag (release.sys); each partition's comm stream waits on all
//    flags and runs the check on the records in rank order, so every
//    partition computes bitwise the same coefficients and stops at the same
//    check.  Slots and flags alternate between two parities.
// Flags are 0/1 toggles (wait == 1, reset to 0): the value a wait expects does
// not depend on the iteration, and every partition's flags return to their
// initial state at the end of a solve.
//
// PBS_TRANSPORT_NCCL keeps the previous transport (grouped ncclSend/Recv on
// the halo stream, ncclAllGather of the pairs on the comm stream); it needs
// one process per GPU.
//
// Per steady p-BiCGSafe iteration j on every partition (S = compute stream,
// H = halo stream, C = comm stream):
//   H: push s                          | C: (check j: publish -> wait flags ->
//   S: K1 As = A s: interior rows,     |     finalize, overlapping K1)
//      wait s halo, boundary rows      |
//   S: wait coefficients(j); K2 (p u w t z y x r) + dots b e f h r of check j+1
//   H: push w
//   S: K3 Aw: interior, wait w halo, boundary; l g s + dots a c d g
//   C: publish check j+1 ; wait every partition's flag ; finalize check j+1
// The check's reduction runs on C while S computes the next A s: the
// pipelined method's single reduction hides behind one SpMV.
//
// Stopping: every partition's device state is identical (same records, same
// check), so the host stops issuing deterministically: before iteration j it
// waits until check j - lag is done and stops if the solve stopped at a check
// <= j - lag.  No agreement collective, no per-chunk host sync.  A non-finite
// SpMV output on one partition rides the reduction as an error flag, so every
// partition stops at the same check.
#include <cuda.h>  // stream memory-op flags; the entry points come from cudaGetDriverEntryPoint
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is loaded at run time

#include <chrono>
#include <functional>

#include "host.h"

constexpr int kMaxRanks = 64;
// a partition's record: 9 compensated pairs, then its first non-finite SpMV
// output (encoded tag + 1, or 0) and that output's global row
constexpr int kRecStride = kPartStride + 2;
// schedule-evidence stamps per iteration i (globaltimer ns): the As product of
// iteration i, its Aw product, and the reduction of check i (publish, then the
// finalize that waits for every partition's record)
enum { kStK1 = 0, kStK3 = 2, kStPub = 4, kStFin = 6, kStampWords = 8 };

// Mailbox of one partition (device memory, IPC-exported): peers write into it.
struct Mailbox {
  unsigned int arrived[kNumVecs][kMaxRanks];  // halo of vector k from peer q landed (toggle)
  unsigned int freed[kNumVecs][kMaxRanks];    // peer q has consumed my push of vector k (toggle, starts 1)
  unsigned int red[2][kMaxRanks];             // record of peer q is in slots[parity][q] (toggle)
  double slots[2][kMaxRanks][kRecStride];
};

// ---- stream memory operations (driver API, resolved at run time)
struct MemOps {
  bool tried = false, ok = false, flush = false;
  std::string err;
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
};

static MemOps& memops(int device) {
  static MemOps m;
  if (m.tried) return m;
  m.tried = true;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", (void**)&m.wait32, 12000, cudaEnableDefault, &q) !=
          cudaSuccess ||
      q != cudaDriverEntryPointSuccess ||
      cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", (void**)&m.write32, 12000, cudaEnableDefault, &q) !=
          cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    m.err = "cuStreamWaitValue32 / cuStreamWriteValue32 unavailable";
    return m;
  }
  int fl = 0;
  cudaDeviceGetAttribute(&fl, cudaDevAttrCanFlushRemoteWrites, device);
  m.flush = fl != 0;
  m.ok = true;
  return m;
}

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
#define PBS_SYM(field, sym)                                         \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, sym)); \
  if (!api.field) {                                                 \
    api.err = std::string("libnccl lacks ") + sym;                  \
    return api;                                                     \
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

// A peer partition as seen from this one.
struct PeerLink {
  double* base = nullptr;  // its workspace base (extended space), mapped here
  long long stride = 0;    // its elements per workspace vector
  Mailbox* mbox = nullptr;
  bool ipc = false;  // opened with cudaIpcOpenMemHandle (closed on destroy)
};

struct pbs_dist {
  pbs_ctx* ctx = nullptr;
  int nranks = 1, rank = 0;
  int transport = PBS_TRANSPORT_P2P;
  pbs_mat* mat = nullptr;  // the partition this link carries (pbs_mat_set_partition)
  cudaStream_t s = nullptr;        // compute (S)
  cudaStream_t comm = nullptr;     // reduction (C): publish, flag waits, finalize
  cudaStream_t hstream = nullptr;  // halo pushes (H)
  cudaEvent_t ev_vec = nullptr, ev_k3 = nullptr, ev_coef = nullptr, ev_halo = nullptr;
  Mailbox* mbox = nullptr;
  std::vector<PeerLink> peers;
  bool connected = false;
  int sm_limit = 0;  // SMs this partition's kernels may fill (0: all)
  int parity = 0;    // reduction slot parity of the next publish
  // NCCL transport
  ncclComm_t halo = nullptr, red = nullptr;
  double* sendbuf = nullptr;
  double* recvbuf = nullptr;
};

// ================================================================ kernels

// K2 of the multi-GPU schedule: block 1 of the iteration (solvers.py:678-701,
// 715), with the five dots of check j+1 that do not need the new s
// (b=(y,y) e=(y,r) f=(r0s,r) h=(r0s,t) r=(r,r), solvers.py:471-481) in the
// same pass, so K3 carries only a c d g.  o and q stay in registers.
static __global__ void __launch_bounds__(kThreads) k2_dots_kernel(VecPtrs V, long long n, SolverState* st,
                                                                  double* parts) {
  if (!gate_after_spine(st)) return;
  const double alpha = st->alpha, beta = st->beta, zeta = st->zeta, eta = st->eta;
  double *__restrict__ x = V.v[VX], *__restrict__ r = V.v[VR], *__restrict__ p = V.v[VP],
         *__restrict__ u = V.v[VU], *__restrict__ t = V.v[VT], *__restrict__ w = V.v[VW],
         *__restrict__ y = V.v[VY], *__restrict__ z = V.v[VZ];
  const double *__restrict__ s = V.v[VS], *__restrict__ as = V.v[VAS], *__restrict__ l = V.v[VL],
               *__restrict__ g = V.v[VG], *__restrict__ r0s = V.v[VR0S];
  DotsT<kDotsK12> d;
  d.zero();
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const double rv = r[i], pv = p[i], uv = u[i], sv = s[i], tv = t[i], yv = y[i];
    const double asv = __ldcs(as + i), lv = l[i], gv = g[i], wv = w[i], zv = z[i], xv = x[i];
    const double pn = asd(rv, beta, pv, uv);               // p = r + beta*(p - u)
    const double o = lc2(1.0, sv, beta, tv);               // o = s + beta*t
    const double un = lcn(zeta, o, eta, yv, beta, uv);     // u = zeta*o + eta*(y + beta*u)
    const double q = lc2(1.0, asv, beta, lv);              // q = As + beta*l
    const double wn = lcn(zeta, q, eta, gv, beta, wv);     // w = zeta*q + eta*(g + beta*w)
    const double tn = lc2(1.0, o, -1.0, wn);               // t = o - w
    const double zn = lc3(zeta, rv, eta, zv, -alpha, un);  // z = zeta*r + eta*z - alpha*u
    const double yn = lc3(zeta, sv, eta, yv, -alpha, wn);  // y = zeta*s + eta*y - alpha*w
    const double xn = lc3(1.0, xv, alpha, pn, 1.0, zn);    // x = x + alpha*p + z
    const double rn = lc3(1.0, rv, -alpha, o, -1.0, yn);   // r = r - alpha*o - y
    p[i] = pn;
    u[i] = un;
    w[i] = wn;
    t[i] = tn;
    z[i] = zn;
    y[i] = yn;
    x[i] = xn;
    r[i] = rn;
    d.add_row(0.0, yn, rn, __ldcs(r0s + i), tn);
  }
  block_reduce9<kThreads, false, kDotsK12>(d.acc, parts + blockIdx.x);
}

// K2 for the row blocks K1 left (EpiK1opp: streamed before the coefficients
// of check j were published): block 1 of the iteration and the b e f h r
// partials of check j+1 over those rows only.  Always launched: its gate
// closes the spine once a check has stopped the solve.
static __global__ void __launch_bounds__(kThreads) k2_deferred_kernel(VecPtrs V, long long n, SolverState* st,
                                                                      const int* rows, const unsigned* count,
                                                                      double* parts) {
  if (!gate_after_spine(st)) return;
  const double alpha = st->alpha, beta = st->beta, zeta = st->zeta, eta = st->eta;
  double *__restrict__ x = V.v[VX], *__restrict__ r = V.v[VR], *__restrict__ p = V.v[VP],
         *__restrict__ u = V.v[VU], *__restrict__ t = V.v[VT], *__restrict__ w = V.v[VW],
         *__restrict__ y = V.v[VY], *__restrict__ z = V.v[VZ];
  const double *__restrict__ s = V.v[VS], *__restrict__ as = V.v[VAS], *__restrict__ l = V.v[VL],
               *__restrict__ g = V.v[VG], *__restrict__ r0s = V.v[VR0S];
  DotsT<kDotsK12> d;
  d.zero();
  const unsigned nb = *count;
  for (unsigned b = blockIdx.x; b < nb; b += gridDim.x) {
    const long long i = (long long)rows[b] + threadIdx.x;
    if (i >= n) continue;
    const double rv = r[i], pv = p[i], uv = u[i], sv = s[i], tv = t[i], yv = y[i];
    const double asv = __ldcs(as + i), lv = l[i], gv = g[i], wv = w[i], zv = z[i], xv = x[i];
    const double pn = asd(rv, beta, pv, uv);
    const double o = lc2(1.0, sv, beta, tv);
    const double un = lcn(zeta, o, eta, yv, beta, uv);
    const double q = lc2(1.0, asv, beta, lv);
    const double wn = lcn(zeta, q, eta, gv, beta, wv);
    const double tn = lc2(1.0, o, -1.0, wn);
    const double zn = lc3(zeta, rv, eta, zv, -alpha, un);
    const double yn = lc3(zeta, sv, eta, yv, -alpha, wn);
    const double xn = lc3(1.0, xv, alpha, pn, 1.0, zn);
    const double rn = lc3(1.0, rv, -alpha, o, -1.0, yn);
    p[i] = pn;
    u[i] = un;
    w[i] = wn;
    t[i] = tn;
    z[i] = zn;
    y[i] = yn;
    x[i] = xn;
    r[i] = rn;
    d.add_row(0.0, yn, rn, __ldcs(r0s + i), tn);
  }
  block_reduce9<kThreads, false, kDotsK12>(d.acc, parts + blockIdx.x);
}

// Where a publish stores this partition's record: one slot and one flag per
// partition of the group (peer mappings; its own mailbox included).
struct PubTargets {
  double* slot[kMaxRanks];
  unsigned int* flag[kMaxRanks];
  int n;
};

// The partition's contribution to check j: its CTA records (partials: the
// dots not in mask2, field-major; partials2: the dots in mask2) reduced to 9
// compensated pairs, plus its error flag, stored into every partition's slot,
// then every partition's flag raised (release at system scope).
static __device__ __forceinline__ void record_error(const SolverState* st, long long row_lo, double* out) {
  if (dev_err(st)) {
    out[0] = (double)st->nf_tag + 1.0;
    out[1] = (double)(row_lo + (long long)st->nf_row);
  } else {
    out[0] = 0.0;
    out[1] = -1.0;
  }
}

static __global__ void __launch_bounds__(288) publish_kernel(const double* partials, int np, const double* partials2,
                                                             int np2, unsigned mask2, const SolverState* st,
                                                             long long row_lo, const __grid_constant__ PubTargets T,
                                                             unsigned long long* stamp) {
  constexpr int TM = 288 / kNumDots;
  __shared__ Ddbl team[kNumDots][TM];
  __shared__ double rec[kRecStride];
  const int t = threadIdx.x;
  if (stamp && t == 0) stamp[0] = gtime();
  {
    const int j = t / TM, l = t % TM;
    if (j < kNumDots) {
      const bool second = (mask2 >> j) & 1u;
      const double* src = (second ? partials2 : partials) + (size_t)(2 * j) * kMaxParts;
      const int n = second ? np2 : np;
      Ddbl acc{0.0, 0.0};
      for (int b = l; b < n; b += TM) acc = dd_add(acc, Ddbl{__ldcg(src + b), __ldcg(src + kMaxParts + b)});
      team[j][l] = acc;
    }
  }
  __syncthreads();
  if (t < kNumDots) {
    Ddbl acc = team[t][0];
    for (int k = 1; k < TM; ++k) acc = dd_add(acc, team[t][k]);
    rec[2 * t] = acc.hi;
    rec[2 * t + 1] = acc.lo;
  } else if (t == kNumDots) {
    record_error(st, row_lo, rec + kPartStride);
  }
  __syncthreads();
  for (int e = t; e < T.n * kRecStride; e += 288) T.slot[e / kRecStride][e % kRecStride] = rec[e % kRecStride];
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  __syncthreads();
  if (t < T.n) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(T.flag[t]), "r"(1u) : "memory");
  if (stamp && t == 0) stamp[1] = gtime();
}

// Check j on every partition's record (rank order, fixed-shape compensated
// sum: every partition computes bitwise the same dots), then the host mirror:
// stop_check, run_all, err, a system fence, iter.  A record with the error
// flag stops the solve on every partition at this check.
static __global__ void __launch_bounds__(288) dist_finalize_kernel(SolverState* st, const double* recs, int nranks,
                                                                   int replaced, unsigned long long* stamp) {
  __shared__ double dots[kNumDots];
  __shared__ SolverState ss;
  __shared__ int any_err;
  if (stamp && threadIdx.x == 0) stamp[0] = gtime();
  state_load<288>(st, &ss);
  // the group's first non-finite SpMV output: the earliest launch (the
  // encoded tag carries the launch sequence), then the lowest global row —
  // what the reference's check_finite after that SpMV would name
  __shared__ double err_tag, err_row;
  if (threadIdx.x == 0) {
    int e = 0;
    double bt = 0.0, br = -1.0;
    for (int q = 0; q < nranks; ++q) {
      const double tg = __ldcg(recs + (size_t)q * kRecStride + kPartStride);
      const double rw = __ldcg(recs + (size_t)q * kRecStride + kPartStride + 1);
      if (tg != 0.0 && (!e || tg < bt || (tg == bt && rw < br))) {
        bt = tg;
        br = rw;
        e = 1;
      }
    }
    any_err = e;
    err_tag = bt;
    err_row = br;
  }
  reduce_parts<288, false>(recs, nranks, 0, dots, nullptr, 0, 0u, kRecStride, 1);  // ends with a barrier
  HostMirror* mirror = ss.mirror;
  __syncthreads();
  if (threadIdx.x == 0) ss.mirror = nullptr;  // the mirror is written below, in order
  __syncthreads();
  if (any_err) {
    if (threadIdx.x == 0) {
      const long long j = ss.iter;
      if (ss.run_all && ss.stop_check < 0) ss.stop_check = j;
      ss.run_all = 0;
      ss.run_spine = 0;
      ss.iter = j + 1;
      state_store(st, &ss);
      st->remote_err = 1;
      st->err_tag = (int)(err_tag - 1.0);
      st->err_row = (long long)err_row;
    }
  } else {
    check_and_publish<288, false>(st, &ss, dots, replaced);
  }
  if (threadIdx.x != 0) return;
  // the coefficients of this check are in the state: let K1's opportunistic
  // epilogue use them
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&st->coef_epoch), "l"((unsigned long long)ss.iter)
               : "memory");
  if (mirror) {
    mirror->stop_check = ss.stop_check;
    mirror->run_all = ss.run_all;
    mirror->err = dev_err(&ss) || any_err ? 1 : 0;
    __threadfence_system();
    mirror->iter = ss.iter;
  }
  if (stamp) stamp[1] = gtime();
}

// NCCL transport: this partition's record (pairs + error flag) into sendbuf
static __global__ void __launch_bounds__(288) pack_record_kernel(const double* partials, int np,
                                                                 const double* partials2, int np2, unsigned mask2,
                                                                 const SolverState* st, long long row_lo,
                                                                 double* out, unsigned long long* stamp) {
  constexpr int TM = 288 / kNumDots;
  __shared__ Ddbl team[kNumDots][TM];
  const int t = threadIdx.x;
  if (stamp && t == 0) stamp[0] = gtime();
  const int j = t / TM, l = t % TM;
  if (j < kNumDots) {
    const bool second = (mask2 >> j) & 1u;
    const double* src = (second ? partials2 : partials) + (size_t)(2 * j) * kMaxParts;
    const int n = second ? np2 : np;
    Ddbl acc{0.0, 0.0};
    for (int b = l; b < n; b += TM) acc = dd_add(acc, Ddbl{__ldcg(src + b), __ldcg(src + kMaxParts + b)});
    team[j][l] = acc;
  }
  __syncthreads();
  if (t < kNumDots) {
    Ddbl acc = team[t][0];
    for (int k = 1; k < TM; ++k) acc = dd_add(acc, team[t][k]);
    out[2 * t] = acc.hi;
    out[2 * t + 1] = acc.lo;
  } else if (t == kNumDots) {
    record_error(st, row_lo, out + kPartStride);
  }
  if (stamp && t == 0) stamp[1] = gtime();
}

// ======================================================= partitions in a solve

struct Part {
  pbs_mat* m = nullptr;
  Workspace* ws = nullptr;
  pbs_dist* D = nullptr;
  Launcher L{nullptr, nullptr, nullptr};
  std::vector<int> send_peers, recv_peers;  // distinct peers
  int np = 0, np2 = 0;                      // records of the next publish
  int seq = 0;                              // SpMV launch sequence (identical on every partition)
  int* defer_rows = nullptr;                // EpiK1opp: blocks left to k2_deferred_kernel, and their count
  unsigned* defer_count = nullptr;
  // records of the dots b e f h r, by iteration parity: K1 of iteration j+1
  // (EpiK1opp) writes its records while the publish of check j+1 still
  // reads those of iteration j
  double* p12buf[2] = {nullptr, nullptr};
  double* p12 = nullptr;
  unsigned long long* stamps = nullptr;     // device [cap][kStampWords]
  long long stamps_cap = 0;
  Part() = default;
};

static unsigned long long* stamp_at(Part& P, long long i, int word) {
  if (!P.stamps || i < 0 || i >= P.stamps_cap) return nullptr;
  return P.stamps + (size_t)i * kStampWords + word;
}

static int eff_sms(const Part& P) { return P.D->sm_limit > 0 ? P.D->sm_limit : P.D->ctx->sms; }

static void mo_wait(Part& P, cudaStream_t s, unsigned int* addr) {
  if (P.L.err) return;
  MemOps& mo = memops(P.D->ctx->device);
  unsigned fl = CU_STREAM_WAIT_VALUE_EQ | (mo.flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
  if (mo.wait32((CUstream)s, (CUdeviceptr)addr, 1u, fl) != CUDA_SUCCESS)
    P.L.err = set_err(P.D->ctx, PBS_ERR_CUDA, "cuStreamWaitValue32 failed");
}

static void mo_write(Part& P, cudaStream_t s, unsigned int* addr, unsigned v) {
  if (P.L.err) return;
  if (memops(P.D->ctx->device).write32((CUstream)s, (CUdeviceptr)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS)
    P.L.err = set_err(P.D->ctx, PBS_ERR_CUDA, "cuStreamWriteValue32 failed");
}

static bool has_halo(const Part& P) { return !P.m->part.sends.empty() || !P.m->part.recvs.empty(); }

// S -> H: vector k is final on S; push its boundary slices into the
// neighbours' halos (copy engines), then raise their arrival flags.
static void push(Part& P, int k) {
  pbs_dist* D = P.D;
  Partition& Pt = P.m->part;
  if (P.L.err || !has_halo(P)) return;
  cudaEventRecord(D->ev_vec, D->s);
  cudaStreamWaitEvent(D->hstream, D->ev_vec, 0);
  if (D->transport == PBS_TRANSPORT_NCCL) {
    NcclApi& A = nccl();
    ncclResult_t r = A.GroupStart();
    for (size_t i = 0; r == ncclSuccess && i < Pt.recvs.size(); i += 3)
      r = A.Recv(P.ws->X.v[k] + Pt.recvs[i + 1], (size_t)Pt.recvs[i + 2], ncclDouble, (int)Pt.recvs[i], D->halo,
                 D->hstream);
    for (size_t i = 0; r == ncclSuccess && i < Pt.sends.size(); i += 4)
      r = A.Send(P.ws->V.v[k] + Pt.sends[i + 1], (size_t)Pt.sends[i + 2], ncclDouble, (int)Pt.sends[i], D->halo,
                 D->hstream);
    ncclResult_t r2 = A.GroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) P.L.err = set_err(D->ctx, PBS_ERR_NCCL, std::string("halo exchange: ") + A.GetErrorString(r));
    cudaEventRecord(D->ev_halo, D->hstream);
    return;
  }
  for (int q : P.send_peers) {
    mo_wait(P, D->hstream, &D->mbox->freed[k][q]);  // the neighbour is done with my previous push
    mo_write(P, D->hstream, &D->mbox->freed[k][q], 0u);
  }
  for (size_t i = 0; i < Pt.sends.size() && !P.L.err; i += 4) {
    const int q = (int)Pt.sends[i];
    const PeerLink& pl = D->peers[q];
    double* dst = pl.base + (size_t)pl.stride * k + Pt.sends[i + 3];
    const double* src = P.ws->V.v[k] + Pt.sends[i + 1];
    if (cudaMemcpyAsync(dst, src, sizeof(double) * Pt.sends[i + 2], cudaMemcpyDeviceToDevice, D->hstream) !=
        cudaSuccess)
      P.L.err = set_err(D->ctx, PBS_ERR_CUDA, "halo copy failed");
  }
  for (int q : P.send_peers) mo_write(P, D->hstream, &D->peers[q].mbox->arrived[k][D->rank], 1u);
}

// S: wait until every halo slice of vector k has landed
static void arrive(Part& P, int k) {
  pbs_dist* D = P.D;
  if (P.L.err || P.m->part.recvs.empty()) return;
  if (D->transport == PBS_TRANSPORT_NCCL) {
    cudaStreamWaitEvent(D->s, D->ev_halo, 0);
    return;
  }
  for (int q : P.recv_peers) {
    mo_wait(P, D->s, &D->mbox->arrived[k][q]);
    mo_write(P, D->s, &D->mbox->arrived[k][q], 0u);
  }
}

// S: the SpMV that reads the halo of vector k is issued; once it has run, the
// senders may overwrite the halo again
static void release(Part& P, int k) {
  pbs_dist* D = P.D;
  if (P.L.err || D->transport == PBS_TRANSPORT_NCCL) return;
  for (int q : P.recv_peers) mo_write(P, D->s, &D->peers[q].mbox->freed[k][D->rank], 1u);
}

// SpMV of vector k (epilogue factory mk(partial_offset)) over the partition's
// rows.  With Partition::split the interior rows [L0, L1) run before the
// halo wait, the boundary rows after it; dot records of the pieces are stored
// one after another (each launch capped so they fit the record buffer).
template <class MakeEpi>
static int halo_spmv(Part& P, int k, int kind, MakeEpi mk0) {
  Partition& Pt = P.m->part;
  Launcher& L = P.L;
  const long long n = P.ws->n;
  const double* x = P.m->stencil ? P.ws->V.v[k] : P.ws->X.v[k];  // stencils address x from the own segment
  // tag the non-finite reports with this SpMV's place in the schedule, so the
  // group can name the first one (a neighbour's NaN halo fails later SpMVs)
  const int seq = ++P.seq;
  auto mk = [&](int off) {
    auto e = mk0(off);
    if (e.tag & 0xff) e.tag = (e.tag & 0xff) | (seq << 8);
    return e;
  };
  if (Pt.recvs.empty()) return spmv_launch(L, x, mk(0), 0, n, kind);
  if (!Pt.split) {
    arrive(P, k);
    const int np = spmv_launch(L, x, mk(0), 0, n, kind);
    release(P, k);
    return np;
  }
  int np = spmv_launch(L, x, mk(0), Pt.L0, Pt.L1, kind);
  arrive(P, k);
  for (int piece = 0; piece < 2 && !L.err; ++piece) {
    const long long lo = piece == 0 ? 0 : Pt.L1, hi = piece == 0 ? Pt.L0 : n;
    if (hi <= lo) continue;
    if (np >= kMaxParts) {
      L.err = set_err(P.D->ctx, PBS_ERR_INVALID, "boundary SpMV pieces exceed the partial-record buffer");
      break;
    }
    L.grid_cap = kMaxParts - np;
    np += spmv_launch(L, x, mk(np), lo, hi, kind);
    L.grid_cap = 0;
  }
  release(P, k);
  return np;
}

// C: publish this partition's record of check i (after ev_k3 on S)
static void publish(Part& P, long long i) {
  pbs_dist* D = P.D;
  if (P.L.err) return;
  cudaEventRecord(D->ev_k3, D->s);
  cudaStreamWaitEvent(D->comm, D->ev_k3, 0);
  const unsigned mask2 = P.np2 ? kDotsK12 : 0u;
  if (D->transport == PBS_TRANSPORT_NCCL) {
    pack_record_kernel<<<1, 288, 0, D->comm>>>(P.ws->partials, P.np, P.p12, P.np2, mask2, P.ws->st,
                                               P.m->part.row_lo, D->sendbuf, stamp_at(P, i, kStPub));
  } else {
    PubTargets T;
    T.n = D->nranks;
    for (int q = 0; q < D->nranks; ++q) {
      T.slot[q] = &D->peers[q].mbox->slots[D->parity][D->rank][0];
      T.flag[q] = &D->peers[q].mbox->red[D->parity][D->rank];
    }
    publish_kernel<<<1, 288, 0, D->comm>>>(P.ws->partials, P.np, P.p12, P.np2, mask2, P.ws->st,
                                           P.m->part.row_lo, T, stamp_at(P, i, kStPub));
  }
  P.L.done(KD);
}

// C: wait for every partition's record of check i, run the check, and let S
// go on (ev_coef)
static void finalize_dist(Part& P, long long i, int replaced) {
  pbs_dist* D = P.D;
  if (P.L.err) return;
  const double* recs;
  if (D->transport == PBS_TRANSPORT_NCCL) {
    ncclResult_t r = nccl().AllGather(D->sendbuf, D->recvbuf, kRecStride, ncclDouble, D->red, D->comm);
    if (r != ncclSuccess) {
      P.L.err = set_err(D->ctx, PBS_ERR_NCCL, std::string("all-gather: ") + nccl().GetErrorString(r));
      return;
    }
    recs = D->recvbuf;
  } else {
    for (int q = 0; q < D->nranks; ++q) {
      mo_wait(P, D->comm, &D->mbox->red[D->parity][q]);
      mo_write(P, D->comm, &D->mbox->red[D->parity][q], 0u);
    }
    recs = &D->mbox->slots[D->parity][0][0];
    D->parity ^= 1;
  }
  dist_finalize_kernel<<<1, 288, 0, D->comm>>>(P.ws->st, recs, D->nranks, replaced, stamp_at(P, i, kStFin));
  P.L.done(KF);
  cudaEventRecord(D->ev_coef, D->comm);
}

static EpiStore epi_store_st(Workspace* ws, int out, int tag, int spine, unsigned long long* stamp) {
  EpiStore e = epi_store(ws, out, tag, spine);
  e.stamp = stamp;
  return e;
}

static EpiDots epi_dots_parts(Workspace* ws, int spine, int off) {
  Mode md;
  EpiDots e = epi_dots(ws, md, spine, 0, 0);
  e.sink.partials = ws->partials + off;
  e.sink.fuse = 0;
  return e;
}

// ------------------------------------------------------ the steps of a solve
// Every wait a step issues is for a signal an earlier step issued (on any
// partition), so issuing the steps step-major over the partitions of a
// loopback group can never queue a wait ahead of the signal it needs.

typedef std::function<void(Part&)> Step;

static void run_steps(std::vector<Part>& parts, const std::vector<Step>& steps) {
  for (const Step& st : steps)
    for (Part& P : parts) {
      if (P.L.err) return;
      st(P);
    }
}

// K1 fuses block 1 opportunistically (EpiK1opp) on large CSR slabs: the
// reduction (~25 us) then covers a small share of K1 and the K2 pass mostly
// disappears (config 4 partitioned, N = 1: 98.6 -> 102.7 it/s).  On small
// slabs a third of the blocks stream before the coefficients exist and the
// fused epilogue's register pressure costs more than the K2 pass it saves
// (config 2, N = 1: 5434 -> 4870 it/s), so they keep the plain product.
// Stencil operators keep it too.  PBS_K1_OPP=0|1 forces either.
static bool k1_opp(const Part& P) {
  static int forced = env_int("PBS_K1_OPP", -1, -1, 1);
  if (P.m->stencil || csr_engine_tpr() || forced == 0) return false;
  return forced == 1 || P.m->nnz >= (64LL << 20);
}

static void k1_step(Part& P, long long j, bool fuse) {
  // room for the comm stream's 1-CTA publish / finalize beside K1: one SM
  // for the persistent staged engines, one CTA slot per SM for the rest
  P.L.sm_limit = eff_sms(P) - 1;
  if (P.L.sm_limit < 1) P.L.sm_limit = 1;
  P.L.leave_room = true;
  P.p12 = P.p12buf[j & 1];
  if (fuse && k1_opp(P)) {
    if (cudaMemsetAsync(P.defer_count, 0, sizeof(unsigned), P.D->s) != cudaSuccess)
      P.L.err = set_err(P.D->ctx, PBS_ERR_CUDA, "defer list reset failed");
    Mode md;
    P.np2 = halo_spmv(P, VS, KK1, [&](int off) {
      EpiK1opp e = epi_k12_fill<EpiK1opp>(P.ws, md);
      e.parts = P.p12 + off;
      e.stamp = stamp_at(P, j, kStK1);
      e.want = (unsigned long long)(j + 1);  // check j's coefficients
      e.defer_rows = P.defer_rows;
      e.defer_count = P.defer_count;
      e.tag = PBS_TAG_AS;
      return e;
    });
  } else {
    halo_spmv(P, VS, KK1, [&](int) { return epi_store_st(P.ws, VAS, PBS_TAG_AS, 1, stamp_at(P, j, kStK1)); });
  }
  P.L.sm_limit = eff_sms(P);
  P.L.leave_room = false;
}

// setup (solvers.py:612-631): r0 = b - A x0, r0s = r0; the pipelined methods
// also s0 = A r0 with the batch of check 0
static void setup_steps(std::vector<Step>& st, bool pipelined) {
  st.push_back([](Part& P) { push(P, VX); });
  st.push_back([](Part& P) { halo_spmv(P, VX, KS, [&](int) { return epi_resid(P.ws, true); }); });
  if (!pipelined) return;
  st.push_back([](Part& P) { push(P, VR); });
  st.push_back([](Part& P) {
    P.np = halo_spmv(P, VR, KS, [&](int off) { return epi_dots_parts(P.ws, 0, off); });
    P.np2 = 0;
  });
  st.push_back([](Part& P) { publish(P, 0); });
  st.push_back([](Part& P) { finalize_dist(P, 0, 0); });
}

// one p-BiCGSafe(-rr) iteration j (solvers.py:639-734); its batch is check j+1
static void iter_steps(std::vector<Step>& st, long long j, bool replace) {
  st.push_back([](Part& P) { push(P, VS); });
  st.push_back([j, replace](Part& P) { k1_step(P, j, !replace); });
  if (!replace) {
    st.push_back([](Part& P) {
      cudaStreamWaitEvent(P.D->s, P.D->ev_coef, 0);  // coefficients of check j
      Launcher& L = P.L;
      const long long nblk = (P.ws->n + kThreads - 1) / kThreads;
      if (k1_opp(P)) {  // only the blocks K1 left
        if (P.np2 >= kMaxParts) {
          L.err = set_err(P.D->ctx, PBS_ERR_INVALID, "K1 records fill the partial-record buffer");
          return;
        }
        L.grid_cap = kMaxParts - P.np2;
        const int g = L.cap_grid(grid_for(L.ctx, (const void*)k2_deferred_kernel, nblk, 2, L.sms()));
        L.grid_cap = 0;
        k2_deferred_kernel<<<g, kThreads, 0, L.s>>>(P.ws->V, P.ws->n, P.ws->st, P.defer_rows, P.defer_count,
                                                    P.p12 + P.np2);
        P.np2 += g;
      } else {
        P.np2 = L.cap_grid(grid_for(L.ctx, (const void*)k2_dots_kernel, nblk, 8, L.sms()));
        k2_dots_kernel<<<P.np2, kThreads, 0, L.s>>>(P.ws->V, P.ws->n, P.ws->st, P.p12);
      }
      L.done(KK2);
    });
    st.push_back([](Part& P) { push(P, VW); });
    st.push_back([j](Part& P) {
      Mode md;
      P.np = halo_spmv(P, VW, KK3, [&](int off) {
        EpiK3s e = epi_k3s(P.ws, md, 0, 0);
        e.sink.partials = P.ws->partials + off;
        e.sink.partials2 = nullptr;
        e.sink.nparts2 = 0;
        e.stamp = stamp_at(P, j, kStK3);
        return e;
      });
    });
  } else {  // residual replacement (solvers.py:676-713)
    st.push_back([](Part& P) {
      cudaStreamWaitEvent(P.D->s, P.D->ev_coef, 0);
      vec_launch(P.L, pou_kernel, P.ws->n, KR, P.ws->V, P.ws->n, P.ws->st);
    });
    struct RS {
      int in, out, tag;
    };
    for (RS r : {RS{VO, VQ, PBS_TAG_AO}, RS{VU, VW, PBS_TAG_AU}}) {
      st.push_back([r](Part& P) { push(P, r.in); });
      st.push_back([r](Part& P) {
        halo_spmv(P, r.in, KRS, [&](int) { return epi_store(P.ws, r.out, r.tag, 0); });
      });
    }
    st.push_back([](Part& P) { vec_launch(P.L, tzyx_kernel, P.ws->n, KR, P.ws->V, P.ws->n, P.ws->st); });
    st.push_back([](Part& P) { push(P, VX); });
    st.push_back([](Part& P) { halo_spmv(P, VX, KRS, [&](int) { return epi_resid(P.ws, false); }); });
    for (RS r : {RS{VT, VL, PBS_TAG_AT}, RS{VY, VG, PBS_TAG_AY}}) {
      st.push_back([r](Part& P) { push(P, r.in); });
      st.push_back([r](Part& P) {
        halo_spmv(P, r.in, KRS, [&](int) { return epi_store(P.ws, r.out, r.tag, 0); });
      });
    }
    st.push_back([](Part& P) { push(P, VR); });
    st.push_back([](Part& P) {
      P.np = halo_spmv(P, VR, KRS, [&](int off) { return epi_dots_parts(P.ws, 0, off); });
    });
  }
  st.push_back([replace](Part& P) {
    if (replace) P.np2 = 0;
  });
  st.push_back([j](Part& P) { publish(P, j + 1); });
  st.push_back([j, replace](Part& P) { finalize_dist(P, j + 1, replace ? 1 : 0); });
}

// one ssBiCGSafe2 iteration j (solvers.py:528-587): s = A r + batch -> check j
// (the reduction follows its producer: nothing to hide it behind), then
// p o u, then w = A u + t z y x r
static void ss_iter_steps(std::vector<Step>& st, long long j) {
  st.push_back([](Part& P) { push(P, VR); });
  st.push_back([j](Part& P) {
    P.np = halo_spmv(P, VR, KK1, [&](int off) {
      EpiDots e = epi_dots_parts(P.ws, 1, off);
      e.stamp = stamp_at(P, j, kStK1);  // the spine product (A r) in the As slot
      return e;
    });
    P.np2 = 0;
  });
  st.push_back([j](Part& P) { publish(P, j); });
  st.push_back([j](Part& P) { finalize_dist(P, j, 0); });
  st.push_back([](Part& P) {
    cudaStreamWaitEvent(P.D->s, P.D->ev_coef, 0);
    vec_launch(P.L, pou_kernel, P.ws->n, KK2, P.ws->V, P.ws->n, P.ws->st);
  });
  st.push_back([](Part& P) { push(P, VU); });
  st.push_back([](Part& P) { halo_spmv(P, VU, KK3, [&](int) { return epi_ss3(P.ws); }); });
}

// ssBiCGSafe2's record after max_iters: plan_dot(r, r) (solvers.py:589)
static void ss_final_steps(std::vector<Step>& st, long long j) {
  st.push_back([](Part& P) {
    Launcher& L = P.L;
    auto& V = P.ws->V.v;
    const long long nblk = (P.ws->n + kThreads - 1) / kThreads;
    P.np = L.cap_grid(grid_for(L.ctx, (const void*)dots9_tree_kernel, nblk, 8, L.sms()));
    dots9_tree_kernel<<<P.np, kThreads, 0, L.s>>>(P.ws->n, V[VS], V[VY], V[VR], V[VR0S], V[VT], P.ws->partials,
                                                  P.ws->st);
    L.done(KD);
    P.np2 = 0;
  });
  st.push_back([j](Part& P) { publish(P, j); });
  st.push_back([j](Part& P) { finalize_dist(P, j, 0); });
}

// =============================================================== group solve

static int init_part(Part& P, pbs_mat* m, const pbs_config* cfg, int method) {
  pbs_ctx* ctx = m->ctx;
  P.m = m;
  P.D = m->part.dist;
  pbs_dist* D = P.D;
  if (!D || !D->connected) return set_err(ctx, PBS_ERR_INVALID, "partition is not connected to its group");
  int rc = ensure_ws(m, cfg->max_iters + 1);
  if (rc) return rc;
  P.ws = m->ws;
  Workspace* ws = P.ws;
  P.L = Launcher{ctx, m, D->s};
  P.L.timing = false;
  P.L.sm_limit = eff_sms(P);
  P.send_peers.clear();
  P.recv_peers.clear();
  for (size_t i = 0; i < m->part.sends.size(); i += 4)
    if (std::find(P.send_peers.begin(), P.send_peers.end(), (int)m->part.sends[i]) == P.send_peers.end())
      P.send_peers.push_back((int)m->part.sends[i]);
  for (size_t i = 0; i < m->part.recvs.size(); i += 3)
    if (std::find(P.recv_peers.begin(), P.recv_peers.end(), (int)m->part.recvs[i]) == P.recv_peers.end())
      P.recv_peers.push_back((int)m->part.recvs[i]);
  cudaStream_t s = D->s;
  SolverState h{};
  h.tol = cfg->tol;
  h.max_iters = cfg->max_iters;
  h.record_history = cfg->record_history ? 1 : 0;
  h.spine_done = method == PBS_METHOD_SSBICGSAFE2 ? 1 : 0;
  h.run_all = 1;
  h.run_spine = 1;
  h.status = -1;
  h.failure_iter = -1;
  h.stop_check = -1;
  h.nf_row = (unsigned long long)kNoError;
  h.hist_rel = ws->hist_rel;
  h.hist_flags = ws->hist_flags;
  h.hist_coef = ws->hist_coef;
  h.mirror = ws->mirror_d;
  ws->mirror_h->iter = 0;
  ws->mirror_h->run_all = 1;
  ws->mirror_h->err = 0;
  ws->mirror_h->stop_check = -1;
  CK(cudaMemcpyAsync(ws->st, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  const int zero_slots[] = {VP, VU, VT, VY, VZ, VG, VL, VW};
  for (int k : zero_slots) CK(cudaMemsetAsync(ws->X.v[k], 0, sizeof(double) * ws->n_ext, s));
  D->parity = 0;
  P.stamps = nullptr;
  P.stamps_cap = 0;
  if (cfg->stamps_out && cfg->stamps_cap > 0) {
    P.stamps_cap = cfg->stamps_cap;
    CK(pool_alloc(ctx, &P.stamps, sizeof(unsigned long long) * kStampWords * P.stamps_cap));
    CK(cudaMemsetAsync(P.stamps, 0, sizeof(unsigned long long) * kStampWords * P.stamps_cap, s));
  }
  const long long nblk = (ws->n + kPipeRows - 1) / kPipeRows;
  CK(pool_alloc(ctx, &P.defer_rows, sizeof(int) * (nblk > 0 ? nblk : 1)));
  CK(pool_alloc(ctx, &P.defer_count, sizeof(unsigned)));
  CK(cudaMemsetAsync(P.defer_count, 0, sizeof(unsigned), s));
  P.p12buf[0] = ws->partials12;
  CK(pool_alloc(ctx, &P.p12buf[1], sizeof(double) * kMaxParts * kPartStride));
  P.p12 = P.p12buf[0];
  // the comm / halo streams start after the state is in place
  CK(cudaEventRecord(D->ev_coef, s));
  CK(cudaStreamWaitEvent(D->comm, D->ev_coef, 0));
  CK(cudaStreamWaitEvent(D->hstream, D->ev_coef, 0));
  return PBS_OK;
}

// wait until partition 0's device finished check c (mirror.iter > c)
static int wait_check(Part& P, long long c) {
  HostMirror* mh = P.ws->mirror_h;
  long long last = mh->iter;
  auto t0 = std::chrono::steady_clock::now();
  while (mh->iter <= c) {
    if (mh->err && mh->stop_check >= 0 && mh->stop_check <= c) return PBS_OK;
    cudaError_t e = cudaStreamQuery(P.D->comm);
    if (e != cudaSuccess && e != cudaErrorNotReady)
      return set_err(P.D->ctx, PBS_ERR_CUDA, std::string("device error during the solve: ") + cudaGetErrorString(e));
    const long long now = mh->iter;
    if (now != last) {
      last = now;
      t0 = std::chrono::steady_clock::now();
    } else if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
      return set_err(P.D->ctx, PBS_ERR_CUDA, "multi-GPU solve made no progress for 120 s (a peer stopped?)");
    }
    std::this_thread::yield();
  }
  return PBS_OK;
}

static int group_solve(std::vector<pbs_mat*>& mats, int method, const pbs_config* cfg, pbs_result* res) {
  pbs_ctx* ctx = mats[0]->ctx;
  const bool pipelined = method == PBS_METHOD_PBICGSAFE || method == PBS_METHOD_PBICGSAFE_RR;
  if (!pipelined && method != PBS_METHOD_SSBICGSAFE2)
    return set_err(ctx, PBS_ERR_UNSUPPORTED, "the multi-GPU schedule runs p-BiCGSafe(-rr) and ssBiCGSafe2");
  if (cfg->reduce_mode != PBS_REDUCE_TREE)
    return set_err(ctx, PBS_ERR_UNSUPPORTED, "multi-GPU solves use the compensated tree reduction");
  if (cfg->trace_fn) return set_err(ctx, PBS_ERR_UNSUPPORTED, "trace_hook is single-GPU only");
  std::vector<Part> parts(mats.size());
  for (size_t p = 0; p < mats.size(); ++p) {
    int rc = init_part(parts[p], mats[p], cfg, method);
    if (rc) return rc;
  }
  Part& P0 = parts[0];
  for (Part& P : parts) CK(cudaEventRecord(P.ws->ev0, P.D->s));
  const bool rr = method == PBS_METHOD_PBICGSAFE_RR;
  const long long cutoff = cfg->rr_cutoff >= 0 ? cfg->rr_cutoff : cfg->max_iters;
  {
    std::vector<Step> st;
    setup_steps(st, pipelined);
    run_steps(parts, st);
  }
  const long long lag = env_int("PBS_DIST_LAG", 6, 1, 64);
  long long j = 0;
  int rc = PBS_OK;
  for (; j < cfg->max_iters; ++j) {
    for (Part& P : parts)
      if (P.L.err) return P.L.err;
    if (j >= lag) {
      const long long c = j - lag;
      rc = wait_check(P0, c);
      if (rc) return rc;
      const long long sc = P0.ws->mirror_h->stop_check;
      if (sc >= 0 && sc <= c) break;  // identical on every partition and rank
    }
    std::vector<Step> st;
    if (pipelined) {
      const bool replace = rr && (j % cfg->rr_epoch == 0) && 0 < j && j < cutoff;
      iter_steps(st, j, replace);
    } else {
      ss_iter_steps(st, j);
    }
    run_steps(parts, st);
  }
  if (!pipelined && j == cfg->max_iters) {
    std::vector<Step> st;
    ss_final_steps(st, j);
    run_steps(parts, st);
  }
  for (Part& P : parts)
    if (P.L.err) return P.L.err;
  for (Part& P : parts) {
    CK(cudaStreamWaitEvent(P.D->s, P.D->ev_coef, 0));
    CK(cudaEventRecord(P.ws->ev1, P.D->s));
  }
  for (Part& P : parts) {
    CK(cudaStreamSynchronize(P.D->s));
    CK(cudaStreamSynchronize(P.D->comm));
    CK(cudaStreamSynchronize(P.D->hstream));
  }
  CK(cudaGetLastError());
  // stamps -> host (ns from the earliest stamp), -1 where a stamp is absent
  if (cfg->stamps_out && P0.stamps) {
    const long long cap = P0.stamps_cap;
    std::vector<unsigned long long> hs((size_t)cap * kStampWords * parts.size());
    for (size_t p = 0; p < parts.size(); ++p)
      CK(cudaMemcpy(hs.data() + (size_t)p * cap * kStampWords, parts[p].stamps,
                    sizeof(unsigned long long) * kStampWords * cap, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ULL;
    auto decode = [](unsigned long long v, int w) -> unsigned long long {
      return (w == kStK1 || w == kStK3) ? (v ? ~v : 0ULL) : v;  // starts of multi-CTA products are complemented
    };
    for (size_t e = 0; e < hs.size(); ++e) {
      const unsigned long long v = decode(hs[e], (int)(e % kStampWords));
      if (v && v < t0) t0 = v;
    }
    for (size_t e = 0; e < hs.size(); ++e) {
      const unsigned long long v = decode(hs[e], (int)(e % kStampWords));
      cfg->stamps_out[e] = v ? (double)(v - t0) : -1.0;
    }
    if (cfg->stamps_count) *cfg->stamps_count = cap;
  }
  for (Part& P : parts) {
    if (P.stamps) pool_free(ctx, P.stamps);
    pool_free(ctx, P.defer_rows);
    pool_free(ctx, P.defer_count);
    pool_free(ctx, P.p12buf[1]);
  }
  // results: every partition's state is identical; a non-finite SpMV
  // output anywhere reached every partition through the next check's records
  // (NonFiniteVectorError with the group's first failure: tag, global row)
  std::vector<std::pair<int, cudaEvent_t>> marks;
  SolverState st0;
  CK(cudaMemcpy(&st0, P0.ws->st, sizeof(st0), cudaMemcpyDeviceToHost));
  if (st0.remote_err) {
    memset(res, 0, sizeof(*res));
    res->status = st0.status;
    res->nonfinite_tag = st0.err_tag & 0xff;
    res->nonfinite_index = st0.err_row;
    return set_err(ctx, PBS_ERR_NONFINITE, "non-finite SpMV output");
  }
  for (Part& P : parts) {  // (a failure no check saw: its own partition names it)
    SolverState sp;
    CK(cudaMemcpy(&sp, P.ws->st, sizeof(sp), cudaMemcpyDeviceToHost));
    if (sp.nf_row != (unsigned long long)kNoError) {
      Launcher L{ctx, P.m, P.D->s};
      return collect_result(P.m, method, cfg, res, L, marks, 0);
    }
  }
  {
    Launcher L{ctx, P0.m, P0.D->s};
    int rc2 = collect_result(P0.m, method, cfg, res, L, marks, 0);
    if (rc2) return rc2;
  }
  long long launches = 0;
  for (Part& P : parts) launches += P.L.launches;
  res->kernel_launches = launches;
  return PBS_OK;
}

// A partitioned solve on this process's partition (one process per GPU):
// b / x0 already in the workspace.
int run_solve_dist(pbs_mat* m, int method, const pbs_config* cfg, pbs_result* res) {
  pbs_dist* D = m->part.dist;
  pbs_ctx* ctx = m->ctx;
  // b / x0 were copied on the context's stream
  CK(cudaEventRecord(D->ev_vec, m->ctx->stream));
  CK(cudaStreamWaitEvent(D->s, D->ev_vec, 0));
  std::vector<pbs_mat*> mats{m};
  return group_solve(mats, method, cfg, res);
}

// ============================================================== C-ABI

PBS_EXPORT int pbs_nccl_unique_id(void* out) {
  NcclApi& A = nccl();
  if (!A.ok) return set_err(nullptr, PBS_ERR_NCCL, A.err);
  ncclUniqueId id;
  ncclResult_t r = A.GetUniqueId(&id);
  if (r != ncclSuccess) return set_err(nullptr, PBS_ERR_NCCL, A.GetErrorString(r));
  memcpy(out, &id, sizeof(id));
  return PBS_OK;
}

PBS_EXPORT int pbs_dist_init(pbs_ctx* ctx, int32_t nranks, int32_t rank, int32_t transport, const void* id_halo,
                             const void* id_red, pbs_dist** out) {
  if (!ctx || !out) return set_err(ctx, PBS_ERR_INVALID, "NULL argument");
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return set_err(ctx, PBS_ERR_INVALID, "bad rank / nranks (at most 64 partitions)");
  if (transport != PBS_TRANSPORT_P2P && transport != PBS_TRANSPORT_NCCL)
    return set_err(ctx, PBS_ERR_INVALID, "unknown transport");
  CK(cudaSetDevice(ctx->device));
  pbs_dist* d = new pbs_dist();
  d->ctx = ctx;
  d->nranks = nranks;
  d->rank = rank;
  d->transport = transport;
  if (transport == PBS_TRANSPORT_NCCL) {
    NcclApi& A = nccl();
    if (!A.ok) {
      delete d;
      return set_err(ctx, PBS_ERR_NCCL, A.err);
    }
    if (!id_halo || !id_red) {
      delete d;
      return set_err(ctx, PBS_ERR_INVALID, "the NCCL transport needs two unique ids");
    }
    ncclUniqueId a, b;
    memcpy(&a, id_halo, sizeof(a));
    memcpy(&b, id_red, sizeof(b));
    ncclResult_t r = A.CommInitRank(&d->halo, nranks, a, rank);
    if (r == ncclSuccess) r = A.CommInitRank(&d->red, nranks, b, rank);
    if (r != ncclSuccess) {
      delete d;
      return set_err(ctx, PBS_ERR_NCCL, std::string("ncclCommInitRank: ") + A.GetErrorString(r));
    }
    CK(cudaMalloc(&d->sendbuf, sizeof(double) * kRecStride));
    CK(cudaMalloc(&d->recvbuf, sizeof(double) * kRecStride * nranks));
  } else {
    MemOps& mo = memops(ctx->device);
    if (!mo.ok) {
      delete d;
      return set_err(ctx, PBS_ERR_UNSUPPORTED, mo.err);
    }
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CK(cudaStreamCreateWithFlags(&d->s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithPriority(&d->comm, cudaStreamNonBlocking, hi));  // the reduction first
  CK(cudaStreamCreateWithPriority(&d->hstream, cudaStreamNonBlocking, hi));
  for (cudaEvent_t* e : {&d->ev_vec, &d->ev_k3, &d->ev_coef, &d->ev_halo})
    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  // mailbox: arrival and reduction flags 0, freed flags 1 (nothing pushed yet)
  CK(cudaMalloc(&d->mbox, sizeof(Mailbox)));
  {
    std::vector<unsigned char> init(sizeof(Mailbox), 0);
    Mailbox* hm = reinterpret_cast<Mailbox*>(init.data());
    for (int k = 0; k < kNumVecs; ++k)
      for (int q = 0; q < kMaxRanks; ++q) hm->freed[k][q] = 1u;
    CK(cudaMemcpy(d->mbox, init.data(), sizeof(Mailbox), cudaMemcpyHostToDevice));
  }
  d->peers.assign(nranks, PeerLink{});
  *out = d;
  return PBS_OK;
}

PBS_EXPORT int pbs_dist_set_sm_limit(pbs_dist* d, int32_t sms) {
  if (!d) return set_err(nullptr, PBS_ERR_INVALID, "dist is NULL");
  if (sms < 0 || sms > d->ctx->sms) return set_err(d->ctx, PBS_ERR_INVALID, "sm limit out of range");
  d->sm_limit = sms;
  return PBS_OK;
}

PBS_EXPORT int pbs_dist_destroy(pbs_dist* d) {
  if (!d) return PBS_OK;
  cudaSetDevice(d->ctx->device);
  for (cudaStream_t s : {d->s, d->comm, d->hstream})
    if (s) cudaStreamSynchronize(s);
  for (PeerLink& pl : d->peers)
    if (pl.ipc) {
      cudaIpcCloseMemHandle(pl.base);
      cudaIpcCloseMemHandle(pl.mbox);
    }
  if (d->halo) nccl().CommDestroy(d->halo);
  if (d->red) nccl().CommDestroy(d->red);
  for (cudaStream_t s : {d->s, d->comm, d->hstream})
    if (s) cudaStreamDestroy(s);
  for (cudaEvent_t e : {d->ev_vec, d->ev_k3, d->ev_coef, d->ev_halo})
    if (e) cudaEventDestroy(e);
  cudaFree(d->mbox);
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

// Rows of a stencil slab that read no halo: [b0, b1) (host scan of the rows
// within one stencil reach of either end)
static void stencil_interior(const pbs_mat* m, long long* b0, long long* b1) {
  const StencilView& S = m->sv;
  const long long n = m->n_rows;
  long long reach = 0;
  for (int p = 0; p < S.npts; ++p) reach = std::max(reach, S.foff[p] < 0 ? -S.foff[p] : S.foff[p]);
  auto reads = [&](long long i, bool left) {
    const long long g = i + S.g0;
    int c[3] = {0, 0, 0};
    if (S.dim == 3) {
      c[0] = (int)(g / S.k2);
      c[1] = (int)((g % S.k2) / S.k);
      c[2] = (int)(g % S.k);
    } else if (S.dim == 2) {
      c[1] = (int)(g / S.k);
      c[2] = (int)(g % S.k);
    } else {
      c[2] = (int)g;
    }
    for (int p = 0; p < S.npts; ++p) {
      bool ok = true;
      for (int a = 3 - S.dim; a < 3; ++a) {
        const int cc = c[a] + S.off[p][a];
        ok = ok && cc >= 0 && cc < S.k;
      }
      if (!ok) continue;
      const long long col = i + S.foff[p];
      if (left ? col < 0 : col >= n) return true;
    }
    return false;
  };
  *b0 = 0;
  for (long long i = 0; i < std::min(n, reach + 1); ++i)
    if (reads(i, true)) *b0 = i + 1;
  *b1 = n;
  for (long long i = n - 1; i >= std::max(0LL, n - reach - 1); --i)
    if (reads(i, false)) *b1 = i;
}

PBS_EXPORT int pbs_mat_set_partition(pbs_mat* m, pbs_dist* dist, int64_t n_global, int64_t row_lo, int64_t hl,
                                     int64_t hr, int32_t nsend, const int64_t* sends, int32_t nrecv,
                                     const int64_t* recvs) {
  if (!m || !dist) return set_err(nullptr, PBS_ERR_INVALID, "NULL argument");
  pbs_ctx* ctx = m->ctx;
  if (dist->ctx != ctx) return set_err(ctx, PBS_ERR_INVALID, "partition and link must share a context");
  const long long pad = hl & 1;
  if (m->n_cols != pad + hl + m->n_rows + hr)
    return set_err(ctx, PBS_ERR_INVALID, "n_cols must equal pad + hl + n_own + hr (extended space)");
  if (m->stencil && (m->sv.xlo != -hl || m->sv.xhi != m->n_rows + hr || m->sv.g0 != row_lo))
    return set_err(ctx, PBS_ERR_INVALID, "stencil slab does not match the partition (pbs_stencil_slab)");
  CK(cudaSetDevice(ctx->device));
  if (m->ws) {  // the workspace layout depends on the partition
    free_ws(m->ws);
    m->ws = nullptr;
  }
  Partition& P = m->part;
  P = Partition{};
  P.dist = dist;
  P.n_global = n_global;
  P.row_lo = row_lo;
  P.hl = hl;
  P.hr = hr;
  P.sends.assign(sends, sends + 4 * (size_t)nsend);
  P.recvs.assign(recvs, recvs + 3 * (size_t)nrecv);
  for (size_t i = 0; i < P.sends.size(); i += 4)
    if (P.sends[i] < 0 || P.sends[i] >= dist->nranks || P.sends[i] == dist->rank || P.sends[i + 1] < 0 ||
        P.sends[i + 1] + P.sends[i + 2] > m->n_rows || P.sends[i + 3] < 0)
      return set_err(ctx, PBS_ERR_INVALID, "halo send outside the own segment");
  for (size_t i = 0; i < P.recvs.size(); i += 3)
    if (P.recvs[i] < 0 || P.recvs[i] >= dist->nranks || P.recvs[i] == dist->rank || P.recvs[i + 1] < 0 ||
        P.recvs[i + 1] + P.recvs[i + 2] > m->n_cols)
      return set_err(ctx, PBS_ERR_INVALID, "halo receive outside the extended space");
  // interior / boundary split of the SpMVs that follow a halo exchange
  {
    const long long n = m->n_rows, own_lo = pad + hl, own_hi = own_lo + n;
    long long b0, b1;  // rows [b0, b1) read no halo column
    if (m->stencil) {
      stencil_interior(m, &b0, &b1);
    } else {
      unsigned long long* d = nullptr;
      unsigned long long h[2] = {0ULL, (unsigned long long)n};
      CK(cudaMalloc(&d, sizeof(h)));
      CK(cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice));
      if (n > 0) halo_rows_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(m->rp, m->ci, n, own_lo, own_hi, d);
      CK(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(d);
      b0 = (long long)h[0];
      b1 = (long long)h[1];
    }
    // PBS_SPLIT_TEST=k (tests): treat the first and last k blocks as boundary
    // rows even without halos, so one GPU exercises the split schedule
    const char* stt = getenv("PBS_SPLIT_TEST");
    const long long force = stt ? atoll(stt) : 0;
    if (force > 0) {
      b0 = std::max(b0, force * kPipeRows);
      b1 = std::min(b1, n - force * kPipeRows);
    }
    P.L0 = (b0 + kPipeRows - 1) / kPipeRows * kPipeRows;
    P.L1 = b1 >= n ? n : b1 / kPipeRows * kPipeRows;
    const char* sp = getenv("PBS_SPLIT");  // PBS_SPLIT=0: wait for the halo, then one SpMV over all rows
    const bool allow = !(sp && atoi(sp) == 0);
    P.split = allow && !P.recvs.empty() && P.L1 > P.L0 && (P.L0 > 0 || P.L1 < n);
  }
  dist->mat = m;
  dist->connected = false;
  return ensure_ws(m, 1024);  // IPC-exportable base; peers map it at connect time
}

// What peers need to map this partition: IPC handles of its workspace base
// and mailbox, its vector stride.
struct DistBlob {
  uint32_t magic, version;
  int32_t rank, nranks;
  cudaIpcMemHandle_t ws;
  cudaIpcMemHandle_t mbox;
  int64_t stride;
  int64_t n_ext;
  int32_t device;
  int32_t pad;
};
static_assert(sizeof(DistBlob) <= PBS_DIST_BLOB_BYTES, "blob too large");
constexpr uint32_t kBlobMagic = 0x50425344u;  // "PBSD"

PBS_EXPORT int pbs_dist_export(pbs_mat* m, void* out) {
  if (!m || !out || !m->part.dist || !m->ws) return set_err(m ? m->ctx : nullptr, PBS_ERR_INVALID, "not a partition");
  pbs_dist* D = m->part.dist;
  pbs_ctx* ctx = m->ctx;
  CK(cudaSetDevice(ctx->device));
  DistBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.version = 1;
  b.rank = D->rank;
  b.nranks = D->nranks;
  CK(cudaIpcGetMemHandle(&b.ws, m->ws->base));
  CK(cudaIpcGetMemHandle(&b.mbox, D->mbox));
  b.stride = (int64_t)m->ws->stride;
  b.n_ext = m->ws->n_ext;
  b.device = ctx->device;
  memset(out, 0, PBS_DIST_BLOB_BYTES);
  memcpy(out, &b, sizeof(b));
  return PBS_OK;
}

// Map every peer's workspace and mailbox (blobs: nranks blobs in rank order,
// this rank's own included and skipped).  The caller barriers afterwards:
// once every rank is connected, any may start pushing.
PBS_EXPORT int pbs_dist_connect(pbs_mat* m, const void* blobs) {
  if (!m || !blobs || !m->part.dist || !m->ws) return set_err(m ? m->ctx : nullptr, PBS_ERR_INVALID, "not a partition");
  pbs_dist* D = m->part.dist;
  pbs_ctx* ctx = m->ctx;
  CK(cudaSetDevice(ctx->device));
  for (int q = 0; q < D->nranks; ++q) {
    DistBlob b;
    memcpy(&b, (const unsigned char*)blobs + (size_t)q * PBS_DIST_BLOB_BYTES, sizeof(b));
    if (b.magic != kBlobMagic || b.rank != q || b.nranks != D->nranks)
      return set_err(ctx, PBS_ERR_INVALID, "malformed partition blob");
    PeerLink& pl = D->peers[q];
    if (q == D->rank) {
      pl.base = m->ws->base;
      pl.stride = (long long)m->ws->stride;
      pl.mbox = D->mbox;
      pl.ipc = false;
      continue;
    }
    if (D->transport == PBS_TRANSPORT_NCCL) continue;  // NCCL moves the data
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, b.ws, cudaIpcMemLazyEnablePeerAccess));
    pl.base = (double*)p;
    CK(cudaIpcOpenMemHandle(&p, b.mbox, cudaIpcMemLazyEnablePeerAccess));
    pl.mbox = (Mailbox*)p;
    pl.stride = b.stride;
    pl.ipc = true;
  }
  D->connected = true;
  return PBS_OK;
}

// Loopback group: the n partitions of one system held by this process (one
// device), linked directly.
PBS_EXPORT int pbs_dist_connect_local(pbs_mat** mats, int32_t n) {
  if (!mats || n < 1) return set_err(nullptr, PBS_ERR_INVALID, "no partitions");
  for (int p = 0; p < n; ++p) {
    pbs_mat* m = mats[p];
    if (!m || !m->part.dist || !m->ws) return set_err(nullptr, PBS_ERR_INVALID, "not a partition");
    pbs_dist* D = m->part.dist;
    if (D->nranks != n || D->rank != p) return set_err(m->ctx, PBS_ERR_INVALID, "partition ranks must be 0..n-1");
    if (D->transport != PBS_TRANSPORT_P2P)
      return set_err(m->ctx, PBS_ERR_INVALID, "a loopback group uses the P2P transport");
    if (m->ctx->device != mats[0]->ctx->device)
      return set_err(m->ctx, PBS_ERR_INVALID, "a loopback group lives on one device");
  }
  for (int p = 0; p < n; ++p) {
    pbs_dist* D = mats[p]->part.dist;
    for (int q = 0; q < n; ++q) {
      PeerLink& pl = D->peers[q];
      pl.base = mats[q]->ws->base;
      pl.stride = (long long)mats[q]->ws->stride;
      pl.mbox = mats[q]->part.dist->mbox;
      pl.ipc = false;
    }
    D->connected = true;
  }
  return PBS_OK;
}

// copy the partitions' own segments of b / x0 in, solve, copy x out
static int group_entry(pbs_mat** mats, int32_t n, int32_t method, const double* const* b, const double* const* x0,
                       const pbs_config* cfg, double* const* x_out, double* hist_rel, uint8_t* hist_flags,
                       double* hist_coef, pbs_result* res, cudaMemcpyKind in_kind, cudaMemcpyKind out_kind) {
  if (!mats || n < 1 || !b) return set_err(nullptr, PBS_ERR_INVALID, "NULL argument");
  pbs_ctx* ctx = mats[0]->ctx;
  if (method < 0 || method > PBS_METHOD_PBICGSTAB) return set_err(ctx, PBS_ERR_INVALID, "unknown method");
  int rc = validate_cfg(ctx, cfg);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  std::vector<pbs_mat*> v(mats, mats + n);
  for (int p = 0; p < n; ++p) {
    pbs_mat* m = v[p];
    if (!m || !m->part.dist) return set_err(ctx, PBS_ERR_INVALID, "not a partition");
    rc = ensure_ws(m, cfg->max_iters + 1);
    if (rc) return rc;
    Workspace* ws = m->ws;
    cudaStream_t s = m->part.dist->s;
    const size_t bytes = sizeof(double) * ws->n;
    CK(cudaMemcpyAsync(ws->V.v[VB], b[p], bytes, in_kind, s));
    if (x0 && x0[p])
      CK(cudaMemcpyAsync(ws->V.v[VX], x0[p], bytes, in_kind, s));
    else
      CK(cudaMemsetAsync(ws->V.v[VX], 0, bytes, s));
  }
  rc = group_solve(v, method, cfg, res);
  if (rc) return rc;
  for (int p = 0; p < n; ++p) {
    Workspace* ws = v[p]->ws;
    if (x_out && x_out[p])
      CK(cudaMemcpyAsync(x_out[p], ws->V.v[VX], sizeof(double) * ws->n, out_kind, v[p]->part.dist->s));
    CK(cudaStreamSynchronize(v[p]->part.dist->s));
  }
  return copy_history(v[0], res, hist_rel, hist_flags, hist_coef);
}

PBS_EXPORT int pbs_solve_group(pbs_mat** mats, int32_t n, int32_t method, const double* const* d_b,
                               const double* const* d_x0, const pbs_config* cfg, double* const* d_x,
                               double* hist_rel, uint8_t* hist_flags, double* hist_coef, pbs_result* res) {
  return group_entry(mats, n, method, d_b, d_x0, cfg, d_x, hist_rel, hist_flags, hist_coef, res,
                     cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice);
}

// partitioned SpMV y = A x over a group (own segments in / out; halos
// exchanged by the group's transport): the parity seam of the slabs
PBS_EXPORT int pbs_spmv_group(pbs_mat** mats, int32_t n, const double* const* d_x, double* const* d_y,
                              int64_t* nonfinite_index) {
  if (!mats || n < 1 || !d_x || !d_y) return set_err(nullptr, PBS_ERR_INVALID, "NULL argument");
  pbs_ctx* ctx = mats[0]->ctx;
  CK(cudaSetDevice(ctx->device));
  std::vector<Part> parts(n);
  for (int p = 0; p < n; ++p) {
    pbs_mat* m = mats[p];
    Part& P = parts[p];
    if (!m->part.dist || !m->part.dist->connected) return set_err(ctx, PBS_ERR_INVALID, "not a connected partition");
    P.m = m;
    P.D = m->part.dist;
    int rc = ensure_ws(m, 4);
    if (rc) return rc;
    P.ws = m->ws;
    P.L = Launcher{ctx, m, P.D->s};
    P.L.sm_limit = eff_sms(P);
    for (size_t i = 0; i < m->part.sends.size(); i += 4)
      if (std::find(P.send_peers.begin(), P.send_peers.end(), (int)m->part.sends[i]) == P.send_peers.end())
        P.send_peers.push_back((int)m->part.sends[i]);
    for (size_t i = 0; i < m->part.recvs.size(); i += 3)
      if (std::find(P.recv_peers.begin(), P.recv_peers.end(), (int)m->part.recvs[i]) == P.recv_peers.end())
        P.recv_peers.push_back((int)m->part.recvs[i]);
    SolverState h{};
    h.run_all = 1;
    h.run_spine = 1;
    h.stop_check = -1;
    h.nf_row = (unsigned long long)kNoError;
    CK(cudaMemcpyAsync(P.ws->st, &h, sizeof(h), cudaMemcpyHostToDevice, P.D->s));
    CK(cudaMemcpyAsync(P.ws->V.v[VTMP], d_x[p], sizeof(double) * P.ws->n, cudaMemcpyDeviceToDevice, P.D->s));
  }
  std::vector<Step> st;
  st.push_back([](Part& P) { push(P, VTMP); });
  st.push_back([d_y](Part& P) {
    const int p = P.D->rank;
    halo_spmv(P, VTMP, KS, [&](int) {
      EpiStore e{};
      e.y = d_y[p];
      e.st = P.ws->st;
      e.tag = PBS_TAG_AX;
      return e;
    });
  });
  run_steps(parts, st);
  for (Part& P : parts)
    if (P.L.err) return P.L.err;
  for (int p = 0; p < n; ++p) {
    Part& P = parts[p];
    unsigned long long row = 0;
    CK(cudaMemcpyAsync(&row, &P.ws->st->nf_row, sizeof(row), cudaMemcpyDeviceToHost, P.D->s));
    CK(cudaStreamSynchronize(P.D->s));
    CK(cudaStreamSynchronize(P.D->hstream));
    if (nonfinite_index) nonfinite_index[p] = row == (unsigned long long)kNoError ? -1 : (int64_t)row;
  }
  CK(cudaGetLastError());
  return PBS_OK;
}
