// common.cuh — shared device-side types of libpbsafe (sm_100a).
//
// Floating-point contract: the whole library is compiled with -fmad=false and
// the update/SpMV arithmetic is written with explicit __dmul_rn/__dadd_rn, so
// every expression rounds exactly like the reference's numba loops
// (kernels.py:95-137: a product rounded, then a sum rounded, left to right).
// SpMV rows accumulate sequentially in ascending column order; only the dot
// batch is reassociated (a fixed-shape tree, or the reference's own
// PartitionPlan chains in PBS_REDUCE_PLAN mode).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pbsafe.h"

namespace pbs {

constexpr int kThreads = 256;          // CTA size of every streaming kernel
constexpr int kChunk = 2048;           // CSR products staged per smem chunk (16 KiB)
constexpr int kNumDots = 9;            // a b c d e f g h r  (reduction.py:32)
constexpr int kPartStride = 2 * kNumDots;  // doubles per partial record (double-double)
// Partial-record buffers hold up to kMaxParts records stored field-major:
// field f of record b at p[f * kMaxParts + b], so a warp reading one field of
// consecutive records is coalesced.
constexpr int kMaxParts = 148 * 16;
constexpr int kMaxStencil = 27;
constexpr long long kNoError = 0x7fffffffffffffffLL;

// dot slots in BATCH_LABELS order; _safe_batch pairs (solvers.py:467-482)
enum Dot { DA = 0, DB, DC, DD, DE, DF, DG, DH, DR };
// dot subsets: the s-independent dots (b e f h r) are final after K12's
// row-local updates, so K12 carries them and K3 only the four that need the
// new s (a c d g)
constexpr unsigned kAllDots = (1u << kNumDots) - 1;
constexpr unsigned kDotsK12 = (1u << DB) | (1u << DE) | (1u << DF) | (1u << DH) | (1u << DR);
constexpr unsigned kDotsK3 = kAllDots & ~kDotsK12;
// the product-type comparators' reduction phases (solvers.py:210-460), in the
// same slots: g = (r0*, Ap); BiCGStab b=(At,t) e=(At,At) c=(r0*,At) d=(t,t);
// GPBi-CG a=(y,y) b=(At,t) c=(y,t) d=(At,y) e=(At,At), then f=(r0*,r) r=(r,r)
constexpr unsigned kDotsProdA = 1u << DG;
constexpr unsigned kDotsStabB = (1u << DB) | (1u << DE) | (1u << DC) | (1u << DD);
constexpr unsigned kDotsGpB = (1u << DA) | (1u << DB) | (1u << DC) | (1u << DD) | (1u << DE);
constexpr unsigned kDotsGpC = (1u << DF) | (1u << DR);
constexpr unsigned kDotsRR = 1u << DR;
// p-BiCGStab (oracle solve_pstab): setup rr=(r,r) g=(r0*,w); omega phase
// b=(q,y) e=(y,y) d=(q,q); beta phase f=(r0*,r) r=(r,r) g=(r0*,w) a=(r0*,s) h=(r0*,z)
constexpr unsigned kDotsPsW = (1u << DR) | (1u << DG);
constexpr unsigned kDotsPsA = (1u << DB) | (1u << DE) | (1u << DD);
constexpr unsigned kDotsPsB = (1u << DF) | (1u << DR) | (1u << DG) | (1u << DA) | (1u << DH);

// Host-visible mirror, written by the finalize kernel through mapped pinned
// memory so the host can stop launching without a device sync.
struct HostMirror {
  volatile long long iter;
  volatile int run_all;
  volatile int err;
  // the check that stopped the solve (-1 while running).  The multi-GPU
  // schedule writes it before iter (with a system fence), so a host that has
  // seen iter > c knows whether the solve stopped at a check <= c; every
  // rank's device state is identical, so every rank takes the same decision.
  volatile long long stop_check;
};

// Device-resident solver state.  Written by the single-CTA finalize kernel
// (the reference's _Run bookkeeping + coefficient step) and by SpMV epilogues
// (non-finite detection); read by every gated kernel.
struct SolverState {
  // configuration
  double tol;
  long long max_iters;
  int record_history;
  int spine_done;  // 1 for ssBiCGSafe2: the iteration's SpMV precedes the check
  // carried scalars (solvers.py:631-632)
  double alpha, beta, zeta, eta;
  double f_prev;
  double r0_norm;
  double dots[kNumDots];
  double omega;  // BiCGStab's step (its coefficient record keeps it in the zeta slot)
  double rr;     // product-type methods: the residual norm^2 of the next check
  // control
  long long iter;       // index of the next check the finalize kernel performs
  int run_all;          // 0 once a check stopped the solve
  int run_spine;        // the spine SpMV (As / Ar) still runs for the stop iteration
  int status;           // -1 running, else PBS_CONVERGED...
  int breakdown;
  int upd;              // BiCGStab: this iteration's x/r update may run (omega passed)
  int stop_stage;       // product-type methods: where the stopping iteration ended
                        // (0 its loop-top check, 1 alpha, 2 omega/zeta, 3 after
                        // the x/r update, 4 complete) -> the reference's tallies
  long long failure_iter;
  long long iterations;
  long long n_records;
  long long stop_check;  // the check that stopped the solve (-1 while running)
  // non-finite SpMV output (NonFiniteVectorError): first row, tag
  unsigned long long nf_row;
  int nf_tag;
  // multi-GPU: the group's first non-finite SpMV output (every partition
  // learns it from the records of the next check): its encoded tag and
  // global row
  int remote_err;
  int err_tag;
  long long err_row;
  // multi-GPU: the finalize of check j publishes its coefficients by setting
  // this to j + 1 (release, after the state is stored); K1's opportunistic
  // epilogue reads it (acquire)
  unsigned long long coef_epoch;
  unsigned int done_ctas;  // last-CTA ticket of the fused finalize (reset by the last CTA)
  // history (device arrays, max_iters+1 slots)
  double* hist_rel;
  unsigned char* hist_flags;
  double* hist_coef;
  HostMirror* mirror;
};

__device__ __forceinline__ bool dev_err(const SolverState* st) {
  return *(volatile const unsigned long long*)&st->nf_row != (unsigned long long)kNoError;
}

// kernels of the iteration body run while no check has stopped the solve
__device__ __forceinline__ bool gate_all(const SolverState* st) {
  return st == nullptr || (!dev_err(st) && st->run_all);
}
// the spine SpMV (As in p-BiCGSafe, Ar in ssBiCGSafe2) also runs on the
// iteration whose check stops the solve (solvers.py:641-643, 530-531)
__device__ __forceinline__ bool gate_spine(const SolverState* st) {
  return st == nullptr || (!dev_err(st) && st->run_spine);
}

__device__ __forceinline__ void report_nonfinite(SolverState* st, int tag, long long row) {
  if (st == nullptr) return;
  atomicMin(&st->nf_row, (unsigned long long)row);
  st->nf_tag = tag;
  if (st->mirror) st->mirror->err = 1;  // lets the host stop launching at once
}

// release/acquire fence (the patterns here — publish a record, then take a
// ticket; take the ticket, then read every record — need no more than
// acq_rel; __threadfence() is the stronger, slower fence.sc)
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// device-wide nanosecond clock (schedule evidence stamps)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// kernels.py:110-137 element expressions, association as written
__device__ __forceinline__ double lc2(double sa, double a, double sb, double b) {
  return add(mul(sa, a), mul(sb, b));
}
__device__ __forceinline__ double lc3(double sa, double a, double sb, double b, double sc, double c) {
  return add(add(mul(sa, a), mul(sb, b)), mul(sc, c));
}
__device__ __forceinline__ double lc4(double sa, double a, double sb, double b, double sc, double c,
                                      double sd, double d) {
  return add(add(add(mul(sa, a), mul(sb, b)), mul(sc, c)), mul(sd, d));
}
__device__ __forceinline__ double lcn(double sa, double a, double sb, double b, double sc, double c) {
  return add(mul(sa, a), mul(sb, add(b, mul(sc, c))));
}
__device__ __forceinline__ double asd(double base, double s, double a, double b) {
  return add(base, mul(s, sub(a, b)));
}
__device__ __forceinline__ double asdd(double base, double s, double a, double w, double b) {
  return add(base, mul(s, sub(a, mul(w, b))));
}

template <int NT, bool NAMED>
__device__ __forceinline__ void block_bar() {
  if (NAMED)
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  else
    __syncthreads();
}

// ---- compensated accumulation of the dot batch --------------------------
// Each dot is carried as a pair (p, s): p the running sum, s the running sum
// of the exact rounding errors of every product (TwoProduct via fma) and of
// every addition into p (TwoSum) — Ogita, Rump & Oishi's Dot2.  The result
// p + s is as accurate as a dot computed in twice the working precision and
// then rounded, i.e. (except in pathological cases) the correctly rounded
// dot, so the batch no longer depends on the reduction order (DESIGN.md,
// iteration-count parity).  Loop-carried dependencies are one add each.
struct Ddbl {
  double hi, lo;  // p, s
};

__device__ __forceinline__ Ddbl two_sum(double a, double b) {
  const double s = add(a, b);
  const double bb = sub(s, a);
  return Ddbl{s, add(sub(a, sub(s, bb)), sub(b, bb))};
}

// accumulate one product a*b into (p, s)
__device__ __forceinline__ Ddbl dot2_step(Ddbl acc, double a, double b) {
#ifdef PBS_PLAIN_DOT  // measurement-only build (tools/build_variants.py): what the compensation costs
  return Ddbl{add(acc.hi, mul(a, b)), acc.lo};
#endif
  const double h = mul(a, b);
  const double r = __fma_rn(a, b, -h);
  const Ddbl t = two_sum(acc.hi, h);
  return Ddbl{t.hi, add(acc.lo, add(t.lo, r))};
}

// combine two partial pairs
__device__ __forceinline__ Ddbl dd_add(Ddbl a, Ddbl b) {
  const Ddbl t = two_sum(a.hi, b.hi);
  return Ddbl{t.hi, add(add(a.lo, b.lo), t.lo)};
}

__device__ __forceinline__ Ddbl dd_shfl_xor(Ddbl v, int o) {
  return Ddbl{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
}

// Block-level reduction of 9 per-thread compensated partials into fields
// 2j, 2j+1 of the CTA's record, out = partials + blockIdx.x (field-major;
// threads 0..8 write, then a release fence so a last-CTA
// reader sees them).  Fixed shape (xor-butterfly in warps, then warps in
// index order): the result depends only on the data-to-thread mapping.
// Only the dots in M are reduced and written.
template <int NT, bool NAMED, unsigned M = kAllDots>
__device__ __forceinline__ void block_reduce9(Ddbl (&acc)[kNumDots], double* out) {
  __shared__ Ddbl red[NT / 32][kNumDots];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kNumDots; ++j) {
    if (!((M >> j) & 1u)) continue;
    Ddbl v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dd_add(v, dd_shfl_xor(v, o));
    if (lane == 0) red[warp][j] = v;
  }
  block_bar<NT, NAMED>();
  if (threadIdx.x < kNumDots && ((M >> threadIdx.x) & 1u)) {
    Ddbl v = red[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) v = dd_add(v, red[w][threadIdx.x]);
    out[(size_t)(2 * threadIdx.x) * kMaxParts] = v.hi;
    out[(size_t)(2 * threadIdx.x + 1) * kMaxParts] = v.lo;
    fence_gpu();
  }
}

}  // namespace pbs
