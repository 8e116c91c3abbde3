// spmv.cuh — SpMV engines with fused epilogues (sm_100a).
//
// Both engines hand each output row to an epilogue: Epi::row(i, y, in[])
// where in[] holds the row's values of the epilogue's kIn input vectors.
//
//  * csr_pipe_kernel — CSR, warp-specialised and TMA-fed.  One CTA per SM:
//    a producer warp streams, per 256-row block, the row_ptr slice, the x
//    windows the block's columns fall in (offset clusters measured at upload:
//    3 plane windows for a 3D stencil) and the epilogue's input segments into
//    a ring of block slots, and the block's contiguous nonzero range of
//    values / int32 col_idx (<=2048-nonzero chunks) into a ring of chunk
//    stages — all with 1-D bulk async copies (cp.async.bulk, completion on
//    mbarriers).  Eight consumer warps own one row each per block, read x and
//    everything else from shared memory (global gathers only for matrices
//    whose offsets are too spread to window) and accumulate the row
//    sequentially in ascending column order
//    (kernels.py:95-100), so the product is bitwise the reference's while HBM
//    sees every matrix byte once with the copy engine keeping it busy.
//  * stencil_spmv_kernel — matrix-free constant-coefficient stencil, one
//    thread per row, neighbours in ascending flattened offset (= CSR column
//    order), out-of-grid neighbours skipped (Dirichlet elimination): bitwise
//    equal to the CSR of the same stencil.
//
// Epilogues (SURVEY §8(d) kernel plan):
//   EpiStore  y = A x                          (rr products, plain SpMV)
//   EpiK12    As = A s -> p u w t z y x r       (K1 fused with the row-local K2, solvers.py:678-715)
//   EpiResid  r = b - A x  (+ r0s = r)         (setup; rr "r = b - A x")
//   EpiK3     Aw -> l, g, s + next 9 dot partials (solvers.py:717-723, 467-482)
//   EpiDots   s = A r + 9 dot partials          (setup s0 = A r0; rr s = A r)
//   EpiSS3    w = A u -> t, z, y, x, r          (ssBiCGSafe2, solvers.py:569-580)
// Epilogues with dot partials finish with a fixed-shape block reduction and,
// when `fuse` is set, the last CTA to finish runs the coefficient check.
#pragma once
#include "common.cuh"
#include "finalize.cuh"
#include "ptx.cuh"

namespace pbs {

// staged-window products in flight per row for the dot-carrying epilogues
// (register-bound; -D overrides for sweeps)
#ifndef PBS_WCB_K12D
#define PBS_WCB_K12D 2
#endif
#ifndef PBS_WCB_K3S
#define PBS_WCB_K3S 4
#endif
#ifndef PBS_WCB_ONE  // the 1-CTA-per-SM instantiation (band mode, long rows)
#define PBS_WCB_ONE 8
#endif
#ifndef PBS_K12D_MINB
#define PBS_K12D_MINB 1
#endif

struct CsrView {
  const long long* rp;
  const int* ci;
  const double* v;
  long long row_lo, row_hi;
  long long n_cols;
  // nullable: per-nonzero index into its row block's staged x windows (built
  // at upload for row_lo == 0); replaces col_idx in the staged engine
  const unsigned short* wc;
};

// Division of a row index i < 2^31 by an invariant d >= 1 with one 32x32->64
// multiply and a shift: m = ceil(2^(31+l) / d), l = ceil(log2 d), s = 31 + l
// gives floor(i * m / 2^s) == i / d for all i < 2^31 (Granlund-Montgomery);
// m < 2^32.  The grid coordinates of every stencil row use it instead of a
// 64-bit division.
struct FastDiv {
  unsigned long long m;
  int s;
  __host__ __device__ __forceinline__ long long div(long long i) const {
    return (long long)(((unsigned long long)(unsigned)i * m) >> s);
  }
};

__host__ inline FastDiv make_fastdiv(long long d) {
  int l = 0;
  while ((1LL << l) < d) ++l;
  const unsigned __int128 two = (unsigned __int128)1 << (31 + l);
  FastDiv f;
  f.m = (unsigned long long)((two + (unsigned __int128)d - 1) / (unsigned __int128)d);
  f.s = 31 + l;
  return f;
}

struct StencilView {
  long long n, k, k2;
  FastDiv dk, dk2;  // i / k, i / k^2
  // boundary masks (offsets are in {-1, 0, 1} per axis): bit p of nlo[a] is
  // clear when point p steps -1 along axis a, of nhi[a] when it steps +1; a
  // row at coordinate 0 (k - 1) on axis a keeps only the points in nlo[a]
  // (nhi[a]) — the Dirichlet elimination as two masks per axis instead of a
  // bounds test per point and axis
  unsigned nlo[3], nhi[3];
  int dim, npts;
  int off[kMaxStencil][3];      // (dz,)dy,dx per point, padded to 3 axes from the left
  long long foff[kMaxStencil];  // flattened offset
  double coef[kMaxStencil];
  long long row_lo, row_hi;
  // row slab of a partitioned grid (pbs_stencil_slab): local row i is grid
  // row i + g0, and x is addressed relative to the slab's own segment, valid
  // on [xlo, xhi) = [-left halo, n + right halo).  Whole grid: 0, [0, n).
  long long g0, xlo, xhi;
  // neighbours of the row at grid coordinates c (padded to 3 axes) that lie
  // in the grid, as a bit mask over the points
  __device__ __forceinline__ unsigned valid_mask(const int (&c)[3], int dim) const {
    const int km1 = (int)k - 1;
    unsigned vm = 0xffffffffu;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a < 3 - dim) continue;
      if (c[a] == 0) vm &= nlo[a];
      if (c[a] == km1) vm &= nhi[a];
    }
    return vm;
  }
};

// ---------------------------------------------------------------- epilogues
//
// Opportunistic epilogues (Epi::kOpp, csr_pipe_kernel only): the producer
// decides per row block whether the epilogue can run now (Epi::ready(): the
// coefficients it needs exist yet), stages the block's epilogue inputs only
// then, and tells the consumers through the block header; the consumers run
// the full epilogue for such blocks and hand the others to Epi::defer().
template <class Epi, class = void>
struct EpiOpp {
  static constexpr bool value = false;
};
template <class Epi>
struct EpiOpp<Epi, decltype((void)Epi::kOpp)> {
  static constexpr bool value = Epi::kOpp;
};

template <unsigned M>
struct DotsT {
  Ddbl acc[kNumDots];
  __device__ void zero() {
#pragma unroll
    for (int j = 0; j < kNumDots; ++j) acc[j] = Ddbl{0.0, 0.0};
  }
  __device__ __forceinline__ void step(int j, double a, double b) {
    if ((M >> j) & 1u) acc[j] = dot2_step(acc[j], a, b);
  }
  // _safe_batch pairs (solvers.py:471-481), compensated (Dot2) accumulation;
  // only the dots in M
  __device__ void add_row(double s, double y, double r, double r0s, double t) {
    step(DA, s, s);
    step(DB, y, y);
    step(DC, s, y);
    step(DD, s, r);
    step(DE, y, r);
    step(DF, r0s, r);
    step(DG, r0s, s);
    step(DH, r0s, t);
    step(DR, r, r);
  }
};
using Dots9 = DotsT<kAllDots>;

// dot-partial sink shared by the epilogues that carry the batch
struct DotSink {
  double* partials;  // nullptr: no partials (PBS_REDUCE_PLAN computes them separately)
  int fuse;          // last CTA runs finalize_tail (check + coefficients)
  int replaced;      // the record this check writes follows a replacement
  int phase;         // finalize phase (kPhSafe: the Safe methods' check)
  // the dots this kernel does not carry: K12's records (mask2 = kDotsK12)
  const double* partials2;
  int nparts2;
  unsigned mask2;
  template <int NT, bool NAMED, unsigned M>
  __device__ void finish(DotsT<M>& d, SolverState* st) {
    if (!partials) return;
    block_reduce9<NT, NAMED, M>(d.acc, partials + blockIdx.x);
    if (fuse) finalize_tail<NT, NAMED>(st, partials, gridDim.x, replaced, partials2, nparts2, mask2, phase);
  }
};

struct EpiStore {
  static constexpr int kIn = 0;
  static constexpr int kInStaged = kIn;  // inputs the staged engines copy into smem
  static constexpr int kWcBatch = 4;  // staged-window products in flight per row
  static constexpr int kMinBlocks = 1;  // direct stencil engine occupancy target
  static constexpr bool kStencilPipe = false;  // staged engine wins (sweep r1)
  static constexpr int kGatherBatch = 8;  // x gathers in flight per row
  double* y;
  SolverState* st;
  int tag;
  int spine;  // gate on run_spine instead of run_all
  // nullable: [start, end] of this product over all CTAs (schedule
  // evidence; the start is stored complemented so both take atomicMax)
  unsigned long long* stamp;
  const double* in[1];
  __device__ bool active() const { return spine ? gate_spine(st) : gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() {
    if (stamp && threadIdx.x == 0) atomicMax(stamp, ~gtime());
  }
  __device__ void row(long long i, double v, const double*) {
    y[i] = v;
    if (tag && !isfinite(v)) report_nonfinite(st, tag, i);
  }
  template <int NT, bool NAMED>
  __device__ void finish() {
    if (!stamp) return;
    block_bar<NT, NAMED>();
    if (threadIdx.x == 0) atomicMax(stamp + 1, gtime());
  }
};

struct EpiResid {  // lincomb2(r, 1.0, b, -1.0, ax) after check_finite(ax)
  static constexpr int kIn = 1;
  static constexpr int kInStaged = kIn;  // inputs the staged engines copy into smem
  static constexpr int kWcBatch = 4;  // staged-window products in flight per row
  static constexpr int kMinBlocks = 1;  // direct stencil engine occupancy target
  static constexpr bool kStencilPipe = false;  // staged engine wins (sweep r1)
  static constexpr int kGatherBatch = 8;  // x gathers in flight per row
  double* r;
  double* r0s;  // nullable: also r0s = r (solvers.py:617)
  SolverState* st;
  int tag;  // PBS_TAG_AX (| launch sequence << 8 in the multi-GPU schedule)
  const double* in[kIn];  // b
  __device__ bool active() const { return gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() {}
  __device__ void row(long long i, double ax, const double* v) {
    if (!isfinite(ax)) report_nonfinite(st, tag, i);
    const double rv = lc2(1.0, v[0], -1.0, ax);
    r[i] = rv;
    if (r0s) r0s[i] = rv;
  }
  template <int NT, bool NAMED>
  __device__ void finish() {}
};

struct EpiDots {  // s = A r, then the batch partials over (s, y, r, r0s, t)
  static constexpr int kIn = 4;
  static constexpr int kInStaged = kIn;  // inputs the staged engines copy into smem
  static constexpr int kWcBatch = 4;  // staged-window products in flight per row
  static constexpr int kMinBlocks = 1;  // direct stencil engine occupancy target
  static constexpr bool kStencilPipe = true;  // staged engine wins (sweep r1)
  static constexpr int kGatherBatch = 2;  // x gathers in flight per row
  double* s;
  SolverState* st;
  int tag;
  int spine;
  DotSink sink;
  unsigned long long* stamp;  // nullable: [~start, end] of the product (see EpiStore)
  const double* in[kIn];  // y r r0s t
  Dots9 d;
  __device__ bool active() const { return spine ? gate_spine(st) : gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() {
    if (stamp && threadIdx.x == 0) atomicMax(stamp, ~gtime());
    d.zero();
  }
  __device__ void row(long long i, double v, const double* in4) {
    s[i] = v;
    if (!isfinite(v)) report_nonfinite(st, tag, i);
    if (sink.partials) d.add_row(v, in4[0], in4[1], in4[2], in4[3]);
  }
  template <int NT, bool NAMED>
  __device__ void finish() {
    if (stamp) {
      block_bar<NT, NAMED>();
      if (threadIdx.x == 0) atomicMax(stamp + 1, gtime());
    }
    sink.finish<NT, NAMED>(d, st);
  }
};

// DOTS: also the partials of the s-independent dots of the next check (b e f
// h r: y, r, t are final here), with r0s read directly, not staged
template <bool DOTS>
struct EpiK12T {  // K1 (As = A s) fused with block 1 of the iteration (row-local K2 updates)
  static constexpr int kIn = DOTS ? 12 : 11;
  static constexpr int kInStaged = 11;  // r0s (DOTS) is loaded by the consumer thread
  // K12 with the dots is only launched by the fused steady iteration, after
  // K3 (writes l g s), the setup's / a replacement iteration's s = A r, or a
  // finalize kernel: r p u t y w z x are final before that kernel starts
  // (sell.cuh: EpiEarly)
  // Measured neutral to slightly negative (config 2: 9.71k vs 9.75-9.9k it/s,
  // profiles/r2/sweeps_sell.md): the early copies compete with the draining
  // kernel for HBM.  Mask kept for the record: 0x737.
  static constexpr unsigned kEarly = 0u;
  static constexpr int kWcBatch = DOTS ? PBS_WCB_K12D : 4;  // staged-window products in flight per row
  static constexpr int kMinBlocks = DOTS ? PBS_K12D_MINB : 1;  // direct stencil engine occupancy target
  static constexpr bool kStencilPipe = false;  // staged engine wins (sweep r1)
  static constexpr int kGatherBatch = DOTS ? 4 : 8;  // x gathers in flight per row
  double* as;  // As is kept for K3
  double *p, *u, *w, *t, *z, *y, *x, *r;
  double *o_out, *q_out;  // nullable (single-step parity)
  double* parts;          // DOTS: partial records of the s-independent dots (kDotsK12)
  SolverState* st;
  const double* in[kIn];  // r p u s t y l g w z x r0s
  double alpha, beta, zeta, eta;
  int full;  // 0: the check stopped the solve; only the spine product runs
  DotsT<kDotsK12> d;
  __device__ bool active() const { return gate_spine(st); }
  __device__ void on_skip() const {}
  __device__ void init() {
    full = gate_all(st);
    if (DOTS) d.zero();
    alpha = st->alpha;
    beta = st->beta;
    zeta = st->zeta;
    eta = st->eta;
  }
  __device__ void row(long long i, double asv, const double* v) {
    as[i] = asv;
    if (!isfinite(asv)) report_nonfinite(st, PBS_TAG_AS, i);
    if (!full) return;
    const double rv = v[0], pv = v[1], uv = v[2], sv = v[3], tv = v[4], yv = v[5];
    const double lv = v[6], gv = v[7], wv = v[8], zv = v[9], xv = v[10];
    const double pn = asd(rv, beta, pv, uv);              // p = r + beta*(p - u)
    const double o = add(sv, mul(beta, tv));               // o = s + beta*t   (1.0 * s is s: no product issued)
    const double un = lcn(zeta, o, eta, yv, beta, uv);    // u = zeta*o + eta*(y + beta*u)
    const double q = add(asv, mul(beta, lv));              // q = As + beta*l
    const double wn = lcn(zeta, q, eta, gv, beta, wv);    // w = zeta*q + eta*(g + beta*w)
    const double tn = sub(o, wn);                          // t = o - w
    const double zn = lc3(zeta, rv, eta, zv, -alpha, un); // z = zeta*r + eta*z - alpha*u
    const double yn = lc3(zeta, sv, eta, yv, -alpha, wn); // y = zeta*s + eta*y - alpha*w
    const double xn = add(add(xv, mul(alpha, pn)), zn);    // x = x + alpha*p + z
    const double rn = sub(add(rv, mul(-alpha, o)), yn);    // r = r - alpha*o - y
    p[i] = pn;
    u[i] = un;
    w[i] = wn;
    t[i] = tn;
    z[i] = zn;
    y[i] = yn;
    x[i] = xn;
    r[i] = rn;
    if (o_out) {
      o_out[i] = o;
      q_out[i] = q;
    }
    if constexpr (DOTS) d.add_row(0.0, yn, rn, v[kIn - 1], tn);  // next check's b e f h r
  }
  template <int NT, bool NAMED>
  __device__ void finish() {
    if constexpr (DOTS) block_reduce9<NT, NAMED, kDotsK12>(d.acc, parts + blockIdx.x);
  }
};
using EpiK12 = EpiK12T<false>;
using EpiK12d = EpiK12T<true>;

// K1 of the multi-GPU schedule (As = A s, overlapping the reduction of check
// j) with block 1 of the iteration fused in opportunistically: the row blocks
// whose producer finds the coefficients of check j already published (the
// finalize has advanced coef_epoch to want) run EpiK12d's epilogue — p u w t
// z y x r and the dots b e f h r of check j+1 — in the same pass; the blocks
// streamed before that only store As and are listed for k2_deferred_kernel.
// On a large slab the reduction (~30 us) covers a few percent of K1, so the
// partitioned iteration streams like the fused single-GPU one.
struct EpiK1opp {
  static constexpr bool kOpp = true;
  static constexpr int kIn = 12;
  static constexpr int kInStaged = 11;  // r0s is loaded by the consumer thread
  static constexpr int kWcBatch = PBS_WCB_K12D;
  static constexpr int kMinBlocks = PBS_K12D_MINB;
  static constexpr bool kStencilPipe = false;
  static constexpr int kGatherBatch = 4;
  double* as;
  double *p, *u, *w, *t, *z, *y, *x, *r;
  double *o_out, *q_out;  // unused (epi_k12_fill sets them)
  double* parts;  // records of this launch's b e f h r partials (kDotsK12)
  SolverState* st;
  const double* in[kIn];  // r p u s t y l g w z x r0s
  unsigned long long* stamp;
  unsigned long long want;  // the coefficients exist once st->coef_epoch >= want
  int* defer_rows;          // first rows of the blocks left to k2_deferred_kernel
  unsigned* defer_count;
  int tag;
  int have, full;
  double alpha, beta, zeta, eta;
  DotsT<kDotsK12> d;
  __device__ bool active() const { return gate_spine(st); }
  __device__ void on_skip() const {}
  __device__ void init() {
    if (stamp && threadIdx.x == 0) atomicMax(stamp, ~gtime());
    d.zero();
    have = 0;
    full = 0;
  }
  __device__ bool ready() const {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&st->coef_epoch) : "memory");
    return v >= want;
  }
  __device__ void row_opp(long long i, double asv, const double* v, bool fused) {
    as[i] = asv;
    if (!isfinite(asv)) report_nonfinite(st, tag, i);
    if (!fused) return;
    if (!have) {  // the producer saw the coefficients published: read them once
      have = 1;
      full = !dev_err(st) && __ldcg(&st->run_all);
      alpha = __ldcg(&st->alpha);
      beta = __ldcg(&st->beta);
      zeta = __ldcg(&st->zeta);
      eta = __ldcg(&st->eta);
    }
    if (!full) return;
    const double rv = v[0], pv = v[1], uv = v[2], sv = v[3], tv = v[4], yv = v[5];
    const double lv = v[6], gv = v[7], wv = v[8], zv = v[9], xv = v[10];
    const double pn = asd(rv, beta, pv, uv);              // p = r + beta*(p - u)
    const double o = add(sv, mul(beta, tv));               // o = s + beta*t   (1.0 * s is s: no product issued)
    const double un = lcn(zeta, o, eta, yv, beta, uv);    // u = zeta*o + eta*(y + beta*u)
    const double q = add(asv, mul(beta, lv));              // q = As + beta*l
    const double wn = lcn(zeta, q, eta, gv, beta, wv);    // w = zeta*q + eta*(g + beta*w)
    const double tn = sub(o, wn);                          // t = o - w
    const double zn = lc3(zeta, rv, eta, zv, -alpha, un); // z = zeta*r + eta*z - alpha*u
    const double yn = lc3(zeta, sv, eta, yv, -alpha, wn); // y = zeta*s + eta*y - alpha*w
    const double xn = add(add(xv, mul(alpha, pn)), zn);    // x = x + alpha*p + z
    const double rn = sub(add(rv, mul(-alpha, o)), yn);    // r = r - alpha*o - y
    p[i] = pn;
    u[i] = un;
    w[i] = wn;
    t[i] = tn;
    z[i] = zn;
    y[i] = yn;
    x[i] = xn;
    r[i] = rn;
    d.add_row(0.0, yn, rn, v[kIn - 1], tn);  // next check's b e f h r
  }
  // engines without the producer's per-block decision defer every row
  __device__ void row(long long i, double asv, const double* v) { row_opp(i, asv, v, false); }
  __device__ void defer(long long r0) {
    const unsigned k = atomicAdd(defer_count, 1u);
    defer_rows[k] = (int)r0;
  }
  template <int NT, bool NAMED>
  __device__ void finish() {
    if (stamp) {
      block_bar<NT, NAMED>();
      if (threadIdx.x == 0) atomicMax(stamp + 1, gtime());
    }
    block_reduce9<NT, NAMED, kDotsK12>(d.acc, parts + blockIdx.x);
  }
};

// block 2 of the pipelined iteration with the dot partials in M of the next
// check's batch: all 9 (kAllDots), the 4 that need the new s (kDotsK3; K12
// carried the rest), or none (0: a separate streaming kernel computes them)
template <unsigned M>
struct EpiK3T {
  static constexpr int kIn = M == kAllDots ? 8 : (M ? 7 : 4);
  static constexpr int kInStaged = kIn;  // inputs the staged engines copy into smem
  // K3 with the four s-dots follows K12 (writes As p u w t z y x r) in the
  // fused iteration and plain (non-programmatic) kernels in the multi-GPU
  // schedule: l g s r0s are final before its predecessor starts
  // (mask 0x4e; off, see EpiK12T)
  static constexpr unsigned kEarly = 0u;
  static constexpr int kWcBatch = M == kAllDots ? 2 : PBS_WCB_K3S;  // staged-window products in flight per row
  static constexpr int kMinBlocks = 1;  // direct stencil engine occupancy target
  static constexpr bool kStencilPipe = true;  // staged engine wins (sweep r1)
  static constexpr int kGatherBatch = 2;  // x gathers in flight per row
  double *l, *g, *s;
  double* q_out;  // nullable (single-step parity: expose q)
  SolverState* st;
  int tag;  // PBS_TAG_AW (| launch sequence << 8 in the multi-GPU schedule)
  DotSink sink;
  const double* in[8];  // As l g s (y r r0s (t))
  unsigned long long* stamp;  // nullable: [~start, end] of the product (see EpiStore)
  double alpha, beta, zeta, eta;
  DotsT<M> d;
  __device__ bool active() const { return gate_all(st); }
  // the stop iteration's spine product (K12) has run: close the spine gate for
  // iterations the host launched ahead
  __device__ void on_skip() const {
    if (!dev_err(st) && !st->run_all) st->run_spine = 0;
  }
  __device__ void init() {
    if (stamp && threadIdx.x == 0) atomicMax(stamp, ~gtime());
    if (M) d.zero();
    alpha = st->alpha;
    beta = st->beta;
    zeta = st->zeta;
    eta = st->eta;
  }
  __device__ void row(long long i, double aw, const double* v) {
    if (!isfinite(aw)) report_nonfinite(st, tag, i);
    const double asv = v[0];
    const double q = add(asv, mul(beta, v[1]));               // q = As + beta*l  (1.0 * As is As)
    const double lv = sub(q, aw);                              // l = q - A w
    const double gv = lc3(zeta, asv, eta, v[2], -alpha, aw);  // g = zeta As + eta g - alpha Aw
    const double sv = sub(add(v[3], mul(-alpha, q)), gv);      // s = s - alpha q - g
    l[i] = lv;
    g[i] = gv;
    s[i] = sv;
    if (q_out) q_out[i] = q;
    if constexpr (M == kAllDots) {
      if (sink.partials) d.add_row(sv, v[4], v[5], v[6], v[7]);
    } else if constexpr (M != 0) {
      if (sink.partials) d.add_row(sv, v[4], v[5], v[6], 0.0);
    }
  }
  template <int NT, bool NAMED>
  __device__ void finish() {
    if (stamp) {
      block_bar<NT, NAMED>();
      if (threadIdx.x == 0) atomicMax(stamp + 1, gtime());
    }
    if constexpr (M != 0) sink.finish<NT, NAMED>(d, st);
  }
};
using EpiK3 = EpiK3T<kAllDots>;
using EpiK3n = EpiK3T<0>;
using EpiK3s = EpiK3T<kDotsK3>;


struct EpiSS3 {  // ssBiCGSafe2 tail: w = A u, then t, z, y, x, r (solvers.py:569-580)
  static constexpr int kIn = 8;
  static constexpr int kInStaged = kIn;  // inputs the staged engines copy into smem
  static constexpr int kWcBatch = 4;  // staged-window products in flight per row
  static constexpr int kMinBlocks = 1;  // direct stencil engine occupancy target
  static constexpr bool kStencilPipe = false;  // staged engine wins (sweep r1)
  static constexpr int kGatherBatch = 8;  // x gathers in flight per row
  double *w, *t, *z, *y, *x, *r;
  SolverState* st;
  int tag;  // PBS_TAG_AU (| launch sequence << 8 in the multi-GPU schedule)
  const double* in[kIn];  // o s u p y z x r
  double alpha, zeta, eta;
  __device__ bool active() const { return gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() {
    alpha = st->alpha;
    zeta = st->zeta;
    eta = st->eta;
  }
  __device__ void row(long long i, double wv, const double* v) {
    if (!isfinite(wv)) report_nonfinite(st, tag, i);
    const double ov = v[0];
    const double yv = lc3(zeta, v[1], eta, v[4], -alpha, wv);  // y = zeta s + eta y - alpha w
    const double zv = lc3(zeta, v[7], eta, v[5], -alpha, v[2]);  // z = zeta r + eta z - alpha u
    w[i] = wv;
    t[i] = lc2(1.0, ov, -1.0, wv);                              // t = o - w
    z[i] = zv;
    y[i] = yv;
    x[i] = lc3(1.0, v[6], alpha, v[3], 1.0, zv);                // x = x + alpha p + z
    r[i] = lc3(1.0, v[7], -alpha, ov, -1.0, yv);                // r = r - alpha o - y
  }
  template <int NT, bool NAMED>
  __device__ void finish() {}
};

// ---- product-type comparators (BiCGStab solvers.py:210-327, GPBi-CG 330-460)

// Ap = A p (check_finite tag "Ap"), then the partials of g = (r0*, Ap)
struct EpiPA {
  static constexpr int kIn = 1;
  static constexpr int kInStaged = kIn;
  static constexpr int kWcBatch = 4;
  static constexpr int kMinBlocks = 1;
  static constexpr bool kStencilPipe = false;
  static constexpr int kGatherBatch = 8;
  double* ap;
  SolverState* st;
  DotSink sink;
  const double* in[kIn];  // r0s
  DotsT<kDotsProdA> d;
  __device__ bool active() const { return gate_all(st); }
  // a stopped solve: the stopping iteration's x/r update has run, so close
  // its gate for iterations the host launched ahead
  __device__ void on_skip() const {
    if (!dev_err(st) && !st->run_all) st->upd = 0;
  }
  __device__ void init() { d.zero(); }
  __device__ void row(long long i, double v, const double* in1) {
    ap[i] = v;
    if (!isfinite(v)) report_nonfinite(st, PBS_TAG_AP, i);
    if (sink.partials) d.step(DG, in1[0], v);
  }
  template <int NT, bool NAMED>
  __device__ void finish() { sink.finish<NT, NAMED>(d, st); }
};

// At = A t (tag "At"), then BiCGStab's b=(At,t) e=(At,At) c=(r0*,At) d=(t,t)
// or GPBi-CG's a=(y,y) b=(At,t) c=(y,t) d=(At,y) e=(At,At)
template <bool GP>
struct EpiProdBT {
  static constexpr int kIn = 2;
  static constexpr int kInStaged = kIn;
  static constexpr int kWcBatch = 4;
  static constexpr int kMinBlocks = 1;
  static constexpr bool kStencilPipe = false;
  static constexpr int kGatherBatch = 8;
  double* at;
  SolverState* st;
  DotSink sink;
  const double* in[kIn];  // t, then r0s (BiCGStab) or y (GPBi-CG)
  DotsT<GP ? kDotsGpB : kDotsStabB> d;
  __device__ bool active() const { return gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() { d.zero(); }
  __device__ void row(long long i, double v, const double* in2) {
    at[i] = v;
    if (!isfinite(v)) report_nonfinite(st, PBS_TAG_AT, i);
    if (!sink.partials) return;
    const double t = in2[0], q = in2[1];
    if constexpr (GP) {
      d.step(DA, q, q);
      d.step(DB, v, t);
      d.step(DC, q, t);
      d.step(DD, v, q);
      d.step(DE, v, v);
    } else {
      d.step(DB, v, t);
      d.step(DE, v, v);
      d.step(DC, q, v);
      d.step(DD, t, t);
    }
  }
  template <int NT, bool NAMED>
  __device__ void finish() { sink.finish<NT, NAMED>(d, st); }
};
using EpiStabB = EpiProdBT<false>;
using EpiGpB = EpiProdBT<true>;

// ---- p-BiCGStab (oracle solve_pstab; Cools & Vanroose's pipelined BiCGStab)

// setup: w = A r (tag "Ar"), then the partials of rr = (r, r), g = (r0*, w)
struct EpiPsW {
  static constexpr int kIn = 2;
  static constexpr int kInStaged = kIn;
  static constexpr int kWcBatch = 4;
  static constexpr int kMinBlocks = 1;
  static constexpr bool kStencilPipe = false;
  static constexpr int kGatherBatch = 8;
  double* w;
  SolverState* st;
  DotSink sink;
  const double* in[kIn];  // r r0s
  DotsT<kDotsPsW> d;
  __device__ bool active() const { return gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() { d.zero(); }
  __device__ void row(long long i, double wv, const double* v) {
    w[i] = wv;
    if (!isfinite(wv)) report_nonfinite(st, PBS_TAG_AR, i);
    if (!sink.partials) return;
    d.step(DR, v[0], v[0]);
    d.step(DG, v[1], wv);
  }
  template <int NT, bool NAMED>
  __device__ void finish() { sink.finish<NT, NAMED>(d, st); }
};

// t = A w (tag "Aw") fused with the row-local p s z q y update and the omega
// phase's partials b = (q, y), e = (y, y), d = (q, q)
struct EpiPsA {
  static constexpr int kIn = 6;
  static constexpr int kInStaged = kIn;
  static constexpr int kWcBatch = 2;  // dot-carrying: register-bound
  static constexpr int kMinBlocks = 1;
  static constexpr bool kStencilPipe = false;
  static constexpr int kGatherBatch = 8;
  double *t, *p, *s, *z, *q, *y;
  SolverState* st;
  DotSink sink;
  const double* in[kIn];  // r p s w z v
  double alpha, beta, omega;
  DotsT<kDotsPsA> d;
  __device__ bool active() const { return gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() {
    d.zero();
    alpha = st->alpha;
    beta = st->beta;
    omega = st->omega;
  }
  __device__ void row(long long i, double tv, const double* v) {
    t[i] = tv;
    if (!isfinite(tv)) report_nonfinite(st, PBS_TAG_AW, i);
    const double rv = v[0], wv = v[3];
    const double pn = asdd(rv, beta, v[1], omega, v[2]);  // p = r + beta*(p - omega*s)
    const double sn = asdd(wv, beta, v[2], omega, v[4]);  // s = w + beta*(s - omega*z)
    const double zn = asdd(tv, beta, v[4], omega, v[5]);  // z = t + beta*(z - omega*v)
    const double qn = lc2(1.0, rv, -alpha, sn);           // q = r - alpha*s
    const double yn = lc2(1.0, wv, -alpha, zn);           // y = w - alpha*z
    p[i] = pn;
    s[i] = sn;
    z[i] = zn;
    q[i] = qn;
    y[i] = yn;
    if (!sink.partials) return;
    d.step(DB, qn, yn);
    d.step(DE, yn, yn);
    d.step(DD, qn, qn);
  }
  template <int NT, bool NAMED>
  __device__ void finish() { sink.finish<NT, NAMED>(d, st); }
};

// v = A z (tag "Az") fused with x, r, w and the beta phase's partials
// f = (r0*, r), r = (r, r), g = (r0*, w), a = (r0*, s), h = (r0*, z)
struct EpiPsB {
  static constexpr int kIn = 8;
  static constexpr int kInStaged = kIn;
  static constexpr int kWcBatch = 2;  // dot-carrying: register-bound
  static constexpr int kMinBlocks = 1;
  static constexpr bool kStencilPipe = false;
  static constexpr int kGatherBatch = 8;
  double *v, *x, *r, *w;
  SolverState* st;
  DotSink sink;
  const double* in[kIn];  // x p q y t r0s s z
  double alpha, omega;
  DotsT<kDotsPsB> d;
  __device__ bool active() const { return gate_all(st); }
  __device__ void on_skip() const {}
  __device__ void init() {
    d.zero();
    alpha = st->alpha;
    omega = st->omega;
  }
  __device__ void row(long long i, double vv, const double* in8) {
    v[i] = vv;
    if (!isfinite(vv)) report_nonfinite(st, PBS_TAG_AZ, i);
    const double qv = in8[2], yv = in8[3];
    x[i] = lc3(1.0, in8[0], alpha, in8[1], omega, qv);   // x = x + alpha*p + omega*q
    const double rn = lc2(1.0, qv, -omega, yv);           // r = q - omega*y
    const double wn = asdd(yv, -omega, in8[4], alpha, vv);  // w = y - omega*(t - alpha*v)
    r[i] = rn;
    w[i] = wn;
    if (!sink.partials) return;
    const double r0 = in8[5];
    d.step(DF, r0, rn);
    d.step(DR, rn, rn);
    d.step(DG, r0, wn);
    d.step(DA, r0, in8[6]);
    d.step(DH, r0, in8[7]);
  }
  template <int NT, bool NAMED>
  __device__ void finish() { sink.finish<NT, NAMED>(d, st); }
};

// --------------------------------------------------- CSR pipelined engine

constexpr int kPipeRows = 256;        // rows per block = consumer threads
constexpr int kPipeChunkMax = 4096;   // nonzeros per chunk stage (runtime <= this)
constexpr int kConsumerWarps = kPipeRows / 32;
constexpr int kPipeThreads = kPipeRows + 32;  // + one producer warp
constexpr int kMaxStages = 8;
constexpr int kMaxWin = 4;            // x windows per row block
constexpr int kMaxWinElems = 4096;    // staged x elements per row block (32 KiB)
constexpr int kBandMaxElems = 16384;  // band mode's circular x buffer, at most (128 KiB)

__host__ __device__ constexpr size_t align128(size_t b) { return (b + 127) / 128 * 128; }

// x windows: every column of row i lies in one of [i + wmin[c], i + wmax[c]]
// (offset clusters measured at upload); for a 256-row block starting at r0 the
// producer stages x[r0 + wmin[c] .. r0 + 255 + wmax[c]] per cluster.  nwin = 0:
// offsets too spread (e.g. wide random bands) -> gather x from global memory.
struct XWin {
  int nwin;
  int wmin[kMaxWin], wmax[kMaxWin];
  int cap[kMaxWin];  // staged elements reserved per cluster (even)
  int total;         // sum of cap
  // band mode (nwin == 0, band_s > 0): every row's offsets lie in
  // [band_lo, band_hi] but the span is too wide for per-block windows.  Each
  // CTA then takes a contiguous run of row blocks and keeps x in a circular
  // shared buffer of band_s doubles, x[g] at g % band_s, adding only each
  // block's new columns.
  int band_s;
  int band_lo, band_hi;
};

struct BlockHdr {
  long long r0, base, end;
  int nr, dr, nch, pad;
  long long ws[kMaxWin];  // first staged column per window (16-byte aligned)
};

struct ChunkHdr {
  long long c0, c1;
  int dv, dci, last, pad;
};

// block slot: header, row_ptr slice, x windows, epilogue inputs
struct BlockLayout {
  size_t rp, xw, ein, bytes;
  __host__ __device__ BlockLayout(int xw_total, int kin) {
    rp = 256;
    xw = rp + align128(sizeof(long long) * (kPipeRows + 2));
    ein = xw + align128(sizeof(double) * (xw_total > 0 ? xw_total : 2));
    bytes = ein + align128(sizeof(double) * (kPipeRows + 2) * (kin > 0 ? kin : 1));
  }
};

// chunk stage: header, values, column stream (ch nonzeros; int32 col_idx or
// u16 window-local columns, colb bytes each, 16-byte-aligned copy slack)
struct ChunkLayout {
  size_t v, ci, bytes;
  __host__ __device__ ChunkLayout(int ch, int colb) {
    v = 128;
    ci = v + align128(sizeof(double) * (ch + 2));
    bytes = ci + align128((size_t)colb * (ch + 32 / colb));
  }
};
constexpr size_t kPipeBarrierBytes = 512;

// Launched with programmatic dependent launch: the CTA comes up while the
// previous kernel drains, the producer streams its first block's nonzeros
// (the matrix does not depend on the previous kernel), and only then does
// every thread wait for the previous grid (griddep_wait) and take the CTA's
// one gate decision.  Consumers release the next kernel's launch once their
// rows are written, before the dot reduction / check tail.
// MINB: resident CTAs per SM the instantiation is compiled for.  2 (96
// registers) is the window-mode default; the 1-CTA layouts (band mode,
// config 4's long rows with extra chunk stages) get their own instantiation
// with the register room for 8 staged products in flight per row
// (profiles/sweeps/r1_band_ilp.log: config 3, 692 -> 615 us per iteration).
template <class Epi, bool SI = true, int MINB = 2>
__global__ void __launch_bounds__(kPipeThreads, MINB) csr_pipe_kernel(CsrView A, const double* __restrict__ x,
                                                                   Epi epi, XWin W, int bslots, int cstages,
                                                                   int chunk) {
  constexpr bool stage_in = SI;
  __shared__ int go;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* cfull = reinterpret_cast<uint64_t*>(smem);
  uint64_t* cempty = cfull + kMaxStages;
  uint64_t* bfull = cempty + kMaxStages;
  uint64_t* bempty = bfull + kMaxStages;
  // stage_in = 0: the epilogue inputs are not staged (their slot space goes
  // to a second resident CTA when x windows are wide, e.g. 27-point rows);
  // consumers load them from global memory while the row's products run
  const BlockLayout BL(W.total, stage_in ? Epi::kInStaged : 0);
  const ChunkLayout CL(chunk, A.wc ? 2 : 4);
  double* xband = reinterpret_cast<double*>(smem + kPipeBarrierBytes);  // band mode only
  unsigned char* blk0 = smem + kPipeBarrierBytes + (size_t)W.band_s * sizeof(double);
  unsigned char* chk0 = blk0 + (size_t)bslots * BL.bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < cstages; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], kConsumerWarps);
    }
    for (int s = 0; s < bslots; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long nrows = A.row_hi - A.row_lo;
  const long long nblk_all = (nrows + kPipeRows - 1) / kPipeRows;
  // blocks of this CTA: strided (blockIdx.x, + gridDim.x, ...) or, in band
  // mode, a contiguous run [first_blk, nblk)
  const bool band = W.band_s > 0;
  long long first_blk = blockIdx.x, nblk = nblk_all, bstep = gridDim.x;
  if (band) {
    const long long per = (nblk_all + gridDim.x - 1) / gridDim.x;
    first_blk = (long long)blockIdx.x * per;
    nblk = min(nblk_all, first_blk + per);
    bstep = 1;
  }

  if (warp == kConsumerWarps) {
    // ----------------------------------------------------------- producer
    // The whole warp: row-block bounds for the next 32 blocks come from one
    // warp-wide load (no dependent load per block), and the block's bulk
    // copies are issued by different lanes in parallel.
    int cs = 0, bs = 0;
    uint32_t cph = 0, bph = 0;
    long long pf_base = 0, pf_end = 0;
    bool gated = false;
    int issued = 0;  // chunk stages filled before the gate
    auto gate = [&]() -> bool {
      gated = true;
      griddep_wait();
      cta_sync2<kPipeThreads>();  // thread 0 (a consumer) has taken the gate decision
      if (go) return true;
      for (int s2 = 0; s2 < issued; ++s2) mbar_wait(&cfull[s2], 0);  // let the early copies land
      return false;
    };
    long long xhi = 0;  // band mode: x staged up to here (exclusive)
    bool opp_ready = false;
    if (nblk <= first_blk && !gate()) return;
    for (long long blk = first_blk, q = 0; blk < nblk; blk += bstep, ++q) {
      const int slot = (int)(q & 31);
      if (slot == 0) {  // prefetch bounds of blocks q .. q+31 of this CTA
        const long long b2 = blk + (long long)lane * bstep;
        if (b2 < nblk) {
          const long long rr0 = A.row_lo + b2 * kPipeRows;
          const long long rr1 = min(A.row_hi, rr0 + kPipeRows);
          pf_base = __ldg(A.rp + rr0);
          pf_end = __ldg(A.rp + rr1);
        }
      }
      const long long base = __shfl_sync(0xffffffffu, pf_base, slot);
      const long long end = __shfl_sync(0xffffffffu, pf_end, slot);
      const long long r0 = A.row_lo + blk * kPipeRows;
      const long long r0a = r0 & ~1LL;
      const int nr = (int)min((long long)kPipeRows, A.row_hi - r0);
      const int dr = (int)(r0 - r0a);
      const long long nch = end > base ? (end - base + chunk - 1) / chunk : 1;
      const uint32_t brp = (uint32_t)(((nr + dr + 2) & ~1) * sizeof(long long));
      const uint32_t bin = (uint32_t)(((nr + dr + 1) & ~1) * sizeof(double));
      // chunk stage c of this block: the block's nonzero range
      auto issue_chunk = [&](long long c) {
        mbar_wait(&cempty[cs], cph ^ 1);
        unsigned char* st = chk0 + (size_t)cs * CL.bytes;
        const long long c0 = base + c * chunk;
        const long long c1 = min(end, c0 + chunk);
        const long long c0a = c0 & ~1LL, c1a = (c1 + 1) & ~1LL;
        // column stream: window-local u16 indices (8 per 16 bytes) or int32
        const long long cal = A.wc ? 7 : 3;
        const long long c0b = c0 & ~cal, c1b = (c1 + cal) & ~cal;
        const uint32_t bv = (uint32_t)((c1a - c0a) * sizeof(double));
        const uint32_t bc = (uint32_t)((c1b - c0b) * (A.wc ? sizeof(unsigned short) : sizeof(int)));
        if (lane == 0) {
          ChunkHdr* h = reinterpret_cast<ChunkHdr*>(st);
          h->c0 = c0;
          h->c1 = c1;
          h->dv = (int)(c0 - c0a);
          h->dci = (int)(c0 - c0b);
          h->last = c == nch - 1;
          mbar_arrive_expect_tx(&cfull[cs], bv + bc);
        }
        __syncwarp();
        if (lane == 0 && bv) bulk_g2s(st + CL.v, A.v + c0a, bv, &cfull[cs]);
        if (lane == 1 && bc)
          bulk_g2s(st + CL.ci, A.wc ? (const void*)(A.wc + c0b) : (const void*)(A.ci + c0b), bc, &cfull[cs]);
        if (++cs == cstages) {
          cs = 0;
          cph ^= 1;
        }
      };
      // first block: the matrix chunks that fit the free stages go before the
      // gate (they do not depend on the previous kernel); the rest follow the
      // block slot, as on every later block (consumers need the slot first)
      long long cfirst = 0;
      if (!gated) {
        cfirst = nch < cstages ? nch : cstages;
        for (long long c = 0; c < cfirst; ++c) issue_chunk(c);
        issued = (int)cfirst;
        if (!gate()) return;
      }
      // an opportunistic epilogue runs (and its inputs are staged) only for
      // blocks whose coefficients already exist (see EpiOpp)
      bool fuse_in = true;
      if constexpr (EpiOpp<Epi>::value) {  // polled until seen once (it never goes back)
        if (!opp_ready) opp_ready = __shfl_sync(0xffffffffu, lane == 0 ? epi.ready() : false, 0);
        fuse_in = opp_ready;
      }
      // x windows of this block (every lane computes them; lane 1+c copies window c)
      long long wlo[kMaxWin];
      uint32_t wbytes[kMaxWin];
      uint32_t total = brp + (stage_in && fuse_in ? Epi::kInStaged * bin : 0u);
#pragma unroll
      for (int c = 0; c < kMaxWin; ++c) {
        wlo[c] = 0x7fffffff;
        wbytes[c] = 0;
        if (c < W.nwin) {
          long long lo = r0 + W.wmin[c], hi = r0 + nr - 1 + W.wmax[c] + 1;
          if (lo < 0) lo = 0;
          if (hi > A.n_cols) hi = A.n_cols;
          if (hi > lo) {  // an empty window (past either end of x) copies nothing
            const long long loa = lo & ~1LL, hia = (hi + 1) & ~1LL;
            wlo[c] = loa;
            wbytes[c] = (uint32_t)((hia - loa) * sizeof(double));
            total += wbytes[c];
          } else {
            wlo[c] = lo & ~1LL;
          }
        }
      }
      // band mode: the block's new columns [xhi, hi), as up to two pieces of
      // the circular buffer (lanes 1 and 2 copy them)
      long long bnd0 = 0, bnd1 = 0;
      uint32_t bb0 = 0, bb1 = 0;
      if (band) {
        long long lo = r0 + W.band_lo, hi = r0 + nr - 1 + W.band_hi + 1;
        if (lo < 0) lo = 0;
        if (hi > A.n_cols) hi = A.n_cols;
        lo &= ~1LL;
        hi = (hi + 1) & ~1LL;
        if (q == 0 || lo >= xhi) xhi = lo;  // first block of the run: fill from lo
        if (hi > xhi) {
          const long long room = W.band_s - xhi % W.band_s;
          const long long n0 = min(hi - xhi, room);
          bnd0 = xhi;
          bb0 = (uint32_t)(n0 * sizeof(double));
          if (hi - xhi > n0) {
            bnd1 = xhi + n0;
            bb1 = (uint32_t)((hi - xhi - n0) * sizeof(double));
          }
          total += bb0 + bb1;
          xhi = hi;
        }
      }
      mbar_wait(&bempty[bs], bph ^ 1);
      unsigned char* bst = blk0 + (size_t)bs * BL.bytes;
      if (lane == 0) {
        BlockHdr* bh = reinterpret_cast<BlockHdr*>(bst);
        bh->r0 = r0;
        bh->base = base;
        bh->end = end;
        bh->nr = nr;
        bh->dr = dr;
        bh->nch = (int)nch;
        bh->pad = fuse_in ? 1 : 0;
#pragma unroll
        for (int c = 0; c < kMaxWin; ++c) bh->ws[c] = wlo[c];
        mbar_arrive_expect_tx(&bfull[bs], total);
      }
      __syncwarp();
      if (lane == 0) {
        bulk_g2s(bst + BL.rp, A.rp + r0a, brp, &bfull[bs]);
      } else if (band && lane <= 2) {
        // the slot of block blk - bslots is free, so no block still being
        // consumed needs the columns these pieces overwrite
        // (band_s >= band span + 2 * 256 + 4, checked at upload)
        if (lane == 1 && bb0) bulk_g2s(xband + bnd0 % W.band_s, x + bnd0, bb0, &bfull[bs]);
        if (lane == 2 && bb1) bulk_g2s(xband + bnd1 % W.band_s, x + bnd1, bb1, &bfull[bs]);
      } else if (lane <= W.nwin) {
        // lane 1+c copies window c (static indexing keeps wlo/wbytes in registers)
        int soff = 0;
#pragma unroll
        for (int cc = 0; cc < kMaxWin; ++cc) {
          if (cc == lane - 1 && wbytes[cc])
            bulk_g2s(bst + BL.xw + (size_t)soff * sizeof(double), x + wlo[cc], wbytes[cc], &bfull[bs]);
          soff += cc < W.nwin ? W.cap[cc] : 0;
        }
      } else if (stage_in && fuse_in && lane >= 8 && lane < 8 + Epi::kInStaged) {
        const int e = lane - 8;
        bulk_g2s(bst + BL.ein + (size_t)e * (kPipeRows + 2) * sizeof(double), epi.in[e] + r0a, bin, &bfull[bs]);
      }
      if (++bs == bslots) {
        bs = 0;
        bph ^= 1;
      }
      for (long long c = cfirst; c < nch; ++c) issue_chunk(c);
    }
    return;
  }

  // ------------------------------------------------------------- consumers
  griddep_wait();
  if (threadIdx.x == 0) {
    go = epi.active();  // one gate decision per CTA
    if (!go && blockIdx.x == 0) epi.on_skip();
  }
  cta_sync2<kPipeThreads>();
  if (!go) return;
  Epi e = epi;
  e.init();
  const int t = threadIdx.x;
  int cs = 0, bs = 0;
  uint32_t cph = 0, bph = 0;
  for (long long blk = first_blk; blk < nblk; blk += bstep) {
    mbar_wait(&bfull[bs], bph);
    const unsigned char* bst = blk0 + (size_t)bs * BL.bytes;
    const BlockHdr* bhp = reinterpret_cast<const BlockHdr*>(bst);
    const int nr = bhp->nr, dr = bhp->dr;
    const long long r0 = bhp->r0;
    const bool fused = !EpiOpp<Epi>::value || bhp->pad;  // the producer's decision for this block
    long long my_s = 0, my_e = 0;
    double inr[Epi::kIn > 0 ? Epi::kIn : 1];
    if (t < nr) {
      const long long* rps = reinterpret_cast<const long long*>(bst + BL.rp);
      my_s = rps[t + dr];
      my_e = rps[t + dr + 1];
      // inputs the producer does not stage: in flight during the row's products
      if (fused) {
#pragma unroll
        for (int k = 0; k < Epi::kIn; ++k)
          if (k >= Epi::kInStaged || !stage_in) inr[k] = __ldg(e.in[k] + r0 + t);
      }
    }
    // staged x windows (or the band buffer), addressed by the window-local
    // column stream
    const double* xw = band ? xband : reinterpret_cast<const double*>(bst + BL.xw);
    double acc = 0.0;
    for (long long c = 0;; ++c) {
      mbar_wait(&cfull[cs], cph);
      const unsigned char* st = chk0 + (size_t)cs * CL.bytes;
      const ChunkHdr h = *reinterpret_cast<const ChunkHdr*>(st);
      if (t < nr) {
        // chunk-local indices: smem addressing stays 32-bit for any nnz
        const double* vs = reinterpret_cast<const double*>(st + CL.v) + h.dv;
        const int lo = (int)(max(my_s, h.c0) - h.c0), hi = (int)(min(my_e, h.c1) - h.c0);
        if (A.wc) {
          // staged window index per nonzero: no window search, half the bytes
          const unsigned short* wcs = reinterpret_cast<const unsigned short*>(st + CL.ci) + h.dci;
          constexpr int U = MINB == 1 ? PBS_WCB_ONE : Epi::kWcBatch;
          for (int k = lo; k < hi; k += U) {
            double vv[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (k + u < hi) {
                vv[u] = vs[k + u];
                xv[u] = xw[wcs[k + u]];
              }
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (k + u < hi) acc = add(acc, mul(vv[u], xv[u]));
          }
        } else {
          // no windows: x gathered from global memory (L2)
          const int* cis = reinterpret_cast<const int*>(st + CL.ci) + h.dci;
          constexpr int U = Epi::kGatherBatch;
          for (int k = lo; k < hi; k += U) {
            double vv[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (k + u < hi) {
                vv[u] = vs[k + u];
                xv[u] = __ldg(x + cis[k + u]);
              }
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (k + u < hi) acc = add(acc, mul(vv[u], xv[u]));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty[cs]);
      if (++cs == cstages) {
        cs = 0;
        cph ^= 1;
      }
      if (h.last) break;
    }
    if (t < nr) {
      const double* ein = reinterpret_cast<const double*>(bst + BL.ein);
      if (stage_in && fused) {
#pragma unroll
        for (int k = 0; k < Epi::kInStaged; ++k) inr[k] = ein[k * (kPipeRows + 2) + t + dr];
      }
      if constexpr (EpiOpp<Epi>::value) {
        e.row_opp(r0 + t, acc, inr, fused);
        if (!fused && t == 0) e.defer(r0);
      } else {
        e.row(r0 + t, acc, inr);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bempty[bs]);
    if (++bs == bslots) {
      bs = 0;
      bph ^= 1;
    }
  }
  griddep_launch();  // rows written: the next kernel may start its prologue
  e.template finish<kPipeRows, true>();
}

// ---------------------------------------------- stencil pipelined engine

// Matrix-free counterpart of csr_pipe_kernel: the producer warp stages, per
// 256-row block, the x windows the stencil reaches (one per offset cluster:
// the z-1 / z / z+1 plane slices of a 3D stencil) and the epilogue inputs
// into a ring of block slots with bulk async copies; consumers compute their
// row from shared memory, neighbours in ascending flattened offset (the CSR
// column order), so the result is bitwise the CSR engine's.
struct StencilWin {
  int pw[kMaxStencil];  // window of each stencil point
  // Blocks whose windows all start in the grid (r0 >= clamp_r0) stage window
  // c from r0 + (wmin[c] & ~1), so row t's neighbour p sits at the staged
  // index t + kfix[p], a constant; only the first blocks (windows clamped at
  // row 0) look the window start up per block.
  int kfix[kMaxStencil];
  long long clamp_r0;
};

// resident CTAs per SM the staged stencil engine is compiled for (register cap)
#ifndef PBS_SPIPE_MINB
#define PBS_SPIPE_MINB 2
#endif

template <class Epi, int DIM, int NP>
__global__ void __launch_bounds__(kPipeThreads, PBS_SPIPE_MINB) stencil_pipe_kernel(const __grid_constant__ StencilView S,
                                                                       const double* __restrict__ x, Epi epi,
                                                                       XWin W, StencilWin SW, int bslots) {
  __shared__ int go;
  griddep_wait();  // PDL: everything here reads the previous kernel's output
  if (threadIdx.x == 0) {
    go = epi.active();
    if (!go && blockIdx.x == 0) epi.on_skip();
  }
  __syncthreads();
  if (!go) return;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem);
  uint64_t* bempty = bfull + kMaxStages;
  const BlockLayout BL(W.total, Epi::kInStaged);
  unsigned char* blk0 = smem + kPipeBarrierBytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < bslots; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long nrows = S.row_hi - S.row_lo;
  const long long nblk = (nrows + kPipeRows - 1) / kPipeRows;
  if (warp == kConsumerWarps) {
    // Every lane owns one copy stream of the slot and works out its own source
    // and size per block (lanes 1..nwin the x windows, lanes 8.. the epilogue
    // inputs); lane 0 writes the header.  One warp computing every window in
    // every lane was the critical path of the staged engines (sell.cuh).
    int bs = 0;
    uint32_t bph = 0;
    const BlockLayout BLp(W.total, Epi::kInStaged);
    const int role_win = lane >= 1 && lane <= W.nwin ? lane - 1 : -1;
    const int role_in = lane >= 8 && lane < 8 + Epi::kInStaged ? lane - 8 : -1;
    long long wmin_l = 0, wmax_l = 0;
    uint32_t dst_l = 0;
    const double* src_l = nullptr;
    if (role_win >= 0) {
      int so = 0;
#pragma unroll
      for (int cc = 0; cc < kMaxWin; ++cc) {
        if (cc == role_win) {
          wmin_l = W.wmin[cc];
          wmax_l = W.wmax[cc];
          dst_l = (uint32_t)(BLp.xw + (size_t)so * sizeof(double));
        }
        so += cc < W.nwin ? W.cap[cc] : 0;
      }
      src_l = x;
    } else if (role_in >= 0) {
      dst_l = (uint32_t)(BLp.ein + (size_t)role_in * (kPipeRows + 2) * sizeof(double));
#pragma unroll
      for (int k = 0; k < Epi::kInStaged; ++k)
        if (k == role_in) src_l = epi.in[k];
    }
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
      const long long r0 = S.row_lo + blk * kPipeRows;
      const long long r0a = r0 & ~1LL;
      const int nr = (int)min((long long)kPipeRows, S.row_hi - r0);
      const int dr = (int)(r0 - r0a);
      const void* src = nullptr;
      uint32_t bytes = 0;
      long long ws_l = 0x7fffffff;  // first staged column of this lane's window
      if (role_win >= 0) {
        long long lo = r0 + wmin_l, hi = r0 + nr + wmax_l;
        if (lo < S.xlo) lo = S.xlo;
        if (hi > S.xhi) hi = S.xhi;
        ws_l = lo & ~1LL;
        if (hi > lo) {
          const long long hia = (hi + 1) & ~1LL;
          src = src_l + ws_l;
          bytes = (uint32_t)((hia - ws_l) * sizeof(double));
        }
      } else if (role_in >= 0) {
        src = src_l + r0a;
        bytes = (uint32_t)(((nr + dr + 1) & ~1) * sizeof(double));
      }
      const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
      mbar_wait(&bempty[bs], bph ^ 1);
      unsigned char* bst = blk0 + (size_t)bs * BLp.bytes;
      BlockHdr* bh = reinterpret_cast<BlockHdr*>(bst);
      if (role_win >= 0) bh->ws[role_win] = ws_l;
      if (lane == 0) {
        bh->r0 = r0;
        bh->nr = nr;
        bh->dr = dr;
      }
      __syncwarp();
      if (lane == 0) {
        if (total)
          mbar_arrive_expect_tx(&bfull[bs], total);
        else
          mbar_arrive(&bfull[bs]);  // unreachable with kIn > 0 or windows
      }
      __syncwarp();
      if (bytes) bulk_g2s(bst + dst_l, src, bytes, &bfull[bs]);
      if (++bs == bslots) {
        bs = 0;
        bph ^= 1;
      }
    }
    return;
  }
  Epi e = epi;
  e.init();
  const int t = threadIdx.x;
  int bs = 0;
  uint32_t bph = 0;
  const int npts = NP > 0 ? NP : S.npts;
  for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    mbar_wait(&bfull[bs], bph);
    const unsigned char* bst = blk0 + (size_t)bs * BL.bytes;
    const BlockHdr* bhp = reinterpret_cast<const BlockHdr*>(bst);
    const int nr = bhp->nr, dr = bhp->dr;
    const long long r0 = bhp->r0;
    if (t < nr) {
      const long long i = r0 + t;
      const long long gi = i + S.g0;  // grid row (slab-local rows are offset)
      int c[3] = {0, 0, 0};
      if (DIM == 3) {
        const long long z = S.dk2.div(gi);
        const long long rem = gi - z * S.k2;
        const long long yy = S.dk.div(rem);
        c[0] = (int)z;
        c[1] = (int)yy;
        c[2] = (int)(rem - yy * S.k);
      } else if (DIM == 2) {
        const long long yy = S.dk.div(gi);
        c[1] = (int)yy;
        c[2] = (int)(gi - yy * S.k);
      } else {
        c[2] = (int)gi;
      }
      const double* xw = reinterpret_cast<const double*>(bst + BL.xw);
      const unsigned vm = S.valid_mask(c, DIM);
      double acc = 0.0;
      if (r0 >= SW.clamp_r0 && !(r0 & 1)) {
        // interior blocks: neighbour p at the constant staged offset t + kfix[p]
        const double* xt = xw + t;
#pragma unroll
        for (int p = 0; p < (NP > 0 ? NP : kMaxStencil); ++p) {
          if (NP == 0 && p >= npts) break;
          if ((vm >> p) & 1u) acc = add(acc, mul(S.coef[p], xt[SW.kfix[p]]));
        }
      } else {
        // window base per cluster: x[col] = xw[col - wsb[w]]
        int wsb[kMaxWin];
        {
          int soff = 0;
#pragma unroll
          for (int cc = 0; cc < kMaxWin; ++cc) {
            wsb[cc] = cc < W.nwin ? (int)bhp->ws[cc] - soff : 0;
            soff += cc < W.nwin ? W.cap[cc] : 0;
          }
        }
#pragma unroll
        for (int p = 0; p < (NP > 0 ? NP : kMaxStencil); ++p) {
          if (NP == 0 && p >= npts) break;
          if ((vm >> p) & 1u) {
            const int col = (int)(i + S.foff[p]);
            acc = add(acc, mul(S.coef[p], xw[col - wsb[SW.pw[p]]]));
          }
        }
      }
      double inr[Epi::kIn > 0 ? Epi::kIn : 1];
#pragma unroll
      for (int k = Epi::kInStaged; k < Epi::kIn; ++k) inr[k] = __ldg(e.in[k] + i);
      const double* ein = reinterpret_cast<const double*>(bst + BL.ein);
#pragma unroll
      for (int k = 0; k < Epi::kInStaged; ++k) inr[k] = ein[k * (kPipeRows + 2) + t + dr];
      e.row(i, acc, inr);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bempty[bs]);
    if (++bs == bslots) {
      bs = 0;
      bph ^= 1;
    }
  }
  griddep_launch();
  e.template finish<kPipeRows, true>();
}

// ------------------------------------------- CSR thread-per-row engine

// One thread per row at full occupancy (no shared memory, so L1 keeps the
// matrix sectors a warp's strided row loads share): each thread loads its
// row's epilogue inputs first, then its nonzeros in batches of U (values,
// col_idx, x gathers all in flight), and accumulates in ascending column
// order — bitwise the reference's row sum.
template <class Epi, bool LATE>
__global__ void __launch_bounds__(kThreads, LATE ? 4 : 1) csr_tpr_kernel(CsrView A, const double* __restrict__ x,
                                                                       Epi epi) {
  __shared__ int go;
  if (threadIdx.x == 0) {
    go = epi.active();
    if (!go && blockIdx.x == 0) epi.on_skip();
  }
  __syncthreads();
  if (!go) return;
  Epi e = epi;
  e.init();
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = A.row_lo + (long long)blockIdx.x * kThreads + threadIdx.x; i < A.row_hi; i += stride) {
    double inr[Epi::kIn > 0 ? Epi::kIn : 1];
    if (!LATE) {
#pragma unroll
      for (int k = 0; k < Epi::kIn; ++k) inr[k] = epi.in[k][i];
    }
    const long long s0 = __ldg(A.rp + i), s1 = __ldg(A.rp + i + 1);
    const int len = (int)(s1 - s0);
    const double* __restrict__ vr = A.v + s0;
    const int* __restrict__ cr = A.ci + s0;
    double acc = 0.0;
    constexpr int U = 8;
    for (int k = 0; k < len; k += U) {
      double vv[U], xv[U];
      int cc[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k + u < len) {
          vv[u] = __ldcs(vr + k + u);
          cc[u] = __ldcs(cr + k + u);
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k + u < len) xv[u] = __ldg(x + cc[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k + u < len) acc = add(acc, mul(vv[u], xv[u]));
    }
    if (LATE) {
#pragma unroll
      for (int k = 0; k < Epi::kIn; ++k) inr[k] = epi.in[k][i];
    }
    e.row(i, acc, inr);
  }
  e.template finish<kThreads, false>();
}

// ------------------------------------------------------ stencil engine

// NP > 0: compile-time point count (fully unrolled); NP == 0: runtime npts
template <class Epi, int DIM, int NP>
__global__ void __launch_bounds__(kThreads, Epi::kMinBlocks) stencil_spmv_kernel(const __grid_constant__ StencilView S,
                                                                const double* __restrict__ x, Epi epi) {
  __shared__ int go;
  griddep_wait();  // PDL: everything here reads the previous kernel's output
  if (threadIdx.x == 0) {
    go = epi.active();  // one gate decision per CTA
    if (!go && blockIdx.x == 0) epi.on_skip();
  }
  __syncthreads();
  if (!go) return;
  Epi e = epi;
  e.init();
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = S.row_lo + (long long)blockIdx.x * kThreads + threadIdx.x; i < S.row_hi; i += stride) {
    const long long gi = i + S.g0;  // grid row (slab-local rows are offset)
    int c[3] = {0, 0, 0};
    if (DIM == 3) {
      const long long z = S.dk2.div(gi);
      const long long rem = gi - z * S.k2;
      const long long yy = S.dk.div(rem);
      c[0] = (int)z;
      c[1] = (int)yy;
      c[2] = (int)(rem - yy * S.k);
    } else if (DIM == 2) {
      const long long yy = S.dk.div(gi);
      c[1] = (int)yy;
      c[2] = (int)(gi - yy * S.k);
    } else {
      c[2] = (int)gi;
    }
    double inr[Epi::kIn > 0 ? Epi::kIn : 1];
#pragma unroll
    for (int k = 0; k < Epi::kIn; ++k) inr[k] = epi.in[k][i];
    const int npts = NP > 0 ? NP : S.npts;
    const unsigned vm = S.valid_mask(c, DIM);
    double acc = 0.0;
#pragma unroll
    for (int p = 0; p < (NP > 0 ? NP : kMaxStencil); ++p) {
      if (NP == 0 && p >= npts) break;
      if ((vm >> p) & 1u) acc = add(acc, mul(S.coef[p], __ldg(x + i + S.foff[p])));
    }
    e.row(i, acc, inr);
  }
  griddep_launch();
  e.template finish<kThreads, false>();
}

}  // namespace pbs
