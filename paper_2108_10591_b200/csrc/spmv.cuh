// spmv.cuh — SpMV engines with fused epilogues (sm_100a).
//
// Two engines feed one epilogue interface (Epi::row(i, y) per output row,
// Epi::finish() once per thread at the end):
//
//  * csr_spmv: a CTA owns 256 consecutive rows at a time (grid-stride over
//    row blocks, grid = SMs x resident CTAs).  The row block's nonzeros are
//    streamed through shared memory in 2048-product chunks: coalesced,
//    evict-first loads of values / int32 col_idx, an L1-cached gather of x,
//    one rounded product per nonzero.  Each thread then sums its own row from
//    shared memory in ascending column order (kernels.py:95-100 order), so
//    the result is bitwise the reference's, while HBM sees each matrix byte
//    once and every lane does useful loads.
//  * stencil_spmv: matrix-free constant-coefficient stencil, one thread per
//    row, neighbours visited in ascending flattened offset (= CSR column
//    order), out-of-grid neighbours skipped (Dirichlet elimination) — bitwise
//    equal to the CSR of the same stencil.
//
// Epilogues (SURVEY §8(d) kernel plan):
//   EpiStore  y = A x                          (K1: As = A s; rr products)
//   EpiResid  r = b - A x  (+ r0s = r)         (setup; rr "r = b - A x")
//   EpiK3     Aw -> l, g, s updates + next 9 dot partials (solvers.py:717-723, 467-482)
//   EpiDots   s = A r + 9 dot partials          (setup s0 = A r0; rr s = A r)
//   EpiSS3    w = A u -> t, z, y, x, r updates  (ssBiCGSafe2, solvers.py:569-580)
#pragma once
#include "common.cuh"

namespace pbs {

struct CsrView {
  const long long* rp;
  const int* ci;
  const double* v;
  long long row_lo, row_hi;
};

struct StencilView {
  long long n, k, k2;
  int dim, npts;
  int off[kMaxStencil][3];     // (dz,)dy,dx per point, padded to 3 axes from the left
  long long foff[kMaxStencil]; // flattened offset
  double coef[kMaxStencil];
  long long row_lo, row_hi;
};

// ---------------------------------------------------------------- epilogues

struct EpiStore {
  double* y;
  SolverState* st;
  int tag;
  int spine;  // gate on run_spine instead of run_all
  __device__ bool active() const { return spine ? gate_spine(st) : gate_all(st); }
  __device__ void row(long long i, double v) {
    y[i] = v;
    if (tag && !isfinite(v)) report_nonfinite(st, tag, i);
  }
  __device__ void finish() {}
};

struct EpiResid {  // lincomb2(r, 1.0, b, -1.0, ax) after check_finite(ax)
  const double* b;
  double* r;
  double* r0s;  // nullable: also r0s = r (solvers.py:617)
  SolverState* st;
  __device__ bool active() const { return gate_all(st); }
  __device__ void row(long long i, double ax) {
    if (!isfinite(ax)) report_nonfinite(st, PBS_TAG_AX, i);
    double rv = lc2(1.0, b[i], -1.0, ax);
    r[i] = rv;
    if (r0s) r0s[i] = rv;
  }
  __device__ void finish() {}
};

struct Dots9 {
  double acc[kNumDots];
  __device__ void zero() {
#pragma unroll
    for (int j = 0; j < kNumDots; ++j) acc[j] = 0.0;
  }
  // _safe_batch pairs (solvers.py:471-481)
  __device__ void add_row(double s, double y, double r, double r0s, double t) {
    acc[DA] = add(acc[DA], mul(s, s));
    acc[DB] = add(acc[DB], mul(y, y));
    acc[DC] = add(acc[DC], mul(s, y));
    acc[DD] = add(acc[DD], mul(s, r));
    acc[DE] = add(acc[DE], mul(y, r));
    acc[DF] = add(acc[DF], mul(r0s, r));
    acc[DG] = add(acc[DG], mul(r0s, s));
    acc[DH] = add(acc[DH], mul(r0s, t));
    acc[DR] = add(acc[DR], mul(r, r));
  }
};

struct EpiDots {  // s = A r, then the batch partials over (s, y, r, r0s, t)
  double* s;
  const double *y, *r, *r0s, *t;
  double* partials;  // nullable: PBS_REDUCE_PLAN computes the batch separately
  SolverState* st;
  int tag;
  int spine;
  Dots9 d;
  __device__ bool active() const { return spine ? gate_spine(st) : gate_all(st); }
  __device__ void init() { d.zero(); }
  __device__ void row(long long i, double v) {
    s[i] = v;
    if (!isfinite(v)) report_nonfinite(st, tag, i);
    if (partials) d.add_row(v, y[i], r[i], r0s[i], t[i]);
  }
  __device__ void finish() {
    if (partials) block_reduce9(d.acc, partials + (size_t)blockIdx.x * kNumDots);
  }
};

struct EpiK3 {  // block 2 of the pipelined iteration, fused with the next batch
  const double* as;
  double *l, *g, *s;
  const double *y, *r, *r0s, *t;
  double* q_out;     // nullable (single-step parity: expose q)
  double* partials;  // nullable (PBS_REDUCE_PLAN)
  SolverState* st;
  double alpha, beta, zeta, eta;
  Dots9 d;
  __device__ bool active() const { return gate_all(st); }
  __device__ void init() {
    d.zero();
    alpha = st->alpha;
    beta = st->beta;
    zeta = st->zeta;
    eta = st->eta;
  }
  __device__ void row(long long i, double aw) {
    if (!isfinite(aw)) report_nonfinite(st, PBS_TAG_AW, i);
    const double asv = as[i];
    const double q = lc2(1.0, asv, beta, l[i]);                  // q = As + beta*l
    const double lv = lc2(1.0, q, -1.0, aw);                     // l = q - A w
    const double gv = lc3(zeta, asv, eta, g[i], -alpha, aw);     // g = zeta As + eta g - alpha Aw
    const double sv = lc3(1.0, s[i], -alpha, q, -1.0, gv);       // s = s - alpha q - g
    l[i] = lv;
    g[i] = gv;
    s[i] = sv;
    if (q_out) q_out[i] = q;
    if (partials) d.add_row(sv, y[i], r[i], r0s[i], t[i]);
  }
  __device__ void finish() {
    if (partials) block_reduce9(d.acc, partials + (size_t)blockIdx.x * kNumDots);
  }
};

struct EpiSS3 {  // ssBiCGSafe2 tail: w = A u, then t, z, y, x, r (solvers.py:569-580)
  double* w;
  const double *o, *s, *u, *p;
  double *t, *z, *y, *x, *r;
  SolverState* st;
  double alpha, zeta, eta;
  __device__ bool active() const { return gate_all(st); }
  __device__ void init() {
    alpha = st->alpha;
    zeta = st->zeta;
    eta = st->eta;
  }
  __device__ void row(long long i, double wv) {
    if (!isfinite(wv)) report_nonfinite(st, PBS_TAG_AU, i);
    const double ov = o[i];
    const double yv = lc3(zeta, s[i], eta, y[i], -alpha, wv);
    const double zv = lc3(zeta, r[i], eta, z[i], -alpha, u[i]);
    w[i] = wv;
    t[i] = lc2(1.0, ov, -1.0, wv);
    z[i] = zv;
    y[i] = yv;
    x[i] = lc3(1.0, x[i], alpha, p[i], 1.0, zv);
    r[i] = lc3(1.0, r[i], -alpha, ov, -1.0, yv);
  }
  __device__ void finish() {}
};

template <class E>
__device__ __forceinline__ auto epi_init(E& e, int) -> decltype(e.init(), void()) { e.init(); }
template <class E>
__device__ __forceinline__ void epi_init(E&, long) {}

// ------------------------------------------------------------------- engines

template <class Epi>
__global__ void __launch_bounds__(kThreads) csr_spmv_kernel(CsrView A, const double* __restrict__ x,
                                                            Epi epi) {
  if (!epi.active()) return;
  Epi e = epi;
  epi_init(e, 0);
  __shared__ double prod[kChunk];
  __shared__ long long srp[kThreads + 1];
  constexpr int U = kChunk / kThreads;
  const int t = threadIdx.x;
  const long long nrows = A.row_hi - A.row_lo;
  const long long nblk = (nrows + kThreads - 1) / kThreads;
  for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const long long r0 = A.row_lo + blk * kThreads;
    const int nr = (int)min((long long)kThreads, A.row_hi - r0);
    for (int i = t; i <= nr; i += kThreads) srp[i] = __ldg(A.rp + r0 + i);
    __syncthreads();
    const long long base = srp[0], end = srp[nr];
    long long my_s = 0, my_e = 0;
    if (t < nr) {
      my_s = srp[t];
      my_e = srp[t + 1];
    }
    double acc = 0.0;
    for (long long c0 = base; c0 < end; c0 += kChunk) {
      const int len = (int)min((long long)kChunk, end - c0);
      double vv[U];
      int cc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = t + u * kThreads;
        if (k < len) {
          vv[u] = __ldcs(A.v + c0 + k);
          cc[u] = __ldcs(A.ci + c0 + k);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = t + u * kThreads;
        if (k < len) prod[k] = mul(vv[u], __ldg(x + cc[u]));
      }
      __syncthreads();
      if (t < nr) {
        const long long lo = max(my_s, c0), hi = min(my_e, c0 + len);
        for (long long k = lo; k < hi; ++k) acc = add(acc, prod[k - c0]);
      }
      __syncthreads();
    }
    if (t < nr) e.row(r0 + t, acc);
  }
  e.finish();
}

// NP > 0: compile-time point count (fully unrolled); NP == 0: runtime npts
template <class Epi, int DIM, int NP>
__global__ void __launch_bounds__(kThreads) stencil_spmv_kernel(const __grid_constant__ StencilView S,
                                                                const double* __restrict__ x, Epi epi) {
  if (!epi.active()) return;
  Epi e = epi;
  epi_init(e, 0);
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = S.row_lo + (long long)blockIdx.x * kThreads + threadIdx.x; i < S.row_hi; i += stride) {
    int c[3] = {0, 0, 0};
    if (DIM == 3) {
      const long long z = i / S.k2;
      const long long rem = i - z * S.k2;
      const long long yy = rem / S.k;
      c[0] = (int)z;
      c[1] = (int)yy;
      c[2] = (int)(rem - yy * S.k);
    } else if (DIM == 2) {
      const long long yy = i / S.k;
      c[1] = (int)yy;
      c[2] = (int)(i - yy * S.k);
    } else {
      c[2] = (int)i;
    }
    const int km1 = (int)S.k - 1;
    double acc = 0.0;
    const int npts = NP > 0 ? NP : S.npts;
#pragma unroll
    for (int p = 0; p < (NP > 0 ? NP : kMaxStencil); ++p) {
      if (NP == 0 && p >= npts) break;
      bool ok = true;
#pragma unroll
      for (int a = 3 - DIM; a < 3; ++a) {
        const int cc = c[a] + S.off[p][a];
        ok = ok && cc >= 0 && cc <= km1;
      }
      if (ok) acc = add(acc, mul(S.coef[p], __ldg(x + i + S.foff[p])));
    }
    e.row(i, acc);
  }
  e.finish();
}

}  // namespace pbs
