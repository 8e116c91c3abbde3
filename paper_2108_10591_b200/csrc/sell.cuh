// sell.cuh — the sliced-ELL form of the staged CSR engine (sm_100a).
//
// csr_pipe_kernel's consumers own one row each and walk its nonzeros in CSR
// order: per row block every thread pays 64-bit row bounds, chunk clipping
// and a predicated variable-length loop — about 300 warp instructions around
// the ~50 a 7-nonzero row needs — and at 16 consumer warps per SM that
// instruction stream, not HBM, bounds the fused kernels (ncu: issue slots 38%
// busy, 0.6 eligible warps per scheduler, profiles/r2/c2_k12_k3_details.csv).
//
// At upload the operator's nonzeros are therefore also laid out per 256-row
// block in level-major ("sliced ELL", slice = the row block) order: level k
// of the block holds the k-th nonzero of each of its 256 rows — value and
// window-local u16 column — padded with a sentinel column where a row is
// shorter than the block's longest.  A block is L x 256 entries, contiguous,
// so the producer still streams it with two 1-D bulk copies per chunk of
// levels, and there is no row_ptr stream at all (8 B per row less per
// product).  Consumer thread t reads entry k * 256 + t: consecutive lanes
// read consecutive shared-memory words (no bank conflicts), the level count
// is CTA-uniform, and the loop has no per-thread bounds.  Each row still sums
// its products sequentially in ascending column order with rounded products
// and rounded adds, so the result is bitwise kernels.py:95-100's.
//
// Used for window-mode operators whose padding is small (stencil-like row
// lengths: configs 1, 2, 4, 5); band mode, gathered x and ragged matrices
// stay on csr_pipe_kernel.
#pragma once
#include "spmv.cuh"

namespace pbs {

constexpr unsigned kSellPad = 0xffffu;  // sentinel column of a padding entry
constexpr int kSellLevMax = 8;          // levels per chunk stage, at most (20 KiB)

struct SellView {
  const double* sv;           // values, level-major per row block
  const unsigned short* sc;   // window-local columns (kSellPad: padding)
  const long long* soff;      // entry offset of each 256-row block (multiples of 256), nblk + 1
  long long row_lo, row_hi;   // row_lo is a multiple of 256
  long long n_cols;
};

struct SellHdr {
  long long r0;
  int nr, levels, fused, pad;
};

// block slot: header, x windows, epilogue inputs
struct SellBlockLayout {
  size_t xw, ein, bytes;
  __host__ __device__ SellBlockLayout(int xw_total, int kin) {
    xw = 128;
    ein = xw + align128(sizeof(double) * (xw_total > 0 ? xw_total : 2));
    bytes = ein + align128(sizeof(double) * kPipeRows * (kin > 0 ? kin : 1));
  }
};

// chunk stage: klev levels of values, then of columns
struct SellChunkLayout {
  size_t ci, bytes;
  __host__ __device__ SellChunkLayout(int klev) {
    ci = sizeof(double) * kPipeRows * (size_t)klev;
    bytes = ci + sizeof(unsigned short) * kPipeRows * (size_t)klev;
  }
};

// N levels of one row, G staged products in flight: columns, values and x
// loads are issued ahead of the rounded product / rounded add chain
template <int N, int G>
__device__ __forceinline__ double sell_levels(const double* __restrict__ vs, const unsigned short* __restrict__ cs,
                                              const double* __restrict__ xw, double acc) {
#pragma unroll
  for (int k0 = 0; k0 < N; k0 += G) {
    unsigned c[G];
    double v[G], xv[G];
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (k0 + u < N) c[u] = cs[(k0 + u) * kPipeRows];
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (k0 + u < N) v[u] = vs[(k0 + u) * kPipeRows];
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (k0 + u < N) xv[u] = c[u] != kSellPad ? xw[c[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (k0 + u < N)
        if (c[u] != kSellPad) acc = add(acc, mul(v[u], xv[u]));
  }
  return acc;
}

template <int G>
__device__ __forceinline__ double sell_chunk(int nk, const double* vs, const unsigned short* cs, const double* xw,
                                             double acc) {
  switch (nk) {  // CTA-uniform
    case 8: return sell_levels<8, G>(vs, cs, xw, acc);
    case 7: return sell_levels<7, G>(vs, cs, xw, acc);
    case 6: return sell_levels<6, G>(vs, cs, xw, acc);
    case 5: return sell_levels<5, G>(vs, cs, xw, acc);
    case 4: return sell_levels<4, G>(vs, cs, xw, acc);
    case 3: return sell_levels<3, G>(vs, cs, xw, acc);
    case 2: return sell_levels<2, G>(vs, cs, xw, acc);
    case 1: return sell_levels<1, G>(vs, cs, xw, acc);
    default: return acc;
  }
}

// Same launch protocol as csr_pipe_kernel (programmatic dependent launch: the
// producer streams the first block's matrix chunks before griddep_wait; one
// gate decision per CTA; consumers release the next grid once their rows are
// written).  MINB: resident CTAs per SM the instantiation is compiled for.
template <class Epi, int MINB = 2>
__global__ void __launch_bounds__(kPipeThreads, MINB) sell_pipe_kernel(SellView A, const double* __restrict__ x,
                                                                    Epi epi, XWin W, int bslots, int cstages,
                                                                    int klev) {
  __shared__ int go;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* cfull = reinterpret_cast<uint64_t*>(smem);
  uint64_t* cempty = cfull + kMaxStages;
  uint64_t* bfull = cempty + kMaxStages;
  uint64_t* bempty = bfull + kMaxStages;
  const SellBlockLayout BL(W.total, Epi::kInStaged);
  const SellChunkLayout CL(klev);
  unsigned char* blk0 = smem + kPipeBarrierBytes;
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
  const int nblk = (int)((nrows + kPipeRows - 1) / kPipeRows);
  const long long gb0 = A.row_lo / kPipeRows;  // first block, counted from row 0

  if (warp == kConsumerWarps) {
    // ----------------------------------------------------------- producer
    int cs = 0, bs = 0;
    uint32_t cph = 0, bph = 0;
    long long pf_off = 0, pf_end = 0;
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
    bool opp_ready = false;
    if (nblk <= (int)blockIdx.x && !gate()) return;
    for (int blk = blockIdx.x, q = 0; blk < nblk; blk += gridDim.x, ++q) {
      const int slot = q & 31;
      if (slot == 0) {  // entry offsets of blocks q .. q+31 of this CTA in one warp-wide load
        const long long b2 = (long long)blk + (long long)lane * gridDim.x;
        if (b2 < nblk) {
          pf_off = __ldg(A.soff + gb0 + b2);
          pf_end = __ldg(A.soff + gb0 + b2 + 1);
        }
      }
      const long long off = __shfl_sync(0xffffffffu, pf_off, slot);
      const long long end = __shfl_sync(0xffffffffu, pf_end, slot);
      const int levels = (int)((end - off) / kPipeRows);
      const int nch = (levels + klev - 1) / klev;
      const long long r0 = A.row_lo + (long long)blk * kPipeRows;
      const int nr = (int)min((long long)kPipeRows, A.row_hi - r0);
      const uint32_t bin = (uint32_t)(((nr + 1) & ~1) * sizeof(double));
      auto issue_chunk = [&](int c) {
        mbar_wait(&cempty[cs], cph ^ 1);
        unsigned char* st = chk0 + (size_t)cs * CL.bytes;
        const int nk = min(klev, levels - c * klev);
        const long long e0 = off + (long long)c * klev * kPipeRows;
        const uint32_t bv = (uint32_t)(nk * kPipeRows * sizeof(double));
        const uint32_t bc = (uint32_t)(nk * kPipeRows * sizeof(unsigned short));
        if (lane == 0) mbar_arrive_expect_tx(&cfull[cs], bv + bc);
        __syncwarp();
        if (lane == 0) bulk_g2s(st, A.sv + e0, bv, &cfull[cs]);
        if (lane == 1) bulk_g2s(st + CL.ci, A.sc + e0, bc, &cfull[cs]);
        if (++cs == cstages) {
          cs = 0;
          cph ^= 1;
        }
      };
      int cfirst = 0;
      if (!gated) {
        cfirst = nch < cstages ? nch : cstages;
        for (int c = 0; c < cfirst; ++c) issue_chunk(c);
        issued = cfirst;
        if (!gate()) return;
      }
      bool fuse_in = true;
      if constexpr (EpiOpp<Epi>::value) {  // polled until seen once (it never goes back)
        if (!opp_ready) opp_ready = __shfl_sync(0xffffffffu, lane == 0 ? epi.ready() : false, 0);
        fuse_in = opp_ready;
      }
      long long wlo[kMaxWin];
      uint32_t wbytes[kMaxWin];
      uint32_t total = fuse_in ? Epi::kInStaged * bin : 0u;
#pragma unroll
      for (int c = 0; c < kMaxWin; ++c) {
        wlo[c] = 0;
        wbytes[c] = 0;
        if (c < W.nwin) {
          long long lo = r0 + W.wmin[c], hi = r0 + nr - 1 + W.wmax[c] + 1;
          if (lo < 0) lo = 0;
          if (hi > A.n_cols) hi = A.n_cols;
          if (hi > lo) {
            const long long loa = lo & ~1LL, hia = (hi + 1) & ~1LL;
            wlo[c] = loa;
            wbytes[c] = (uint32_t)((hia - loa) * sizeof(double));
            total += wbytes[c];
          }
        }
      }
      mbar_wait(&bempty[bs], bph ^ 1);
      unsigned char* bst = blk0 + (size_t)bs * BL.bytes;
      if (lane == 0) {
        SellHdr* bh = reinterpret_cast<SellHdr*>(bst);
        bh->r0 = r0;
        bh->nr = nr;
        bh->levels = levels;
        bh->fused = fuse_in ? 1 : 0;
        if (total)
          mbar_arrive_expect_tx(&bfull[bs], total);
        else
          mbar_arrive(&bfull[bs]);
      }
      __syncwarp();
      if (lane >= 1 && lane <= W.nwin) {
        int soff = 0;
#pragma unroll
        for (int cc = 0; cc < kMaxWin; ++cc) {
          if (cc == lane - 1 && wbytes[cc])
            bulk_g2s(bst + BL.xw + (size_t)soff * sizeof(double), x + wlo[cc], wbytes[cc], &bfull[bs]);
          soff += cc < W.nwin ? W.cap[cc] : 0;
        }
      } else if (fuse_in && lane >= 8 && lane < 8 + Epi::kInStaged) {
        const int e = lane - 8;
        bulk_g2s(bst + BL.ein + (size_t)e * kPipeRows * sizeof(double), epi.in[e] + r0, bin, &bfull[bs]);
      }
      if (++bs == bslots) {
        bs = 0;
        bph ^= 1;
      }
      for (int c = cfirst; c < nch; ++c) issue_chunk(c);
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
  constexpr int G = MINB == 1 ? 8 : 4;
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    mbar_wait(&bfull[bs], bph);
    const unsigned char* bst = blk0 + (size_t)bs * BL.bytes;
    const SellHdr* bhp = reinterpret_cast<const SellHdr*>(bst);
    const int nr = bhp->nr, levels = bhp->levels;
    const long long r0 = bhp->r0;
    const bool fused = !EpiOpp<Epi>::value || bhp->fused;  // the producer's decision for this block
    double inr[Epi::kIn > 0 ? Epi::kIn : 1];
    if (t < nr && fused) {  // inputs the producer does not stage: in flight during the row's products
#pragma unroll
      for (int k = Epi::kInStaged; k < Epi::kIn; ++k) inr[k] = __ldg(e.in[k] + r0 + t);
    }
    const double* xw = reinterpret_cast<const double*>(bst + BL.xw);
    double acc = 0.0;
    for (int l0 = 0; l0 < levels; l0 += klev) {
      mbar_wait(&cfull[cs], cph);
      const unsigned char* st = chk0 + (size_t)cs * CL.bytes;
      const int nk = min(klev, levels - l0);
      // rows past the matrix end hold only padding entries
      acc = sell_chunk<G>(nk, reinterpret_cast<const double*>(st) + t,
                          reinterpret_cast<const unsigned short*>(st + CL.ci) + t, xw, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty[cs]);
      if (++cs == cstages) {
        cs = 0;
        cph ^= 1;
      }
    }
    if (t < nr) {
      const double* ein = reinterpret_cast<const double*>(bst + BL.ein);
      if (fused) {
#pragma unroll
        for (int k = 0; k < Epi::kInStaged; ++k) inr[k] = ein[k * kPipeRows + t];
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

}  // namespace pbs
