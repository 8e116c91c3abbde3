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
// of the block holds the k-th nonzero of each of its 256 rows, padded where a
// row is shorter than the block's longest.  A u8 length per row tells the
// consumer which levels to add: a padded product is formed but never added,
// so signed zeros and non-finite x stay exactly the reference's.  A block is
// L x 256 entries, contiguous, so the matrix stream is one or two 1-D bulk
// copies per chunk of levels, and there is no row_ptr stream (8 B per row
// less per product).  Consumer thread t reads entry k * 256 + t: consecutive
// lanes read consecutive shared-memory words, the level count is CTA-uniform,
// and the loop has no per-thread bounds.  Each row still sums its products
// sequentially in ascending column order with rounded products and rounded
// adds: bitwise kernels.py:95-100's row sum.
//
// Three value streams (SellView / kSell*), chosen at upload (core.cu):
//   kSellF64    f64 value + u16 window-local column per entry (10 B).
//   kSellDictV  at most 256 distinct f64 bit patterns in the operator
//               (constant-coefficient discretisations: 7 or 27): a u8 index
//               into a dictionary the CTA keeps in shared memory + the u16
//               column (3 B).  The f64 looked up is the uploaded bit pattern.
//   kSellPairs  also at most 256 distinct (value, staged column - row slot)
//               pairs (every interior row of a stencil repeats the same
//               ones): one u8 per entry into a dictionary of 16-byte pairs
//               (1 B); one LDS.128 gives the value and the x address.
//
// Two producer warps: one streams the matrix chunks (and runs ahead of the
// grid dependency), one fills the block slots with one copy stream per lane.
//
// Used for window-mode operators whose padding is small (stencil-like row
// lengths: configs 1, 2, 4, 5); band mode, gathered x and ragged matrices
// stay on csr_pipe_kernel.
#pragma once
#include "spmv.cuh"

namespace pbs {

constexpr int kSellMaxLen = 255;        // longest row the u8 row lengths can hold
constexpr int kSellLevMax = 8;          // levels per chunk stage, at most (20 KiB)
constexpr int kSellLevMaxPair = 32;     // pair dictionary: 256 B per level
constexpr int kSellDict = 256;          // dictionary entries (u8 value indices)
constexpr int kSellThreads = kPipeRows + 64;  // + two producer warps (block slots, matrix stream)

// value stream of the layout: f64 values, u8 value-dictionary indices (+ the
// u16 column stream either way), or u8 (value, relative column) pair indices
enum { kSellF64 = 0, kSellDictV = 1, kSellPairs = 2 };

struct SellPair {
  double v;
  int rel;  // staged x index of the entry minus the row's index in its block
  int pad;
};

struct SellView {
  const double* sv;           // values, level-major per row block (null with a dictionary)
  const unsigned char* svi;   // dictionary modes: index of each entry's value / pair
  const void* dict;           // kSellDict doubles (kSellDictV) or SellPairs (kSellPairs)
  const unsigned short* sc;   // window-local columns (0 in padding entries)
  const unsigned char* slen;  // nonzeros per row, 256 per row block (0 past the last row)
  const long long* soff;      // entry offset of each 256-row block (multiples of 256), nblk + 1
  long long row_lo, row_hi;   // row_lo is a multiple of 256
  long long n_cols;
};

struct SellHdr {
  long long r0;
  int nr, levels, fused, pad;
};

// block slot: header, row lengths, x windows, epilogue inputs
struct SellBlockLayout {
  size_t len, xw, ein, bytes;
  __host__ __device__ SellBlockLayout(int xw_total, int kin) {
    len = 128;
    xw = len + kPipeRows;
    ein = xw + align128(sizeof(double) * (xw_total > 0 ? xw_total : 2));
    bytes = ein + align128(sizeof(double) * kPipeRows * (kin > 0 ? kin : 1));
  }
};

// chunk stage: klev levels of values (vb bytes each: f64, or u8 dictionary
// indices), then of columns
struct SellChunkLayout {
  size_t ci, bytes;
  __host__ __device__ SellChunkLayout(int klev, int mode) {
    ci = (size_t)(mode == kSellF64 ? 8 : 1) * kPipeRows * (size_t)klev;
    bytes = ci + (mode == kSellPairs ? 0 : sizeof(unsigned short) * kPipeRows * (size_t)klev);
  }
};

// acc + p when level k of the chunk is one of the row's (k < rem), as a
// predicated rounded add (no select on the result)
__device__ __forceinline__ double sell_add_if(double acc, double p, int k, int rem) {
  asm("{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %2, %3;\n\t@q add.rn.f64 %0, %0, %1;\n\t}"
      : "+d"(acc)
      : "d"(p), "r"(k), "r"(rem));
  return acc;
}

// N levels of one row, G staged products in flight: columns, values and x
// loads are issued ahead of the rounded product / rounded add chain; rem =
// the row's nonzeros left at this chunk's first level
template <int N, int G, int MODE>
__device__ __forceinline__ double sell_levels(const void* __restrict__ vsv, const unsigned short* __restrict__ cs,
                                              const double* __restrict__ xw, const void* __restrict__ dictv,
                                              int t, double acc, int rem) {
  const double* vs = reinterpret_cast<const double*>(vsv);
  const unsigned char* vi = reinterpret_cast<const unsigned char*>(vsv);
  const double* dict = reinterpret_cast<const double*>(dictv);
  const int4* pairs = reinterpret_cast<const int4*>(dictv);
  const double* xt = xw + t;
#pragma unroll
  for (int k0 = 0; k0 < N; k0 += G) {
    double v[G], xv[G];
    if constexpr (MODE == kSellPairs) {
      unsigned pi[G];
      int4 e[G];
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (k0 + u < N) pi[u] = vi[(k0 + u) * kPipeRows];
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (k0 + u < N) e[u] = pairs[pi[u]];  // one 16-byte load: value and relative x index
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (k0 + u < N) {
          v[u] = __hiloint2double(e[u].y, e[u].x);
          xv[u] = xt[e[u].z];
        }
    } else {
      unsigned c[G];
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (k0 + u < N) c[u] = cs[(k0 + u) * kPipeRows];
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (k0 + u < N) v[u] = MODE == kSellDictV ? dict[vi[(k0 + u) * kPipeRows]] : vs[(k0 + u) * kPipeRows];
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (k0 + u < N) xv[u] = xw[c[u]];
    }
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (k0 + u < N) acc = sell_add_if(acc, mul(v[u], xv[u]), k0 + u, rem);
  }
  return acc;
}

// nk <= 8 levels starting at vs / cs (already offset to the thread's column)
template <int G, int MODE>
__device__ __forceinline__ double sell_chunk8(int nk, const unsigned char* vs, const unsigned short* cs,
                                              const double* xw, const void* dict, int t, double acc, int rem) {
  switch (nk) {  // CTA-uniform
    case 8: return sell_levels<8, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    case 7: return sell_levels<7, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    case 6: return sell_levels<6, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    case 5: return sell_levels<5, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    case 4: return sell_levels<4, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    case 3: return sell_levels<3, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    case 2: return sell_levels<2, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    case 1: return sell_levels<1, G, MODE>(vs, cs, xw, dict, t, acc, rem);
    default: return acc;
  }
}

// a chunk stage of nk levels (up to klev: 8, or 32 with the pair dictionary)
template <int G, int MODE>
__device__ __forceinline__ double sell_chunk(int nk, const unsigned char* vs, const unsigned short* cs,
                                             const double* xw, const void* dict, int t, double acc, int rem) {
  constexpr size_t vb = MODE == kSellF64 ? sizeof(double) : 1;
  if constexpr (MODE == kSellPairs) {
    int k0 = 0;
    for (; k0 + 8 <= nk; k0 += 8)
      acc = sell_levels<8, G, MODE>(vs + (size_t)k0 * kPipeRows * vb, cs, xw, dict, t, acc, rem - k0);
    return sell_chunk8<G, MODE>(nk - k0, vs + (size_t)k0 * kPipeRows * vb, cs, xw, dict, t, acc, rem - k0);
  } else {
    return sell_chunk8<G, MODE>(nk, vs, cs, xw, dict, t, acc, rem);
  }
}

// Epi::kEarly: bit k set when staged input k is not written by the kernel
// that precedes this epilogue's kernel in the schedules that launch it with
// programmatic dependent launch, so its copy may precede griddep_wait.
template <class Epi, class = void>
struct EpiEarly {
  static constexpr unsigned value = 0;
};
template <class Epi>
struct EpiEarly<Epi, decltype((void)Epi::kEarly)> {
  static constexpr unsigned value = Epi::kEarly;
};

// One lane's copy stream of a block slot: lane 0 the row lengths, lanes
// 1..nwin the x windows, lanes 8.. the epilogue inputs.
struct SellLaneStream {
  int role_win, role_in;
  int wmin, wmax;
  uint32_t dst;       // offset in the block slot
  const double* base;
  template <class Epi>
  __device__ void init(int lane, const XWin& W, const SellBlockLayout& BL, const Epi& epi, const double* x) {
    role_win = lane >= 1 && lane <= W.nwin ? lane - 1 : -1;
    role_in = lane >= 8 && lane < 8 + Epi::kInStaged ? lane - 8 : -1;
    wmin = wmax = 0;
    dst = (uint32_t)BL.len;
    base = nullptr;
    if (role_win >= 0) {
      int so = 0;
#pragma unroll
      for (int cc = 0; cc < kMaxWin; ++cc) {
        if (cc == role_win) {
          wmin = W.wmin[cc];
          wmax = W.wmax[cc];
          dst = (uint32_t)(BL.xw + (size_t)so * sizeof(double));
        }
        so += cc < W.nwin ? W.cap[cc] : 0;
      }
      base = x;
    } else if (role_in >= 0) {
      dst = (uint32_t)(BL.ein + (size_t)role_in * kPipeRows * sizeof(double));
#pragma unroll
      for (int k = 0; k < Epi::kInStaged; ++k)
        if (k == role_in) base = epi.in[k];
    }
  }
  // source and size of this lane's copy for the block of rows [r0, r0 + nr)
  __device__ __forceinline__ uint32_t stream(int lane, int r0, int nr, int ncols, const unsigned char* slen_blk,
                                             bool inputs, const void** src) const {
    if (lane == 0) {
      *src = slen_blk;
      return kPipeRows;
    }
    if (role_win >= 0) {
      int lo = r0 + wmin, hi = r0 + nr + wmax;
      if (lo < 0) lo = 0;
      if (hi > ncols) hi = ncols;
      if (hi <= lo) return 0;
      const int loa = lo & ~1, hia = (hi + 1) & ~1;
      *src = base + loa;
      return (uint32_t)((hia - loa) * sizeof(double));
    }
    if (role_in >= 0 && inputs) {
      *src = base + r0;
      return (uint32_t)(((nr + 1) & ~1) * sizeof(double));
    }
    return 0;
  }
};

// Same launch protocol as csr_pipe_kernel (programmatic dependent launch: the
// producer streams the first block's matrix chunks before griddep_wait; one
// gate decision per CTA; consumers release the next grid once their rows are
// written).  MINB: resident CTAs per SM the instantiation is compiled for.
template <class Epi, int MINB = 2, int MODE = kSellF64>
__global__ void __launch_bounds__(kSellThreads, MINB) sell_pipe_kernel(SellView A, const double* __restrict__ x,
                                                                    Epi epi, XWin W, int bslots, int cstages,
                                                                    int klev, int pf) {
  __shared__ int go;
  __shared__ __align__(16) double dict_s[MODE == kSellPairs ? 2 * kSellDict : (MODE == kSellDictV ? kSellDict : 2)];
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* cfull = reinterpret_cast<uint64_t*>(smem);
  uint64_t* cempty = cfull + kMaxStages;
  uint64_t* bfull = cempty + kMaxStages;
  uint64_t* bempty = bfull + kMaxStages;
  const SellBlockLayout BL(W.total, Epi::kInStaged);
  const SellChunkLayout CL(klev, MODE);
  // the dictionary belongs to the operator: read ahead of the grid dependency
  if (MODE != kSellF64 && threadIdx.x < kSellDict) {
    const double* dg = reinterpret_cast<const double*>(A.dict);
    if (MODE == kSellPairs) {
      dict_s[2 * threadIdx.x] = __ldg(dg + 2 * threadIdx.x);
      dict_s[2 * threadIdx.x + 1] = __ldg(dg + 2 * threadIdx.x + 1);
    } else {
      dict_s[threadIdx.x] = __ldg(dg + threadIdx.x);
    }
  }
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

  if (warp == kConsumerWarps + 1) {
    // ------------------------------------------- producer of the matrix stream
    // The block's levels, klev per chunk stage.  Nothing here depends on the
    // previous kernel, so the first chunks are in flight before the gate.
    int cs = 0;
    uint32_t cph = 0;
    long long pf_off = 0, pf_end = 0;
    bool gated = false;
    int issued = 0;  // chunk stages filled before the gate
    auto gate = [&]() -> bool {
      gated = true;
      griddep_wait();
      cta_sync2<kSellThreads>();  // thread 0 (a consumer) has taken the gate decision
      if (go) return true;
      for (int s2 = 0; s2 < issued; ++s2) mbar_wait(&cfull[s2], 0);  // let the early copies land
      return false;
    };
    SellLaneStream LS;
    LS.init(lane, W, BL, epi, x);
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
      const int levels = (int)((end - off) >> 8);
      for (int l0 = 0; l0 < levels; l0 += klev) {
        if (!gated && issued == cstages && !gate()) return;  // the next stage needs the consumers
        mbar_wait(&cempty[cs], cph ^ 1);
        if (lane == 0) {
          unsigned char* st = chk0 + (size_t)cs * CL.bytes;
          const int nk = min(klev, levels - l0);
          const long long e0 = off + (long long)l0 * kPipeRows;
          const uint32_t bv = (uint32_t)(nk * kPipeRows * (MODE == kSellF64 ? sizeof(double) : 1));
          const uint32_t bc = MODE == kSellPairs ? 0u : (uint32_t)(nk * kPipeRows * sizeof(unsigned short));
          mbar_arrive_expect_tx(&cfull[cs], bv + bc);
          bulk_g2s(st, MODE == kSellF64 ? (const void*)(A.sv + e0) : (const void*)(A.svi + e0), bv, &cfull[cs]);
          if (MODE != kSellPairs) bulk_g2s(st + CL.ci, A.sc + e0, bc, &cfull[cs]);
        }
        if (!gated) ++issued;
        if (++cs == cstages) {
          cs = 0;
          cph ^= 1;
        }
      }
      if (!gated && !gate()) return;  // first block's chunks are in flight
      // This warp has slack (one or two copies per block): it asks L2 for what
      // the slot producer will copy for the block `pf` steps ahead, so that
      // copy finds its lines in L2 instead of paying the DRAM latency inside
      // the slot's turnaround.  (L2 is the coherence point: a line prefetched
      // before its producer kernel's last write is updated in place.)
      if (pf > 0) {
        const long long bp = (long long)blk + (long long)pf * gridDim.x;
        if (bp < nblk) {
          const int r0p = (int)A.row_lo + (int)bp * kPipeRows;
          const int nrp = min(kPipeRows, (int)A.row_hi - r0p);
          const void* srcp = nullptr;
          const uint32_t bp_bytes =
              LS.stream(lane, r0p, nrp, (int)A.n_cols, A.slen + (gb0 + bp) * kPipeRows, true, &srcp);
          if (bp_bytes) bulk_prefetch_l2(srcp, bp_bytes);
        }
      }
    }
    if (!gated) gate();
    return;
  }

  if (warp == kConsumerWarps) {
    // --------------------------------------------- producer of the block slots
    // Every lane owns one copy stream of the slot and works out its own
    // source and size per block: lane 0 the row lengths, lanes 1..nwin the x
    // windows, lanes 8.. the epilogue inputs.  (One warp computing all of it,
    // and the matrix stream too, set the kernel's pace: ncu showed the
    // producer never waiting on a free slot while the consumers waited on
    // data at half the HBM rate.)
    int bs = 0;
    uint32_t bph = 0;
    long long pf_off = 0, pf_end = 0;
    bool opp_ready = false;
    SellLaneStream LS;
    LS.init(lane, W, BL, epi, x);
    const int row_lo = (int)A.row_lo, row_hi = (int)A.row_hi, ncols = (int)A.n_cols;
    // Early streams: the row lengths (the operator's) and the epilogue inputs
    // the previous kernel of the schedule does not write (Epi::kEarly).  For
    // the first bslots blocks they go out before griddep_wait, while that
    // kernel drains and runs its check tail; the x windows and the other
    // inputs follow once it has completed.
    constexpr unsigned kEarly = EpiOpp<Epi>::value ? 0u : EpiEarly<Epi>::value;
    const bool lane_early = lane == 0 || (LS.role_in >= 0 && ((kEarly >> LS.role_in) & 1u));
    // phase 0: every stream of the block; 1: header, expected bytes and the
    // early streams; 2: the late streams of a block issued with phase 1
    auto issue = [&](int blk, int q, int phase) {
      const int slot = q & 31;
      if (slot == 0 && phase != 2) {  // entry offsets of blocks q .. q+31 of this CTA
        const long long b2 = (long long)blk + (long long)lane * gridDim.x;
        if (b2 < nblk) {
          pf_off = __ldg(A.soff + gb0 + b2);
          pf_end = __ldg(A.soff + gb0 + b2 + 1);
        }
      }
      const long long off = __shfl_sync(0xffffffffu, pf_off, slot);
      const long long end = __shfl_sync(0xffffffffu, pf_end, slot);
      const int levels = (int)((end - off) >> 8);
      const int r0 = row_lo + blk * kPipeRows;
      const int nr = min(kPipeRows, row_hi - r0);
      bool fuse_in = true;
      if constexpr (EpiOpp<Epi>::value) {  // polled until seen once (it never goes back)
        if (!opp_ready) opp_ready = __shfl_sync(0xffffffffu, lane == 0 ? epi.ready() : false, 0);
        fuse_in = opp_ready;
      }
      const void* src = nullptr;
      const uint32_t bytes = LS.stream(lane, r0, nr, ncols, A.slen + (gb0 + blk) * kPipeRows, fuse_in, &src);
      const int sl = phase == 2 ? q : bs;  // phase 2 only runs for q < bslots
      unsigned char* bst = blk0 + (size_t)sl * BL.bytes;
      if (phase != 2) {
        const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
        mbar_wait(&bempty[bs], bph ^ 1);
        if (lane == 0) {
          SellHdr* bh = reinterpret_cast<SellHdr*>(bst);
          bh->r0 = r0;
          bh->nr = nr;
          bh->levels = levels;
          bh->fused = fuse_in ? 1 : 0;
          mbar_arrive_expect_tx(&bfull[bs], total);
        }
        __syncwarp();
      }
      const bool mine = phase == 0 || ((phase == 1) == lane_early);
      if (bytes && mine) bulk_g2s(bst + LS.dst, src, bytes, &bfull[sl]);
      if (phase != 2 && ++bs == bslots) {
        bs = 0;
        bph ^= 1;
      }
    };
    int npre = 0;
    if (kEarly)
      for (int blk = blockIdx.x; blk < nblk && npre < bslots; blk += gridDim.x, ++npre) issue(blk, npre, 1);
    griddep_wait();  // the previous kernel's vectors are final from here on
    if (kEarly) {
      for (int q = 0; q < npre; ++q) issue((int)blockIdx.x + q * (int)gridDim.x, q, 2);
    } else if (nblk > (int)blockIdx.x) {
      // the first block goes out before the CTA's gate decision (thread 0's
      // read of the solver state and the barrier behind it)
      issue(blockIdx.x, 0, 0);
      npre = 1;
    }
    cta_sync2<kSellThreads>();
    if (!go) {  // the gate says stop: let what was issued land
      for (int q = 0; q < npre; ++q) mbar_wait(&bfull[q], 0);
      return;
    }
    for (int blk = (int)blockIdx.x + npre * (int)gridDim.x, q = npre; blk < nblk; blk += gridDim.x, ++q) issue(blk, q, 0);
    return;
  }

  // ------------------------------------------------------------- consumers
  griddep_wait();
  if (threadIdx.x == 0) {
    go = epi.active();  // one gate decision per CTA
    if (!go && blockIdx.x == 0) epi.on_skip();
  }
  cta_sync2<kSellThreads>();
  if (!go) return;
  Epi e = epi;
  e.init();
  const int t = threadIdx.x;
  int cs = 0, bs = 0;
  uint32_t cph = 0, bph = 0;
#ifndef PBS_SELL_G  // staged products in flight per row at 2 CTAs/SM (-D override for sweeps)
#define PBS_SELL_G 4
#endif
  constexpr int G = MINB == 1 ? 8 : PBS_SELL_G;
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
    const int len = reinterpret_cast<const unsigned char*>(bst + BL.len)[t];  // 0 past the last row
    double acc = 0.0;
    for (int l0 = 0; l0 < levels; l0 += klev) {
      mbar_wait(&cfull[cs], cph);
      const unsigned char* st = chk0 + (size_t)cs * CL.bytes;
      const int nk = min(klev, levels - l0);
      acc = sell_chunk<G, MODE>(nk, st + (size_t)t * (MODE == kSellF64 ? sizeof(double) : 1),
                                reinterpret_cast<const unsigned short*>(st + CL.ci) + t, xw, dict_s, t, acc, len - l0);
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
