// zmarch.cuh — z-marching matrix-free engine for 3D stencils (sm_100a).
//
// The staged stencil engine (stencil_pipe_kernel) copies, per 256-row block,
// the three plane windows its rows reach: for a 27-point stencil on a 384^2
// plane that is ~3 x 1026 doubles for 256 rows, so every x element crosses
// L2 -> SM about twelve times and the plain product (config 4's K1) is bound
// by L2 bandwidth at 0.15 of the HBM roofline.  This engine tiles the grid in
// (y, x) and marches along z instead: a CTA owns a 15 x 32 column of the
// grid over a run of planes and keeps the halo'd tile of the planes z-1, z,
// z+1 (17 x 36 doubles each) in a ring of shared-memory stages that the
// copy engine fills ahead (one cp.async.bulk per tile row, completion on the
// stage's mbarrier).  Each x element is staged ~1.1 times.  Thread (ty, tx)
// computes grid row (z, y0 + ty, x0 + tx) — its neighbours in ascending
// flattened offset (the CSR column order), out-of-grid neighbours skipped —
// so the row sum is bitwise the CSR engine's; the epilogue's inputs for the
// next plane are loaded while the current plane computes (coalesced: a warp
// is one tile row of 32 consecutive x).
//
// Geometry: rows [row_lo, row_hi) must be whole planes; x is addressed from
// the slab's own segment, planes [zx_lo, zx_hi) present (a partition's halo
// planes included); the grid's edge length k must be even (16-byte-aligned
// tile-row copies).
#pragma once
#include <cuda.h>  // CUtensorMap (the map is encoded on the host through the driver entry point)

#include <type_traits>

#include "spmv.cuh"

namespace pbs {

constexpr int kZmTY = 15, kZmTX = 32;  // 15 rows: with the producer warp a CTA is 16 warps (register file split evenly)
constexpr int kZmThreads = kZmTY * kZmTX;  // consumers: one thread per tile column position
constexpr int kZmWarps = kZmThreads / 32;
constexpr int kZmCTA = kZmThreads + 32;     // + one producer warp
constexpr int kZmMaxRing = 16;
// RPT rows per consumer thread along x (2 for the light epilogues: the
// neighbours of the pair come from 4 staged values per line instead of 6, and
// the two row sums are independent chains)
template <int RPT>
struct ZmShape {
  static constexpr int TX = kZmTX * RPT;                   // tile width
  static constexpr int RowW = TX + 4;                      // staged doubles per tile row: x in [x0-2, x0+TX+2)
  static constexpr int Plane = (kZmTY + 2) * RowW;         // doubles of one staged plane tile (the TMA box)
  static constexpr uint32_t PlaneBytes = Plane * sizeof(double);
  static constexpr int Stage = (Plane * 8 + 127) / 128 * 128 / 8;  // stage stride in doubles (128-byte aligned)
};

// 3-D tiled TMA load of one plane tile: box (TX+4, TY+2, 1) at (x, y, z) of
// the tensor map; out-of-range elements arrive as zeros (never read: their
// neighbours are masked out)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int cx, int cy, int cz, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cx), "r"(cy), "r"(cz), "r"(smem_u32(bar))
      : "memory");
}

struct ZmGeom {
  int tiles_y, tiles_x;
  int z_lo, z_hi;   // planes of rows [row_lo, row_hi) (slab-local)
  int zx_lo, zx_hi; // planes of x present (slab-local; the halo planes of a partition)
  int zchunk;       // planes per work item
  int ring;         // shared-memory plane stages
  long long gz0;    // grid plane of slab-local plane 0
};

// resident CTAs per SM the instantiation is compiled for: the light
// epilogues without dot accumulators run two 512-thread CTAs per SM (64
// registers), the rest one
template <class Epi>
__host__ __device__ constexpr int zm_minb() {
  return (std::is_same<Epi, EpiStore>::value || std::is_same<Epi, EpiResid>::value ||
          std::is_same<Epi, EpiK3n>::value)
             ? 2
             : 1;
}

// rows per consumer thread (the engine supports 2: a pair's neighbours come
// from 4 staged values per line instead of 6, two independent row chains).
// One everywhere: the plain 27-point product is bound by the FP64 pipe (the
// bitwise row sum is 27 DMUL + 27 DADD per row, ~9e12 DP instructions/s on
// B200, 340 us for config 4), and two rows per thread measured no faster
// (573 vs 531 us, the partitioned schedule's K1).
template <class Epi>
__host__ __device__ constexpr int zm_rpt() {
  return 1;
}

// neighbour p of the 7- and 27-point stencils in ascending flattened offset
// (the CSR column order): (dz, dy, dx) in {-1, 0, 1}^3
template <int NP>
__host__ __device__ constexpr int zm_off(int p, int axis) {
  if (NP == 27) return axis == 0 ? p / 9 - 1 : (axis == 1 ? (p / 3) % 3 - 1 : p % 3 - 1);
  // 7-point star: (-1,0,0) (0,-1,0) (0,0,-1) (0,0,0) (0,0,1) (0,1,0) (1,0,0)
  return axis == 0 ? (p == 0 ? -1 : (p == 6 ? 1 : 0))
                   : (axis == 1 ? (p == 1 ? -1 : (p == 5 ? 1 : 0)) : (p == 2 ? -1 : (p == 4 ? 1 : 0)));
}

// register cap: the whole register file split between the resident CTAs
template <class Epi>
__host__ __device__ constexpr int zm_maxreg() {
  return zm_minb<Epi>() == 2 ? 64 : 128;
}

template <class Epi, int NP>
__global__ void __launch_bounds__(kZmCTA) __maxnreg__(zm_maxreg<Epi>())
    stencil_zm_kernel(const __grid_constant__ StencilView S, const __grid_constant__ CUtensorMap xmap, Epi epi,
                      ZmGeom G) {
  constexpr int RPT = zm_rpt<Epi>();
  using Sh = ZmShape<RPT>;
  constexpr int kZmRowW = Sh::RowW, kZmStage = Sh::Stage, TXE = Sh::TX;
  constexpr uint32_t kZmPlaneBytes = Sh::PlaneBytes;
  __shared__ int go;
  griddep_wait();  // PDL: everything here reads the previous kernel's output
  if (threadIdx.x == 0) {
    go = epi.active();
    if (!go && blockIdx.x == 0) epi.on_skip();
  }
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kZmMaxRing;
  double* ring = reinterpret_cast<double*>(smem + 256);  // stages 128-byte aligned (TMA destination)
  const int t = threadIdx.x, lane = t & 31;
  if (t == 0) {
    for (int s = 0; s < G.ring; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kZmWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (!go) return;
  const long long k = S.k, k2 = S.k2;
  const int ki = (int)k;
  if (t == kZmThreads) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
  const int ntiles = G.tiles_y * G.tiles_x;
  const int nchunks = (G.z_hi - G.z_lo + G.zchunk - 1) / G.zchunk;
  const int items = ntiles * nchunks;
  // The planes a CTA stages form one stream across its work items (item it:
  // planes za-1 .. zb), filled by the producer warp through a ring of stages
  // (full: staged; empty: every consumer warp is done with it), so the next
  // item's first planes arrive while the current item computes.
  if (t >= kZmThreads) {
    // producer warp: one 3-D TMA per plane tile, issued by lane 0
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int tile = it % ntiles, chunk = it / ntiles;
        const int y0 = (tile / G.tiles_x) * kZmTY, x0 = (tile % G.tiles_x) * TXE;
        const int za = G.z_lo + chunk * G.zchunk, zb = min(G.z_hi, za + G.zchunk);
        for (int zl = za - 1; zl <= zb; ++zl) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kZmPlaneBytes);
          tma_load_3d(ring + (size_t)s * kZmStage, &xmap, x0 - 2, y0 - 1, zl - G.zx_lo, &full[s]);
          if (++s == G.ring) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }
  Epi e = epi;
  e.init();
  const int ty = t / kZmTX, tx = t % kZmTX;
  // stage / phase of the current item's first plane (loads advance both)
  int s = 0;
  uint32_t ph = 0;
  constexpr unsigned kAll = (1u << NP) - 1u;
  const int ctr = (ty + 1) * kZmRowW + RPT * tx + 2;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int tile = it % ntiles, chunk = it / ntiles;
    const int y0 = (tile / G.tiles_x) * kZmTY, x0 = (tile % G.tiles_x) * TXE;
    const int za = G.z_lo + chunk * G.zchunk, zb = min(G.z_hi, za + G.zchunk);
    const int y = y0 + ty, xx = x0 + RPT * tx;  // this thread's rows: x = xx .. xx + RPT - 1
    bool live[RPT];
    unsigned vm_yx[RPT];  // in-grid neighbours as far as y and x decide (z per plane below)
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      live[r] = y < ki && xx + r < ki;
      vm_yx[r] = kAll;
      if (y == 0) vm_yx[r] &= S.nlo[1];
      if (y == ki - 1) vm_yx[r] &= S.nhi[1];
      if (xx + r == 0) vm_yx[r] &= S.nlo[2];
      if (xx + r == ki - 1) vm_yx[r] &= S.nhi[2];
    }
    const long long rowoff = (long long)y * k + xx;
    double nin[RPT][Epi::kIn > 0 ? Epi::kIn : 1];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
      if (live[r]) {
#pragma unroll
        for (int j = 0; j < Epi::kIn; ++j) nin[r][j] = __ldg(e.in[j] + (long long)za * k2 + rowoff + r);
      }
    // stages of the planes below / at / above the centre, and their phases
    int s0 = s, s1 = s + 1, s2 = s + 2;
    uint32_t p0 = ph, p1 = ph, p2 = ph;
    if (s1 >= G.ring) s1 -= G.ring, p1 ^= 1;
    if (s2 >= G.ring) s2 -= G.ring, p2 ^= 1;
    mbar_wait(&full[s0], p0);
    mbar_wait(&full[s1], p1);
    for (int z = za; z < zb; ++z) {
      double inr[RPT][Epi::kIn > 0 ? Epi::kIn : 1];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
#pragma unroll
        for (int j = 0; j < Epi::kIn; ++j) inr[r][j] = nin[r][j];
        if (live[r] && z + 1 < zb) {  // the next plane's epilogue inputs, in flight during this one
#pragma unroll
          for (int j = 0; j < Epi::kIn; ++j) nin[r][j] = __ldg(e.in[j] + (long long)(z + 1) * k2 + rowoff + r);
        }
      }
      mbar_wait(&full[s2], p2);
      const long long gz = z + G.gz0;
      unsigned vm[RPT];
      bool interior = true;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        vm[r] = vm_yx[r];
        if (gz == 0) vm[r] &= S.nlo[0];
        if (gz == k - 1) vm[r] &= S.nhi[0];
        interior = interior && vm[r] == kAll && live[r];
      }
      const double* pl0 = ring + (size_t)s0 * kZmStage + ctr;
      const double* pl1 = ring + (size_t)s1 * kZmStage + ctr;
      const double* pl2 = ring + (size_t)s2 * kZmStage + ctr;
      double acc[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) acc[r] = 0.0;
      // each row's neighbours in ascending flattened offset; the points come
      // grouped by (dz, dy) line, and a line's staged values are loaded once
      // for all the thread's rows
      double w[RPT + 2];
      if (interior) {  // no predicates
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const int dz = zm_off<NP>(p, 0), dy = zm_off<NP>(p, 1), dx = zm_off<NP>(p, 2);
          if (p == 0 || dz != zm_off<NP>(p - 1, 0) || dy != zm_off<NP>(p - 1, 1)) {
            const double* ln = (dz < 0 ? pl0 : (dz == 0 ? pl1 : pl2)) + dy * kZmRowW;
#pragma unroll
            for (int q = 0; q < RPT + 2; ++q) w[q] = ln[q - 1];
          }
#pragma unroll
          for (int r = 0; r < RPT; ++r) acc[r] = add(acc[r], mul(S.coef[p], w[dx + 1 + r]));
        }
      } else {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const int dz = zm_off<NP>(p, 0), dy = zm_off<NP>(p, 1), dx = zm_off<NP>(p, 2);
          if (p == 0 || dz != zm_off<NP>(p - 1, 0) || dy != zm_off<NP>(p - 1, 1)) {
            const double* ln = (dz < 0 ? pl0 : (dz == 0 ? pl1 : pl2)) + dy * kZmRowW;
#pragma unroll
            for (int q = 0; q < RPT + 2; ++q) w[q] = ln[q - 1];
          }
#pragma unroll
          for (int r = 0; r < RPT; ++r)
            if ((vm[r] >> p) & 1u) acc[r] = add(acc[r], mul(S.coef[p], w[dx + 1 + r]));
        }
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (live[r]) e.row((long long)z * k2 + rowoff + r, acc[r], inr[r]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s0]);  // this warp is done with the plane below
      s0 = s1, p0 = p1;
      s1 = s2, p1 = p2;
      if (++s2 == G.ring) s2 = 0, p2 ^= 1;
    }
    // the last two planes of the item are released at its end
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty[s0]);
      mbar_arrive(&empty[s1]);
    }
    s = s2, ph = p2;  // the next item's first plane follows this item's last
  }
  griddep_launch();
  e.template finish<kZmThreads, true>();
}

}  // namespace pbs
