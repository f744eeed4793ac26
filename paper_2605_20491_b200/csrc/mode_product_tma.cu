// Mode-k eigenbasis transform, Blackwell-native pipeline: TMA (cp.async.bulk.tensor) tiles into
// 128B-swizzled shared memory, mbarrier full/empty handshakes, one producer warp and eight
// FP64-DMMA consumer warps (warp specialisation), 128-bit fragment loads.
//
// Same contraction as mode_product.cu (proj/src/tensor.cpp:31-84, mode_product :105-134) with the
// same fused epilogues (operators.cpp:36,57,68-71,102); this kernel serves the two geometries that
// carry ~all of the FLOPs at scale:
//   STRIDED  pre % 128 == 0: X tile = 8 TMA boxes of [BK k][16 rows] (3-D tensor map pre x nk x post)
//   CONTIG   pre == 1:       X tile = 2 TMA boxes of [128 rows][16 k] (2-D tensor map nk x rows)
// and the per-axis matrix (B operand) = BN/16 boxes of [BK k][16 cols] (2-D, zero-padded lda x kp).
// Everything else (complex axis 0 with pre = 2, odd strides) runs the cp.async kernel.
//
// Fragment layout (why 128-bit loads are conflict free): with 128B swizzle the 16-byte chunk c of
// smem row y sits at chunk c ^ (y & 7). A thread loads one 16-byte chunk = two consecutive rows (or
// k values) and feeds them to two different 8x8x4 DMMA tiles; the lane -> row map is permuted so
// that the 8 lanes of each quarter-warp touch 8 distinct chunks:
//   STRIDED / matrix boxes (row = k): chunk(g) = (g&1)*4 + (g>>1)  (k varies in bits 0-1)
//   CONTIG X box (row = tile row):    row(g)   = (g&1)*4 + (g>>1), chunk spans an aligned 4-block
//   CONTIG matrix box (k = 2t+s):     chunk(g) = g                   (k varies in bits 1-2)
// The permutation is undone in the epilogue (row / column maps below). The contraction index may be
// permuted freely as long as both operands agree, which the CONTIG path uses (lane t holds k = 2t, 2t+1).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "epilogue.cuh"
#include "kronop_internal.cuh"

namespace kronop_dev {

namespace {

constexpr int BM = 128;
#ifndef KRONOP_TMA_BK
#define KRONOP_TMA_BK 32  // k per stage (A/B experiments: -DKRONOP_TMA_BK=16 -DKRONOP_TMA_STAGES=6)
#endif
#ifndef KRONOP_TMA_STAGES
#define KRONOP_TMA_STAGES 3
#endif
constexpr int BK = KRONOP_TMA_BK;
constexpr int STAGES = KRONOP_TMA_STAGES;
constexpr int NCONS = 8;                 // DMMA warps; warp 0 lane 0 also drives TMA
constexpr int NTHREADS = NCONS * 32;
constexpr int BOX_STRIDED_BYTES = BK * 128;  // [BK rows][16 doubles]
constexpr int BOX_CONTIG_BYTES = BM * 128;   // [BM rows][16 doubles]

enum { TL_STRIDED = 0, TL_CONTIG = 1, TL_CPLX0 = 2 };
// TL_CPLX0: pre == 2 (axis 0 of an interleaved complex field). X viewed as the 2-D tensor
// (2 nk doubles per row, post rows); a box is [64 q][8 j x (re, im)] = 128 B rows, so one 128-bit
// fragment load returns (re, im) of one (q, j): the re row and the im row of the pass are the two
// DMMA tiles of a pair, exactly like the STRIDED pairing (rows r = c + 2q).
constexpr int BOX_CPLX0_BYTES = (BM / 2) * 128;

template <int BN>
struct Cfg {
  static constexpr int WARPS_N = BN == 128 ? 4 : 2;
  static constexpr int WARPS_M = NCONS / WARPS_N;
  static constexpr int WTM = BM / WARPS_M;  // 64 | 32
  static constexpr int WTN = BN / WARPS_N;  // 32
  static constexpr int RT = WTM / 8;
  static constexpr int CT = WTN / 8;
  static constexpr int X_BYTES = BM * BK * 8;
  static constexpr int A_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = X_BYTES + A_BYTES;
  // + per-warp tables of the spectral-divide epilogue (EK_DIV): row lambda partial sums (WTM)
  //   and column eigenvalues (WTN) of the warp's current tile
  static constexpr int WTAB = WTM + WTN;
  static constexpr int SMEM =
      STAGES * STAGE_BYTES + 1024 /*align*/ + 64 /*barriers*/ + NCONS * WTAB * 8;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// multicast variants (thread-block clusters of CL CTAs along N share the X tile)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
      "cluster [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, int c0, int c1,
                                               int c2, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
      "cluster [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// arrive on the mbarrier at the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

__device__ __forceinline__ double2 lds128(const char* base, uint32_t byte_off) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y)
               : "r"(smem_u32(base) + byte_off));
  return v;
}
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int chS(int g) { return ((g & 1) << 2) | (g >> 1); }

// Epilogue specialisations (compile-time, so each kernel carries only its own epilogue code: the
// general one, with every kind behind runtime branches, is large enough to miss in the
// instruction cache when unrolled over 64 accumulators per thread):
//   EK_GENERIC  every EpiParams kind (runtime dispatch; out-of-line per-element helpers)
//   EK_STORE    plain store
//   EK_MUL / EK_PHASE  the spectral multiply (apply) / phase (propagate: one sincos per (re, im)
//               pair, both outputs from it) on the last real-view axis, same tables as EK_DIV
//   EK_AXPY     + diag u - sigma u (FullOperator::apply's last pass): a row's u / diag loads are
//               issued together before its stores (y may alias u, so the compiler cannot)
//   EK_DIV      spectral divide on the last real-view axis (the solve's fused pass): per-warp
//               tables of the row lambda partial sums and column eigenvalues, built before the K
//               loop, and the divisions of one row batch issued together (div_rn_fast)
//   EK_SPLIT    plain store into the destination parts of a slab exchange (SplitDst): the
//               per-column destination is resolved once per tile, the rows stay coalesced
enum { EK_GENERIC = 0, EK_STORE = 1, EK_DIV = 2, EK_MUL = 3, EK_PHASE = 4, EK_AXPY = 5,
       EK_SPLIT = 6 };

struct TArgs {
  double* y;
  int x2d;  // STRIDED with post == 1: X is the 2-D (pre x nk) tensor map
  long long pre, post, R;
  long long ldy;  // q-stride of Y
  long long ycol;  // stride of the output index i in Y (pre, or R for a rotated pass)
  int rot;         // eigenvalue rows = full row index r (rotated pass)
  int nk, m;
  int ntiles_n;
  long long ntiles_m;
  EpiParams ep;
  SplitDst split;  // EK_SPLIT
};

template <int BN, int LOADER>
__device__ __forceinline__ int row_map(int j, int g) {
  // row (within the warp tile) of MMA row g of row-tile j
  if (LOADER == TL_STRIDED || LOADER == TL_CPLX0) return (j >> 1) * 16 + 2 * chS(g) + (j & 1);
  return j * 8 + chS(g);
}
template <int BN, int LOADER>
__device__ __forceinline__ int col_map(int jc, int n) {
  if (LOADER == TL_CONTIG) return (jc >> 1) * 16 + 2 * n + (jc & 1);
  return (jc >> 1) * 16 + 2 * chS(n) + (jc & 1);
}

template <int BN, int LOADER, int CL, int EK>
__global__ void __launch_bounds__(NTHREADS, 1)
    mode_product_tma_kernel(const __grid_constant__ CUtensorMap tmx,
                            const __grid_constant__ CUtensorMap tma, const TArgs args) {
  using C = Cfg<BN>;
  if (args.ep.active && *args.ep.active == 0) return;  // whole CTA: before any barrier init
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  double* s_tab = reinterpret_cast<double*>(smem + STAGES * C::STAGE_BYTES + 64);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int KT = (args.nk + BK - 1) / BK;
  // Persistent CTAs over the tile sequence T = blockIdx.x + lt * gridDim.x with the N-tiles of
  // a row panel consecutive in T: the ~148 tiles in flight cover ~148 / ntiles_n panels, whose X
  // rows (1 MB each at n = 1024) stay L2-resident while all N-tiles of the panel consume them, so
  // X is read from HBM once (a CTA walking all N-tiles of its own panel keeps 148 panels live,
  // more than L2, and re-reads X ntiles_n times). The per-axis matrix stays L2-resident. The
  // k-stage counter `it` runs across tiles, so the producer streams the next tile's first stages
  // while the consumers run the current tile's epilogue.
  //
  // Clusters (CL > 1): the CL CTAs of a cluster take CL consecutive N-tiles of the same row
  // panel in lockstep; each CTA issues 1/CL of the X boxes of a stage as a TMA multicast to the
  // whole cluster, so X crosses L2 -> SM once per cluster, and a stage is refilled only after
  // all CL x 8 consumer warps of the cluster released it (remote mbarrier arrivals).
  //
  // Round 2: the tile sequence is cut into UNITS of NSUB consecutive N-tiles of one row panel
  // (NSUB = 4 when a panel has a multiple of 4 N-tiles, e.g. 8 at n = 1024): CTA cid takes units
  // cid, cid + ncl, ... and walks each unit's N-tiles back to back, so a panel's X rows are
  // consumed by 2 CTAs within a few tile times (interleaving single tiles let the CTAs drift
  // apart over the ~440 tiles each processes, and a panel's 8 consumers then spread beyond what
  // L2 holds: ncu measured 33 GB of DRAM reads per 1024^3 pass against 8.6 GB algorithmic).
  const uint32_t crank = CL > 1 ? cluster_rank() : 0;
  const long long cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int ngroups = args.ntiles_n / CL;
  const int nsub = (CL == 1 && ngroups % 4 == 0) ? 4 : 1;
  const int upp = ngroups / nsub;  // units per panel
  const long long total_units = args.ntiles_m * upp;
  const long long my_units = cid < total_units ? (total_units - 1 - cid) / ncl + 1 : 0;
  const long long my_tiles = my_units * nsub;
  const long long total_it = my_tiles * KT;
  // local tile lt -> (row panel, N-group)
  auto tile_pos = [&](long long lt, long long& panel, int& grp) {
    const long long j = lt / nsub;
    const int sub = static_cast<int>(lt - j * nsub);
    const long long u = cid + j * ncl;
    panel = u / upp;
    grp = static_cast<int>(u - panel * upp) * nsub + sub;
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS * CL);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (CL > 1)
    cluster_sync();  // peers' barriers are initialised before any remote arrive / multicast
  else
    __syncthreads();

  // ------------------------------------------------------------------ producer state --
  // Lane 0 of warp 0 is the TMA producer (a dedicated producer warp would cap the DMMA warps at
  // 168 registers): it refills slot (it + STAGES - 1) % STAGES once all eight warps released it.
  const bool producer = tid == 0;
  long long p_tile = -1;  // local tile index the producer state below describes
  long long p_row0 = 0;
  int p_col0 = 0;
  int box_p[BM / 16], box_q[BM / 16];
  auto producer_tile = [&](long long lt) {
    p_tile = lt;
    long long panel;
    int grp;
    tile_pos(lt, panel, grp);
    p_row0 = panel * BM;
    p_col0 = (grp * CL + static_cast<int>(crank)) * BN;
    if (LOADER == TL_STRIDED && !args.x2d) {
      // (p, q) of each 16-row box (pre % 16 == 0: a box never straddles two q)
      long long q = p_row0 / args.pre;
      long long pp = p_row0 - q * args.pre;
#pragma unroll
      for (int b = 0; b < BM / 16; ++b) {
        box_p[b] = static_cast<int>(pp);
        box_q[b] = static_cast<int>(q);
        pp += 16;
        if (pp >= args.pre) {
          pp -= args.pre;
          ++q;
        }
      }
    }
  };
  // producer cursor: (local tile, k tile, ring slot, ring phase) advanced incrementally (no
  // 64-bit divisions on the producer's critical path)
  long long c_lt = 0;
  int c_kt = 0, c_slot = 0;
  uint32_t c_phase = 0;
  auto issue = [&]() {
    if (c_lt != p_tile) producer_tile(c_lt);
    const int s = c_slot;
    const int kt = c_kt;
    mbar_wait(&empty[s], c_phase ^ 1);
    if (++c_slot == STAGES) {
      c_slot = 0;
      c_phase ^= 1;
    }
    if (++c_kt == KT) {
      c_kt = 0;
      ++c_lt;
    }
    unsigned char* xs = smem + s * C::STAGE_BYTES;
    unsigned char* as = xs + C::X_BYTES;
    mbar_expect_tx(&full[s], C::STAGE_BYTES);
    const int k0 = kt * BK;
    constexpr uint16_t mask = static_cast<uint16_t>((1u << CL) - 1u);
    auto x2 = [&](void* dst, int c0, int c1, int b) {
      if (CL == 1)
        tma_load_2d(dst, &tmx, c0, c1, &full[s]);
      else if (b % CL == static_cast<int>(crank))
        tma_load_2d_mc(dst, &tmx, c0, c1, &full[s], mask);
    };
    if (LOADER == TL_STRIDED) {
#pragma unroll
      for (int b = 0; b < BM / 16; ++b) {
        if (args.x2d) {
          x2(xs + b * BOX_STRIDED_BYTES, static_cast<int>(p_row0) + 16 * b, k0, b);
        } else if (CL == 1) {
          tma_load_3d(xs + b * BOX_STRIDED_BYTES, &tmx, box_p[b], k0, box_q[b], &full[s]);
        } else if (b % CL == static_cast<int>(crank)) {
          tma_load_3d_mc(xs + b * BOX_STRIDED_BYTES, &tmx, box_p[b], k0, box_q[b], &full[s],
                         mask);
        }
      }
    } else if (LOADER == TL_CONTIG) {
#pragma unroll
      for (int h = 0; h < BK / 16; ++h)
        x2(xs + h * BOX_CONTIG_BYTES, k0 + 16 * h, static_cast<int>(p_row0), h);
    } else {
#pragma unroll
      for (int h = 0; h < BK / 8; ++h)
        x2(xs + h * BOX_CPLX0_BYTES, 2 * (k0 + 8 * h), static_cast<int>(p_row0 >> 1), h);
    }
#pragma unroll
    for (int c = 0; c < BN / 16; ++c)
      tma_load_2d(as + c * BOX_STRIDED_BYTES, &tma, p_col0 + 16 * c, k0, &full[s]);
  };
  if (producer) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmx) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tma) : "memory");
    for (long long it = 0; it < STAGES - 1 && it < total_it; ++it) issue();
  }

  // ---------------------------------------------------------------- DMMA consumers --
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int cs = chS(g);
  const EpiParams& ep = args.ep;
  const long long pre = args.pre, R = args.R, ycol = args.ycol;
  const int m = args.m;
  const bool spectral =
      ep.kind == EPI_SPEC_MUL || ep.kind == EPI_SPEC_DIV || ep.kind == EPI_SPEC_PHASE;
  long long it = 0;
  int slot = 0;
  uint32_t phase = 0;
  for (long long lt = 0; lt < my_tiles; ++lt) {
    long long panel;
    int grp;
    tile_pos(lt, panel, grp);
    const long long row0 = panel * BM;
    const int col0 = (grp * CL + static_cast<int>(crank)) * BN;
    double* w_rowlam = s_tab + warp * C::WTAB;
    double* w_collam = w_rowlam + C::WTM;
    if (EK == EK_DIV || EK == EK_MUL || EK == EK_PHASE) {
      // this warp's rows / columns of the tile: one index decomposition per row (32-bit: TMA
      // passes have R < 2^31) and one eigenvalue load per column, latency hidden behind the
      // first stage's wait; the warp owns its table (no CTA barrier couples the warps)
      __syncwarp();
#pragma unroll
      for (int k = lane; k < C::WTM; k += 32) {
        const long long r = row0 + wm * C::WTM + k;
        w_rowlam[k] = r < R ? lambda_partial_low_ext(ep, args.rot ? r : r % pre, ep.axis) : 0.0;
      }
      const int c = col0 + wn * C::WTN + lane;
      w_collam[lane] = c < m ? ep.lam[ep.axis][c] : 0.0;
      __syncwarp();
    }
    double acc[C::RT][C::CT][2];
#pragma unroll
    for (int i = 0; i < C::RT; ++i)
#pragma unroll
      for (int j = 0; j < C::CT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt, ++it) {
      if (producer && it + STAGES - 1 < total_it) issue();
      const int s = slot;
      mbar_wait(&full[s], phase);
      if (++slot == STAGES) {
        slot = 0;
        phase ^= 1;
      }
      const char* xs = reinterpret_cast<const char*>(smem + s * C::STAGE_BYTES);
      const char* as = xs + C::X_BYTES;
      if (LOADER == TL_STRIDED || LOADER == TL_CPLX0) {
#pragma unroll
        for (int k4 = 0; k4 < BK / 4; ++k4) {
          const int kk = k4 * 4 + t;
          const uint32_t rowoff = kk * 128 + ((cs ^ (kk & 7)) << 4);
          double af[C::RT], bf[C::CT];
#pragma unroll
          for (int bb = 0; bb < C::RT / 2; ++bb) {
            double2 v;
            if (LOADER == TL_STRIDED) {
              v = lds128(xs, (wm * (C::RT / 2) + bb) * BOX_STRIDED_BYTES + rowoff);
            } else {
              const int ql = wm * (C::WTM / 2) + bb * 8 + cs;  // ql & 7 == chS(g)
              v = lds128(xs, (kk >> 3) * BOX_CPLX0_BYTES + ql * 128 + (((kk & 7) ^ cs) << 4));
            }
            af[2 * bb] = v.x;
            af[2 * bb + 1] = v.y;
          }
#pragma unroll
          for (int cc = 0; cc < C::CT / 2; ++cc) {
            const double2 w = lds128(as, (wn * (C::CT / 2) + cc) * BOX_STRIDED_BYTES + rowoff);
            bf[2 * cc] = w.x;
            bf[2 * cc + 1] = w.y;
          }
#pragma unroll
          for (int i = 0; i < C::RT; ++i)
#pragma unroll
            for (int j = 0; j < C::CT; ++j) dmma884(acc[i][j], af[i], bf[j]);
        }
      } else {
#pragma unroll
        for (int kb = 0; kb < BK / 8; ++kb) {
          double a0[C::RT], a1[C::RT];
          const int h = kb >> 1;
          const int chunk = ((kb & 1) << 2) | t;
#pragma unroll
          for (int rt = 0; rt < C::RT; ++rt) {
            const int row = wm * C::WTM + rt * 8 + cs;  // row & 7 == chS(g)
            const double2 v =
                lds128(xs, h * BOX_CONTIG_BYTES + row * 128 + ((chunk ^ (row & 7)) << 4));
            a0[rt] = v.x;  // k = kb*8 + 2t
            a1[rt] = v.y;  // k = kb*8 + 2t + 1
          }
#pragma unroll
          for (int sstep = 0; sstep < 2; ++sstep) {
            const int kk = kb * 8 + 2 * t + sstep;
            const uint32_t rowoff = kk * 128 + ((g ^ (kk & 7)) << 4);
            double bf[C::CT];
#pragma unroll
            for (int cc = 0; cc < C::CT / 2; ++cc) {
              const double2 w = lds128(as, (wn * (C::CT / 2) + cc) * BOX_STRIDED_BYTES + rowoff);
              bf[2 * cc] = w.x;
              bf[2 * cc + 1] = w.y;
            }
#pragma unroll
            for (int i = 0; i < C::RT; ++i)
#pragma unroll
              for (int j = 0; j < C::CT; ++j) dmma884(acc[i][j], sstep ? a1[i] : a0[i], bf[j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        if (CL == 1) {
          mbar_arrive(&empty[s]);
        } else {
#pragma unroll
          for (int q = 0; q < CL; ++q) mbar_arrive_cluster(&empty[s], q);
        }
      }
    }

    // --------------------------------------------------------------------- epilogue --
    if (EK == EK_DIV) {
      // lambda = (lo + L_axis[i]) in axis order (direct_sum_grid), true division by
      // (lambda - shift) (operators.cpp:56-57): a row's 2 CT divisions are in flight together
#pragma unroll
      for (int j = 0; j < C::RT; ++j) {
        const int lr = row_map<BN, LOADER>(j, g);
        const long long r = row0 + wm * C::WTM + lr;
        const bool rok = r < R;
        const long long q = rok ? r / pre : 0;
        const long long ybase = (rok ? r - q * pre : 0) + q * args.ldy;
        const double lam_lo = w_rowlam[lr];
        double qv[C::CT][2], dv[C::CT][2];
        bool all_ok = true;
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int lc = col_map<BN, LOADER>(jc, 2 * t + v);
            dv[jc][v] = __dsub_rn(__dadd_rn(lam_lo, w_collam[lc]), ep.shift);
            bool ok;
            qv[jc][v] = div_rn_fast(acc[j][jc][v], dv[jc][v], ok);
            all_ok = all_ok && ok;
          }
        if (!all_ok) {
#pragma unroll
          for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
            for (int v = 0; v < 2; ++v) qv[jc][v] = __ddiv_rn(acc[j][jc][v], dv[jc][v]);
        }
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int i = col0 + wn * C::WTN + col_map<BN, LOADER>(jc, 2 * t + v);
            if (rok && i < m) args.y[ybase + ycol * static_cast<long long>(i)] = qv[jc][v];
          }
      }
    } else if (EK == EK_MUL) {
#pragma unroll
      for (int j = 0; j < C::RT; ++j) {
        const int lr = row_map<BN, LOADER>(j, g);
        const long long r = row0 + wm * C::WTM + lr;
        const bool rok = r < R;
        const long long q = rok ? r / pre : 0;
        const long long ybase = (rok ? r - q * pre : 0) + q * args.ldy;
        const double lam_lo = w_rowlam[lr];
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int lc = col_map<BN, LOADER>(jc, 2 * t + v);
            const int i = col0 + wn * C::WTN + lc;
            const double ls = __dsub_rn(__dadd_rn(lam_lo, w_collam[lc]), ep.shift);
            if (rok && i < m)
              args.y[ybase + ycol * static_cast<long long>(i)] = __dmul_rn(acc[j][jc][v], ls);
          }
      }
    } else if (EK == EK_PHASE) {
      // rows j (re) and j + 1 (im) of a pair are the same spatial point (paired row maps, even
      // pre, BM-aligned tiles): one sincos of -(lambda - shift) dt serves both (operators.cpp:68-71)
#pragma unroll
      for (int j = 0; j < C::RT; j += 2) {
        const int lr = row_map<BN, LOADER>(j, g);
        const long long r = row0 + wm * C::WTM + lr;
        const bool rok = r < R;  // R and r are even: the partner row r + 1 is in range too
        const long long q = rok ? r / pre : 0;
        const long long ybase = (rok ? r - q * pre : 0) + q * args.ldy;
        const double lam_lo = w_rowlam[lr];
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int lc = col_map<BN, LOADER>(jc, 2 * t + v);
            const int i = col0 + wn * C::WTN + lc;
            const double ls = __dsub_rn(__dadd_rn(lam_lo, w_collam[lc]), ep.shift);
            const double phase = __dmul_rn(-ls, ep.dt);
            double sn, cs;
            sincos(phase, &sn, &cs);
            const double re = acc[j][jc][v], im = acc[j + 1][jc][v];
            if (rok && i < m) {
              const long long yi = ybase + ycol * static_cast<long long>(i);
              args.y[yi] = __dsub_rn(__dmul_rn(re, cs), __dmul_rn(im, sn));
              args.y[yi + 1] = __dadd_rn(__dmul_rn(re, sn), __dmul_rn(im, cs));
            }
          }
      }
    } else if (EK == EK_AXPY) {
      // (acc + diag .* u) - sigma u (operators.cpp:102; ground_state.cpp:70-72)
#pragma unroll
      for (int j = 0; j < C::RT; ++j) {
        const long long r = row0 + wm * C::WTM + row_map<BN, LOADER>(j, g);
        const bool rok = r < R;
        const long long rr = rok ? r : 0;
        const long long q = rr / pre;
        const long long ybase = rr - q * pre + q * args.ldy;
        long long yi[C::CT][2];
        double uu[C::CT][2], dg[C::CT][2];
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int i = col0 + wn * C::WTN + col_map<BN, LOADER>(jc, 2 * t + v);
            const bool ok = rok && i < m;
            yi[jc][v] = ok ? ybase + ycol * static_cast<long long>(i) : -1;
            uu[jc][v] = ok ? ep.u[yi[jc][v]] : 0.0;
            dg[jc][v] = (ok && ep.diag) ? ep.diag[ep.cplx ? (yi[jc][v] >> 1) : yi[jc][v]] : 0.0;
          }
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            double val = acc[j][jc][v];
            if (ep.diag) val = __dadd_rn(val, __dmul_rn(dg[jc][v], uu[jc][v]));
            if (ep.sigma != 0.0) val = __dsub_rn(val, __dmul_rn(ep.sigma, uu[jc][v]));
            if (yi[jc][v] >= 0) args.y[yi[jc][v]] = val;
          }
      }
    } else if (EK == EK_SPLIT) {
      // destination of each of the thread's columns (one range lookup per column per tile)
      double* cb[C::CT][2];
      long long cqv[C::CT][2];
#pragma unroll
      for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int i = col0 + wn * C::WTN + col_map<BN, LOADER>(jc, 2 * t + v);
          int k = 0;
          while (k + 1 < args.split.parts && i >= args.split.i0[k + 1]) ++k;
          cb[jc][v] = i < m ? args.split.dst[k] + (i - args.split.i0[k]) * args.split.ccol[k]
                            : nullptr;
          cqv[jc][v] = args.split.cq[k];
        }
#pragma unroll
      for (int j = 0; j < C::RT; ++j) {
        const long long r = row0 + wm * C::WTM + row_map<BN, LOADER>(j, g);
        if (r >= R) continue;
        const long long q = r / pre;
        const long long p = r - q * pre;
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            if (cb[jc][v]) cb[jc][v][p + q * cqv[jc][v]] = acc[j][jc][v];
      }
      // the stores may go to another GPU (NVLink peer memory, possibly mapped from another
      // process): order them before whatever signals the peer next (the exchange barrier)
      __threadfence_system();
    } else {
#pragma unroll
      for (int j = 0; j < C::RT; ++j) {
        const long long r = row0 + wm * C::WTM + row_map<BN, LOADER>(j, g);
        const bool rok = r < R;
        const long long rr = rok ? r : 0;
        const long long q = rr / pre;
        const long long p = rr - q * pre;
        const long long ybase = p + q * args.ldy;
        const double lam_lo =
            (EK == EK_GENERIC && spectral) ? lambda_partial_low_ext(ep, args.rot ? rr : p, ep.axis)
                                            : 0.0;
#pragma unroll
        for (int jc = 0; jc < C::CT; ++jc) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int i = col0 + wn * C::WTN + col_map<BN, LOADER>(jc, 2 * t + v);
            const bool ok = rok && i < m;
            double val = acc[j][jc][v];
            const long long yi = ybase + ycol * static_cast<long long>(ok ? i : 0);
            if (EK == EK_GENERIC) {
              if (spectral) {
                // PHASE: the re/im partner (row r ^ 1) is this thread's tile j ^ 1 (paired maps)
                const double other = ep.kind == EPI_SPEC_PHASE ? acc[j ^ 1][jc][v] : 0.0;
                val = spectral_epilogue_ext(ep, val, other, lam_lo, ep.axis, ok ? i : -1, q, p);
              } else if (ep.kind == EPI_AXPY_DIAG && ok) {
                const double uu = ep.u[yi];
                if (ep.diag)
                  val = __dadd_rn(val, __dmul_rn(ep.diag[ep.cplx ? (yi >> 1) : yi], uu));
                if (ep.sigma != 0.0) val = __dsub_rn(val, __dmul_rn(ep.sigma, uu));
              } else if (ep.kind == EPI_BPHASE) {  // partner = tile j ^ 1, as for the phase
                const double other = acc[j ^ 1][jc][v];
                if (ok) val = bphase_rotate(val, other, ep.diag, yi >> 1, ep.dt, (j & 1) != 0);
              }
            }
            if (ok) args.y[yi] = val;
          }
        }
      }
    }
  }
  if (CL > 1) cluster_sync();  // no CTA leaves while peers may still arrive on its barriers
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    KCUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      fail(KRONOP_ERUNTIME, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims,
            const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base),
                                 dims, strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(KRONOP_ERUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

template <int BN, int LOADER>
void set_attr_tma() {
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 1, EK_GENERIC>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 1, EK_STORE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 1, EK_DIV>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 1, EK_MUL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 1, EK_AXPY>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 1, EK_SPLIT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  if (LOADER != TL_CONTIG)
    KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 1, LOADER != TL_CONTIG ? EK_PHASE : EK_GENERIC>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 2, EK_GENERIC>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  KCUDA(cudaFuncSetAttribute(mode_product_tma_kernel<BN, LOADER, 4, EK_GENERIC>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
}

// Largest grid (multiple of CL, <= #SMs) of co-resident CL-CTA clusters, 0 if none fit.
template <int BN, int LOADER, int CL>
int cluster_grid(int num_sms) {
  static int grid = [num_sms] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms / CL * CL));
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = Cfg<BN>::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, mode_product_tma_kernel<BN, LOADER, CL, EK_GENERIC>,
                                       &cfg) !=
        cudaSuccess) {
      (void)cudaGetLastError();
      return 0;
    }
    return n * CL < num_sms ? n * CL : num_sms / CL * CL;
  }();
  return grid;
}

template <int BN, int LOADER, int CL>
void launch_cl(cudaStream_t s, int blocks, const CUtensorMap& tmx, const CUtensorMap& tmA,
               const TArgs& ta) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = Cfg<BN>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KCUDA(cudaLaunchKernelEx(&cfg, mode_product_tma_kernel<BN, LOADER, CL, EK_GENERIC>, tmx, tmA,
                           ta));
}

// Cluster size. Default 1: measured on B200 (profiles/r01_tma_cluster_experiment.json), 2-CTA
// clusters with X multicast cut the 1024^3 pass's DRAM reads from 33-43 GB to 14-19 GB (8.6 GB
// algorithmic) but run 5% slower (a stage is refilled only when both CTAs released it, and 3
// stages of 64 KB leave no slack), 4-CTA clusters reach 10 GB but lose 20-40% (fewer co-resident
// CTAs). The pass is DMMA-bound, so time wins: KRONOP_TMA_CLUSTER=2|4 selects the cluster path.
template <int BN, int LOADER>
void launch_tma(cudaStream_t s, int num_sms, long long ntiles_m, int ntiles_n,
                const CUtensorMap& tmx, const CUtensorMap& tmA, const TArgs& ta) {
  static const int forced = [] {
    const char* e = getenv("KRONOP_TMA_CLUSTER");
    return e ? atoi(e) : 0;
  }();
  const long long tiles = ntiles_m * ntiles_n;
  int cl = 1;
  for (int c : {4, 2}) {
    if (c != forced || ta.split.parts > 0) continue;  // the cluster kernels store plainly
    if (ntiles_n % c != 0 || tiles < 4LL * num_sms) continue;
    const int g = c == 4 ? cluster_grid<BN, LOADER, 4>(num_sms) : cluster_grid<BN, LOADER, 2>(num_sms);
    if (g >= num_sms - (forced ? num_sms : 0) && g > 0) {
      cl = c;
      break;
    }
  }
  if (cl == 4) {
    launch_cl<BN, LOADER, 4>(s, cluster_grid<BN, LOADER, 4>(num_sms), tmx, tmA, ta);
  } else if (cl == 2) {
    launch_cl<BN, LOADER, 2>(s, cluster_grid<BN, LOADER, 2>(num_sms), tmx, tmA, ta);
  } else {
    const long long blocks = tiles < num_sms ? tiles : num_sms;  // one CTA per SM
    const EpiParams& ep = ta.ep;
    const dim3 grid(static_cast<unsigned>(blocks));
    const bool last_axis = ep.axis + 1 == ep.ndims && ep.lam[ep.axis] != nullptr;
    if (ta.split.parts > 0)
      mode_product_tma_kernel<BN, LOADER, 1, EK_SPLIT><<<grid, NTHREADS, Cfg<BN>::SMEM, s>>>(
          tmx, tmA, ta);
    else if (ep.kind == EPI_STORE)
      mode_product_tma_kernel<BN, LOADER, 1, EK_STORE><<<grid, NTHREADS, Cfg<BN>::SMEM, s>>>(
          tmx, tmA, ta);
    else if (ep.kind == EPI_SPEC_DIV && last_axis)
      mode_product_tma_kernel<BN, LOADER, 1, EK_DIV><<<grid, NTHREADS, Cfg<BN>::SMEM, s>>>(
          tmx, tmA, ta);
    else if (ep.kind == EPI_SPEC_MUL && last_axis)
      mode_product_tma_kernel<BN, LOADER, 1, EK_MUL><<<grid, NTHREADS, Cfg<BN>::SMEM, s>>>(
          tmx, tmA, ta);
    else if (ep.kind == EPI_SPEC_PHASE && last_axis && ep.cplx && LOADER != TL_CONTIG)
      mode_product_tma_kernel<BN, LOADER, 1, LOADER != TL_CONTIG ? EK_PHASE : EK_GENERIC>
          <<<grid, NTHREADS, Cfg<BN>::SMEM, s>>>(tmx, tmA, ta);
    else if (ep.kind == EPI_AXPY_DIAG)
      mode_product_tma_kernel<BN, LOADER, 1, EK_AXPY><<<grid, NTHREADS, Cfg<BN>::SMEM, s>>>(
          tmx, tmA, ta);
    else
      mode_product_tma_kernel<BN, LOADER, 1, EK_GENERIC><<<grid, NTHREADS, Cfg<BN>::SMEM, s>>>(
          tmx, tmA, ta);
  }
}

}  // namespace

void prime_mode_product_tma_kernels() {
  set_attr_tma<128, TL_CPLX0>();
  set_attr_tma<64, TL_CPLX0>();
  set_attr_tma<128, TL_STRIDED>();
  set_attr_tma<128, TL_CONTIG>();
  set_attr_tma<64, TL_STRIDED>();
  set_attr_tma<64, TL_CONTIG>();
}

bool mode_product_tma_eligible(const double* x, const PassShape& ps) {
  if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return false;
  if (ps.pre * ps.post > 0x7fffffffLL) return false;  // TMA coordinates are 32-bit
  if (ps.ldx_eff() % 2 != 0) return false;           // q-stride * 8 must be 16-B aligned
  if (ps.pre == 1) return true;                       // CONTIG: row stride ldx
  if (ps.pre == 2) return true;                       // complex axis 0 (TL_CPLX0), rows of ldx
  if (ps.pre % 2 != 0) return false;                  // k stride pre * 8 must be 16-B aligned
  return ps.post == 1 || ps.pre % 16 == 0;            // a 16-row box never straddles two q
}

void launch_mode_product_tma(cudaStream_t s, const double* x, double* y, const double* a_pad,
                             int lda, const PassShape& ps, const EpiParams& ep) {
  TArgs ta;
  ta.y = y;
  ta.x2d = 0;
  ta.pre = ps.pre;
  ta.post = ps.post;
  ta.R = ps.pre * ps.post;
  ta.ldy = ps.ldy_eff();
  ta.ycol = ps.ycol ? ps.ycol : ps.pre;
  ta.rot = ps.rot;
  ta.split = ps.split ? *ps.split : SplitDst{};
  param_check(!ps.split || (ep.kind == EPI_STORE && !ps.rot && ps.split->parts >= 1 &&
                            ps.split->parts <= kMaxSplit),
              "mode_product: exchange-fused store needs a plain, unrotated pass");
  param_check(!ps.rot || ep.axis + 1 >= ep.ndims || (ep.kind != EPI_SPEC_MUL &&
              ep.kind != EPI_SPEC_DIV && ep.kind != EPI_SPEC_PHASE),
              "mode_product: rotated pass with a spectral epilogue must be on the last axis");
  ta.nk = ps.nk;
  ta.m = ps.m;
  ta.ep = ep;
  const int bn = ps.m > 64 ? 128 : 64;
  ta.ntiles_n = (ps.m + bn - 1) / bn;
  ta.ntiles_m = (ta.R + BM - 1) / BM;
  CUtensorMap tmx, tmA;
  const int kp = pad_up(ps.nk, kMatPadK);
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(lda), static_cast<cuuint64_t>(kp)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(lda) * 8};
    const cuuint32_t box[2] = {16, BK};
    encode(&tmA, a_pad, 2, dims, str, box);
  }
  const bool contig = ps.pre == 1;
  const bool cplx0 = ps.pre == 2;
  if (cplx0) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * ps.nk),
                                static_cast<cuuint64_t>(ps.post)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(ps.ldx_eff()) * 8};
    const cuuint32_t box[2] = {16, BM / 2};
    encode(&tmx, x, 2, dims, str, box);
  } else if (contig) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ps.nk), static_cast<cuuint64_t>(ta.R)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(ps.ldx_eff()) * 8};
    const cuuint32_t box[2] = {16, BM};
    encode(&tmx, x, 2, dims, str, box);
  } else if (ps.post == 1) {
    ta.x2d = 1;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ps.pre), static_cast<cuuint64_t>(ps.nk)};
    const cuuint64_t str[1] = {static_cast<cuuint64_t>(ps.pre) * 8};
    const cuuint32_t box[2] = {16, BK};
    encode(&tmx, x, 2, dims, str, box);
  } else {
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(ps.pre), static_cast<cuuint64_t>(ps.nk),
                                static_cast<cuuint64_t>(ps.post)};
    const cuuint64_t str[2] = {static_cast<cuuint64_t>(ps.pre) * 8,
                               static_cast<cuuint64_t>(ps.ldx_eff()) * 8};
    const cuuint32_t box[3] = {16, BK, 1};
    encode(&tmx, x, 3, dims, str, box);
  }
  static int num_sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  if (cplx0) {
    if (bn == 128)
      launch_tma<128, TL_CPLX0>(s, num_sms, ta.ntiles_m, ta.ntiles_n, tmx, tmA, ta);
    else
      launch_tma<64, TL_CPLX0>(s, num_sms, ta.ntiles_m, ta.ntiles_n, tmx, tmA, ta);
  } else if (bn == 128) {
    if (contig)
      launch_tma<128, TL_CONTIG>(s, num_sms, ta.ntiles_m, ta.ntiles_n, tmx, tmA, ta);
    else
      launch_tma<128, TL_STRIDED>(s, num_sms, ta.ntiles_m, ta.ntiles_n, tmx, tmA, ta);
  } else {
    if (contig)
      launch_tma<64, TL_CONTIG>(s, num_sms, ta.ntiles_m, ta.ntiles_n, tmx, tmA, ta);
    else
      launch_tma<64, TL_STRIDED>(s, num_sms, ta.ntiles_m, ta.ntiles_n, tmx, tmA, ta);
  }
  KCUDA(cudaGetLastError());
}

}  // namespace kronop_dev
