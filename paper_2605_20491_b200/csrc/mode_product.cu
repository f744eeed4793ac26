// Mode-k eigenbasis transform on B200 (sm_100a): FP64 tensor-core (DMMA) GEMM pass with fused
// spectral / V2 epilogues.
//
// Reference hot loop this replaces: contract_first_axis / contract_inner_axis
// (proj/src/tensor.cpp:31-84) called by mode_product (tensor.cpp:105-134), plus the pointwise loops
// fused into the epilogue: x(lambda - shift) (operators.cpp:36), /(lambda - shift)
// (operators.cpp:57), exp(-i(lambda - shift)dt) (operators.cpp:68-71), + V2 u (operators.cpp:102),
// - sigma u (ground_state.cpp:70-72).
//
// B200 facts that shape the kernel (profiles/r01_fp64_instr_peak.txt): tcgen05 has no f64 kind, so
// FP64 tensor math is the warp-level DMMA (SASS DMMA.8x8x4; mma.sync m8n8k4 .f64), measured at
// 37 TFLOP/s peak (DFMA 34). A pass at n = 1024 has arithmetic intensity n/8 = 128 flop/B, far
// above the HBM ridge (~6 flop/B), so the kernel is built to keep the DMMA pipe busy:
//   * 128 x BN x 16 CTA tiles, 8 warps, 64x32 (or 32x32) warp tiles = 32 (16) independent DMMAs
//     per k-step per warp; accumulators stay in registers;
//   * 4-stage cp.async.cg (LDGSTS, L2-only) producer pipeline into padded shared memory laid out
//     so every fragment load is 2 wavefronts (the minimum for 32 x 8 B);
//   * per-axis matrices live on device zero-padded to (128, 16) multiples, so B-operand loads
//     carry no predicates; X loads zero-fill out-of-range rows/columns;
//   * 1-D grid, N-tiles fastest, so the 8 CTAs that share an X panel run together and the panel
//     is read from HBM once and served from L2 for the other 7.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "epilogue.cuh"
#include "kronop_internal.cuh"

namespace kronop_dev {
namespace {

constexpr int BM = 128;
#ifndef KRONOP_BK
#define KRONOP_BK 32
#endif
#ifndef KRONOP_STAGES
#define KRONOP_STAGES 3
#endif
constexpr int BK = KRONOP_BK;          // contraction depth per pipeline stage
constexpr int STAGES = KRONOP_STAGES;  // cp.async pipeline depth
constexpr int NTHREADS = 256;

enum LoaderKind : int { LD_CONTIG = 0, LD_STRIDED_R = 1, LD_STRIDED_K = 2 };

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_size));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_size));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int BN>
struct TileCfg {
  static constexpr int WARPS_N = BN == 128 ? 4 : 2;
  static constexpr int WARPS_M = 8 / WARPS_N;
  static constexpr int WTM = BM / WARPS_M;  // 64 or 32
  static constexpr int WTN = BN / WARPS_N;  // 32
  static constexpr int RB = WTM / 8;
  static constexpr int CB = WTN / 8;
  // A-tile row stride (doubles) = 4 mod 16: the 16 lanes of each half-warp phase of a 64-bit
  // fragment load (g = 0..3 or 4..7, t = 0..3 at t*S + g) hit 16 distinct bank pairs.
  static constexpr int SAN = BN + 4;
};

template <int LOADER>
struct XLayout {
  // CONTIG: [BM][BK+4] (k fastest); strided: [BK][BM+4] (rows fastest). Both strides are
  // 4 mod 16 doubles => conflict-free 64-bit fragment loads (see TileCfg::SAN).
  static constexpr int STRIDE = LOADER == LD_CONTIG ? BK + 4 : BM + 4;
  static constexpr int ELEMS = LOADER == LD_CONTIG ? BM * (BK + 4) : BK * (BM + 4);
};

template <int BN, int LOADER>
constexpr int smem_bytes() {
  return STAGES * (XLayout<LOADER>::ELEMS + BK * TileCfg<BN>::SAN) * 8;
}

struct KArgs {
  const double* x;
  double* y;
  const double* a;
  int lda;
  long long pre, post, R;  // R = pre * post rows
  long long ldx, ldy;      // q-strides of X and Y
  int nk, m;
  int ntiles_n;
  long long ntiles_m;
  EpiParams ep;
};

__device__ __forceinline__ long long x_row_base(long long r, long long pre, long long ldx) {
  // X(r, j) lives at x_row_base(r) + pre * j (r = p + pre * q flattened; ldx = q-stride).
  const long long q = r / pre;
  return (r - q * pre) + q * ldx;
}

template <int BN, int LOADER, int VEC>
__global__ void __launch_bounds__(NTHREADS, 1) mode_product_kernel(const KArgs args) {
  if (args.ep.active && *args.ep.active == 0) return;
  using TC = TileCfg<BN>;
  using XL = XLayout<LOADER>;
  extern __shared__ __align__(128) double smem[];
  double* sx = smem;                                   // STAGES * XL::ELEMS
  double* sa = smem + STAGES * XL::ELEMS;              // STAGES * BK * SAN

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / TC::WARPS_N, wn = warp % TC::WARPS_N;

  const long long bid = blockIdx.x;
  const int ntile = static_cast<int>(bid % args.ntiles_n);
  const long long mtile = bid / args.ntiles_n;
  const long long row0 = mtile * BM;
  const int col0 = ntile * BN;

  const long long pre = args.pre, R = args.R;
  const int nk = args.nk;
  const double* __restrict__ x = args.x;
  const double* __restrict__ a = args.a;
  const int lda = args.lda;
  const int KT = (nk + BK - 1) / BK;

  // ---- per-thread load plan (fixed over the K loop) ----
  constexpr int XCH = BM * BK / VEC / NTHREADS;  // X chunks per thread per stage
  long long xoff[XCH];
  int xsm[XCH];   // smem offset (doubles) within a stage
  int xk[XCH];    // k offset within the tile
  bool xrow_ok[XCH];
#pragma unroll
  for (int s = 0; s < XCH; ++s) {
    const int c = tid + NTHREADS * s;
    int r, k;
    if (LOADER == LD_CONTIG) {
      constexpr int CPR = BK / VEC;  // chunks per row
      k = (c % CPR) * VEC;
      r = c / CPR;
    } else if (LOADER == LD_STRIDED_R) {
      constexpr int CPK = BM / VEC;  // chunks per k
      r = (c % CPK) * VEC;
      k = c / CPK;
    } else {
      k = c % BK;
      r = (c / BK) * VEC;
    }
    const long long grow = row0 + r;
    xrow_ok[s] = grow < R;
    const long long gr = xrow_ok[s] ? grow : 0;
    xoff[s] = LOADER == LD_CONTIG ? gr * args.ldx : x_row_base(gr, pre, args.ldx);
    xk[s] = k;
    xsm[s] = LOADER == LD_CONTIG ? r * XL::STRIDE + k : k * XL::STRIDE + r;
  }
  constexpr int ACH = BK * BN / 2 / NTHREADS;  // A chunks (16 B) per thread per stage
  int aoff[ACH], asm_[ACH], akk[ACH];
#pragma unroll
  for (int s = 0; s < ACH; ++s) {
    const int c = tid + NTHREADS * s;
    const int nn = (c % (BN / 2)) * 2;
    const int k = c / (BN / 2);
    aoff[s] = (col0 + nn) + lda * k;
    asm_[s] = k * TC::SAN + nn;
    akk[s] = k;
  }

  auto load_stage = [&](int slot, int kt) {
    const int k0 = kt * BK;
    double* dx = sx + slot * XL::ELEMS;
#pragma unroll
    for (int s = 0; s < XCH; ++s) {
      const int kg = k0 + xk[s];
      const bool ok = xrow_ok[s] && kg < nk;
      const long long go = xoff[s] + (LOADER == LD_CONTIG ? (long long)kg : pre * kg);
      const double* src = x + (ok ? go : 0);
      if (VEC == 2)
        cp_async16(dx + xsm[s], src, ok);
      else
        cp_async8(dx + xsm[s], src, ok);
    }
    double* da = sa + slot * (BK * TC::SAN);
    const double* ak = a + (long long)lda * k0;
    // matrix columns past nk are zero-filled, never read: the padded device copy holds
    // pad_up(nk, 16) columns but a BK = 32 stage can reach further (and 0 * NaN garbage from
    // whatever lies beyond the allocation would poison the sum)
#pragma unroll
    for (int s = 0; s < ACH; ++s) {
      const bool ok = k0 + akk[s] < nk;
      cp_async16(da + asm_[s], ok ? ak + aoff[s] : a, ok);
    }
  };

  double acc[TC::RB][TC::CB][2];
#pragma unroll
  for (int i = 0; i < TC::RB; ++i)
#pragma unroll
    for (int j = 0; j < TC::CB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nkt = kt + STAGES - 1;
      if (nkt < KT) load_stage(nkt % STAGES, nkt);
      cp_async_commit();
    }
    const int slot = kt % STAGES;
    const double* cx = sx + slot * XL::ELEMS;
    const double* ca = sa + slot * (BK * TC::SAN);
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int kk = k4 * 4 + t;
      double af[TC::RB], bf[TC::CB];
#pragma unroll
      for (int rb = 0; rb < TC::RB; ++rb) {
        const int row = wm * TC::WTM + rb * 8 + g;
        af[rb] = LOADER == LD_CONTIG ? cx[row * XL::STRIDE + kk] : cx[kk * XL::STRIDE + row];
      }
#pragma unroll
      for (int cb = 0; cb < TC::CB; ++cb) bf[cb] = ca[kk * TC::SAN + wn * TC::WTN + cb * 8 + g];
#pragma unroll
      for (int rb = 0; rb < TC::RB; ++rb)
#pragma unroll
        for (int cb = 0; cb < TC::CB; ++cb) dmma884(acc[rb][cb], af[rb], bf[cb]);
    }
  }
  cp_async_wait<0>();

  // ---------------------------------------------------------------- epilogue --
  const EpiParams& ep = args.ep;
  const int m = args.m;
  const long long mstride = args.ldy;  // output row base: (r % pre) + ldy*(r / pre)
#pragma unroll
  for (int rb = 0; rb < TC::RB; ++rb) {
    const long long r = row0 + wm * TC::WTM + rb * 8 + g;
    const bool rok = r < R;
    const long long rr = rok ? r : 0;
    const long long q = rr / pre;
    const long long p = rr - q * pre;
    const long long ybase = p + q * mstride;
    double lam_lo = 0.0;
    const int pass_axis = ep.axis;
    if (ep.kind == EPI_SPEC_MUL || ep.kind == EPI_SPEC_DIV || ep.kind == EPI_SPEC_PHASE)
      lam_lo = lambda_partial_low_ext(ep, p, pass_axis);
#pragma unroll
    for (int cb = 0; cb < TC::CB; ++cb) {
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = col0 + wn * TC::WTN + cb * 8 + 2 * t + v;
        const bool ok = rok && i < m;
        double val = acc[rb][cb][v];
        const long long yi = ybase + pre * (long long)(ok ? i : 0);
        switch (ep.kind) {
          case EPI_SPEC_MUL:
          case EPI_SPEC_DIV:
          case EPI_SPEC_PHASE: {
            // re/im rows are adjacent (leading re/im axis): partner lane holds row r ^ 1
            const double other =
                ep.kind == EPI_SPEC_PHASE ? __shfl_xor_sync(0xffffffffu, val, 4) : 0.0;
            val = spectral_epilogue_ext(ep, val, other, lam_lo, pass_axis, ok ? i : -1, q, p);
            break;
          }
          case EPI_AXPY_DIAG: {
            if (ok) {
              const double uu = ep.u[yi];
              if (ep.diag) {
                const long long si = ep.cplx ? (yi >> 1) : yi;
                val = __dadd_rn(val, __dmul_rn(ep.diag[si], uu));
              }
              if (ep.sigma != 0.0) val = __dsub_rn(val, __dmul_rn(ep.sigma, uu));
            }
            break;
          }
          case EPI_BPHASE: {
            const double other = __shfl_xor_sync(0xffffffffu, val, 4);
            if (ok) val = bphase_rotate(val, other, ep.diag, yi >> 1, ep.dt, (p & 1) != 0);
            break;
          }
          default:
            break;
        }
        if (ok) args.y[yi] = val;
      }
    }
  }
}

template <int BN, int LOADER, int VEC>
void set_attr() {
  KCUDA(cudaFuncSetAttribute(mode_product_kernel<BN, LOADER, VEC>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem_bytes<BN, LOADER>()));
}

template <int BN, int LOADER, int VEC>
void launch_cfg(cudaStream_t s, const KArgs& ka) {
  constexpr int SMEM = smem_bytes<BN, LOADER>();
  const long long blocks = ka.ntiles_m * ka.ntiles_n;
  mode_product_kernel<BN, LOADER, VEC><<<static_cast<unsigned>(blocks), NTHREADS, SMEM, s>>>(ka);
  KCUDA(cudaGetLastError());
}

template <int BN>
void dispatch_loader(cudaStream_t s, const KArgs& ka, int loader, int vec) {
  if (loader == LD_CONTIG) {
    if (vec == 2) launch_cfg<BN, LD_CONTIG, 2>(s, ka);
    else launch_cfg<BN, LD_CONTIG, 1>(s, ka);
  } else if (loader == LD_STRIDED_R) {
    if (vec == 2) launch_cfg<BN, LD_STRIDED_R, 2>(s, ka);
    else launch_cfg<BN, LD_STRIDED_R, 1>(s, ka);
  } else {
    if (vec == 2) launch_cfg<BN, LD_STRIDED_K, 2>(s, ka);
    else launch_cfg<BN, LD_STRIDED_K, 1>(s, ka);
  }
}

}  // namespace

// Opt every kernel instantiation into its dynamic shared memory size once per device, before any
// stream capture (cudaFuncSetAttribute is not a stream operation).
void prime_mode_product_kernels() {
  set_attr<128, LD_CONTIG, 1>();
  set_attr<128, LD_CONTIG, 2>();
  set_attr<128, LD_STRIDED_R, 1>();
  set_attr<128, LD_STRIDED_R, 2>();
  set_attr<128, LD_STRIDED_K, 1>();
  set_attr<128, LD_STRIDED_K, 2>();
  set_attr<64, LD_CONTIG, 1>();
  set_attr<64, LD_CONTIG, 2>();
  set_attr<64, LD_STRIDED_R, 1>();
  set_attr<64, LD_STRIDED_R, 2>();
  set_attr<64, LD_STRIDED_K, 1>();
  set_attr<64, LD_STRIDED_K, 2>();
}

bool mode_product_tma_enabled() {
  static const bool no_tma = [] {
    const char* e = getenv("KRONOP_DISABLE_TMA");  // A/B switch for profiling the cp.async kernel
    return e && e[0] == '1';
  }();
  return !no_tma;
}

void launch_mode_product(cudaStream_t s, const double* x, double* y, const double* a_pad, int lda,
                         const PassShape& ps, const EpiParams& ep) {
  param_check(ps.nk >= 1 && ps.m >= 1 && ps.pre >= 1 && ps.post >= 1,
              "mode_product: empty pass shape");
  param_check(lda >= pad_up(ps.m, kMatPadM), "mode_product: matrix leading dimension too small");
  if (mode_product_tma_enabled() && mode_product_tma_eligible(x, ps)) {
    launch_mode_product_tma(s, x, y, a_pad, lda, ps, ep);
    return;
  }
  param_check((ps.ycol == 0 || ps.ycol == ps.pre) && !ps.rot,
              "mode_product: rotated output needs the TMA kernel");
  KArgs ka;
  ka.x = x;
  ka.y = y;
  ka.a = a_pad;
  ka.lda = lda;
  ka.pre = ps.pre;
  ka.post = ps.post;
  ka.R = ps.pre * ps.post;
  ka.nk = ps.nk;
  ka.m = ps.m;
  ka.ldx = ps.ldx_eff();
  ka.ldy = ps.ldy_eff();
  ka.ep = ep;
  const int bn = ps.m > 64 ? 128 : 64;
  ka.ntiles_n = (ps.m + bn - 1) / bn;
  ka.ntiles_m = (ka.R + BM - 1) / BM;
  const bool x16 = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  int loader, vec;
  if (ps.pre == 1) {
    loader = LD_CONTIG;
    vec = (x16 && ps.ldx_eff() % 2 == 0) ? 2 : 1;
  } else {
    loader = ps.pre >= 32 ? LD_STRIDED_R : LD_STRIDED_K;
    vec = (x16 && ps.pre % 2 == 0 && ps.ldx_eff() % 2 == 0) ? 2 : 1;
  }
  if (ep.kind == EPI_SPEC_PHASE)
    param_check(ep.cplx && ps.pre % 2 == 0, "mode_product: phase epilogue needs complex data");
  if (bn == 128)
    dispatch_loader<128>(s, ka, loader, vec);
  else
    dispatch_loader<64>(s, ka, loader, vec);
}

}  // namespace kronop_dev
