// FP64 emulation on the INT8 tensor cores (Ozaki scheme): the separable
// solve (-Delta + V1 - shift)^{-1} b (operators.cpp:42-61) with every per-axis transform computed
// as a sum of exact INT8 x INT8 -> INT32 products on tcgen05 (kind::i8, TMEM accumulators).
//
// Splitting. Every row of an operand (a K-run of the field, or a row of an axis matrix) gets a
// power-of-two exponent e with max|x| < 2^e and is cut into S signed 8-bit slices by repeated
// rounding with the base 254 (|t| <= 127 at every step, so no slice ever needs -128 or 128):
//     t_0 = 127 x 2^-e,  a_s = rint(t_s),  t_{s+1} = 254 (t_s - a_s),   a_s in [-127, 127],
//     x = 2^e / 127 * sum_{s<S} a_s 254^-s + r,     |r| <= 2^e / 127 * 254^-(S-1) / 2.
// (Every operand is signed: the tcgen05 kind::i8 path as measured here gave wrong products for
// unsigned slices >= 128 under mixed s8 / u8 descriptors, so no unsigned slices are used.) A dot
// product of two split rows is then
//     sum_k x_k y_k = 2^(ex+ey) / 127^2 * sum_{g<S} 254^-g G_g,
//     G_g = sum_{s+t=g} sum_k a_s[k] b_t[k]   (exact in INT32: |G_g| <= S 127^2 K < 2^31)
// with the products s + t >= S (weight <= 254^-S) dropped: S(S+1)/2 INT8 products, error
// ~ K 254^-(S-1) max|x| max|y| per output. S = 7 carries ~55 bits, the FP64 DGEMM bound (the
// splitting and the FP64 Horner combination add only FP64 roundings of the parts).
//
// Layout. Split operands are stored pre-tiled in the exact shared-memory image the MMA reads:
// per (row panel of P rows, K-block of 32 bytes) one contiguous block of S slices, each slice in
// the canonical no-swizzle K-major UMMA layout (8-row x 16-byte core matrices, K-adjacent core
// matrices 128 B apart, 8-row groups 256 B apart). A pipeline stage is then two plain bulk copies
// (cp.async.bulk, S x 4 KB of X slices for 128 rows + S x 2 KB of matrix slices for 64 outputs).
//
// Pass kernel (persistent, one CTA per SM): warp 0 = bulk-copy producer over a 4-stage ring;
// warp 1 = TMEM allocator + single-thread MMA issuer: per stage, S(S+1)/2 tcgen05.mma
// (M = 128 rows, N = 64 outputs, K = 32) into S INT32 accumulators (group g at TMEM columns
// 64 g .. +64: 448 columns for S = 7); warps 2-9 = epilogue: Horner-combine the groups in FP64
// (exact INT32 -> FP64, weights 254^-g), scale by 2^(ex+ey) / 127^2, the fused spectral divide
// in FP64 (__ddiv_rn of the axis-order lambda sum, as mode_product_tma.cu), and the FP64 store of
// the rotated output Y[i * R + r] (the contracted axis moves to the slow end, as in tc_lowp.cu).
// A separate HBM-bound kernel splits each pass's FP64 output for the next pass.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "context.cuh"
#include "kronop_internal.cuh"
#include "vector_ops.cuh"

namespace kronop_dev {

namespace {

constexpr int OZ_BM = 128;  // field rows per tile (MMA M)
constexpr int OZ_BN = 64;   // outputs per tile (MMA N)
constexpr int OZ_BK = 32;   // K bytes per stage = one MMA
constexpr int OZ_STAGES = 5;
constexpr int OZ_KMAX = 3200;  // 8 staged rows of the split kernel in 227 KB (INT32 exact to 16384)
constexpr int OZ_THREADS = 320;
constexpr int OZ_EPI_WARPS = 8;
constexpr int OZ_TMEM_COLS = 512;
constexpr int OZ_PAIR = 2 * OZ_BM;  // rows of a 2-SM pair tile; field slices are padded to it

template <int S>
struct OzGeom {
  static constexpr int A_SLICE = OZ_BM * OZ_BK;  // 4 KB
  static constexpr int B_SLICE = OZ_BN * OZ_BK;  // 2 KB
  static constexpr int A = S * A_SLICE;
  static constexpr int B = S * B_SLICE;
  static constexpr int STAGE = A + B;
  static constexpr int SMEM = OZ_STAGES * STAGE + 1024 + 256;
};

struct OzArgs {
  const int8_t* xs;  // tiled slices of the field rows   [R/128][KB][S][128 x 32]
  const int* xe;     // row exponents (R padded)
  const int8_t* bs;  // tiled slices of the matrix rows  [m/64][KB][S][64 x 32]
  const int* be;     // output-row exponents
  double* y;
  long long R;
  int K, KB, m, ntn;
  long long ntm;
  int epi;  // 0 store, 1 divide by / 2 multiply by (lambda - shift), 3 complex phase
  double shift, dt;
  int axpy, cplx;      // last pass: + diag .* u - sigma u (operators.cpp:102)
  const double* diag;  // spatial (real), may be null
  const double* u;     // the transform's input, final layout
  double sigma;
  int nlow;
  int lowext[KRONOP_MAX_DIM];
  const double* lowlam[KRONOP_MAX_DIM];
  const double* lamlast;
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// K-major, no-swizzle UMMA descriptor (cute/arch/mma_sm100_desc.hpp SmemDescriptor; canonical
// layout ((8,m),(T,2)):((1T,SBO),(1,LBO)) of cute/atom/mma_traits_sm100.hpp): LBO = 128 B between
// the two K-adjacent core matrices, SBO = 256 B between 8-row groups, version 1, layout 0.
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(256 >> 4) << 32) | (1ull << 46);
}
// The same descriptor split in halves: the low word carries the start address, so the slices of
// a stage are reached by adding (offset >> 4) to one precomputed word (addresses < 256 KB: no
// carry out of the 14-bit field).
constexpr uint32_t kOzDescHi = (256 >> 4) | (1u << 14);
__device__ __forceinline__ uint32_t oz_desc_lo(uint32_t saddr) {
  return ((saddr >> 4) & 0x3FFF) | ((128 >> 4) << 16);
}
__device__ __forceinline__ uint64_t oz_desc_of(uint32_t lo) {
  return (static_cast<uint64_t>(kOzDescHi) << 32) | lo;
}
// one lane of a converged warp (elect.sync): the MMA warp runs its loop converged and only the
// issue is single-threaded, so the descriptors stay in uniform registers
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, %1;\n@px mov.s32 %0, 1;\n}\n"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}
// instruction descriptor: S8 x S8 -> S32, K-major A and B, N = 64, M = 128
__host__ __device__ constexpr uint32_t oz_idesc() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((OZ_BN >> 3) << 17) | ((OZ_BM >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(oz_idesc()), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Epilogue, part 1: Horner-combine this warp's 32 x 32 block of the S group accumulators
// (TMEM lane quadrant q, column half hc) from the smallest weight: acc = acc / 254 + G_g.
template <int S>
__device__ __forceinline__ void oz_drain(uint32_t tmem, int q, int hc, double (&acc)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.0;
#pragma unroll 1
  for (int g = S - 1; g >= 0; --g) {
    uint32_t v[32];
    tmem_ld32(tmem + g * OZ_BN + hc * 32 + (static_cast<uint32_t>(32 * q) << 16), v);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      acc[j] = fma(acc[j], 1.0 / 254.0, static_cast<double>(static_cast<int>(v[j])));
  }
}

// Row exponent marking a row (field run or matrix row) that holds a NaN / Inf: the slices of such
// a row are meaningless, so every output that contracts it is stored as NaN -- FP64 arithmetic
// (and the reference's Eigen GEMM) propagates non-finite values the same way.
constexpr int OZ_NONFINITE = 1 << 29;

// Epilogue, part 2: scale by 2^(ex+ey) / 127^2, the spectral divide (lambda summed in axis order
// from 0.0, minus the shift, IEEE divide: operators.cpp:57), rotated FP64 store y[col * R + r].
__device__ __forceinline__ void oz_store(const OzArgs& a, long long r, int c0, int lane,
                                         const double (&acc)[32]) {
  const bool live = r < a.R;
  const int er = live ? a.xe[r] : 0;
  double lam_low = 0.0;
  if (a.epi != 0 && live) {  // axes below the contracted one, in axis order from 0.0
    long long rr = a.cplx ? (r >> 1) : r;  // complex: rows are (re, im) pairs
    for (int j = 0; j < a.nlow; ++j) {
      const long long idx = rr % a.lowext[j];
      rr /= a.lowext[j];
      lam_low = __dadd_rn(lam_low, a.lowlam[j][idx]);
    }
  }
  const int ecol = c0 + lane < a.m ? a.be[c0 + lane] : 0;
  // this chunk's 32 column eigenvalues: one coalesced load, then broadcast by shuffle (a load
  // per element would serialise behind the stores, which may alias)
  const double lamc = a.epi != 0 && c0 + lane < a.m ? a.lamlast[c0 + lane] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {  // uniform (shuffles); stores predicated
    const int col = c0 + j;
    const int ec = __shfl_sync(0xffffffffu, ecol, j);
    const double lj = __shfl_sync(0xffffffffu, lamc, j);
    const int E = er + ec;  // 2^(ex+ey) / 127^2: exponent bits directly when in normal range
    const double v0 = acc[j] * (1.0 / 16129.0);
    double val = (E > -1000 && E < 1000)
                     ? v0 * __longlong_as_double(static_cast<long long>(1023 + E) << 52)
                     : ldexp(v0, E);
    if (er == OZ_NONFINITE || ec == OZ_NONFINITE) val = __longlong_as_double(0x7ff8000000000000LL);
    if (a.epi == 3) {  // partner row (re <-> im) is the neighbouring lane; as epilogue.cuh
      const double other = __shfl_xor_sync(0xffffffffu, val, 1);
      if (live && col < a.m) {
        const double ls = __dsub_rn(__dadd_rn(lam_low, lj), a.shift);
        double sn, cs;
        sincos(__dmul_rn(-ls, a.dt), &sn, &cs);
        const bool is_im = (r & 1) != 0;
        const double re = is_im ? other : val, im = is_im ? val : other;
        val = is_im ? __dadd_rn(__dmul_rn(re, sn), __dmul_rn(im, cs))
                    : __dsub_rn(__dmul_rn(re, cs), __dmul_rn(im, sn));
      }
    } else if ((a.epi == 1 || a.epi == 2) && live && col < a.m) {
      const double ls = __dsub_rn(__dadd_rn(lam_low, lj), a.shift);
      val = a.epi == 1 ? __ddiv_rn(val, ls) : __dmul_rn(val, ls);
    }
    const long long yi = static_cast<long long>(col) * a.R + r;
    if (a.axpy && live && col < a.m) {  // as the DMMA epilogue: (val + diag u) - sigma u
      const double uu = a.u[yi];
      if (a.diag) val = __dadd_rn(val, __dmul_rn(a.diag[a.cplx ? (yi >> 1) : yi], uu));
      if (a.sigma != 0.0) val = __dsub_rn(val, __dmul_rn(a.sigma, uu));
    }
    if (live && col < a.m) a.y[yi] = val;
  }
}

template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_pass_kernel(const OzArgs a) {
  using G = OzGeom<S>;
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + OZ_STAGES * G::STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* tfull = empty + OZ_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(tfull, 1);
    mb_init(tempty, OZ_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(OZ_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const long long tiles = a.ntm * a.ntn;  // output tiles fastest: CTAs share the row panel in L2
  if (warp == 0) {
    if (lane == 0) {  // producer
      long long it = 0;
      for (long long T = blockIdx.x; T < tiles; T += gridDim.x) {
        const long long tp = T / a.ntn;
        const long long tn = T - tp * a.ntn;
        const int8_t* xa = a.xs + tp * a.KB * static_cast<long long>(G::A);
        const int8_t* xb = a.bs + tn * a.KB * static_cast<long long>(G::B);
        for (int kb = 0; kb < a.KB; ++kb, ++it) {
          const int s = static_cast<int>(it % OZ_STAGES);
          const uint32_t ph = static_cast<uint32_t>((it / OZ_STAGES) & 1);
          mb_wait(&empty[s], ph ^ 1);
          unsigned char* st = sm + s * G::STAGE;
          mb_expect_tx(&full[s], G::STAGE);
          bulk_g2s(st, xa + static_cast<long long>(kb) * G::A, G::A, &full[s]);
          bulk_g2s(st + G::A, xb + static_cast<long long>(kb) * G::B, G::B, &full[s]);
        }
      }
    }
  } else if (warp == 1) {  // MMA warp (converged; one elected lane issues)
    long long it = 0, lt = 0;
    for (long long T = blockIdx.x; T < tiles; T += gridDim.x, ++lt) {
      mb_wait(tempty, static_cast<uint32_t>((lt & 1) ^ 1));
      tc_fence_after();
      for (int kb = 0; kb < a.KB; ++kb, ++it) {
        const int s = static_cast<int>(it % OZ_STAGES);
        const uint32_t ph = static_cast<uint32_t>((it / OZ_STAGES) & 1);
        mb_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t sa = su32(sm + s * G::STAGE);
        const uint32_t la = oz_desc_lo(sa), lb = oz_desc_lo(sa + G::A);
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < S; ++i)
#pragma unroll
            for (int j = 0; j < S - i; ++j)  // slice pair (i, j) -> group i + j
              umma_i8(tmem + (i + j) * OZ_BN, oz_desc_of(la + ((i * G::A_SLICE) >> 4)),
                      oz_desc_of(lb + ((j * G::B_SLICE) >> 4)), (kb | i) != 0);
          umma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(tfull);
      __syncwarp();
    }
  } else {  // epilogue warps 2..9: TMEM lane quadrant warp % 4, column half (warp - 2) / 4
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    long long lt = 0;
    for (long long T = blockIdx.x; T < tiles; T += gridDim.x, ++lt) {
      const long long tp = T / a.ntn;
      const int tn = static_cast<int>(T - tp * a.ntn);
      const long long r = tp * OZ_BM + 32 * q + lane;
      const int c0 = tn * OZ_BN + hc * 32;
      mb_wait(tfull, static_cast<uint32_t>(lt & 1));
      tc_fence_after();
      double acc[32];
      oz_drain<S>(tmem, q, hc, acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(tempty);  // accumulators free: next tile's MMAs overlap the stores
      oz_store(a, r, c0, lane, acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(OZ_TMEM_COLS));
  }
}

// ------------------------------------------------------------------ 2-SM (cta_group::2) --
// A CTA pair computes a 256-row x 64-output tile with tcgen05.mma.cta_group::2 (M = 256, N = 64,
// K = 32) issued by the leader: each CTA stages its own 128 rows of field slices (S x 4 KB) and
// its 32-output half of the matrix slices (S x 1 KB) per stage, so per SM the tensor core reads
// 5 KB of shared memory per 128 x 64 x 32 block instead of 6 KB, and the matrix crosses L2 -> SM
// once per pair. Protocol as tc2_pass_kernel (tc_lowp.cu): both CTAs' TMA loads (a 2-D byte view
// of the tiled buffers, 128-byte rows, no swizzle) complete on the leader's full barrier, the
// leader's commits multicast to both CTAs' empty / accumulator-full barriers, and both CTAs'
// epilogue warps release the leader's accumulator-empty barrier.
template <int S>
struct Oz2Geom {
  static constexpr int A_SLICE = OZ_BM * OZ_BK;        // 4 KB
  static constexpr int B_SLICE = (OZ_BN / 2) * OZ_BK;  // 1 KB
  static constexpr int A = S * A_SLICE;
  static constexpr int B = S * B_SLICE;
  static constexpr int STAGE = A + B;
  static constexpr int STAGES = (200 * 1024) / STAGE < 8 ? (200 * 1024) / STAGE : 8;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};
constexpr uint32_t kOzPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's barrier

__host__ __device__ constexpr uint32_t oz2_idesc() {  // S8 x S8 -> S32, M = 256 (pair), N = 64
  return (2u << 4) | (1u << 7) | (1u << 10) | ((OZ_BN >> 3) << 17) | ((OZ_PAIR >> 4) << 24);
}
__device__ __forceinline__ void umma2_i8(uint32_t d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n}\n" ::"r"(d),
      "l"(da), "l"(db), "r"(oz2_idesc()), "r"(acc), "r"(0u));
}
__device__ __forceinline__ void umma2_commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n" ::"r"(su32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}
__device__ __forceinline__ void tma_rows_2sm(void* dst, const CUtensorMap* map, int row,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(dst)),
      "l"(map), "r"(0), "r"(row), "r"(su32(bar) & kOzPeerMask)
      : "memory");
}
__device__ __forceinline__ void mb_arrive_rank(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(su32(bar)),
      "r"(rank)
      : "memory");
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz2_pass_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tb,
                    const OzArgs a) {
  using G = Oz2Geom<S>;
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + G::STAGES * G::STAGE);
  uint64_t* empty = full + G::STAGES;
  uint64_t* tfull = empty + G::STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = cl_rank();
  const bool leader = crank == 0;
  if (tid == 0) {
    for (int s = 0; s < G::STAGES; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(tfull, 1);
    mb_init(tempty, 2 * OZ_EPI_WARPS);  // the epilogue warps of both CTAs
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(OZ_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cl_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const long long pair_tm = a.ntm / 2;  // 256-row panels (field slices padded to them)
  const long long tiles = pair_tm * a.ntn;
  const long long t0 = blockIdx.x / 2, tstep = gridDim.x / 2;
  if (warp == 0) {
    if (lane == 0) {  // producer (both CTAs): byte-view rows of 128 B
      long long it = 0;
      for (long long T = t0; T < tiles; T += tstep) {
        const long long tp = T / a.ntn;
        const long long tn = T - tp * a.ntn;
        const long long arow0 = (tp * 2 + crank) * a.KB * (G::A / 128);
        const long long brow0 = (tn * 2 + crank) * a.KB * (G::B / 128);
        for (int kb = 0; kb < a.KB; ++kb, ++it) {
          const int s = static_cast<int>(it % G::STAGES);
          mb_wait(&empty[s], static_cast<uint32_t>((it / G::STAGES) & 1) ^ 1);
          unsigned char* st = sm + s * G::STAGE;
          if (leader) mb_expect_tx(&full[s], 2 * G::STAGE);  // both CTAs' bytes land on it
          tma_rows_2sm(st, &tx, static_cast<int>(arow0 + kb * (G::A / 128)), &full[s]);
          tma_rows_2sm(st + G::A, &tb, static_cast<int>(brow0 + kb * (G::B / 128)), &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // MMA warp of the leader (converged; one elected lane issues)
      long long it = 0, lt = 0;
      for (long long T = t0; T < tiles; T += tstep, ++lt) {
        mb_wait(tempty, static_cast<uint32_t>((lt & 1) ^ 1));
        tc_fence_after();
        for (int kb = 0; kb < a.KB; ++kb, ++it) {
          const int s = static_cast<int>(it % G::STAGES);
          mb_wait(&full[s], static_cast<uint32_t>((it / G::STAGES) & 1));
          tc_fence_after();
          const uint32_t sa = su32(sm + s * G::STAGE);
          const uint32_t la = oz_desc_lo(sa), lb = oz_desc_lo(sa + G::A);
          if (elect_one()) {
#pragma unroll
            for (int i = 0; i < S; ++i)
#pragma unroll
              for (int j = 0; j < S - i; ++j)
                umma2_i8(tmem + (i + j) * OZ_BN, oz_desc_of(la + ((i * G::A_SLICE) >> 4)),
                         oz_desc_of(lb + ((j * G::B_SLICE) >> 4)), (kb | i) != 0);
            umma2_commit_mc(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) umma2_commit_mc(tfull);
        __syncwarp();
      }
    }
  } else {  // epilogue warps, both CTAs: this CTA's 128 rows x 64 outputs
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    long long lt = 0;
    for (long long T = t0; T < tiles; T += tstep, ++lt) {
      const long long tp = T / a.ntn;
      const int tn = static_cast<int>(T - tp * a.ntn);
      const long long r = (tp * 2 + crank) * OZ_BM + 32 * q + lane;
      const int c0 = tn * OZ_BN + hc * 32;
      mb_wait(tfull, static_cast<uint32_t>(lt & 1));
      tc_fence_after();
      double acc[32];
      oz_drain<S>(tmem, q, hc, acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive_rank(tempty, 0);  // the leader's barrier
      oz_store(a, r, c0, lane, acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  cl_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(OZ_TMEM_COLS));
  }
}

// One 16-byte chunk of a row: t holds 127 x 2^-e; S slices a_s = rint(t), t = 254 (t - a_s).
// rint by the 1.5 * 2^52 shifter: y = t + M rounds t to the nearest integer (ties to even, as
// rint) into the low mantissa bits, so the INT8 value is the low word of y (|t| <= 127) and
// y - M is rint(t) as a double: three FP64 adds / one multiply per slice, no conversions.
template <int S>
__device__ __forceinline__ void split16(double (&t)[16], uint32_t (&w)[S][4]) {
  constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
#pragma unroll
  for (int s = 0; s < S; ++s) {
#pragma unroll
    for (int q = 0; q < 4; ++q) w[s][q] = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double y = __dadd_rn(t[u], kShift);
      const double f = __dsub_rn(y, kShift);
      t[u] = __dmul_rn(__dsub_rn(t[u], f), 254.0);
      w[s][u >> 2] |= (static_cast<uint32_t>(__double2loint(y)) & 0xFFu) << (8 * (u & 3));
    }
  }
}

// Tiled byte offset of (row rr of its P-row panel, 16-byte chunk c of K) within slice 0 of the
// panel's K-block c / 2; slice s adds s * P * 32.
template <int P>
__device__ __forceinline__ long long tile_off(long long p, int KB, int S, int rr, int c) {
  return ((p * KB + (c >> 1)) * S) * static_cast<long long>(P * OZ_BK) + (rr >> 3) * 256 +
         (c & 1) * 128 + (rr & 7) * 16;
}

// Field rows (contiguous K-runs): a block stages 8 rows (one 8-row core-matrix group) in shared
// memory with one coalesced read, takes the row maxima, and writes the slices so that 8 lanes
// fill one 128-byte core matrix. Chunks are staged 17 doubles apart and rows ld = 4 (mod 16)
// doubles apart, so the 32 lanes (8 rows x 4 chunks) of a chunk read hit 16 distinct bank pairs:
// the 2-wavefront minimum. HBM-bound: 8 B read and
// S B written per element.
template <int S>
__global__ void __launch_bounds__(256) k_oz_split_rows(const double* __restrict__ x, long long R,
                                                       int K, int KB, long long Rp, int gather,
                                                       long long ldr, long long off,
                                                       int8_t* __restrict__ out,
                                                       int* __restrict__ ex) {
  extern __shared__ double srow[];
  __shared__ int sexp[8];
  const int Kp = KB * OZ_BK;
  const int nch = KB * 2;
  const int ld = nch * 17 + ((4 - nch) & 15);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (long long r0 = blockIdx.x * 8LL; r0 < Rp; r0 += gridDim.x * 8LL) {
    // stage: warp w loads row r0 + w
    {
      const long long r = r0 + warp;
      // gather (interleaved complex field, component c fastest in memory): row r = (q, c) with
      // c = r / (R / 2) the slow part of the row index, element k at x[(q K + k) 2 + c]
      const long long Rh = R >> 1;
      const long long rq = gather ? (r < R ? r % Rh : 0) : r;
      const long long rc = gather ? (r < R ? r / Rh : 0) : 0;
      double amax = 0.0;
      bool nonfinite = false;
      for (int k0 = 0; k0 < Kp; k0 += 256) {  // 8 independent loads in flight per lane
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = k0 + u * 32 + lane;
          v[u] = (r < R && k < K)
                     ? __ldcs(gather ? x + (rq * ldr + off + k) * 2 + rc : x + r * ldr + off + k)
                     : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = k0 + u * 32 + lane;
          if (k < Kp) {
            const bool fin = isfinite(v[u]);
            nonfinite = nonfinite || !fin;
            srow[warp * ld + (k >> 4) * 17 + (k & 15)] = fin ? v[u] : 0.0;
            amax = fmax(amax, fin ? fabs(v[u]) : 0.0);
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      nonfinite = __any_sync(0xffffffffu, nonfinite);
      int e = 0;
      if (amax > 0.0) frexp(amax, &e);  // amax < 2^e
      if (lane == 0) {
        sexp[warp] = e;
        if (r < Rp) ex[r] = nonfinite ? OZ_NONFINITE : e;
      }
    }
    __syncthreads();
    const long long p = r0 / OZ_BM;
    const int rr0 = static_cast<int>(r0 - p * OZ_BM);
    for (int item = tid; item < 8 * nch; item += 256) {
      const int rw = item & 7, c = item >> 3;
      const int e = sexp[rw];
      const double sc = ldexp(127.0, -e);
      double t[16];
      if (e > -900) {  // 127 x 2^-e is finite: one exact-scale multiply
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = srow[rw * ld + c * 17 + u] * sc;
      } else {  // rows of (near-)subnormals
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = ldexp(srow[rw * ld + c * 17 + u], -e) * 127.0;
      }
      uint32_t w[S][4];
      split16<S>(t, w);
      int8_t* base = out + tile_off<OZ_BM>(p, KB, S, rr0 + rw, c);
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2)
        *reinterpret_cast<uint4*>(base + s2 * static_cast<long long>(OZ_BM * OZ_BK)) =
            make_uint4(w[s2][0], w[s2][1], w[s2][2], w[s2][3]);
    }
    __syncthreads();
  }
}

// Axis matrices (element (i, k) at M[i + lda k], rows i = outputs), split once per operator:
// one warp per row, strided reads (small, cached).
template <int S, int P>
__global__ void __launch_bounds__(256) k_oz_split_mat(const double* __restrict__ M, int lda,
                                                      int m, int K, int KB, int mp,
                                                      int8_t* __restrict__ out,
                                                      int* __restrict__ ex) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int nch = KB * 2;
  for (int r = w0; r < mp; r += nw) {
    double amax = 0.0;
    bool nonfinite = false;
    if (r < m)
      for (int k = lane; k < K; k += 32) {
        const double v = M[r + static_cast<long long>(lda) * k];
        nonfinite = nonfinite || !isfinite(v);
        amax = fmax(amax, isfinite(v) ? fabs(v) : 0.0);
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    nonfinite = __any_sync(0xffffffffu, nonfinite);
    int e = 0;
    if (amax > 0.0) frexp(amax, &e);
    if (lane == 0) ex[r] = nonfinite ? OZ_NONFINITE : e;
    const int p = r / P, rr = r - p * P;
    const double sc = ldexp(127.0, -e);
    for (int c = lane; c < nch; c += 32) {
      double t[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = c * 16 + u;
        double v = (r < m && k < K) ? M[r + static_cast<long long>(lda) * k] : 0.0;
        if (!isfinite(v)) v = 0.0;  // the row is marked OZ_NONFINITE
        t[u] = e > -900 ? v * sc : ldexp(v, -e) * 127.0;
      }
      uint32_t w[S][4];
      split16<S>(t, w);
      int8_t* base = out + tile_off<P>(p, KB, S, rr, c);
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2)
        *reinterpret_cast<uint4*>(base + s2 * static_cast<long long>(P * OZ_BK)) =
            make_uint4(w[s2][0], w[s2][1], w[s2][2], w[s2][3]);
    }
  }
}

template <int S>
void oz_split_rows(cudaStream_t st, const double* x, long long R, int K, int gather, int8_t* out,
                   int* ex, long long ldr = -1, long long off = 0) {
  // row r of K values starts at x + r * ldr + off (ldr = K: contiguous runs); the even / odd
  // halves of a folded axis are the sub-runs [0, ne) and [ne, n) of rows of length n
  const int KB = (K + OZ_BK - 1) / OZ_BK;
  const long long Rp = (R + OZ_PAIR - 1) / OZ_PAIR * OZ_PAIR;  // whole 256-row pair panels
  const int nch = KB * 2;
  const size_t smem = static_cast<size_t>(8) * (nch * 17 + ((4 - nch) & 15)) * sizeof(double);
  if (smem > 48 * 1024) ensure_smem_attr(reinterpret_cast<const void*>(k_oz_split_rows<S>), smem);
  const long long groups = Rp / 8;
  const int per_sm = smem <= 72 * 1024 ? 3 : 1;
  const int blocks = static_cast<int>(groups < 148LL * per_sm * 4 ? groups : 148LL * per_sm * 4);
  k_oz_split_rows<S><<<blocks, 256, smem, st>>>(x, R, K, KB, Rp, gather, ldr < 0 ? K : ldr, off,
                                                 out, ex);
  KCUDA(cudaGetLastError());
}

// P = 64 (1-SM kernel: one 64-output tile per block) or 32 (2-SM kernel: each CTA of the pair
// stages its 32-output half of the tile)
template <int S>
void oz_split_mat(cudaStream_t st, const double* M, int lda, int m, int K, int P, int8_t* out,
                  int* ex) {
  const int KB = (K + OZ_BK - 1) / OZ_BK;
  const int mp = (m + OZ_BN - 1) / OZ_BN * OZ_BN;
  const int blocks = (mp + 7) / 8;
  if (P == 32)
    k_oz_split_mat<S, 32><<<blocks, 256, 0, st>>>(M, lda, m, K, KB, mp, out, ex);
  else
    k_oz_split_mat<S, OZ_BN><<<blocks, 256, 0, st>>>(M, lda, m, K, KB, mp, out, ex);
  KCUDA(cudaGetLastError());
}

template <int S>
void oz_pass(cudaStream_t st, OzArgs a) {
  using G = OzGeom<S>;
  ensure_smem_attr(reinterpret_cast<const void*>(oz_pass_kernel<S>), G::SMEM);
  const int sms = device_sm_count();
  const long long tiles = a.ntm * a.ntn;
  const unsigned grid = static_cast<unsigned>(tiles < sms ? tiles : sms);
  oz_pass_kernel<S><<<grid, OZ_THREADS, G::SMEM, st>>>(a);
  KCUDA(cudaGetLastError());
}

PFN_cuTensorMapEncodeTiled_v12000 oz_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    KCUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr));
    if (qr != cudaDriverEntryPointSuccess || !p)
      fail(KRONOP_ERUNTIME, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D byte view of a tiled slice buffer: rows of 128 bytes, box = one CTA's stage part
void oz_encode_rows(CUtensorMap* map, const void* base, size_t bytes, int box_rows) {
  const cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(bytes / 128)};
  const cuuint64_t str[1] = {128};
  const cuuint32_t box[2] = {128, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = oz_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base),
                                    dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(KRONOP_ERUNTIME, "cuTensorMapEncodeTiled (Ozaki slices) failed");
}

template <int S>
void oz2_pass(cudaStream_t st, OzArgs a, size_t xbytes, size_t bbytes) {
  using G = Oz2Geom<S>;
  ensure_smem_attr(reinterpret_cast<const void*>(oz2_pass_kernel<S>), G::SMEM);
  const int sms = device_sm_count();
  CUtensorMap tx, tb;
  oz_encode_rows(&tx, a.xs, xbytes, G::A / 128);
  oz_encode_rows(&tb, a.bs, bbytes, G::B / 128);
  const long long pairs = (a.ntm / 2) * a.ntn;
  const long long g = 2 * (pairs < sms / 2 ? pairs : sms / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(g));
  cfg.blockDim = dim3(OZ_THREADS);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KCUDA(cudaLaunchKernelEx(&cfg, oz2_pass_kernel<S>, tx, tb, a));
}

// bytes of a tiled slice buffer: rows padded to `pad`, K to whole 32-byte blocks
inline size_t oz_slice_bytes(long long rows, int K, int pad, int S) {
  const long long Rp = (rows + pad - 1) / pad * pad;
  const long long KB = (K + OZ_BK - 1) / OZ_BK;
  return static_cast<size_t>(Rp * KB * OZ_BK * S);
}

// KRONOP_OZ_2SM=0 selects the 1-SM kernel (M = 128); default: CTA pairs (M = 256)
bool oz_two_sm() {
  static const bool v = [] {
    const char* e = getenv("KRONOP_OZ_2SM");
    return !(e && e[0] == '0');
  }();
  return v;
}

template <int S>
void sep_ozaki_impl(kronop_ctx& ctx, kronop_op& op, const double* b, double* x, int cplx, int epi,
                    double shift, double dt, const double* diag, double sigma) {
  param_check(!op.folded, "solve_lowp: dense operators only");
  const long long N = op.N;
  const bool propagate = cplx != 0;  // complex field (the gather / pairing below)
  const int cf = propagate ? 2 : 1;  // complex: 2 real rows per fibre
  cudaStream_t st = ctx.stream;
  const bool two = oz_two_sm();
  const int bpan = two ? OZ_BN / 2 : OZ_BN;  // matrix panel rows per CTA
  const int key = S * 2 + (two ? 1 : 0);
  void** of = op.oz_fwd;
  void** ob = op.oz_bwd;
  if (!of[0] || op.oz_slices != key) {  // split copies of the transforms, made once per mode
    for (int a = 0; a < KRONOP_MAX_DIM; ++a)
      for (void** p : {&of[a], &ob[a]})
        if (*p) {
          KCUDA(cudaFree(*p));
          *p = nullptr;
        }
    for (int a = 0; a < op.d; ++a) {
      const int n = op.n[a];
      const size_t sb = oz_slice_bytes(n, n, OZ_BN, S);
      const long long mp = (n + OZ_BN - 1) / OZ_BN * OZ_BN;
      for (int dir = 0; dir < 2; ++dir) {
        void* p = nullptr;
        KCUDA(cudaMalloc(&p, sb + mp * sizeof(int)));
        // matrix element (i, k) at M[i + lda * k]: rows i (outputs), contraction k
        oz_split_mat<S>(st, dir == 0 ? op.fwd[a] : op.bwd[a], op.lda[a], n, n, bpan,
                        static_cast<int8_t*>(p), reinterpret_cast<int*>(static_cast<char*>(p) + sb));
        (dir == 0 ? of : ob)[a] = p;
      }
    }
    op.oz_slices = key;
  }
  // workspace: one FP64 field (scratch[0]) + the current pass's slices and row exponents
  size_t need = 0;
  for (int a = 0; a < op.d; ++a) {
    const long long R = cf * (N / op.n[a]);
    const size_t v = oz_slice_bytes(R, op.n[a], OZ_PAIR, S) +
                     ((R + OZ_PAIR - 1) / OZ_PAIR * OZ_PAIR) * sizeof(int);
    need = v > need ? v : need;
  }
  const size_t need_d = (need + 7) / 8 + 16;
  ensure_scratch(ctx, need_d > static_cast<size_t>(cf * N) ? need_d : static_cast<size_t>(cf * N));
  double* f = ctx.scratch[0];
  int8_t* xs = reinterpret_cast<int8_t*>(ctx.scratch[1]);
  const double* cur = b;
  int k = 0;
  for (int dir = 0; dir < 2; ++dir)
    for (int a = 0; a < op.d; ++a, ++k) {
      const bool last = dir == 1 && a == op.d - 1;
      const int n = op.n[a];
      const long long R = cf * (N / n);
      const size_t xb = oz_slice_bytes(R, n, OZ_PAIR, S);
      int* xe = reinterpret_cast<int*>(xs + xb);
      // complex: the first pass of each direction reads the interleaved layout (re/im fastest)
      oz_split_rows<S>(st, cur, R, n, propagate && a == 0 ? 1 : 0, xs, xe);
      OzArgs oa{};
      oa.cplx = cplx;
      if (last && (diag != nullptr || sigma != 0.0)) {
        oa.axpy = 1;
        oa.diag = diag;
        oa.u = b;
        oa.sigma = sigma;
      }
      if (dir == 0 && a == op.d - 1) {
        oa.epi = epi;
        oa.dt = dt;
        oa.shift = shift;
        oa.nlow = op.d - 1;
        for (int j = 0; j < op.d - 1; ++j) {
          oa.lowext[j] = op.n[j];
          oa.lowlam[j] = op.lam[j];
        }
        oa.lamlast = op.lam[a];
      }
      const void* mat = dir == 0 ? of[a] : ob[a];
      const size_t mb = oz_slice_bytes(n, n, OZ_BN, S);
      oa.xs = xs;
      oa.xe = xe;
      oa.bs = static_cast<const int8_t*>(mat);
      oa.be = reinterpret_cast<const int*>(static_cast<const char*>(mat) + mb);
      oa.y = last ? x : f;
      oa.R = R;
      oa.K = n;
      oa.KB = (n + OZ_BK - 1) / OZ_BK;
      oa.m = n;
      oa.ntn = (n + OZ_BN - 1) / OZ_BN;
      oa.ntm = (R + OZ_PAIR - 1) / OZ_PAIR * 2;  // 128-row panels, even count
      if (two)
        oz2_pass<S>(st, oa, xb, mb);
      else
        oz_pass<S>(st, oa);
      ctx.ws.launches += 2;
      cur = f;
    }
}

// The even/odd folded operator (kronop_op_create_folded) on the INT8 path: per axis the fold
// kernel (vector_ops.cu) puts the axis in [even half | odd half] order, the split kernel reads
// the two sub-runs as separate rows with their own exponents, and two INT8 passes with the
// half-size matrices write the two mode blocks of the rotated output (the folded mode order the
// lambda arrays use). Backward passes write the two physical halves and the unfold kernel
// (with the FullOperator AXPY on the last axis) restores the axis. Half the INT8 products of the
// dense operator, plus one fold / unfold HBM pass per axis.
template <int S>
void sep_ozaki_folded_impl(kronop_ctx& ctx, kronop_op& op, const double* in, double* out,
                           int cplx, int epi, double shift, double dt, const double* diag,
                           double sigma) {
  const long long N = op.N;
  const int cf = cplx ? 2 : 1;
  cudaStream_t st = ctx.stream;
  const bool two = oz_two_sm();
  const int bpan = two ? OZ_BN / 2 : OZ_BN;
  const int key = 1000 + S * 2 + (two ? 1 : 0);
  void** se[2] = {op.oz_fwd, op.oz_bwd};  // even blocks
  void** so[2] = {op.oz_fo, op.oz_bo};    // odd blocks
  if (!op.oz_fwd[0] || op.oz_slices != key) {
    for (int a = 0; a < KRONOP_MAX_DIM; ++a)
      for (void** p : {&op.oz_fwd[a], &op.oz_bwd[a], &op.oz_fo[a], &op.oz_bo[a]})
        if (*p) {
          KCUDA(cudaFree(*p));
          *p = nullptr;
        }
    for (int a = 0; a < op.d; ++a)
      for (int dir = 0; dir < 2; ++dir)
        for (int h = 0; h < 2; ++h) {
          const int m = h == 0 ? op.ne[a] : op.no[a];
          if (m == 0) continue;
          const double* M = dir == 0 ? (h == 0 ? op.fe[a] : op.fo[a]) : (h == 0 ? op.be[a] : op.bo[a]);
          const int lda = h == 0 ? op.lda_e[a] : op.lda_o[a];
          const size_t sb = oz_slice_bytes(m, m, OZ_BN, S);
          const long long mp = (m + OZ_BN - 1) / OZ_BN * OZ_BN;
          void* p = nullptr;
          KCUDA(cudaMalloc(&p, sb + mp * sizeof(int)));
          oz_split_mat<S>(st, M, lda, m, m, bpan, static_cast<int8_t*>(p),
                          reinterpret_cast<int*>(static_cast<char*>(p) + sb));
          (h == 0 ? se : so)[dir][a] = p;
        }
    op.oz_slices = key;
  }
  size_t need = 0;
  for (int a = 0; a < op.d; ++a) {
    const long long R = cf * (N / op.n[a]);
    const size_t v = oz_slice_bytes(R, op.ne[a], OZ_PAIR, S) +
                     ((R + OZ_PAIR - 1) / OZ_PAIR * OZ_PAIR) * sizeof(int);
    need = v > need ? v : need;
  }
  const size_t need_d = (need + 7) / 8 + 16;
  ensure_scratch(ctx, need_d > static_cast<size_t>(cf * N) ? need_d : static_cast<size_t>(cf * N));
  double* fa = ctx.scratch[0];                                  // folded input of a pass
  int8_t* xs = reinterpret_cast<int8_t*>(ctx.scratch[1]);      // slices + row exponents
  double* fb = ensure_tmp(ctx, static_cast<size_t>(cf * N));   // pass output
  auto half_pass = [&](const double* src, double* dst, int a, int dir, int h, bool spectral) {
    const int n = op.n[a];
    const int m = h == 0 ? op.ne[a] : op.no[a];
    if (m == 0) return;
    const long long off = h == 0 ? 0 : op.ne[a];
    const long long R = cf * (N / n);
    const size_t xb = oz_slice_bytes(R, m, OZ_PAIR, S);
    int* xe = reinterpret_cast<int*>(xs + xb);
    oz_split_rows<S>(st, src, R, m, cplx && a == 0 ? 1 : 0, xs, xe, n, off);
    OzArgs oa{};
    oa.cplx = cplx;
    if (spectral) {
      oa.epi = epi;
      oa.dt = dt;
      oa.shift = shift;
      oa.nlow = op.d - 1;
      for (int j = 0; j < op.d - 1; ++j) {
        oa.lowext[j] = op.n[j];
        oa.lowlam[j] = op.lam[j];
      }
      oa.lamlast = op.lam[a] + off;
    }
    const void* mat = (h == 0 ? se : so)[dir][a];
    const size_t mb = oz_slice_bytes(m, m, OZ_BN, S);
    oa.xs = xs;
    oa.xe = xe;
    oa.bs = static_cast<const int8_t*>(mat);
    oa.be = reinterpret_cast<const int*>(static_cast<const char*>(mat) + mb);
    oa.y = dst + off * R;
    oa.R = R;
    oa.K = m;
    oa.KB = (m + OZ_BK - 1) / OZ_BK;
    oa.m = m;
    oa.ntn = (m + OZ_BN - 1) / OZ_BN;
    oa.ntm = (R + OZ_PAIR - 1) / OZ_PAIR * 2;
    if (two)
      oz2_pass<S>(st, oa, xb, mb);
    else
      oz_pass<S>(st, oa);
    ctx.ws.launches += 2;
  };
  const double* cur = in;
  for (int a = 0; a < op.d; ++a) {  // forward: fold the (fastest) axis, two half passes
    const int n = op.n[a];
    const long long pre = cplx && a == 0 ? 2 : 1;
    launch_fold(st, ctx.ws, cur, fa, pre, n, cf * N / (n * pre));
    for (int h = 0; h < 2; ++h) half_pass(fa, fb, a, 0, h, a == op.d - 1);
    cur = fb;
  }
  for (int a = 0; a < op.d; ++a) {  // backward: two half passes, unfold the (slowest) axis
    const int n = op.n[a];
    for (int h = 0; h < 2; ++h) half_pass(fb, fa, a, 1, h, false);
    const bool last = a == op.d - 1;
    launch_unfold(st, ctx.ws, fa, last ? out : fb, cf * N / n, n, 1, last ? diag : nullptr,
                  last ? in : nullptr, last ? sigma : 0.0, cplx);
  }
}

}  // namespace

// Any separable transform on the INT8 path: cplx (interleaved complex field), epi 1 divide /
// 2 multiply by (lambda - shift) / 3 phase, optional last-pass AXPY (+ diag u - sigma u).
void sep_ozaki(kronop_ctx& ctx, kronop_op& op, const double* in, double* out, int cplx, int epi,
               double shift, double dt, const double* diag, double sigma, int slices) {
  for (int a = 0; a < op.d; ++a)
    param_check(op.n[a] <= OZ_KMAX, "Ozaki mode needs extents <= 3200");
  if (op.folded) {
    if (slices == 5)
      sep_ozaki_folded_impl<5>(ctx, op, in, out, cplx, epi, shift, dt, diag, sigma);
    else if (slices == 6)
      sep_ozaki_folded_impl<6>(ctx, op, in, out, cplx, epi, shift, dt, diag, sigma);
    else
      sep_ozaki_folded_impl<7>(ctx, op, in, out, cplx, epi, shift, dt, diag, sigma);
    return;
  }
  if (slices == 5)
    sep_ozaki_impl<5>(ctx, op, in, out, cplx, epi, shift, dt, diag, sigma);
  else if (slices == 6)
    sep_ozaki_impl<6>(ctx, op, in, out, cplx, epi, shift, dt, diag, sigma);
  else
    sep_ozaki_impl<7>(ctx, op, in, out, cplx, epi, shift, dt, diag, sigma);
}

// kronop_op_set_precision: everything a later (possibly graph-captured) call would allocate or
// initialise - the split matrices, the workspace for complex fields, the kernels' attributes -
// is done here, by one throw-away transform of a zero field.
void ozaki_prepare(kronop_ctx& ctx, kronop_op& op, int slices) {
  // one throw-away REAL transform splits the matrices and sizes the workspace for the real
  // drivers (PCG, inverse iteration, GPE capture graphs and must not allocate); a complex field
  // grows it later, outside any capture. In + out = 2 N doubles (a complex warm-up took 6 N).
  const size_t n = static_cast<size_t>(op.N);
  double* z = nullptr;
  KCUDA(cudaMallocAsync(&z, 2 * n * sizeof(double), ctx.stream));
  KCUDA(cudaMemsetAsync(z, 0, n * sizeof(double), ctx.stream));
  sep_ozaki(ctx, op, z, z + n, 0, 2, op.shift, 0.0, nullptr, 0.0, slices);
  KCUDA(cudaFreeAsync(z, ctx.stream));
  KCUDA(cudaStreamSynchronize(ctx.stream));
}

// (-Delta + V1 - shift)^{-1} b with FP64 accuracy from INT8 tensor-core products (Ozaki scheme,
// `slices` 8-bit slices per operand: 5, 6 or 7). Real fields, FP64 device in and out.
void sep_solve_ozaki(kronop_ctx& ctx, kronop_op& op, const double* b, double* x, int slices) {
  for (int a = 0; a < op.d; ++a)
    param_check(op.n[a] <= OZ_KMAX, "solve_lowp: Ozaki mode needs extents <= 3200");
  sep_ozaki(ctx, op, b, x, 0, 1, op.shift, 0.0, nullptr, 0.0, slices);
}

// exp(-i dt (-Delta + V1 - shift)) psi (operators.cpp:63-75) on the same INT8 path: complex
// interleaved FP64 in and out; re and im travel as separate real rows through the transforms
// (the matrices are real) and meet again in the phase epilogue of the last forward pass.
void sep_propagate_ozaki(kronop_ctx& ctx, kronop_op& op, const double* psi, double dt, double* out,
                         int slices) {
  for (int a = 0; a < op.d; ++a)
    param_check(op.n[a] <= OZ_KMAX, "propagate_lowp: Ozaki mode needs extents <= 3200");
  sep_ozaki(ctx, op, psi, out, 1, 3, op.shift, dt, nullptr, 0.0, slices);
}

}  // namespace kronop_dev
