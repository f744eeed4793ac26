// Reduced-precision transforms on the 5th-generation tensor cores (tcgen05 + TMEM): the BF16
// variant of the separable solve (the paper's FP32 / TF32 / BF16 rows), as a
// separately reported alternative path. FP64 has no tcgen05 kind, so the
// north-star path stays on DMMA (mode_product_tma.cu); this file is the Blackwell tensor-core
// path for the precisions that have one.
//
// One pass contracts the FASTEST axis of a BF16 field viewed as X[R rows][K] (K contiguous) with
// the axis matrix B[m][K] (K contiguous): D[r][i] = sum_k X[r][k] B[i][k], FP32 accumulation in
// TMEM, and writes Y[i * R + r] (the contracted axis moves to the slow end: after d passes the
// layout is the original again, as in fused_rot.cu). Both operands are K-major, the canonical
// UMMA layout, loaded by TMA with 128-byte swizzle.
//
// Per CTA (persistent, one per SM, 6 warps): warp 0 lane 0 = TMA producer (4-stage ring of
// 48 KB: A 128 x 64, B 256 x 64 bf16); warp 1 = TMEM allocator + single-thread tcgen05.mma
// issuer (M = 128, N = 256, K = 16 per instruction, 4 per stage) with tcgen05.commit releasing
// smem stages and publishing finished accumulators; warps 2-5 = epilogue (tcgen05.ld 32x32b, the
// fused spectral divide / multiply, BF16 or FP64 stores of the rotated output). Two TMEM
// accumulator buffers (2 x 256 columns) let the epilogue of tile i overlap the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "context.cuh"
#include "kronop_internal.cuh"

namespace kronop_dev {

namespace {

constexpr int TC_BM = 128, TC_BN = 256, TC_STAGES = 4;
// a stage holds 128-byte rows of K: 64 BF16 or 32 TF32 (FP32 storage) values
constexpr int TC_ROW = 128;
constexpr int TC_A_BYTES = TC_BM * TC_ROW;  // 16 KB
constexpr int TC_B_BYTES = TC_BN * TC_ROW;  // 32 KB
constexpr int TC_STAGE = TC_A_BYTES + TC_B_BYTES;

enum { PREC_BF16 = 1, PREC_TF32 = 2 };
template <int PREC>
struct TcTraits;
template <>
struct TcTraits<PREC_BF16> {
  using T = __nv_bfloat16;
  static constexpr int BK = 64;      // elements per 128-byte row
  static constexpr int UK = 16;      // K per tcgen05.mma (32 bytes)
  static constexpr uint32_t FMT = 1; // BF16 in the instruction descriptor
};
template <>
struct TcTraits<PREC_TF32> {
  using T = float;
  static constexpr int BK = 32;
  static constexpr int UK = 8;
  static constexpr uint32_t FMT = 2; // TF32
};
constexpr int TC_THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (2 per TMEM quadrant)
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_SMEM = TC_STAGES * TC_STAGE + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TC_TMEM_COLS = 512;  // two 128 x 256 FP32 accumulators

struct TcArgs {
  void* y;
  long long R;  // rows (product of the other axes)
  int K;        // contracted extent
  int m;        // output extent
  int ntn;      // N tiles
  long long ntm;
  int epi;      // 0 store, 1 divide by (lambda - shift), 2 multiply
  double shift;
  int nlow;                              // axes below (row decomposition) for lambda
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
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma2d_mc(void* dst, const CUtensorMap* map, int c0, int c1,
                                         uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
      "cluster [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(su32(bar)), "h"(mask)
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
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// one lane of a converged warp: the MMA warps run their loops converged and only the issue is
// single-threaded, so descriptors stay in uniform registers (a lane-0 branch made the compiler
// wrap every tcgen05.mma in an ELECT / BRA.U.ANY loop; see ozaki.cu)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, %1;\n@px mov.s32 %0, 1;\n}\n"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}
// K-major, 128-byte-swizzled UMMA shared-memory descriptor (cute/arch/mma_sm100_desc.hpp layout):
// start >> 4 | LBO 1 | SBO 1024 B (8-row groups) | version 1 (Blackwell) | SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) |
         (1ull << 46) | (2ull << 61);
}
// instruction descriptor: FMT x FMT -> FP32, K-major A and B, M = 128, N = 256
template <int PREC>
__host__ __device__ constexpr uint32_t idesc() {
  return (1u << 4) | (TcTraits<PREC>::FMT << 7) | (TcTraits<PREC>::FMT << 10) |
         ((TC_BN >> 3) << 17) | ((TC_BM >> 4) << 24);
}
template <int PREC>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  if constexpr (PREC == PREC_BF16)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc<PREC>()), "r"(acc));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc<PREC>()), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   su32(bar))
               : "memory");
}
// arrive on the barrier at this offset in every CTA of `mask` once the issued MMAs completed
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n" ::"r"(su32(bar)),
      "h"(mask)
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

// TF32 operands are stored pre-rounded (round to nearest): the tensor core drops the low 13
// mantissa bits, which would otherwise truncate (a systematic bias that compounds over passes)
__device__ __forceinline__ float round_tf32(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
// CL = 2: the two CTAs of a cluster take vertically adjacent 128-row panels with the same
// 256-column tile; each loads one 128-row half of the B tile as a TMA multicast into both, so the
// matrix crosses L2 -> SM once per pair (B traffic halves); a stage is refilled only when both
// CTAs' MMAs have read it (multicast tcgen05.commit into both empty barriers).
template <int PREC, int OUT_F64, int CL>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_pass_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tb,
                   const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + TC_STAGES * TC_STAGE);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], CL);
    }
    for (int b = 0; b < 2; ++b) {
      mb_init(&tfull[b], 1);
      mb_init(&tempty[b], TC_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (CL > 1) cl_sync();  // the peer's barriers exist before any multicast / remote commit
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // tile sequence: T over (row-panel group, column tile); a CL-cluster shares one T
  const uint32_t crank = CL > 1 ? cl_rank() : 0;
  const long long tiles = ((a.ntm + CL - 1) / CL) * a.ntn;
  const long long t0 = blockIdx.x / CL, tstep = gridDim.x / CL;
  constexpr int BK = TcTraits<PREC>::BK;
  const int KB = (a.K + BK - 1) / BK;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tx) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tb) : "memory");
      long long it = 0;
      for (long long T = t0; T < tiles; T += tstep) {
        const long long tg = T / a.ntn;
        const int row0 = static_cast<int>((tg * CL + crank) * TC_BM);
        const int col0 = static_cast<int>(T - tg * a.ntn) * TC_BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = static_cast<int>(it % TC_STAGES);
          const uint32_t ph = static_cast<uint32_t>((it / TC_STAGES) & 1);
          mb_wait(&empty[s], ph ^ 1);
          unsigned char* st = sm + s * TC_STAGE;
          mb_expect_tx(&full[s], TC_STAGE);
          tma2d(st, &tx, kb * BK, row0, &full[s]);
          if (CL == 1)
            tma2d(st + TC_A_BYTES, &tb, kb * BK, col0, &full[s]);
          else  // this CTA's 128-row half of the B tile, into both CTAs
            tma2d_mc(st + TC_A_BYTES + crank * (TC_B_BYTES / 2), &tb, kb * BK,
                     col0 + static_cast<int>(crank) * (TC_BN / 2), &full[s], 0x3);
        }
      }
    }
  } else if (warp == 1) {
    {  // MMA warp (converged; one elected lane issues)
      long long it = 0, lt = 0;
      for (long long T = t0; T < tiles; T += tstep, ++lt) {
        const int b = static_cast<int>(lt & 1);
        const uint32_t tph = static_cast<uint32_t>((lt >> 1) & 1);
        mb_wait(&tempty[b], tph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + b * TC_BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = static_cast<int>(it % TC_STAGES);
          const uint32_t ph = static_cast<uint32_t>((it / TC_STAGES) & 1);
          mb_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = su32(sm + s * TC_STAGE), sb = sa + TC_A_BYTES;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / TcTraits<PREC>::UK; ++kk)  // 32 bytes of K per instruction
              umma<PREC>(d, umma_desc(sa + kk * 32), umma_desc(sb + kk * 32), (kb | kk) != 0);
            if (CL == 1)
              umma_commit(&empty[s]);  // smem stage free once these MMAs have read it
            else
              umma_commit_mc(&empty[s], 0x3);  // ... in both CTAs (the peer multicasts into it)
          }
          __syncwarp();
        }
        if (elect_one()) umma_commit(&tfull[b]);  // accumulator b complete
        __syncwarp();
      }
    }
  } else {  // epilogue warps 2..9: TMEM lane quadrant = warp % 4, column half = (warp - 2) / 4
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    long long lt = 0;
    for (long long T = t0; T < tiles; T += tstep, ++lt) {
      const int b = static_cast<int>(lt & 1);
      const uint32_t tph = static_cast<uint32_t>((lt >> 1) & 1);
      const long long tg = T / a.ntn;
      const long long r = (tg * CL + crank) * TC_BM + 32 * q + lane;
      const int col0 = static_cast<int>(T - tg * a.ntn) * TC_BN;
      double lam_low = 0.0;
      if (a.epi != 0 && r < a.R) {  // axes below the contracted one, in axis order from 0.0
        long long rr = r;
        for (int j = 0; j < a.nlow; ++j) {
          const long long idx = rr % a.lowext[j];
          rr /= a.lowext[j];
          lam_low = __dadd_rn(lam_low, a.lowlam[j][idx]);
        }
      }
      const float lam_low_f = static_cast<float>(__dsub_rn(lam_low, a.shift));
      mb_wait(&tfull[b], tph);
      tc_fence_after();
      for (int c = hc * (TC_BN / 64); c < (hc + 1) * (TC_BN / 64); ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + b * TC_BN + c * 32 + (static_cast<uint32_t>(32 * q) << 16), v);
        if (a.epi == 0) {  // plain pass: no per-element arithmetic beyond the conversion
          if (r < a.R) {
            const int cb = col0 + c * 32;
            const int nj = a.m - cb < 32 ? a.m - cb : 32;
            long long gi = static_cast<long long>(cb) * a.R + r;
#pragma unroll
            for (int j = 0; j < 32; ++j, gi += a.R) {
              if (j >= nj) break;
              const float val = __uint_as_float(v[j]);
              if (OUT_F64)
                static_cast<double*>(a.y)[gi] = static_cast<double>(val);
              else if (PREC == PREC_BF16)
                static_cast<__nv_bfloat16*>(a.y)[gi] = __float2bfloat16_rn(val);
              else
                static_cast<float*>(a.y)[gi] = round_tf32(val);
            }
          }
          continue;
        }
        // lambda of this chunk's 32 columns: one coalesced load, then broadcast by shuffle
        float lam_c = 0.0f;
        if (a.epi != 0) {
          const int cl_ = col0 + c * 32 + lane;
          lam_c = cl_ < a.m ? static_cast<float>(a.lamlast[cl_]) : 1.0f;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {  // uniform (shuffles); stores predicated
          const int col = col0 + c * 32 + j;
          float val = __uint_as_float(v[j]);
          if (a.epi != 0) {
            // low-precision modes: lambda in FP32 and the fast FP32 divide (2 ulp) - the
            // exact FP64 sum / IEEE divide made this pass epilogue-bound (7.3 vs 2.0 ms)
            const float ls = lam_low_f + __shfl_sync(0xffffffffu, lam_c, j);
            val = a.epi == 1 ? __fdividef(val, ls) : val * ls;
          }
          if (r < a.R && col < a.m) {
            const long long gi = static_cast<long long>(col) * a.R + r;
            if (OUT_F64)
              static_cast<double*>(a.y)[gi] = static_cast<double>(val);
            else if (PREC == PREC_BF16)
              static_cast<__nv_bfloat16*>(a.y)[gi] = __float2bfloat16_rn(val);
            else
              static_cast<float*>(a.y)[gi] = round_tf32(val);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(&tempty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cl_sync();  // the peer may still multicast / commit into this CTA until it is done
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(TC_TMEM_COLS));
  }
}

__device__ __forceinline__ void cvt(double v, __nv_bfloat16& o) { o = __double2bfloat16(v); }
__device__ __forceinline__ void cvt(double v, float& o) { o = round_tf32(static_cast<float>(v)); }

template <class T>
__global__ void k_f64_to_lowp(const double* __restrict__ x, T* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    cvt(x[i], y[i]);
}

// padded column-major f64 matrix (lda) -> row-major low-precision [m][k]
template <class T>
__global__ void k_mat_to_lowp(const double* __restrict__ a, int lda, int m, int k,
                              T* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * k; e += gridDim.x * blockDim.x) {
    const int i = e / k, kk = e - i * k;
    cvt(a[i + static_cast<long long>(lda) * kk], out[e]);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    KCUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr));
    if (qr != cudaDriverEntryPointSuccess || !p) fail(KRONOP_ERUNTIME, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void encode_lowp_2d(CUtensorMap* map, const void* base, long long inner, long long outer,
                    int box_inner, int box_outer, int esize) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t str[1] = {static_cast<cuuint64_t>(inner) * esize};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tc_encode_fn()(map, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                    2, const_cast<void*>(base),
                                    dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(KRONOP_ERUNTIME, "cuTensorMapEncodeTiled (low precision) failed");
}

template <int PREC, int OUT_F64, int CL>
void tc_launch(cudaStream_t s, unsigned grid, const CUtensorMap& tx, const CUtensorMap& tb,
               const TcArgs& a) {
  ensure_smem_attr(reinterpret_cast<const void*>(tc_pass_kernel<PREC, OUT_F64, CL>), TC_SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = TC_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KCUDA(cudaLaunchKernelEx(&cfg, tc_pass_kernel<PREC, OUT_F64, CL>, tx, tb, a));
}

template <int PREC>
void tc_pass(cudaStream_t s, const void* x, const void* bmat, void* y, long long R, int K, int m,
             bool out_f64, TcArgs a) {
  using T = typename TcTraits<PREC>::T;
  // KRONOP_TC_CLUSTER=2: B tile multicast across a CTA pair. Measured at 1024^3: no change
  // (BF16 solve 19.8 -> 20.4 ms, TF32 30.1 -> 29.9 ms): each SM still receives its full 48 KB
  // stage, which is what bounds the pass, so the default stays 1.
  static const int cl = [] {
    const char* e = getenv("KRONOP_TC_CLUSTER");
    return e && e[0] == '2' ? 2 : 1;
  }();
  // cta_group::2 pairs by default (1024^3: BF16 solve 16.0 -> 14.8 ms, TF32 26.8 -> 23.8 ms);
  // KRONOP_TC_2SM=0 selects the 1-SM kernel
  static const bool two_sm = [] {
    const char* e = getenv("KRONOP_TC_2SM");
    return !(e && e[0] == '0');
  }();
  if (two_sm) {
    CUtensorMap tx2, tb2;
    encode_lowp_2d(&tx2, x, K, R, TcTraits<PREC>::BK, TC_BM, sizeof(T));
    encode_lowp_2d(&tb2, bmat, K, m, TcTraits<PREC>::BK, TC_BN / 2, sizeof(T));
    a.y = y;
    a.R = R;
    a.K = K;
    a.m = m;
    a.ntn = (m + TC_BN - 1) / TC_BN;
    a.ntm = (R + TC_BM - 1) / TC_BM;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long pairs = ((a.ntm + 1) / 2) * a.ntn;
    const long long g = 2 * (pairs < sms / 2 ? pairs : sms / 2);
    if (out_f64)
      tc2_launch<PREC, 1>(s, static_cast<unsigned>(g), tx2, tb2, a);
    else
      tc2_launch<PREC, 0>(s, static_cast<unsigned>(g), tx2, tb2, a);
    return;
  }
  CUtensorMap tx, tb;
  encode_lowp_2d(&tx, x, K, R, TcTraits<PREC>::BK, TC_BM, sizeof(T));
  encode_lowp_2d(&tb, bmat, K, m, TcTraits<PREC>::BK, cl == 2 ? TC_BN / 2 : TC_BN, sizeof(T));
  a.y = y;
  a.R = R;
  a.K = K;
  a.m = m;
  a.ntn = (m + TC_BN - 1) / TC_BN;
  a.ntm = (R + TC_BM - 1) / TC_BM;
  const int sms = device_sm_count();
  const long long tiles = ((a.ntm + cl - 1) / cl) * a.ntn * cl;  // CTAs worth of work
  long long g = tiles < sms ? tiles : sms;
  g = g / cl * cl;
  if (g < cl) g = cl;
  const unsigned grid = static_cast<unsigned>(g);
  if (cl == 2) {
    if (out_f64)
      tc_launch<PREC, 1, 2>(s, grid, tx, tb, a);
    else
      tc_launch<PREC, 0, 2>(s, grid, tx, tb, a);
  } else {
    if (out_f64)
      tc_launch<PREC, 1, 1>(s, grid, tx, tb, a);
    else
      tc_launch<PREC, 0, 1>(s, grid, tx, tb, a);
  }
}

template <int PREC>
void sep_solve_lowp_impl(kronop_ctx& ctx, kronop_op& op, const double* b, double* x) {
  using T = typename TcTraits<PREC>::T;
  param_check(!op.folded, "solve_lowp: dense operators only");
  for (int a = 0; a < op.d; ++a)
    param_check(op.n[a] % 8 == 0 && op.n[a] >= 16, "solve_lowp: extents must be multiples of 8");
  const long long N = op.N;
  cudaStream_t s = ctx.stream;
  void** lf = PREC == PREC_BF16 ? op.lp_fwd : op.tf_fwd;
  void** lb = PREC == PREC_BF16 ? op.lp_bwd : op.tf_bwd;
  if (!lf[0]) {  // low-precision copies of the transforms (row-major [out][k]), made once
    for (int a = 0; a < op.d; ++a) {
      const int n = op.n[a];
      for (int dir = 0; dir < 2; ++dir) {
        void* p = nullptr;
        KCUDA(cudaMalloc(&p, static_cast<size_t>(n) * n * sizeof(T)));
        k_mat_to_lowp<T><<<256, 256, 0, s>>>(dir == 0 ? op.fwd[a] : op.bwd[a], op.lda[a], n, n,
                                             static_cast<T*>(p));
        KCUDA(cudaGetLastError());
        (dir == 0 ? lf : lb)[a] = p;
      }
    }
  }
  ensure_scratch(ctx, static_cast<size_t>(N * sizeof(T) / 8 + 16));  // two low-precision fields
  T* f0 = reinterpret_cast<T*>(ctx.scratch[0]);
  T* f1 = reinterpret_cast<T*>(ctx.scratch[1]);
  k_f64_to_lowp<T><<<kEltBlocks, 256, 0, s>>>(b, f0, N);
  KCUDA(cudaGetLastError());
  ctx.ws.launches += 1;
  const T* cur = f0;
  int k = 0;
  for (int dir = 0; dir < 2; ++dir)
    for (int a = 0; a < op.d; ++a, ++k) {
      const bool last = dir == 1 && a == op.d - 1;
      T* dst = (k % 2 == 0) ? f1 : f0;
      TcArgs ta{};
      if (dir == 0 && a == op.d - 1) {
        ta.epi = 1;
        ta.shift = op.shift;
        ta.nlow = op.d - 1;
        for (int j = 0; j < op.d - 1; ++j) {
          ta.lowext[j] = op.n[j];
          ta.lowlam[j] = op.lam[j];
        }
        ta.lamlast = op.lam[a];
      }
      const int n = op.n[a];
      tc_pass<PREC>(s, cur, dir == 0 ? lf[a] : lb[a],
                    last ? static_cast<void*>(x) : static_cast<void*>(dst), N / n, n, n, last, ta);
      ctx.ws.launches += 1;
      cur = dst;
    }
}

// ------------------------------------------------------------- 2-SM (cta_group::2) --
// A CTA pair computes a 256 x 256 tile with tcgen05.mma.cta_group::2 issued by the leader (rank
// 0): each CTA stages its own 128 rows of A and 128 of the 256 B rows (N split), so per SM a
// stage is 32 KB for twice the FLOPs of the 1-SM kernel's 48 KB stage (6 stages fit). Both CTAs'
// TMA loads complete on the leader's full barrier; the leader's commits multicast to both CTAs'
// empty / accumulator-full barriers; both CTAs' epilogue warps release the leader's
// accumulator-empty barrier. Protocol as in cute/arch/copy_sm100_tma.hpp (SM100_TMA_2SM_LOAD),
// cute/arch/mma_sm100_umma.hpp (SM100_MMA_*_2x1SM_SS), cute/arch/tmem_allocator_sm100.hpp.
constexpr int T2_STAGES = 6;
constexpr int T2_A = TC_BM * TC_ROW;         // 16 KB
constexpr int T2_B = (TC_BN / 2) * TC_ROW;   // 16 KB (this CTA's half of N)
constexpr int T2_STAGE = T2_A + T2_B;
constexpr int T2_SMEM = T2_STAGES * T2_STAGE + 1024 + 256;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's barrier

template <int PREC>
__host__ __device__ constexpr uint32_t idesc2() {  // M = 256 (pair), N = 256
  return (1u << 4) | (TcTraits<PREC>::FMT << 7) | (TcTraits<PREC>::FMT << 10) |
         ((TC_BN >> 3) << 17) | ((256 >> 4) << 24);
}
__device__ __forceinline__ void tma2d_2sm(void* dst, const CUtensorMap* map, int c0, int c1,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(su32(bar) & kPeerMask)
      : "memory");
}
template <int PREC>
__device__ __forceinline__ void umma2(uint32_t d, uint64_t da, uint64_t db, uint32_t acc) {
  if constexpr (PREC == PREC_BF16)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n}\n" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc2<PREC>()), "r"(acc), "r"(0u));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n}\n" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc2<PREC>()), "r"(acc), "r"(0u));
}
__device__ __forceinline__ void umma2_commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n" ::"r"(su32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}
__device__ __forceinline__ void mb_arrive_rank(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(su32(bar)),
      "r"(rank)
      : "memory");
}

template <int PREC, int OUT_F64>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc2_pass_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tb,
                    const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + T2_STAGES * T2_STAGE);
  uint64_t* empty = full + T2_STAGES;
  uint64_t* tfull = empty + T2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = cl_rank();
  const bool leader = crank == 0;
  if (tid == 0) {
    for (int s = 0; s < T2_STAGES; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mb_init(&tfull[b], 1);
      mb_init(&tempty[b], 2 * TC_EPI_WARPS);  // the epilogue warps of both CTAs of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cl_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const long long pair_tm = (a.ntm + 1) / 2;  // 256-row panels
  const long long tiles = pair_tm * a.ntn;
  const long long t0 = blockIdx.x / 2, tstep = gridDim.x / 2;
  constexpr int BK = TcTraits<PREC>::BK;
  const int KB = (a.K + BK - 1) / BK;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs)
      long long it = 0;
      for (long long T = t0; T < tiles; T += tstep) {
        const long long tg = T / a.ntn;
        const int row0 = static_cast<int>((tg * 2 + crank) * TC_BM);
        const int col0 = static_cast<int>(T - tg * a.ntn) * TC_BN + static_cast<int>(crank) * (TC_BN / 2);
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = static_cast<int>(it % T2_STAGES);
          mb_wait(&empty[s], static_cast<uint32_t>((it / T2_STAGES) & 1) ^ 1);
          unsigned char* st = sm + s * T2_STAGE;
          if (leader) mb_expect_tx(&full[s], 2 * T2_STAGE);  // both CTAs' bytes land on it
          tma2d_2sm(st, &tx, kb * BK, row0, &full[s]);
          tma2d_2sm(st + T2_A, &tb, kb * BK, col0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // MMA warp of the leader (converged; one elected lane issues)
      long long it = 0, lt = 0;
      for (long long T = t0; T < tiles; T += tstep, ++lt) {
        const int b = static_cast<int>(lt & 1);
        mb_wait(&tempty[b], static_cast<uint32_t>((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + b * TC_BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = static_cast<int>(it % T2_STAGES);
          mb_wait(&full[s], static_cast<uint32_t>((it / T2_STAGES) & 1));
          tc_fence_after();
          const uint32_t sa = su32(sm + s * T2_STAGE), sb = sa + T2_A;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / TcTraits<PREC>::UK; ++kk)
              umma2<PREC>(d, umma_desc(sa + kk * 32), umma_desc(sb + kk * 32), (kb | kk) != 0);
            umma2_commit_mc(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) umma2_commit_mc(&tfull[b]);
        __syncwarp();
      }
    }
  } else {  // epilogue warps, both CTAs: this CTA's 128 rows x 256 columns
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    long long lt = 0;
    for (long long T = t0; T < tiles; T += tstep, ++lt) {
      const int b = static_cast<int>(lt & 1);
      const long long tg = T / a.ntn;
      const long long r = (tg * 2 + crank) * TC_BM + 32 * q + lane;
      const int col0 = static_cast<int>(T - tg * a.ntn) * TC_BN;
      double lam_low = 0.0;
      if (a.epi != 0 && r < a.R) {
        long long rr = r;
        for (int j = 0; j < a.nlow; ++j) {
          const long long idx = rr % a.lowext[j];
          rr /= a.lowext[j];
          lam_low = __dadd_rn(lam_low, a.lowlam[j][idx]);
        }
      }
      const float lam_low_f = static_cast<float>(__dsub_rn(lam_low, a.shift));
      mb_wait(&tfull[b], static_cast<uint32_t>((lt >> 1) & 1));
      tc_fence_after();
      for (int c = hc * (TC_BN / 64); c < (hc + 1) * (TC_BN / 64); ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + b * TC_BN + c * 32 + (static_cast<uint32_t>(32 * q) << 16), v);
        if (a.epi == 0) {  // plain pass: no per-element arithmetic beyond the conversion
          if (r < a.R) {
            const int cb = col0 + c * 32;
            const int nj = a.m - cb < 32 ? a.m - cb : 32;
            long long gi = static_cast<long long>(cb) * a.R + r;
#pragma unroll
            for (int j = 0; j < 32; ++j, gi += a.R) {
              if (j >= nj) break;
              const float val = __uint_as_float(v[j]);
              if (OUT_F64)
                static_cast<double*>(a.y)[gi] = static_cast<double>(val);
              else if (PREC == PREC_BF16)
                static_cast<__nv_bfloat16*>(a.y)[gi] = __float2bfloat16_rn(val);
              else
                static_cast<float*>(a.y)[gi] = round_tf32(val);
            }
          }
          continue;
        }
        // lambda of this chunk's 32 columns: one coalesced load, then broadcast by shuffle
        float lam_c = 0.0f;
        if (a.epi != 0) {
          const int cl_ = col0 + c * 32 + lane;
          lam_c = cl_ < a.m ? static_cast<float>(a.lamlast[cl_]) : 1.0f;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {  // uniform (shuffles); stores predicated
          const int col = col0 + c * 32 + j;
          float val = __uint_as_float(v[j]);
          if (a.epi != 0) {
            const float ls = lam_low_f + __shfl_sync(0xffffffffu, lam_c, j);
            val = __fdividef(val, ls);
          }
          if (r < a.R && col < a.m) {
            const long long gi = static_cast<long long>(col) * a.R + r;
            if (OUT_F64)
              static_cast<double*>(a.y)[gi] = static_cast<double>(val);
            else if (PREC == PREC_BF16)
              static_cast<__nv_bfloat16*>(a.y)[gi] = __float2bfloat16_rn(val);
            else
              static_cast<float*>(a.y)[gi] = round_tf32(val);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive_rank(&tempty[b], 0);  // the leader's barrier
    }
  }
  tc_fence_before();
  __syncthreads();
  cl_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(TC_TMEM_COLS));
  }
}

template <int PREC, int OUT_F64>
void tc2_launch(cudaStream_t s, unsigned grid, const CUtensorMap& tx, const CUtensorMap& tb,
                const TcArgs& a) {
  ensure_smem_attr(reinterpret_cast<const void*>(tc2_pass_kernel<PREC, OUT_F64>), T2_SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = T2_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KCUDA(cudaLaunchKernelEx(&cfg, tc2_pass_kernel<PREC, OUT_F64>, tx, tb, a));
}

// ---------------------------------------------------------------- FP32 via 3xTF32 --
// The paper's FP32 row on tensor cores: every field value is carried as a pair (hi, lo) of
// TF32-rounded floats (x ~ hi + lo, ~22 significant bits), every matrix likewise, and each
// product is formed as hi*hi + hi*lo + lo*hi (the lo*lo term is below FP32 rounding) by three
// tcgen05.mma kind::tf32 into one FP32 TMEM accumulator. Stage = A_hi, A_lo (128 x 32) and
// B_hi, B_lo (128 x 32) = 64 KB, 3 stages; N = 128 per tile, two 128-column accumulators.
constexpr int T3_BN = 128;
constexpr int T3_A = TC_BM * TC_ROW;   // 16 KB per A half
constexpr int T3_B = T3_BN * TC_ROW;   // 16 KB per B half
constexpr int T3_STAGE = 2 * T3_A + 2 * T3_B;
constexpr int T3_STAGES = 3;
constexpr int T3_SMEM = T3_STAGES * T3_STAGE + 1024 + 256;
constexpr int T3_TMEM_COLS = 256;
constexpr uint32_t kIdesc3 =
    (1u << 4) | (2u << 7) | (2u << 10) | ((T3_BN >> 3) << 17) | ((TC_BM >> 4) << 24);

__device__ __forceinline__ void umma_tf32_n128(uint32_t d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(da), "l"(db), "r"(kIdesc3), "r"(acc));
}

template <int OUT_F64>
__global__ void __launch_bounds__(TC_THREADS, 1)
    t3_pass_kernel(const __grid_constant__ CUtensorMap txh, const __grid_constant__ CUtensorMap txl,
                   const __grid_constant__ CUtensorMap tbh, const __grid_constant__ CUtensorMap tbl,
                   const TcArgs a, float* __restrict__ ylo) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + T3_STAGES * T3_STAGE);
  uint64_t* empty = full + T3_STAGES;
  uint64_t* tfull = empty + T3_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < T3_STAGES; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mb_init(&tfull[b], 1);
      mb_init(&tempty[b], TC_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(T3_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const long long tiles = a.ntm * a.ntn;
  constexpr int BK = 32;
  const int KB = (a.K + BK - 1) / BK;
  if (warp == 0) {
    if (lane == 0) {
      long long it = 0;
      for (long long T = blockIdx.x; T < tiles; T += gridDim.x) {
        const long long tm = T / a.ntn;
        const int row0 = static_cast<int>(tm * TC_BM);
        const int col0 = static_cast<int>(T - tm * a.ntn) * T3_BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = static_cast<int>(it % T3_STAGES);
          const uint32_t ph = static_cast<uint32_t>((it / T3_STAGES) & 1);
          mb_wait(&empty[s], ph ^ 1);
          unsigned char* st = sm + s * T3_STAGE;
          mb_expect_tx(&full[s], T3_STAGE);
          tma2d(st, &txh, kb * BK, row0, &full[s]);
          tma2d(st + T3_A, &txl, kb * BK, row0, &full[s]);
          tma2d(st + 2 * T3_A, &tbh, kb * BK, col0, &full[s]);
          tma2d(st + 2 * T3_A + T3_B, &tbl, kb * BK, col0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      long long it = 0, lt = 0;
      for (long long T = blockIdx.x; T < tiles; T += gridDim.x, ++lt) {
        const int b = static_cast<int>(lt & 1);
        mb_wait(&tempty[b], static_cast<uint32_t>((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + b * T3_BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = static_cast<int>(it % T3_STAGES);
          mb_wait(&full[s], static_cast<uint32_t>((it / T3_STAGES) & 1));
          tc_fence_after();
          const uint32_t ah = su32(sm + s * T3_STAGE), al = ah + T3_A, bh = ah + 2 * T3_A,
                         bl = bh + T3_B;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t o = kk * 32;
            umma_tf32_n128(d, umma_desc(al + o), umma_desc(bh + o), (kb | kk) != 0);  // lo*hi
            umma_tf32_n128(d, umma_desc(ah + o), umma_desc(bl + o), 1);               // hi*lo
            umma_tf32_n128(d, umma_desc(ah + o), umma_desc(bh + o), 1);               // hi*hi
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[b]);
      }
    }
  } else {
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    long long lt = 0;
    for (long long T = blockIdx.x; T < tiles; T += gridDim.x, ++lt) {
      const int b = static_cast<int>(lt & 1);
      const long long tm = T / a.ntn;
      const long long r = tm * TC_BM + 32 * q + lane;
      const int col0 = static_cast<int>(T - tm * a.ntn) * T3_BN;
      double lam_low = 0.0;
      if (a.epi != 0 && r < a.R) {
        long long rr = r;
        for (int j = 0; j < a.nlow; ++j) {
          const long long idx = rr % a.lowext[j];
          rr /= a.lowext[j];
          lam_low = __dadd_rn(lam_low, a.lowlam[j][idx]);
        }
      }
      const float lam_low_f = static_cast<float>(__dsub_rn(lam_low, a.shift));
      mb_wait(&tfull[b], static_cast<uint32_t>((lt >> 1) & 1));
      tc_fence_after();
      for (int c = hc * (T3_BN / 64); c < (hc + 1) * (T3_BN / 64); ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + b * T3_BN + c * 32 + (static_cast<uint32_t>(32 * q) << 16), v);
        if (a.epi == 0) {  // plain pass
          if (r < a.R) {
            const int cb = col0 + c * 32;
            const int nj = a.m - cb < 32 ? a.m - cb : 32;
            long long gi = static_cast<long long>(cb) * a.R + r;
#pragma unroll
            for (int j = 0; j < 32; ++j, gi += a.R) {
              if (j >= nj) break;
              const float val = __uint_as_float(v[j]);
              if (OUT_F64) {
                static_cast<double*>(a.y)[gi] = static_cast<double>(val);
              } else {
                const float hi = round_tf32(val);
                static_cast<float*>(a.y)[gi] = hi;
                ylo[gi] = round_tf32(val - hi);
              }
            }
          }
          continue;
        }
        // lambda of this chunk's 32 columns: one coalesced load, then broadcast by shuffle
        float lam_c = 0.0f;
        if (a.epi != 0) {
          const int cl_ = col0 + c * 32 + lane;
          lam_c = cl_ < a.m ? static_cast<float>(a.lamlast[cl_]) : 1.0f;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {  // uniform (shuffles); stores predicated
          const int col = col0 + c * 32 + j;
          float val = __uint_as_float(v[j]);
          if (a.epi != 0) {
            const float ls = lam_low_f + __shfl_sync(0xffffffffu, lam_c, j);
            val = __fdividef(val, ls);
          }
          if (r < a.R && col < a.m) {
            const long long gi = static_cast<long long>(col) * a.R + r;
            if (OUT_F64) {
              static_cast<double*>(a.y)[gi] = static_cast<double>(val);
            } else {
              const float hi = round_tf32(val);
              static_cast<float*>(a.y)[gi] = hi;
              ylo[gi] = round_tf32(val - hi);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(&tempty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(T3_TMEM_COLS));
  }
}

__global__ void k_f64_to_split(const double* __restrict__ x, float* __restrict__ hi,
                               float* __restrict__ lo, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double v = x[i];
    const float h = round_tf32(static_cast<float>(v));
    hi[i] = h;
    lo[i] = round_tf32(static_cast<float>(v - static_cast<double>(h)));
  }
}

__global__ void k_mat_to_split(const double* __restrict__ a, int lda, int m, int k,
                               float* __restrict__ hi, float* __restrict__ lo) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * k; e += gridDim.x * blockDim.x) {
    const int i = e / k, kk = e - i * k;
    const double v = a[i + static_cast<long long>(lda) * kk];
    const float h = round_tf32(static_cast<float>(v));
    hi[e] = h;
    lo[e] = round_tf32(static_cast<float>(v - static_cast<double>(h)));
  }
}

void t3_pass(cudaStream_t s, const float* xh, const float* xl, const float* bh, const float* bl,
             void* y, float* ylo, long long R, int K, int m, bool out_f64, TcArgs a) {
  CUtensorMap txh, txl, tbh, tbl;
  encode_lowp_2d(&txh, xh, K, R, 32, TC_BM, 4);
  encode_lowp_2d(&txl, xl, K, R, 32, TC_BM, 4);
  encode_lowp_2d(&tbh, bh, K, m, 32, T3_BN, 4);
  encode_lowp_2d(&tbl, bl, K, m, 32, T3_BN, 4);
  a.y = y;
  a.R = R;
  a.K = K;
  a.m = m;
  a.ntn = (m + T3_BN - 1) / T3_BN;
  a.ntm = (R + TC_BM - 1) / TC_BM;
  ensure_smem_attr(reinterpret_cast<const void*>(t3_pass_kernel<0>), T3_SMEM);
  ensure_smem_attr(reinterpret_cast<const void*>(t3_pass_kernel<1>), T3_SMEM);
  const int sms = device_sm_count();
  const long long tiles = a.ntm * a.ntn;
  const unsigned grid = static_cast<unsigned>(tiles < sms ? tiles : sms);
  if (out_f64)
    t3_pass_kernel<1><<<grid, TC_THREADS, T3_SMEM, s>>>(txh, txl, tbh, tbl, a, ylo);
  else
    t3_pass_kernel<0><<<grid, TC_THREADS, T3_SMEM, s>>>(txh, txl, tbh, tbl, a, ylo);
  KCUDA(cudaGetLastError());
}

void sep_solve_3xtf32(kronop_ctx& ctx, kronop_op& op, const double* b, double* x) {
  param_check(!op.folded, "solve_lowp: dense operators only");
  for (int a = 0; a < op.d; ++a)
    param_check(op.n[a] % 8 == 0 && op.n[a] >= 16, "solve_lowp: extents must be multiples of 8");
  const long long N = op.N;
  cudaStream_t s = ctx.stream;
  if (!op.f3_fwd[0]) {  // (hi, lo) pairs of the transforms, row-major [out][k], made once
    for (int a = 0; a < op.d; ++a) {
      const int n = op.n[a];
      for (int dir = 0; dir < 2; ++dir) {
        void* p = nullptr;
        KCUDA(cudaMalloc(&p, static_cast<size_t>(n) * n * 2 * sizeof(float)));
        float* hp = static_cast<float*>(p);
        k_mat_to_split<<<256, 256, 0, s>>>(dir == 0 ? op.fwd[a] : op.bwd[a], op.lda[a], n, n, hp,
                                           hp + static_cast<size_t>(n) * n);
        KCUDA(cudaGetLastError());
        (dir == 0 ? op.f3_fwd : op.f3_bwd)[a] = p;
      }
    }
  }
  ensure_scratch(ctx, static_cast<size_t>(N + 16));  // (hi, lo) FP32 pairs = one double each
  float* h0 = reinterpret_cast<float*>(ctx.scratch[0]);
  float* l0 = h0 + N;
  float* h1 = reinterpret_cast<float*>(ctx.scratch[1]);
  float* l1 = h1 + N;
  k_f64_to_split<<<kEltBlocks, 256, 0, s>>>(b, h0, l0, N);
  KCUDA(cudaGetLastError());
  ctx.ws.launches += 1;
  const float *ch = h0, *cl = l0;
  int k = 0;
  for (int dir = 0; dir < 2; ++dir)
    for (int a = 0; a < op.d; ++a, ++k) {
      const bool last = dir == 1 && a == op.d - 1;
      float* dh = (k % 2 == 0) ? h1 : h0;
      float* dl = (k % 2 == 0) ? l1 : l0;
      TcArgs ta{};
      if (dir == 0 && a == op.d - 1) {
        ta.epi = 1;
        ta.shift = op.shift;
        ta.nlow = op.d - 1;
        for (int j = 0; j < op.d - 1; ++j) {
          ta.lowext[j] = op.n[j];
          ta.lowlam[j] = op.lam[j];
        }
        ta.lamlast = op.lam[a];
      }
      const int n = op.n[a];
      const float* mh = static_cast<const float*>(dir == 0 ? op.f3_fwd[a] : op.f3_bwd[a]);
      t3_pass(s, ch, cl, mh, mh + static_cast<size_t>(n) * n,
              last ? static_cast<void*>(x) : static_cast<void*>(dh), dl, N / n, n, n, last, ta);
      ctx.ws.launches += 1;
      ch = dh;
      cl = dl;
    }
}

}  // namespace

// (-Delta + V1 - shift)^{-1} b in BF16 or TF32 (FP32 storage) on tcgen05, FP32 accumulation
// (real field, every extent a multiple of 8 for the 16-byte TMA row pitch). b, x: FP64 device.
void sep_solve_lowp(kronop_ctx& ctx, kronop_op& op, const double* b, double* x, int precision) {
  if (precision == PREC_BF16)
    sep_solve_lowp_impl<PREC_BF16>(ctx, op, b, x);
  else if (precision == PREC_TF32)
    sep_solve_lowp_impl<PREC_TF32>(ctx, op, b, x);
  else
    sep_solve_3xtf32(ctx, op, b, x);
}

}  // namespace kronop_dev
