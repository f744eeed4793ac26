// Kronecker-factored propagate for small extents (BASELINE config 5: 9D n = 9 complex128).
//
// The reference propagates with forward transforms on every axis, one pointwise phase and
// backward transforms (operators.cpp:63-75):
//   psi' = T (e^{-i (lambda - shift) dt} . T^{-1} psi),  lambda = sum_a lambda_a (tensor.cpp:196-209)
// Because the operator is a Kronecker SUM, its exponential is a Kronecker PRODUCT of the per-axis
// exponentials:
//   e^{-i (sum_a A_a - shift) dt} = e^{i shift dt} (x)_a E_a,   E_a = T_a diag(e^{-i lambda_a dt}) T_a^{-1}
// so the same map is d complex n x n mode products instead of 2d real ones plus a phase pass. The
// flop count is the same (a complex x complex mode product is four real ones, a real x complex
// one two), but a 9D propagate then moves the field through HBM 3 times (groups of three axes)
// instead of 7 (3 forward groups, the phase pass, 3 backward groups), and no sincos runs per
// element. The E_a are formed on the host in extended precision from the operator's own T, T^{-1}
// and lambda (capi.cu, kron_prop_matrix); the result agrees with the transform / phase / transform
// sequence to rounding (tests/test_gpu_kron.py compares both with the oracle).
//
// Kernel (one launch per group of f <= 3 consecutive axes with the same extent N <= 10):
// * Rotating layout as fused_rot.cu: the group is the fastest axes after re/im, a tile = QT
//   consecutive values q of the other axes = QT contiguous planes of F = N^f complex values, and the
//   output moves the group to the slowest end (complex index q + Q g), so after all groups the
//   layout is the caller's again. Tiles arrive by cp.async.bulk (mbarrier complete_tx) into a
//   3-stage ring; one CTA per SM, walking a contiguous range of tiles.
// * The planes sit in shared memory with a pitch PPC = F + pad (complex units) chosen so that the
//   16-byte (re, im) loads of every axis are bank-conflict free (the last axis walks q fastest, so
//   its stores to HBM are runs of QT pairs).
// * DFMA, one thread per complex fiber: the N inputs in registers, 4 N^2 DFMA against E_a, whose
//   entries are KERNEL PARAMETERS read as constant-bank operands (uniform across the warp), so the
//   matrix costs neither registers nor shared-memory loads (the T-form kernel held the real matrix
//   in 2 N^2 registers, which capped it at 2 warps per SM sub-partition).
// * The first f-1 axes are applied in place; the last axis writes its outputs straight from
//   registers to HBM, optionally times the split-step B phase e^{-i factor B} (pointwise_phase,
//   splitting.cpp:44-51) of the NEXT B step, which the caller fuses into the last group.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "kronop_internal.cuh"

namespace kronop_dev {

namespace {

// One CTA per SM with a 3-deep ring (one tile in compute, two in flight) measured fastest:
// 9D n = 9 propagate 10.3 ms vs 11.9 ms for two CTAs x 2 stages and 10.5 ms for 1 x 4
// (tools/microbench/kron_bench.py; profiles/r02_kron_variants.json).
#ifndef KRONOP_KR_CTAS
#define KRONOP_KR_CTAS 1
#endif
#ifndef KRONOP_KR_STAGES
#define KRONOP_KR_STAGES 3
#endif
#ifndef KRONOP_KR_TILE
#define KRONOP_KR_TILE 6144
#endif
constexpr int KR_TILE_MAX = KRONOP_KR_TILE;  // doubles per stage before padding (48 KB)
constexpr int KR_MAXN = 10;
constexpr int KD_MAXN = 32;

__host__ __device__ constexpr int kr_pow(int n, int f) { return f == 0 ? 1 : n * kr_pow(n, f - 1); }
__host__ __device__ constexpr int kr_qt(int F, int q) {
  return (2 * (2 * q) * F <= KR_TILE_MAX && q < 256) ? kr_qt(F, 2 * q) : q;
}
__host__ __device__ constexpr int kr_round32(int v) { return (v + 31) / 32 * 32; }

template <int N, int NF>
struct KronCfg {
  static constexpr int F = kr_pow(N, NF);    // group extent (complex values per plane)
  static constexpr int QT = kr_qt(F, 1);     // planes per tile (power of two)
  static constexpr int PL = F / N;           // last axis' complex stride = fibers per plane
  static constexpr int FIB = QT * PL;        // complex fibers per axis per tile
  static constexpr int THREADS = FIB >= 1024 ? 1024 : (kr_round32(FIB) < 64 ? 64 : kr_round32(FIB));
  // plane pitch: 8 lanes of a 16-byte access phase see QT planes x (8 / QT) fibers on the last
  // axis, so the pitch must be = 8 / QT (mod 8) for QT <= 8 and odd beyond
  static constexpr int TGT = QT >= 8 ? 1 : 8 / QT;
  static constexpr int PPC = F + ((TGT - F % 8) % 8 + 8) % 8;
  static constexpr int STAGE = 2 * QT * PPC;  // doubles
};

template <int N, int NF>
struct KronArgs {
  const double* x;
  double* y;
  long long Q;       // N_total / F
  long long ntiles;
  const double* bfield;  // B phase in the last group's store (null = B == 1)
  double bfactor;
  int bphase;
  // B phase of the step BEFORE this propagate, applied to the tile as it is read (first group
  // only): pre[i] = (cos, sin) of -factor B_i, the table of k_phase's operations; null = none
  const double2* pre;
  double2 E[NF][N][N];  // E_j(i, k) = (re, im): output i, input k
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// psi * (cos, sin) with the operations of k_phase (vector_ops.cu), so a B phase applied here is
// bit-identical to the standalone pass
__device__ __forceinline__ double2 kr_rotate(double2 v, double2 cs) {
  return make_double2(__dsub_rn(__dmul_rn(v.x, cs.x), __dmul_rn(v.y, cs.y)),
                      __dadd_rn(__dmul_rn(v.x, cs.y), __dmul_rn(v.y, cs.x)));
}

// Bulk loads of tile `tile` (thread 0): one copy when the planes are unpadded, else one per plane.
template <int N, int NF>
__device__ __forceinline__ void kr_issue(const KronArgs<N, NF>& A, long long tile, double* dst,
                                         uint64_t* bar) {
  using C = KronCfg<N, NF>;
  const long long q0 = tile * C::QT;
  const int qv = static_cast<int>(A.Q - q0 < C::QT ? A.Q - q0 : C::QT);
  const double* src = A.x + 2LL * C::F * q0;
  mbar_expect_tx(bar, static_cast<uint32_t>(qv) * C::F * 16u);
  if constexpr (C::PPC == C::F) {
    bulk_load(dst, src, static_cast<uint32_t>(qv) * C::F * 16u, bar);
  } else {
    for (int qi = 0; qi < qv; ++qi)
      bulk_load(dst + 2 * C::PPC * qi, src + 2LL * C::F * qi, C::F * 16u, bar);
  }
}

// out_i = sum_k E_J(i, k) x_k, complex; E from the parameter space (uniform constant loads, 128
// bits = one complex entry). Each of the 2N accumulators is one fma chain in k order.
//
// FOLD (every E_a commutes with the reflection R: i -> N-1-i, i.e. the axis' operator is parity
// symmetric -- a symmetric box [-L, L] with an even V1, as every config-5 axis): E maps even
// vectors to even and odd to odd, so with s_k = x_k + x_{N-1-k}, d_k = x_k - x_{N-1-k} (k < M =
// N/2) and s_M = x_M (odd N)
//   a = Ae s,  b = Ao d,   out_i = a_i + b_i,  out_{N-1-i} = a_i - b_i,  out_M = a_M (odd N)
// with Ae_ik = (E_ik + E_i,N-1-k) / 2 (k < M), Ae_iM = E_iM and Ao_ik = (E_ik - E_i,N-1-k) / 2:
// (M + N%2)^2 + M^2 complex products instead of N^2 (41 vs 81 at N = 9). The host forms Ae, Ao
// (stored in E[J] as [Ae | Ao], row-major) and picks this form only when R E R = E to rounding.
template <int N, int NF, int J>
__device__ __forceinline__ double2 kr_e(const KronArgs<N, NF>& A, int flat) {
  return A.E[J][flat / N][flat % N];
}

template <int N, int NF, int J, bool FOLD>
__device__ __forceinline__ void kr_contract(const KronArgs<N, NF>& A, const double2 (&x)[N],
                                            double (&re)[N], double (&im)[N]) {
  if constexpr (!FOLD) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      re[i] = 0.0;
      im[i] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double2 e = A.E[J][i][k];  // one 128-bit uniform constant load
        re[i] = fma(e.x, x[k].x, re[i]);
        re[i] = fma(-e.y, x[k].y, re[i]);
        im[i] = fma(e.x, x[k].y, im[i]);
        im[i] = fma(e.y, x[k].x, im[i]);
      }
  } else {
    constexpr int M = N / 2, ME = M + N % 2;
    double2 sv[ME], dv[M > 0 ? M : 1];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      sv[k] = make_double2(x[k].x + x[N - 1 - k].x, x[k].y + x[N - 1 - k].y);
      dv[k] = make_double2(x[k].x - x[N - 1 - k].x, x[k].y - x[N - 1 - k].y);
    }
    if constexpr (N % 2) sv[M] = x[M];
    double ar[ME], ai[ME], br[M > 0 ? M : 1], bi[M > 0 ? M : 1];
#pragma unroll
    for (int i = 0; i < ME; ++i) ar[i] = ai[i] = 0.0;
#pragma unroll
    for (int i = 0; i < M; ++i) br[i] = bi[i] = 0.0;
#pragma unroll
    for (int k = 0; k < ME; ++k)
#pragma unroll
      for (int i = 0; i < ME; ++i) {
        const double2 e = kr_e<N, NF, J>(A, i * ME + k);
        ar[i] = fma(e.x, sv[k].x, ar[i]);
        ar[i] = fma(-e.y, sv[k].y, ar[i]);
        ai[i] = fma(e.x, sv[k].y, ai[i]);
        ai[i] = fma(e.y, sv[k].x, ai[i]);
      }
#pragma unroll
    for (int k = 0; k < M; ++k)
#pragma unroll
      for (int i = 0; i < M; ++i) {
        const double2 e = kr_e<N, NF, J>(A, ME * ME + i * M + k);
        br[i] = fma(e.x, dv[k].x, br[i]);
        br[i] = fma(-e.y, dv[k].y, br[i]);
        bi[i] = fma(e.x, dv[k].y, bi[i]);
        bi[i] = fma(e.y, dv[k].x, bi[i]);
      }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      re[i] = ar[i] + br[i];
      im[i] = ai[i] + bi[i];
      re[N - 1 - i] = ar[i] - br[i];
      im[N - 1 - i] = ai[i] - bi[i];
    }
    if constexpr (N % 2) {
      re[M] = ar[M];
      im[M] = ai[M];
    }
  }
}

// Group axis J < NF - 1, in place: fibers (lo < P, hg < H, qi) at lo + P N hg + PPC qi.
template <int N, int NF, int J, bool FOLD>
__device__ __forceinline__ void kr_axis(const KronArgs<N, NF>& A, double* buf, long long q0,
                                        int qv, int tid) {
  using C = KronCfg<N, NF>;
  constexpr int P = kr_pow(N, J);
  constexpr int H = C::F / (P * N);
  double2* b2 = reinterpret_cast<double2*>(buf);
#pragma unroll 1
  for (int f = tid; f < C::FIB; f += C::THREADS) {
    const int lo = f % P, hi = f / P;
    const int hg = hi % H, qi = hi / H;
    double2* p = b2 + lo + hg * (P * N) + qi * C::PPC;
    double2 x[N];
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = p[k * P];
    if (J == 0 && A.pre && qi < qv) {  // the preceding B phase, on the original-layout input
      const double2* ph = A.pre + (q0 + qi) * C::F + lo + hg * (P * N);
#pragma unroll
      for (int k = 0; k < N; ++k) x[k] = kr_rotate(x[k], __ldg(ph + k * P));
    }
    double re[N], im[N];
    kr_contract<N, NF, J, FOLD>(A, x, re, im);
#pragma unroll
    for (int i = 0; i < N; ++i) p[i * P] = make_double2(re[i], im[i]);
  }
}

// Last group axis (J = NF - 1, stride PL), q fastest across the lanes; outputs go to HBM with the
// group at the slowest end: complex index (q0 + qi) + Q (lo + PL i).
template <int N, int NF, bool FOLD, bool BPH>
__device__ __forceinline__ void kr_last(const KronArgs<N, NF>& A, const double* buf, long long q0,
                                        int qv, int tid) {
  using C = KronCfg<N, NF>;
  constexpr int P = C::PL;
  const double2* b2 = reinterpret_cast<const double2*>(buf);
  double2* y2 = reinterpret_cast<double2*>(A.y);
#pragma unroll 1
  for (int f = tid; f < C::FIB; f += C::THREADS) {
    const int qi = f % C::QT, lo = f / C::QT;
    if (qi >= qv) continue;
    const double2* p = b2 + lo + qi * C::PPC;
    double2 x[N];
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = p[k * P];
    if (NF == 1 && A.pre) {  // one-axis group: this is also the first axis
      const double2* ph = A.pre + (q0 + qi) * C::F + lo;
#pragma unroll
      for (int k = 0; k < N; ++k) x[k] = kr_rotate(x[k], __ldg(ph + k * P));
    }
    double re[N], im[N];
    kr_contract<N, NF, NF - 1, FOLD>(A, x, re, im);
    const long long o = q0 + qi + A.Q * lo;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const long long oi = o + A.Q * P * i;
      double vr = re[i], vi = im[i];
      if constexpr (BPH) {  // pointwise_phase (splitting.cpp:44-51), the operations of k_phase
        const double phase = A.bfield ? __dmul_rn(-A.bfactor, A.bfield[oi]) : -A.bfactor;
        double sn, cs;
        sincos(phase, &sn, &cs);
        const double r0 = vr, i0 = vi;
        vr = __dsub_rn(__dmul_rn(r0, cs), __dmul_rn(i0, sn));
        vi = __dadd_rn(__dmul_rn(r0, sn), __dmul_rn(i0, cs));
      }
      y2[oi] = make_double2(vr, vi);
    }
  }
}

template <int N, int NF, int J, bool FOLD>
__device__ __forceinline__ void kr_inplace_axes(const KronArgs<N, NF>& A, double* buf, long long q0,
                                                int qv, int tid) {
  if constexpr (J < NF - 1) {
    kr_axis<N, NF, J, FOLD>(A, buf, q0, qv, tid);
    __syncthreads();
    kr_inplace_axes<N, NF, J + 1, FOLD>(A, buf, q0, qv, tid);
  }
}

// Persistent CTA over a contiguous range of tiles, STAGES-deep ring of bulk-loaded stages.
// There is no CTA barrier at the end of a tile: the last warp to finish with a stage refills it,
// so fast warps start the next tile's first axis while slow ones still store. (A software-
// pipelined variant -- the last axis of tile t after the first axis of tile t+1, split-phase
// mbarriers between the axes -- measured slower, 15.1 vs 12.5 ms per 9D propagate: with two
// tiles in compute the 2-stage ring has no stage left to prefetch into.)
template <int N, int NF, bool FOLD, bool BPH>
__global__ void __launch_bounds__(KronCfg<N, NF>::THREADS, KRONOP_KR_CTAS)
    kron_rot_kernel(const __grid_constant__ KronArgs<N, NF> A) {
  using C = KronCfg<N, NF>;
  constexpr int STAGES = KRONOP_KR_STAGES;
  constexpr int WARPS = C::THREADS / 32;
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * C::STAGE);
  int* done = reinterpret_cast<int*>(full + STAGES);  // warps finished with a stage
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // Each CTA walks a contiguous range of tiles: its writes then complete whole lines of every
  // output run over consecutive tiles (the rotating copy measured 2.5 -> 3.1 TB/s at QT = 4
  // against the interleaved order, tools/microbench/rot_copy.cu).
  const long long per = (A.ntiles + gridDim.x - 1) / gridDim.x;
  const long long t0 = blockIdx.x * per;
  const long long t1 = t0 + per < A.ntiles ? t0 + per : A.ntiles;
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s)
      if (t0 + s < t1) kr_issue(A, t0 + s, sm + s * C::STAGE, &full[s]);
  for (int it = 0;; ++it) {
    const long long tile = t0 + it;
    if (tile >= t1) break;
    const int s = it % STAGES;
    double* buf = sm + s * C::STAGE;
    // A warp runs at most one tile ahead of the slowest (the next tile's first axis barrier
    // waits for every warp; one-axis groups: the refill waits for every warp), so the phase it
    // waits for is never two ahead of the barrier's.
    mbar_wait(&full[s], (it / STAGES) & 1);
    const long long q0 = tile * C::QT;
    const int qv = static_cast<int>(A.Q - q0 < C::QT ? A.Q - q0 : C::QT);
    kr_inplace_axes<N, NF, 0, FOLD>(A, buf, q0, qv, tid);
    kr_last<N, NF, FOLD, BPH>(A, buf, q0, qv, tid);
    const long long next = tile + STAGES;
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[s], 1) == WARPS - 1) {
        done[s] = 0;
        __threadfence_block();
        if (next < t1) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          kr_issue(A, next, buf, &full[s]);
        }
      }
    }
  }
}

// Paired-tile variant (groups whose tile has QT < 8 planes, i.e. 9D n = 9: 64-byte output runs).
// A CTA takes its tiles two at a time: both tiles' group axes, the last one included, are applied
// in place in shared memory, then the pair is written out as F runs of 2 QT consecutive q
// (128 bytes at QT = 4) -- the rotating copy moved 3.1 TB/s with 64-byte runs and 4.5 TB/s with
// 128-byte ones (tools/microbench/rot_copy.cu). 4 stages: one pair in compute, the next in flight.
// Stages sit one complex apart (pitch STAGE + 2 doubles) so the 16-byte reads of the write-out,
// 8 lanes = one g over 4 planes of each tile, are bank-conflict free.
#ifndef KRONOP_KR_PAIR
#define KRONOP_KR_PAIR 1
#endif
// KRONOP_KR_PAIR_HALVES = 2: the CTA has two halves of C::THREADS threads, each contracting one
// tile of the pair at the same time (named barriers per half), all threads writing the pair out
// (build knob; at 704 threads the contraction gets 80 registers and spills ~900 bytes, so the
// default is one team of 11 warps)
#ifndef KRONOP_KR_PAIR_HALVES
#define KRONOP_KR_PAIR_HALVES 1
#endif
template <int N, int NF>
struct KronPairCfg {
  using C = KronCfg<N, NF>;
  static constexpr int STAGES = 4;
  static constexpr int PITCH = C::STAGE + 2;  // doubles between stages
  static constexpr int HALVES = KRONOP_KR_PAIR_HALVES;
  static constexpr int THREADS = HALVES * C::THREADS;
};

// the group's axes of one tile, in place, by C::THREADS threads (htid) synchronising on their
// own named barrier (id 1 + half) -- or the whole CTA when the pair is done by one team
template <int N, int NF, int J, bool FOLD, int HALVES>
__device__ __forceinline__ void kr_axes_team(const KronArgs<N, NF>& A, double* buf, long long q0,
                                             int qv, int htid, int half) {
  using C = KronCfg<N, NF>;
  kr_axis<N, NF, J, FOLD>(A, buf, q0, qv, htid);
  if constexpr (HALVES == 1)
    __syncthreads();
  else
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + half), "n"(C::THREADS) : "memory");
  if constexpr (J + 1 < NF) kr_axes_team<N, NF, J + 1, FOLD, HALVES>(A, buf, q0, qv, htid, half);
}

template <int N, int NF, bool FOLD, bool BPH>
__global__ void __launch_bounds__(KronPairCfg<N, NF>::THREADS, 1)
    kron_rot_pair_kernel(const __grid_constant__ KronArgs<N, NF> A) {
  using C = KronCfg<N, NF>;
  using PC = KronPairCfg<N, NF>;
  constexpr int STAGES = PC::STAGES;
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * PC::PITCH);
  const int tid = threadIdx.x;
  const int half = PC::HALVES == 1 ? 0 : tid / C::THREADS;
  const int htid = tid - half * C::THREADS;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // contiguous, even-aligned tile range per CTA (a pair's first q is a multiple of 2 QT)
  long long per = (A.ntiles + gridDim.x - 1) / gridDim.x;
  per += per & 1;
  const long long t0 = blockIdx.x * per;
  const long long t1 = t0 + per < A.ntiles ? t0 + per : A.ntiles;
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s)
      if (t0 + s < t1) kr_issue(A, t0 + s, sm + s * PC::PITCH, &full[s]);
  for (int it = 0;; it += 2) {
    const long long tile = t0 + it;
    if (tile >= t1) break;
    const int nt = tile + 1 < t1 ? 2 : 1;
    const long long q0 = tile * C::QT;
    for (int u = PC::HALVES == 1 ? 0 : half; u < nt; u += PC::HALVES) {
      const int s = (it + u) % STAGES;
      double* buf = sm + s * PC::PITCH;
      mbar_wait(&full[s], ((it + u) / STAGES) & 1);
      const long long qu = q0 + u * C::QT;
      const int qv = static_cast<int>(A.Q - qu < C::QT ? A.Q - qu : C::QT);
      // every group axis, the last one included, in place
      kr_axes_team<N, NF, 0, FOLD, PC::HALVES>(A, buf, qu, qv, htid, half);
    }
    if constexpr (PC::HALVES > 1) __syncthreads();  // both tiles contracted
    // write-out: item = (g, qq), qq = 2 QT consecutive q fastest; 16 bytes per item
    const int qn = static_cast<int>(A.Q - q0 < nt * C::QT ? A.Q - q0 : nt * C::QT);
    const double2* b0 = reinterpret_cast<const double2*>(sm + (it % STAGES) * PC::PITCH);
    const double2* b1 = reinterpret_cast<const double2*>(sm + ((it + 1) % STAGES) * PC::PITCH);
    double2* y2 = reinterpret_cast<double2*>(A.y);
    constexpr int QQ = 2 * C::QT;
#pragma unroll 4
    for (int e = tid; e < C::F * QQ; e += PC::THREADS) {
      const int qq = e % QQ, g = e / QQ;
      if (qq >= qn) continue;
      const int qi = qq % C::QT;
      double2 v = (qq < C::QT ? b0 : b1)[qi * C::PPC + g];
      const long long oi = q0 + qq + A.Q * g;
      if constexpr (BPH) {  // pointwise_phase (splitting.cpp:44-51), the operations of k_phase
        const double phase = A.bfield ? __dmul_rn(-A.bfactor, A.bfield[oi]) : -A.bfactor;
        double sn, cs;
        sincos(phase, &sn, &cs);
        v = kr_rotate(v, make_double2(cs, sn));
      }
      y2[oi] = v;
    }
    __syncthreads();  // both stages read (generic proxy) before their refills
    if (tid == 0)
      for (int u = 0; u < 2; ++u)
        if (tile + u + STAGES < t1) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          const int s = (it + u) % STAGES;
          kr_issue(A, tile + u + STAGES, sm + s * PC::PITCH, &full[s]);
        }
  }
}

template <int N, int NF, bool FOLD, bool BPH>
void launch_kron(cudaStream_t s, const double* x, double* y, long long Ntot, const double* E,
                 const double* bfield, double bfactor, int bphase, const double* pre) {
  using C = KronCfg<N, NF>;
  KronArgs<N, NF> a;
  std::memset(&a, 0, sizeof(a));
  a.x = x;
  a.y = y;
  a.Q = Ntot / C::F;
  a.ntiles = (a.Q + C::QT - 1) / C::QT;
  a.bfield = bfield;
  a.bfactor = bfactor;
  a.bphase = bphase;
  a.pre = reinterpret_cast<const double2*>(pre);
  std::memcpy(a.E, E, sizeof(a.E));
  if constexpr (KRONOP_KR_PAIR && NF >= 2 && C::QT < 8 &&
                KronPairCfg<N, NF>::STAGES * KronPairCfg<N, NF>::PITCH * 8 + 64 <= 227 * 1024) {
    using PC = KronPairCfg<N, NF>;
    const size_t smem = static_cast<size_t>(PC::STAGES) * PC::PITCH * sizeof(double) +
                        PC::STAGES * sizeof(uint64_t);
    ensure_smem_attr(reinterpret_cast<const void*>(kron_rot_pair_kernel<N, NF, FOLD, BPH>), smem);
    const long long cap = device_sm_count();
    const long long grid = (a.ntiles + 1) / 2 < cap ? (a.ntiles + 1) / 2 : cap;
    kron_rot_pair_kernel<N, NF, FOLD, BPH>
        <<<static_cast<unsigned>(grid), PC::THREADS, smem, s>>>(a);
    KCUDA(cudaGetLastError());
    return;
  }
  const size_t smem = static_cast<size_t>(KRONOP_KR_STAGES) * C::STAGE * sizeof(double) +
                      KRONOP_KR_STAGES * sizeof(uint64_t) + KRONOP_KR_STAGES * sizeof(int);
  ensure_smem_attr(reinterpret_cast<const void*>(kron_rot_kernel<N, NF, FOLD, BPH>), smem);
  const long long cap = static_cast<long long>(device_sm_count()) * KRONOP_KR_CTAS;
  const long long grid = a.ntiles < cap ? a.ntiles : cap;
  kron_rot_kernel<N, NF, FOLD, BPH><<<static_cast<unsigned>(grid), C::THREADS, smem, s>>>(a);
  KCUDA(cudaGetLastError());
}

template <int N, bool FOLD>
void launch_kron_f(cudaStream_t s, int f, const double* x, double* y, long long Ntot,
                   const double* E, const double* bfield, double bfactor, int bphase,
                   const double* pre) {
  if (f == 1 && bphase)
    launch_kron<N, 1, FOLD, true>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
  else if (f == 1)
    launch_kron<N, 1, FOLD, false>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
  else if (f == 2 && bphase)
    launch_kron<N, 2, FOLD, true>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
  else if (f == 2)
    launch_kron<N, 2, FOLD, false>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
  else if (bphase)
    launch_kron<N, 3, FOLD, true>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
  else
    launch_kron<N, 3, FOLD, false>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
}

template <int N>
void launch_kron_n(cudaStream_t s, int f, bool fold, const double* x, double* y, long long Ntot,
                   const double* E, const double* bfield, double bfactor, int bphase,
                   const double* pre) {
  if (fold)
    launch_kron_f<N, true>(s, f, x, y, Ntot, E, bfield, bfactor, bphase, pre);
  else
    launch_kron_f<N, false>(s, f, x, y, Ntot, E, bfield, bfactor, bphase, pre);
}

// ------------------------------------------------------------------------------------------
// Extents 11..32 (config 5: 6D n = 29): the same rotating group launch on the FP64 tensor cores.
// Only the parity-folded form (every axis R-symmetric): per complex fiber the blocks
// Ae ((M+c) x (M+c)) and Ao (M x M) are real 2(M+c) x 2(M+c) and 2M x 2M matrices over the
// interleaved (re, im) components,
//   [Re -Im]
//   [Im  Re]  per complex entry,
// contracted with mma.sync.m8n8k4.f64 (DMMA): 8 fibers per warp step (A = fiber components from
// shared memory, B = matrix fragments staged once per CTA in fragment order), K = 2(M+c) / 2M
// padded to 4, N padded to 8. At n = 29 that is 8 x 4 + 7 x 4 = 60 DMMA per 8 fibers against
// 15 x 8 = 120 for the dense complex 58 x 58 matrix, and the same flops as ONE of the two real
// 29 x 29 passes of the transform form -- so the fold halves the tensor work of a propagate on
// top of the halved HBM traffic. Fold / unfold run in the warp that owns the fibers: s, d are
// formed in place in shared memory (s_k at position k, d_k at N-1-k), and the outputs
// y_i = a_i + b_i, y_{N-1-i} = a_i - b_i are formed from the accumulators, which hold a_i and b_i
// of the same (fiber, i, re/im) in the same lane.
#ifndef KRONOP_KD_STAGES
#define KRONOP_KD_STAGES 3
#endif
#ifndef KRONOP_KD_WARPS
#define KRONOP_KD_WARPS 16
#endif
// the CTA's warps form KD_GROUPS groups that take alternate tiles, each synchronising on its own
// named barrier, so one group's fold / unfold and barrier waits overlap the other's DMMA
#ifndef KRONOP_KD_GROUPS
#define KRONOP_KD_GROUPS 2
#endif
constexpr int KD_SMEM_BUDGET = 220 * 1024;

__host__ __device__ constexpr int kd_me(int n) { return n / 2 + n % 2; }
__host__ __device__ constexpr int kd_frag(int n) {  // fragment doubles per axis (Ae + Ao blocks)
  return ((2 * kd_me(n) + 3) / 4) * ((2 * kd_me(n) + 7) / 8) * 32 +
         ((2 * (n / 2) + 3) / 4) * ((2 * (n / 2) + 7) / 8) * 32;
}
__host__ __device__ constexpr int kd_qt(int n, int nf, int q) {
  return (q < 64 && KRONOP_KD_STAGES * 2 * (2 * q) * kr_pow(n, nf) * 8 + nf * kd_frag(n) * 8 + 256 <=
                        KD_SMEM_BUDGET)
             ? kd_qt(n, nf, 2 * q)
             : q;
}

template <int N, int NF>
struct KronDCfg {
  static constexpr int F = kr_pow(N, NF);
  static constexpr int QT = kd_qt(N, NF, 1);
  static constexpr int PL = F / N;
  static constexpr int FIB = QT * PL;
  static constexpr int M = N / 2, ME = kd_me(N);
  static constexpr int K4A = (2 * ME + 3) / 4, NTA = (2 * ME + 7) / 8;
  static constexpr int K4B = (2 * M + 3) / 4, NTB = (2 * M + 7) / 8;
  static constexpr int FRAG_A = K4A * NTA * 32, FRAG_B = K4B * NTB * 32;
  static constexpr int FRAG = FRAG_A + FRAG_B;
  static constexpr int STAGE = 2 * QT * F;  // doubles
  static constexpr int THREADS = 32 * KRONOP_KD_WARPS;
};

template <int N, int NF>
struct KronDArgs {
  const double* x;
  double* y;
  long long Q;
  long long ntiles;
  const double* bfield;
  double bfactor;
  int bphase;
  const double2* pre;  // as KronArgs::pre
  double2 E[NF][kd_me(N) * kd_me(N) + (N / 2) * (N / 2)];  // per axis [Ae | Ao], row-major
};

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// One warp step on 8 fibers (g = lane / 4) of one axis: fold in place, the two block products,
// unfold; in place (LAST = false) or to HBM with the group at the slow end (LAST = true).
#ifndef KRONOP_KD_G
#define KRONOP_KD_G 1  // fiber octets per warp step (B fragments reused across them)
#endif
template <int N, int NF, int J, bool LAST>
__device__ __forceinline__ void kd_step(const KronDArgs<N, NF>& A, double* buf, const double* frag,
                                        int f0, long long q0, int qv, int lane) {
  using C = KronDCfg<N, NF>;
  constexpr int G = KRONOP_KD_G;
  constexpr int FW = 8 * G;        // fibers per warp step
  constexpr int P = kr_pow(N, J);  // complex stride of the axis
  constexpr int H = C::F / (P * N);
  constexpr int M = C::M, ME = C::ME;
  const int g = lane >> 2, t = lane & 3;
  auto base_of = [&](int f, int& qi, int& lo) {  // complex offset of fiber f's element 0
    if constexpr (LAST) {
      qi = f % C::QT;
      lo = f / C::QT;
      return lo + qi * C::F;
    } else {
      lo = f % P;
      const int hi = f / P;
      qi = hi / H;
      return lo + (hi % H) * (P * N) + qi * C::F;
    }
  };
  double2* b2 = reinterpret_cast<double2*>(buf);
  // fold: (x_k, x_{N-1-k}) -> (s_k, d_k) for the warp's fibers; on the group's first axis the
  // preceding B phase (A.pre) is applied to the inputs first, the center element included
  const bool pre = J == 0 && A.pre != nullptr;
  constexpr int ITER = (FW * ME + 31) / 32;
  if (pre) {
    // the table entries of all the lane's items are loaded first (2 ITER loads in flight), then
    // the fold: one global-load latency per warp step instead of one per item
    double2 pu[ITER], pv[ITER];
#pragma unroll
    for (int j = 0; j < ITER; ++j) {
      const int it = lane + 32 * j, gg = it / ME, k = it - gg * ME;
      const int f = f0 + gg;
      pu[j] = pv[j] = make_double2(1.0, 0.0);
      if (it < FW * ME && f < C::FIB) {
        int qi, lo;
        const int fb = base_of(f, qi, lo);
        if (qi < qv) {
          // tile-local complex offset fb + k P is the global one minus q0 F (plane pitch F)
          const double2* ph = A.pre + q0 * C::F + fb;
          pu[j] = __ldg(ph + k * P);
          if (k < M) pv[j] = __ldg(ph + (N - 1 - k) * P);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < ITER; ++j) {
      const int it = lane + 32 * j, gg = it / ME, k = it - gg * ME;
      const int f = f0 + gg;
      if (it < FW * ME && f < C::FIB) {
        int qi, lo;
        double2* p = b2 + base_of(f, qi, lo);
        const double2 u = kr_rotate(p[k * P], pu[j]);
        if (k < M) {
          const double2 v = kr_rotate(p[(N - 1 - k) * P], pv[j]);
          p[k * P] = make_double2(u.x + v.x, u.y + v.y);
          p[(N - 1 - k) * P] = make_double2(u.x - v.x, u.y - v.y);
        } else {
          p[k * P] = u;  // center (odd N), phased
        }
      }
    }
  } else {
    // the lane's pairs are loaded in batches before they are folded (ILP over the
    // shared-memory latency; the loop form stalled on each LDS)
    constexpr int IT2 = (FW * M + 31) / 32;
    constexpr int BATCH = 2;  // pairs in flight per lane (more spilled at 128 registers)
#pragma unroll
    for (int j0 = 0; j0 < IT2; j0 += BATCH) {
      double2 uu[BATCH], vv[BATCH];
      int off[BATCH];
#pragma unroll
      for (int jj = 0; jj < BATCH; ++jj) {
        const int it = lane + 32 * (j0 + jj), gg = it / M, k = it - gg * M;
        const int f = f0 + gg;
        off[jj] = -1;
        if (j0 + jj < IT2 && it < FW * M && f < C::FIB) {
          int qi, lo;
          off[jj] = base_of(f, qi, lo) + k * P;
          uu[jj] = b2[off[jj]];
          vv[jj] = b2[off[jj] + (N - 1 - 2 * k) * P];
        }
      }
#pragma unroll
      for (int jj = 0; jj < BATCH; ++jj) {
        if (off[jj] >= 0) {
          const int k = (lane + 32 * (j0 + jj)) % M;
          b2[off[jj]] = make_double2(uu[jj].x + vv[jj].x, uu[jj].y + vv[jj].y);
          b2[off[jj] + (N - 1 - 2 * k) * P] =
              make_double2(uu[jj].x - vv[jj].x, uu[jj].y - vv[jj].y);
        }
      }
    }
  }
  __syncwarp();
  bool fok[G];
  int qis[G], los[G], fbs[G];
  const double* src[G];
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    const int f = f0 + 8 * gg + g;
    fok[gg] = f < C::FIB;
    fbs[gg] = base_of(fok[gg] ? f : f0, qis[gg], los[gg]);
    src[gg] = buf + 2 * fbs[gg];
  }
  double acc_a[G][C::NTA][2], acc_b[G][C::NTB][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
#pragma unroll
    for (int nt = 0; nt < C::NTA; ++nt) acc_a[gg][nt][0] = acc_a[gg][nt][1] = 0.0;
#pragma unroll
    for (int nt = 0; nt < C::NTB; ++nt) acc_b[gg][nt][0] = acc_b[gg][nt][1] = 0.0;
  }
  const double* fa = frag + lane;
#pragma unroll
  for (int kk = 0; kk < C::K4A; ++kk) {
    const int kap = 4 * kk + t, k = kap >> 1;
    double a[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) a[gg] = k < ME ? src[gg][2 * P * k + (kap & 1)] : 0.0;
#pragma unroll
    for (int nt = 0; nt < C::NTA; ++nt) {
      const double b = fa[(kk * C::NTA + nt) * 32];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) dmma884(acc_a[gg][nt], a[gg], b);
    }
  }
  const double* fbg = frag + C::FRAG_A + lane;
#pragma unroll
  for (int kk = 0; kk < C::K4B; ++kk) {
    const int kap = 4 * kk + t, k = kap >> 1;
    double a[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
      a[gg] = k < M ? src[gg][2 * P * (N - 1 - k) + (kap & 1)] : 0.0;
#pragma unroll
    for (int nt = 0; nt < C::NTB; ++nt) {
      const double b = fbg[(kk * C::NTB + nt) * 32];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) dmma884(acc_b[gg][nt], a[gg], b);
    }
  }
  __syncwarp();  // every lane has read its fibers before any output overwrites them
  double2* y2 = reinterpret_cast<double2*>(A.y);
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    if (!fok[gg]) continue;
    if constexpr (LAST) {
      if (qis[gg] >= qv) continue;
    }
    auto put = [&](int i, double re, double im) {
      if constexpr (LAST) {
        const long long oi = q0 + qis[gg] + A.Q * (los[gg] + static_cast<long long>(P) * i);
        if (A.bphase) {  // pointwise_phase (splitting.cpp:44-51), the operations of k_phase
          const double phase = A.bfield ? __dmul_rn(-A.bfactor, A.bfield[oi]) : -A.bfactor;
          double sn, cs;
          sincos(phase, &sn, &cs);
          const double r0 = re, i0 = im;
          re = __dsub_rn(__dmul_rn(r0, cs), __dmul_rn(i0, sn));
          im = __dadd_rn(__dmul_rn(r0, sn), __dmul_rn(i0, cs));
        }
        y2[oi] = make_double2(re, im);
      } else {
        b2[fbs[gg] + i * P] = make_double2(re, im);
      }
    };
#pragma unroll
    for (int nt = 0; nt < C::NTA; ++nt) {
      const int i = 4 * nt + t;
      if (i < M) {
        put(i, acc_a[gg][nt][0] + acc_b[gg][nt][0], acc_a[gg][nt][1] + acc_b[gg][nt][1]);
        put(N - 1 - i, acc_a[gg][nt][0] - acc_b[gg][nt][0], acc_a[gg][nt][1] - acc_b[gg][nt][1]);
      } else if (i < ME) {
        put(i, acc_a[gg][nt][0], acc_a[gg][nt][1]);
      }
    }
  }
}

template <int N, int NF, int J>
__device__ __forceinline__ void kd_axis(const KronDArgs<N, NF>& A, double* buf, const double* frag,
                                        long long q0, int qv, int gwarp, int lane, int grp) {
  using C = KronDCfg<N, NF>;
  constexpr bool LAST = J == NF - 1;
  constexpr int GW = KRONOP_KD_WARPS / KRONOP_KD_GROUPS;  // warps per group
  for (int f0 = gwarp * 8 * KRONOP_KD_G; f0 < C::FIB; f0 += 8 * KRONOP_KD_G * GW)
    kd_step<N, NF, J, LAST>(A, buf, frag + J * C::FRAG, f0, q0, qv, lane);
  if constexpr (!LAST) {
    if constexpr (KRONOP_KD_GROUPS == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(32 * GW) : "memory");
    kd_axis<N, NF, J + 1>(A, buf, frag, q0, qv, gwarp, lane, grp);
  }
}

template <int N, int NF>
__global__ void __launch_bounds__(32 * KRONOP_KD_WARPS, 1)
    kron_dmma_kernel(const __grid_constant__ KronDArgs<N, NF> A) {
  using C = KronDCfg<N, NF>;
  constexpr int STAGES = KRONOP_KD_STAGES;
  constexpr int WARPS = KRONOP_KD_WARPS;
  extern __shared__ __align__(128) double sm[];
  double* frag = sm + STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(frag + NF * C::FRAG);
  int* done = reinterpret_cast<int*>(full + STAGES);  // warps of the group finished with a stage
  // loads issued per stage: a group can reach the next use of a stage before the other group has
  // consumed and refilled it, when the mbarrier would still show the parity of the use before
  // (phases two apart look alike) -- so it first waits until the load it needs has been issued
  int* issued = done + STAGES;
  constexpr int GROUPS = KRONOP_KD_GROUPS, GW = WARPS / GROUPS;
  static_assert(WARPS % GROUPS == 0 && STAGES >= GROUPS, "warp groups");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / GW, gwarp = warp - grp * GW;
  // B fragments: frag[j][(kk NT + nt) 32 + lane] = Mreal(8 nt + lane / 4, 4 kk + lane % 4)
  for (int j = 0; j < NF; ++j)
    for (int e = tid; e < C::FRAG; e += C::THREADS) {
      const bool blk_a = e < C::FRAG_A;
      const int ee = blk_a ? e : e - C::FRAG_A;
      const int nts = blk_a ? C::NTA : C::NTB, dim = blk_a ? C::ME : C::M;
      const int ln = ee & 31, rest = ee >> 5, nt = rest % nts, kk = rest / nts;
      const int nu = 8 * nt + (ln >> 2), kap = 4 * kk + (ln & 3);
      const int i = nu >> 1, k = kap >> 1, co = nu & 1, ci = kap & 1;
      double v = 0.0;
      if (i < dim && k < dim) {
        const double2 z = blk_a ? A.E[j][i * C::ME + k] : A.E[j][C::ME * C::ME + i * C::M + k];
        v = co == ci ? z.x : (co == 0 ? -z.y : z.y);
      }
      frag[j * C::FRAG + e] = v;
    }
  const long long per = (A.ntiles + gridDim.x - 1) / gridDim.x;
  const long long t0 = blockIdx.x * per;
  const long long t1 = t0 + per < A.ntiles ? t0 + per : A.ntiles;
  auto issue = [&](long long tile, double* dst, uint64_t* bar) {
    const long long q0 = tile * C::QT;
    const int qv = static_cast<int>(A.Q - q0 < C::QT ? A.Q - q0 : C::QT);
    mbar_expect_tx(bar, static_cast<uint32_t>(qv) * C::F * 16u);
    bulk_load(dst, A.x + 2LL * C::F * q0, static_cast<uint32_t>(qv) * C::F * 16u, bar);
  };
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0;
      issued[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s)
      if (t0 + s < t1) {
        issue(t0 + s, sm + s * C::STAGE, &full[s]);
        issued[s] = 1;
      }
  for (int kt = 0;; ++kt) {
    const int it = kt * GROUPS + grp;  // this group's tiles
    const long long tile = t0 + it;
    if (tile >= t1) break;
    const int s = it % STAGES;
    double* buf = sm + s * C::STAGE;
    if constexpr (GROUPS > 1) {
      if (lane == 0)
        while (*reinterpret_cast<volatile int*>(&issued[s]) <= it / STAGES) {
        }
      __syncwarp();
    }
    mbar_wait(&full[s], (it / STAGES) & 1);
    const long long q0 = tile * C::QT;
    const int qv = static_cast<int>(A.Q - q0 < C::QT ? A.Q - q0 : C::QT);
    kd_axis<N, NF, 0>(A, buf, frag, q0, qv, gwarp, lane, grp);
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[s], 1) == GW - 1) {
        done[s] = 0;
        __threadfence_block();
        if (tile + STAGES < t1) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue(tile + STAGES, buf, &full[s]);
          __threadfence_block();
          atomicAdd(&issued[s], 1);
        }
      }
    }
  }
}

template <int N, int NF>
void launch_kron_dmma(cudaStream_t s, const double* x, double* y, long long Ntot, const double* E,
                      const double* bfield, double bfactor, int bphase, const double* pre) {
  using C = KronDCfg<N, NF>;
  KronDArgs<N, NF> a;
  std::memset(&a, 0, sizeof(a));
  a.x = x;
  a.y = y;
  a.Q = Ntot / C::F;
  a.ntiles = (a.Q + C::QT - 1) / C::QT;
  a.bfield = bfield;
  a.bfactor = bfactor;
  a.bphase = bphase;
  a.pre = reinterpret_cast<const double2*>(pre);
  // E: per axis the N x N slot of the caller's buffer holds [Ae | Ao] (kron_fold_blocks)
  constexpr int BLK = C::ME * C::ME + C::M * C::M;
  for (int j = 0; j < NF; ++j)
    std::memcpy(&a.E[j][0], E + static_cast<size_t>(j) * N * N * 2, BLK * sizeof(double2));
  const size_t smem = (static_cast<size_t>(KRONOP_KD_STAGES) * C::STAGE + NF * C::FRAG) *
                          sizeof(double) +
                      KRONOP_KD_STAGES * (sizeof(uint64_t) + 2 * sizeof(int));
  ensure_smem_attr(reinterpret_cast<const void*>(kron_dmma_kernel<N, NF>), smem);
  const long long cap = device_sm_count();
  const long long grid = a.ntiles < cap ? a.ntiles : cap;
  kron_dmma_kernel<N, NF><<<static_cast<unsigned>(grid), C::THREADS, smem, s>>>(a);
  KCUDA(cudaGetLastError());
}

template <int N>
void launch_kron_dmma_n(cudaStream_t s, int f, const double* x, double* y, long long Ntot,
                        const double* E, const double* bfield, double bfactor, int bphase,
                   const double* pre) {
  if (f == 1)
    launch_kron_dmma<N, 1>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
  else
    launch_kron_dmma<N, 2>(s, x, y, Ntot, E, bfield, bfactor, bphase, pre);
}

// ------------------------------------------------------------------------------------------
// Real fields, transform form (solve / apply / FullOperator apply of the small-extent operators,
// e.g. the config-5 ground states by inverse iteration): the same rotating group launch on DFMA
// with the REAL axis matrix (T^{-1} forward, T backward) as kernel parameters, one thread per
// real fiber, 8 planes per tile (64-byte output runs), 1 CTA x 3 stages over a contiguous tile
// range. Epilogues: the spectral divide / multiply on the last forward group (lambda summed in
// axis order from 0.0: the axes below the group per q, then the group axes -- direct_sum_grid
// tensor.cpp:196-209) and the V2 / sigma AXPY on the last backward group (operators.cpp:102),
// the operations and accumulation order of fused_rot.cu's DFMA path, so results are identical.
constexpr int KRE_STORE = 0, KRE_DIV = 1, KRE_MUL = 2, KRE_AXPY = 3;

template <int N, int NF>
struct KronRCfg {
  static constexpr int F = kr_pow(N, NF);
  static constexpr int QT = kr_qt(F, 1) * 2 > 256 ? 256 : kr_qt(F, 1) * 2;  // 8 B elements
  static constexpr int PL = F / N;
  static constexpr int FIB = QT * PL;
  static constexpr int THREADS = FIB >= 1024 ? 1024 : (kr_round32(FIB) < 64 ? 64 : kr_round32(FIB));
  // planes unpadded: a tile is ONE contiguous chunk (8-byte elements: a per-plane bulk copy of
  // an odd-extent plane would be neither a 16-byte multiple nor 16-byte aligned)
  static constexpr int PPR = F;
  static constexpr int STAGE = QT * PPR;
};

template <int N, int NF>
struct KronRArgs {
  const double* x;
  double* y;
  long long Q, ntiles;
  double shift, sigma;
  const double* diag;  // AXPY: V2 (null = none), original layout
  const double* u;     // AXPY: the operator's input, original layout
  const double* lam_g[3];
  int nq;
  long long qext[KRONOP_MAX_DIM];
  const double* lam_q[KRONOP_MAX_DIM];
  double M[NF][N][N];  // M_j(i, k): output i, input k
};

template <int N, int NF, int J>
__device__ __forceinline__ void kre_contract(const KronRArgs<N, NF>& A, const double (&x)[N],
                                             double (&o)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) o[i] = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = fma(A.M[J][i][k], x[k], o[i]);
}

template <int N, int NF, int J>
__device__ __forceinline__ void kre_axis(const KronRArgs<N, NF>& A, double* buf, int tid) {
  using C = KronRCfg<N, NF>;
  constexpr int P = kr_pow(N, J);
  constexpr int H = C::F / (P * N);
#pragma unroll 1
  for (int f = tid; f < C::FIB; f += C::THREADS) {
    const int lo = f % P, hi = f / P;
    const int hg = hi % H, qi = hi / H;
    double* p = buf + lo + hg * (P * N) + qi * C::PPR;
    double x[N], o[N];
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = p[k * P];
    kre_contract<N, NF, J>(A, x, o);
#pragma unroll
    for (int i = 0; i < N; ++i) p[i * P] = o[i];
  }
}

template <int N, int NF, int J>
__device__ __forceinline__ void kre_inplace(const KronRArgs<N, NF>& A, double* buf, int tid) {
  if constexpr (J < NF - 1) {
    kre_axis<N, NF, J>(A, buf, tid);
    __syncthreads();
    kre_inplace<N, NF, J + 1>(A, buf, tid);
  }
}

template <int N, int NF, int EPI>
__device__ __forceinline__ void kre_last(const KronRArgs<N, NF>& A, const double* buf,
                                         const double* lam_low, long long q0, int qv, int tid) {
  using C = KronRCfg<N, NF>;
  constexpr int P = C::PL;
#pragma unroll 1
  for (int f = tid; f < C::FIB; f += C::THREADS) {
    const int qi = f % C::QT, lo = f / C::QT;
    if (qi >= qv) continue;
    const double* p = buf + lo + qi * C::PPR;
    double x[N], o[N];
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = p[k * P];
    kre_contract<N, NF, NF - 1>(A, x, o);
    const long long ob = q0 + qi + A.Q * lo;
    double lam_lo_g = 0.0;
    if constexpr (EPI == KRE_DIV || EPI == KRE_MUL) {
      // the group axes below the last one, in axis order after the axes below the group
      lam_lo_g = lam_low[qi];
      int r = lo;
#pragma unroll
      for (int j = 0; j < NF - 1; ++j) {
        lam_lo_g = __dadd_rn(lam_lo_g, A.lam_g[j][r % N]);
        r /= N;
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const long long oi = ob + A.Q * P * i;
      double v = o[i];
      if constexpr (EPI == KRE_DIV || EPI == KRE_MUL) {
        const double ls = __dsub_rn(__dadd_rn(lam_lo_g, A.lam_g[NF - 1][i]), A.shift);
        v = EPI == KRE_MUL ? __dmul_rn(v, ls) : __ddiv_rn(v, ls);
      } else if constexpr (EPI == KRE_AXPY) {
        const double uu = A.u[oi];
        if (A.diag) v = __dadd_rn(v, __dmul_rn(A.diag[oi], uu));
        if (A.sigma != 0.0) v = __dsub_rn(v, __dmul_rn(A.sigma, uu));
      }
      A.y[oi] = v;
    }
  }
}

template <int N, int NF, int EPI>
__global__ void __launch_bounds__(KronRCfg<N, NF>::THREADS, 1)
    kron_real_kernel(const __grid_constant__ KronRArgs<N, NF> A) {
  using C = KronRCfg<N, NF>;
  constexpr int STAGES = 3;
  constexpr int WARPS = C::THREADS / 32;
  extern __shared__ __align__(128) double sm[];
  double* lam_low2 = sm + STAGES * C::STAGE;  // 2 x QT: lambda of the axes below, per tile
  uint64_t* full = reinterpret_cast<uint64_t*>(lam_low2 + 2 * C::QT);
  int* done = reinterpret_cast<int*>(full + STAGES);
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const long long per = (A.ntiles + gridDim.x - 1) / gridDim.x;
  const long long t0 = blockIdx.x * per;
  const long long t1 = t0 + per < A.ntiles ? t0 + per : A.ntiles;
  auto issue = [&](long long tile, double* dst, uint64_t* bar) {
    const long long q0 = tile * C::QT;
    const int qv = static_cast<int>(A.Q - q0 < C::QT ? A.Q - q0 : C::QT);
    // one bulk copy of an even number of doubles (16-byte multiple; the tile start is 16-byte
    // aligned since QT F is even or the tile is the first); an odd last element (partial last
    // tile) through the generic proxy before the arrive
    const uint32_t doubles = static_cast<uint32_t>(qv) * C::F;
    const double* src = A.x + static_cast<long long>(C::F) * q0;
    if (doubles & 1u) dst[doubles - 1] = src[doubles - 1];
    const uint32_t bulk = (doubles & ~1u) * 8u;
    mbar_expect_tx(bar, bulk);
    if (bulk) bulk_load(dst, src, bulk, bar);
  };
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s)
      if (t0 + s < t1) issue(t0 + s, sm + s * C::STAGE, &full[s]);
  for (int it = 0;; ++it) {
    const long long tile = t0 + it;
    if (tile >= t1) break;
    const int s = it % STAGES;
    double* buf = sm + s * C::STAGE;
    const long long q0 = tile * C::QT;
    const int qv = static_cast<int>(A.Q - q0 < C::QT ? A.Q - q0 : C::QT);
    double* lam_low = lam_low2 + (it & 1) * C::QT;
    if constexpr (EPI == KRE_DIV || EPI == KRE_MUL) {
      if (tid < qv) {  // lambda of the axes below the group, axis order from 0.0
        long long q = q0 + tid;
        double lam = 0.0;
        for (int j = 0; j < A.nq; ++j) {
          const long long e = A.qext[j];
          const long long idx = q % e;
          q /= e;
          lam = __dadd_rn(lam, A.lam_q[j][idx]);
        }
        lam_low[tid] = lam;
      }
    }
    mbar_wait(&full[s], (it / STAGES) & 1);
    kre_inplace<N, NF, 0>(A, buf, tid);
    if constexpr (NF == 1 && (EPI == KRE_DIV || EPI == KRE_MUL)) __syncthreads();  // lam_low
    kre_last<N, NF, EPI>(A, buf, lam_low, q0, qv, tid);
    const long long next = tile + STAGES;
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[s], 1) == WARPS - 1) {
        done[s] = 0;
        __threadfence_block();
        if (next < t1) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue(next, buf, &full[s]);
        }
      }
    }
  }
}

template <int N, int NF, int EPI>
void launch_kron_real(cudaStream_t s, const KronRealLaunch& L) {
  using C = KronRCfg<N, NF>;
  KronRArgs<N, NF> a;
  std::memset(&a, 0, sizeof(a));
  a.x = L.x;
  a.y = L.y;
  a.Q = L.Ntot / C::F;
  a.ntiles = (a.Q + C::QT - 1) / C::QT;
  a.shift = L.shift;
  a.sigma = L.sigma;
  a.diag = L.diag;
  a.u = L.u;
  for (int j = 0; j < NF; ++j) a.lam_g[j] = L.lam_g[j];
  a.nq = L.nq;
  for (int j = 0; j < L.nq; ++j) {
    a.qext[j] = L.qext[j];
    a.lam_q[j] = L.lam_q[j];
  }
  for (int j = 0; j < NF; ++j)
    for (int i = 0; i < N; ++i)
      for (int k = 0; k < N; ++k) a.M[j][i][k] = L.M[(j * N + i) * N + k];
  const size_t smem = (3 * static_cast<size_t>(C::STAGE) + 2 * C::QT) * sizeof(double) +
                      3 * (sizeof(uint64_t) + sizeof(int));
  ensure_smem_attr(reinterpret_cast<const void*>(kron_real_kernel<N, NF, EPI>), smem);
  const long long cap = device_sm_count();
  const long long grid = a.ntiles < cap ? a.ntiles : cap;
  kron_real_kernel<N, NF, EPI><<<static_cast<unsigned>(grid), C::THREADS, smem, s>>>(a);
  KCUDA(cudaGetLastError());
}

template <int N, int NF>
void launch_kron_real_e(cudaStream_t s, const KronRealLaunch& L) {
  switch (L.epi) {
    case KRE_DIV: launch_kron_real<N, NF, KRE_DIV>(s, L); break;
    case KRE_MUL: launch_kron_real<N, NF, KRE_MUL>(s, L); break;
    case KRE_AXPY: launch_kron_real<N, NF, KRE_AXPY>(s, L); break;
    default: launch_kron_real<N, NF, KRE_STORE>(s, L); break;
  }
}

template <int N>
void launch_kron_real_n(cudaStream_t s, const KronRealLaunch& L) {
  if (L.f == 1)
    launch_kron_real_e<N, 1>(s, L);
  else if (L.f == 2)
    launch_kron_real_e<N, 2>(s, L);
  else
    launch_kron_real_e<N, 3>(s, L);
}

}  // namespace

bool kron_group_supported(int n, int f) {
  return (n >= 2 && n <= KR_MAXN && f >= 1 && f <= 3) ||
         (n > KR_MAXN && n <= KD_MAXN && f >= 1 && f <= 2);
}
bool kron_group_needs_fold(int n) { return n > KR_MAXN; }

bool kron_real_supported(int n, int f) { return n >= 2 && n <= KR_MAXN && f >= 1 && f <= 3; }

void launch_kron_real_group(cudaStream_t s, const KronRealLaunch& L) {
  param_check(kron_real_supported(L.n, L.f), "small-extent real transform: unsupported group");
  param_check((reinterpret_cast<uintptr_t>(L.x) & 15u) == 0,
              "small-extent real transform: input must be 16-byte aligned");
  switch (L.n) {
    case 2: launch_kron_real_n<2>(s, L); break;
    case 3: launch_kron_real_n<3>(s, L); break;
    case 4: launch_kron_real_n<4>(s, L); break;
    case 5: launch_kron_real_n<5>(s, L); break;
    case 6: launch_kron_real_n<6>(s, L); break;
    case 7: launch_kron_real_n<7>(s, L); break;
    case 8: launch_kron_real_n<8>(s, L); break;
    case 9: launch_kron_real_n<9>(s, L); break;
    default: launch_kron_real_n<10>(s, L); break;
  }
}

void launch_kron_group(cudaStream_t s, const double* x, double* y, int n, int f, bool fold,
                       long long Ntot, const double* E, const double* bfield, double bfactor,
                       int bphase, const double* pre) {
  param_check(kron_group_supported(n, f), "kron propagate: unsupported group");
  param_check(fold || n <= KR_MAXN, "kron propagate: extents > 10 need parity-symmetric axes");
  param_check((reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (reinterpret_cast<uintptr_t>(y) & 15u) == 0,
              "kron propagate: fields must be 16-byte aligned");
  switch (n) {
    case 2: launch_kron_n<2>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 3: launch_kron_n<3>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 4: launch_kron_n<4>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 5: launch_kron_n<5>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 6: launch_kron_n<6>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 7: launch_kron_n<7>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 8: launch_kron_n<8>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 9: launch_kron_n<9>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    case 10: launch_kron_n<10>(s, f, fold, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
#define KD_CASE(NN) \
  case NN: launch_kron_dmma_n<NN>(s, f, x, y, Ntot, E, bfield, bfactor, bphase, pre); break;
    KD_CASE(11) KD_CASE(12) KD_CASE(13) KD_CASE(14) KD_CASE(15) KD_CASE(16) KD_CASE(17)
    KD_CASE(18) KD_CASE(19) KD_CASE(20) KD_CASE(21) KD_CASE(22) KD_CASE(23) KD_CASE(24)
    KD_CASE(25) KD_CASE(26) KD_CASE(27) KD_CASE(28) KD_CASE(29) KD_CASE(30) KD_CASE(31)
    KD_CASE(32)
#undef KD_CASE
    default: break;
  }
}

}  // namespace kronop_dev
