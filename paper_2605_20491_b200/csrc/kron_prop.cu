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
//   2-stage ring; two CTAs per SM.
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

#ifndef KRONOP_KR_CTAS
#define KRONOP_KR_CTAS 2
#endif
#ifndef KRONOP_KR_STAGES
#define KRONOP_KR_STAGES 2
#endif
constexpr int KR_TILE_MAX = 6144;  // complex doubles x 2 per stage before padding (48 KB)
constexpr int KR_MAXN = 10;

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
  static constexpr int THREADS = FIB >= 512 ? 512 : (kr_round32(FIB) < 64 ? 64 : kr_round32(FIB));
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
  double E[NF][N][N][2];  // E_j(i, k) = (re, im): output i, input k
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

// out_i = sum_k E_J(i, k) x_k, complex; E from the parameter space (constant-bank operands).
// Each of the 2N accumulators is one fma chain in k order.
template <int N, int NF, int J>
__device__ __forceinline__ void kr_contract(const KronArgs<N, NF>& A, const double2 (&x)[N],
                                            double (&re)[N], double (&im)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    re[i] = 0.0;
    im[i] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double er = A.E[J][i][k][0], ei = A.E[J][i][k][1];
      re[i] = fma(er, x[k].x, re[i]);
      re[i] = fma(-ei, x[k].y, re[i]);
      im[i] = fma(er, x[k].y, im[i]);
      im[i] = fma(ei, x[k].x, im[i]);
    }
}

// Group axis J < NF - 1, in place: fibers (lo < P, hg < H, qi) at lo + P N hg + PPC qi.
template <int N, int NF, int J>
__device__ __forceinline__ void kr_axis(const KronArgs<N, NF>& A, double* buf, int tid) {
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
    double re[N], im[N];
    kr_contract<N, NF, J>(A, x, re, im);
#pragma unroll
    for (int i = 0; i < N; ++i) p[i * P] = make_double2(re[i], im[i]);
  }
}

// Last group axis (J = NF - 1, stride PL), q fastest across the lanes; outputs go to HBM with the
// group at the slowest end: complex index (q0 + qi) + Q (lo + PL i).
template <int N, int NF>
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
    double re[N], im[N];
    kr_contract<N, NF, NF - 1>(A, x, re, im);
    const long long o = q0 + qi + A.Q * lo;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const long long oi = o + A.Q * P * i;
      double vr = re[i], vi = im[i];
      if (A.bphase) {  // pointwise_phase (splitting.cpp:44-51), the operations of k_phase
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

template <int N, int NF, int J>
__device__ __forceinline__ void kr_inplace_axes(const KronArgs<N, NF>& A, double* buf, int tid) {
  if constexpr (J < NF - 1) {
    kr_axis<N, NF, J>(A, buf, tid);
    __syncthreads();
    kr_inplace_axes<N, NF, J + 1>(A, buf, tid);
  }
}

template <int N, int NF>
__global__ void __launch_bounds__(KronCfg<N, NF>::THREADS, KRONOP_KR_CTAS)
    kron_rot_kernel(const __grid_constant__ KronArgs<N, NF> A) {
  using C = KronCfg<N, NF>;
  constexpr int STAGES = KRONOP_KR_STAGES;
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * C::STAGE);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) {
      const long long tile = blockIdx.x + static_cast<long long>(s) * gridDim.x;
      if (tile < A.ntiles) kr_issue(A, tile, sm + s * C::STAGE, &full[s]);
    }
  for (int it = 0;; ++it) {
    const long long tile = blockIdx.x + static_cast<long long>(it) * gridDim.x;
    if (tile >= A.ntiles) break;
    const int s = it % STAGES;
    double* buf = sm + s * C::STAGE;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const long long q0 = tile * C::QT;
    const int qv = static_cast<int>(A.Q - q0 < C::QT ? A.Q - q0 : C::QT);
    kr_inplace_axes<N, NF, 0>(A, buf, tid);
    kr_last<N, NF>(A, buf, q0, qv, tid);
    __syncthreads();  // every thread is done with the stage (generic proxy) before the refill
    if (tid == 0) {
      const long long next = tile + static_cast<long long>(STAGES) * gridDim.x;
      if (next < A.ntiles) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        kr_issue(A, next, buf, &full[s]);
      }
    }
  }
}

template <int N, int NF>
void launch_kron(cudaStream_t s, const double* x, double* y, long long Ntot, const double* E,
                 const double* bfield, double bfactor, int bphase) {
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
  std::memcpy(a.E, E, sizeof(a.E));
  const size_t smem = static_cast<size_t>(KRONOP_KR_STAGES) * C::STAGE * sizeof(double) +
                      KRONOP_KR_STAGES * sizeof(uint64_t);
  ensure_smem_attr(reinterpret_cast<const void*>(kron_rot_kernel<N, NF>), smem);
  const long long cap = static_cast<long long>(device_sm_count()) * KRONOP_KR_CTAS;
  const long long grid = a.ntiles < cap ? a.ntiles : cap;
  kron_rot_kernel<N, NF><<<static_cast<unsigned>(grid), C::THREADS, smem, s>>>(a);
  KCUDA(cudaGetLastError());
}

template <int N>
void launch_kron_n(cudaStream_t s, int f, const double* x, double* y, long long Ntot,
                   const double* E, const double* bfield, double bfactor, int bphase) {
  if (f == 1)
    launch_kron<N, 1>(s, x, y, Ntot, E, bfield, bfactor, bphase);
  else if (f == 2)
    launch_kron<N, 2>(s, x, y, Ntot, E, bfield, bfactor, bphase);
  else
    launch_kron<N, 3>(s, x, y, Ntot, E, bfield, bfactor, bphase);
}

}  // namespace

bool kron_group_supported(int n, int f) { return n >= 2 && n <= KR_MAXN && f >= 1 && f <= 3; }

void launch_kron_group(cudaStream_t s, const double* x, double* y, int n, int f, long long Ntot,
                       const double* E, const double* bfield, double bfactor, int bphase) {
  param_check(kron_group_supported(n, f), "kron propagate: unsupported group");
  param_check((reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (reinterpret_cast<uintptr_t>(y) & 15u) == 0,
              "kron propagate: fields must be 16-byte aligned");
  switch (n) {
    case 2: launch_kron_n<2>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    case 3: launch_kron_n<3>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    case 4: launch_kron_n<4>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    case 5: launch_kron_n<5>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    case 6: launch_kron_n<6>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    case 7: launch_kron_n<7>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    case 8: launch_kron_n<8>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    case 9: launch_kron_n<9>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
    default: launch_kron_n<10>(s, f, x, y, Ntot, E, bfield, bfactor, bphase); break;
  }
}

}  // namespace kronop_dev
