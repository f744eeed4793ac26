// Small-extent, high-dimensional transforms with a rotating layout (BASELINE config 5: 6D n = 29,
// 9D n = 9; every operator whose axes all have n <= 32).
//
// A group of f <= 3 consecutive axes (fused extent F = n_0 ... n_{f-1} <= 1024) is contracted per
// HBM round trip, and the group's axes move to the SLOWEST end of the layout on the way out:
//   in : [c][g_0 .. g_{f-1}][rest]      (c = re/im, extent C = 2 for complex, 1 for real)
//   out: [c][rest][g_0 .. g_{f-1}]
// so the next group's axes are again the fastest after c. After all groups the layout is back in
// the original order (a full rotation), which is why a transform (forward groups, spectral
// epilogue, backward groups) ends in the caller's layout. What this buys over contracting a group
// in place (an earlier design, measured 149 / 64 ms for 6D / 9D, since removed): every tile a CTA reads is ONE contiguous chunk of the field
// ([Qt q][F][C], moved by a single cp.async.bulk into shared memory), and every tile it writes is
// F runs of C * Qt contiguous doubles (64 B or more) stored straight from the DMMA accumulators of
// the group's last axis - no strided 32-byte rows and no second shared-memory pass.
//
// Per CTA (persistent, one per SM, 16 warps): the group's matrices are staged once, tiles stream
// through a 3-deep ring of shared-memory stages (mbarrier complete_tx), the first f-1 axes are
// applied in place on the FP64 tensor cores (8 fibers x 4 k per mma.sync.m8n8k4, matrix fragments
// in registers), the last axis writes its outputs to global memory with the fused epilogue
// (spectral multiply / divide / phase on the last forward group, V2 / sigma AXPY on the last
// backward group).
//
// Same contraction as proj/src/tensor.cpp:105-145 per axis and the same epilogues as
// operators.cpp:36,57,68-71,102 (eigenvalues summed in axis order from 0.0, direct_sum_grid
// tensor.cpp:196-209).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kronop_internal.cuh"

namespace kronop_dev {

namespace {

// threads per CTA: 16 warps for the DMMA path (latency hiding), 8 for the DFMA path (the n x n
// matrix lives in registers: 2 n^2 + O(n) registers per thread)
template <int DN>
// (n = 9: 7 warps, so the 648 fibers an axis of a 9D tile holds split into 3 nearly full rounds)
__host__ __device__ constexpr int rt_threads_default() { return DN == 9 ? 224 : DN > 0 ? 256 : 512; }
constexpr int RT_MAXF = 3;
constexpr int RT_STAGES = 3;
constexpr int RT_TILE = 8192;  // doubles per stage (64 KB)
// Compile-time knobs of the DFMA path (n <= 10), for A/B builds (tools/build_variant.py):
// threads per CTA (0 = rt_threads_default), co-resident CTAs per SM, stages, doubles per stage.
// Default: two 4-warp CTAs per SM with 2 stages of 48 KB each (the n x n matrix in registers
// caps a CTA at ~224 registers per thread, so two CTAs is the most the register file holds; one
// CTA's store phase overlaps the other's contraction). Measured (tools/microbench/rot_bench.py,
// profiles/r02_rot_variants.json): 9D n = 9 propagate 27.15 -> 25.73 ms, 9D solve 17.3 -> 15.6
// ms vs one 7-warp CTA with 3 x 64 KB stages; 96-thread CTAs and 4 stages were no better.
#ifndef KRONOP_DF_THREADS
#define KRONOP_DF_THREADS 128
#endif
#ifndef KRONOP_DF_CTAS
#define KRONOP_DF_CTAS 2
#endif
#ifndef KRONOP_DF_STAGES
#define KRONOP_DF_STAGES 2
#endif
#ifndef KRONOP_DF_TILE
#define KRONOP_DF_TILE 6144
#endif
// the same knobs for the DMMA path (n > 10), for A/B builds
#ifndef KRONOP_DM_THREADS
#define KRONOP_DM_THREADS 512
#endif
#ifndef KRONOP_DM_CTAS
#define KRONOP_DM_CTAS 1
#endif
#ifndef KRONOP_DM_STAGES
#define KRONOP_DM_STAGES 3
#endif
#ifndef KRONOP_DM_TILE
#define KRONOP_DM_TILE 8192
#endif
// DMMA path: the CTA's warps form KRONOP_DM_GROUPS independent groups that take alternate tiles,
// each synchronising on its own named barrier, so one group's store phase and barrier waits
// overlap the other's contraction (two CTAs per SM do not fit the shared memory)
#ifndef KRONOP_DM_GROUPS
#define KRONOP_DM_GROUPS 2
#endif
template <int DN>
__host__ __device__ constexpr int rt_threads() {
  return DN > 0 ? (KRONOP_DF_THREADS > 0 ? KRONOP_DF_THREADS : rt_threads_default<DN>())
                : KRONOP_DM_THREADS;
}
template <int DN>
__host__ __device__ constexpr int rt_ctas() { return DN > 0 ? KRONOP_DF_CTAS : KRONOP_DM_CTAS; }
template <int DN>
__host__ __device__ constexpr int rt_stages() {
  return DN > 0 ? KRONOP_DF_STAGES : KRONOP_DM_STAGES;
}
template <int DN>
__host__ __device__ constexpr int rt_tile() { return DN > 0 ? KRONOP_DF_TILE : KRONOP_DM_TILE; }

struct RotArgs {
  const double* x;
  double* y;
  int C;                 // 1 real, 2 complex
  int f;                 // axes in the group
  int n[RT_MAXF];        // group extents, fastest first
  int F;                 // fused extent
  long long Q;           // N / F (count of the other axes' multi-indices)
  int Qt;                // q per tile; C * Qt = CQt is a power of two >= 8
  int lcq;               // log2(CQt)
  long long ntiles;
  const double* a[RT_MAXF];
  int lda[RT_MAXF];
  int kpat[RT_MAXF];     // k permutation per axis (kidx)
  int uniform;           // every group axis has the same matrix
  float inv_n[RT_MAXF];  // 1 / n_j (fast_div)
  int epi;               // EPI_STORE / EPI_SPEC_* / EPI_AXPY_DIAG
  double shift, dt, sigma;
  const double* diag;
  const double* u;
  const double* lam_g[RT_MAXF];  // eigenvalues of the group axes (spectral)
  int nq;                        // axes below the group in original order (spectral lambda_low)
  long long qext[KRONOP_MAX_DIM];
  const double* lam_q[KRONOP_MAX_DIM];
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

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// exact q = v / S for v < 2^22 through a float reciprocal
__device__ __forceinline__ int fast_div(int v, int S, float invS) {
  int o = __float2int_rz(static_cast<float>(v) * invS);
  o -= (o * S > v);
  o += ((o + 1) * S <= v);
  return o;
}

// Issue the bulk load of tile `tile` into `dst` (thread 0 only).
__device__ __forceinline__ void issue_tile(const RotArgs& A, long long tile, double* dst,
                                           uint64_t* bar) {
  const long long q0 = tile * A.Qt;
  const long long qv = A.Q - q0 < A.Qt ? A.Q - q0 : A.Qt;
  const uint32_t doubles = static_cast<uint32_t>(qv * A.C * A.F);
  const uint32_t bulk = (doubles & ~1u) * 8u;  // multiple of 16 B
  const double* src = A.x + q0 * A.C * A.F;
  if (doubles & 1u) dst[doubles - 1] = src[doubles - 1];  // odd tail, generic proxy (before arrive)
  mbar_expect_tx(bar, bulk);
  if (bulk) bulk_load(dst, src, bulk, bar);
}

// k-index permutations of the DMMA contraction (both operands use the same one, so any bijection
// of k is valid): pattern 0 = 4 kk + t; pattern 1 = 8 (kk/2) + 2 t + kk%2 (K4 even), which makes
// the 4 t-lanes of a fragment load hit strides 0, 2S, 4S, 6S - conflict free for the 6D/9D
// strides (chosen per axis on the host by counting bank wavefronts).
__device__ __forceinline__ int kidx(int pat, int t, int kk) {
  return pat == 0 ? 4 * kk + t : 8 * (kk >> 1) + 2 * t + (kk & 1);
}

// In-place contraction of one group axis on the staged tile: fibers = all (lo < S, hi) with the
// axis at stride S; each warp takes 8 x G fibers per step on DMMA (k = fiber element, n = output
// index). The axis' B fragments come from shared memory (fragment order, conflict free) once per
// tile, so only one axis' matrix occupies registers.
template <int K4, int NT, int G, int THREADS>
__device__ __forceinline__ void axis_inplace(double* tile, const double* frag, const int (&koff)[K4],
                                             int m, int S, int nfib, int warp, int lane) {
  const int t = lane & 3, g = lane >> 2;
  const double* fl = frag + lane;
  const float invS = 1.0f / static_cast<float>(S);
  const int Sm = S * m;
  for (int f0 = warp * 8 * G; f0 < nfib; f0 += 8 * G * (THREADS / 32)) {
    const double* src[G];
    bool fok[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const int fib = f0 + 8 * gg + g;
      fok[gg] = fib < nfib;
      const int fb = fok[gg] ? fib : f0;
      src[gg] = tile + fb + fast_div(fb, S, invS) * (Sm - S);
    }
    double acc[G][NT][2];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[gg][nt][0] = acc[gg][nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < K4; ++kk) {
      double a[G], b[NT];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) a[gg] = src[gg][koff[kk]];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = fl[(kk * NT + nt) * 32];  // conflict free
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int gg = 0; gg < G; ++gg) dmma884(acc[gg][nt], a[gg], b[nt]);
    }
    __syncwarp();
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      double* dst = const_cast<double*>(src[gg]);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int n = 8 * nt + 2 * t + v;
          if (fok[gg] && n < m) dst[n * S] = acc[gg][nt][v];
        }
    }
  }
}

// Small extents (n <= 10): the DMMA tiles would be mostly padding (n = 9 fills 42% of a K12 x N16
// tile), so each thread contracts whole fibers with DFMA: it reads its n inputs, forms the n
// outputs against the matrix (shared memory, row-major with an even row pitch, read as 16-byte
// broadcasts) and writes them back in place.
template <int N>
__device__ __forceinline__ void load_matrix(double (&M)[N][N], const double* mat) {
  constexpr int NP = (N + 1) & ~1;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int k = 0; k < N; ++k) M[i][k] = mat[i * NP + k];
}

template <int N, int THREADS>
__device__ __forceinline__ void axis_dfma(double* tile, const double (&M)[N][N], int S, int nfib,
                                          int tid) {
  const float invS = 1.0f / static_cast<float>(S);
  const int Sm = S * N;
  for (int f = tid; f < nfib; f += THREADS) {
    double* p = tile + f + fast_div(f, S, invS) * (Sm - S);
    double x[N];
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = p[k * S];
    // k-outer: N independent accumulation chains advance together (ILP N); each output is still
    // fma(M[i][N-1], x[N-1], ... fma(M[i][0], x[0], 0)) in k order
    double acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = fma(M[i][k], x[k], acc[i]);
#pragma unroll
    for (int i = 0; i < N; ++i) p[i * S] = acc[i];  // in place: the inputs are in registers
  }
}

// The same with the stride and fiber count known at compile time (isotropic three-axis group,
// C known, C Qt = 8): the fiber -> address map is a division by a constant and the strided
// loads / stores take immediate offsets (the runtime version spent ~25% of its issue slots on
// the float-reciprocal division and address arithmetic, profiles/r02_rot9.json).
template <int N, int THREADS, int S, int NFIB>
__device__ __forceinline__ void axis_dfma_ct(double* tile, const double (&M)[N][N], int tid) {
  constexpr int Sm = S * N;
#pragma unroll 1
  for (int f = tid; f < NFIB; f += THREADS) {
    double* p = tile + f + (f / S) * (Sm - S);
    double x[N];
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = p[k * S];
    double acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = fma(M[i][k], x[k], acc[i]);
#pragma unroll
    for (int i = 0; i < N; ++i) p[i * S] = acc[i];
  }
}

// lambda of one output: the axes below the group (lam_low, per q), then the group axes in order
// (axis order from 0.0, direct_sum_grid tensor.cpp:196-209).
template <int NF>
__device__ __forceinline__ double group_lambda(const RotArgs& A, double lam_low, int glin) {
  double lam = lam_low;
#pragma unroll
  for (int j = 0; j < NF; ++j) {
    int ij = glin;
    if (j + 1 < NF) {
      const int q = fast_div(glin, A.n[j], A.inv_n[j]);
      ij = glin - q * A.n[j];
      glin = q;
    }
    lam = __dadd_rn(lam, A.lam_g[j][ij]);
  }
  return lam;
}

// Store the contracted tile with the group moved to the slow end: element (c, g, q0 + qi) goes
// to c + C (q0 + qi) + C Q g. Threads walk (qi fastest, then g) so each group of Qt threads
// writes one run of C * Qt contiguous doubles; complex fields move (re, im) pairs as 16-byte
// units (one sincos per pair for the phase). Epilogues: spectral (last forward group) or the
// V2 / sigma AXPY (last backward group).
template <int NF, int THREADS>
__device__ __forceinline__ void store_tile(const RotArgs& A, const double* tile, long long q0,
                                           int qv, const double* lam_low, int tid) {
  const int C = A.C, F = A.F, Qt = A.Qt;
  const long long CQ = static_cast<long long>(C) * A.Q;
  const int units = Qt * F;  // (re, im) pairs or real scalars
  const bool spectral = A.epi == EPI_SPEC_MUL || A.epi == EPI_SPEC_DIV || A.epi == EPI_SPEC_PHASE;
  const int lq = __ffs(Qt) - 1;  // Qt is a power of two
#pragma unroll 4
  for (int u = tid; u < units; u += THREADS) {
    const int g = u >> lq;
    const int qi = u & (Qt - 1);
    if (qi >= qv) continue;  // partial last tile only
    const long long gi = static_cast<long long>(C) * (q0 + qi) + CQ * g;
    const double* sp = tile + C * (g + F * qi);
    if (C == 2) {
      double2 v = *reinterpret_cast<const double2*>(sp);
      if (spectral) {
        const double lam = group_lambda<NF>(A, lam_low[qi], g);
        const double ls = __dsub_rn(lam, A.shift);
        if (A.epi == EPI_SPEC_MUL) {
          v.x = __dmul_rn(v.x, ls);
          v.y = __dmul_rn(v.y, ls);
        } else if (A.epi == EPI_SPEC_DIV) {
          v.x = __ddiv_rn(v.x, ls);
          v.y = __ddiv_rn(v.y, ls);
        } else {  // operators.cpp:68-71: psi * complex(cos, sin) of -(lambda - shift) dt
          const double phase = __dmul_rn(-ls, A.dt);
          double sn, cs;
          sincos(phase, &sn, &cs);
          const double re = v.x, im = v.y;
          v.x = __dsub_rn(__dmul_rn(re, cs), __dmul_rn(im, sn));
          v.y = __dadd_rn(__dmul_rn(re, sn), __dmul_rn(im, cs));
        }
      } else if (A.epi == EPI_BPHASE) {  // pointwise_phase (splitting.cpp:44-51), as k_phase
        const double phase = A.diag ? __dmul_rn(-A.dt, A.diag[gi >> 1]) : -A.dt;
        double sn, cs;
        sincos(phase, &sn, &cs);
        const double re = v.x, im = v.y;
        v.x = __dsub_rn(__dmul_rn(re, cs), __dmul_rn(im, sn));
        v.y = __dadd_rn(__dmul_rn(re, sn), __dmul_rn(im, cs));
      } else if (A.epi == EPI_AXPY_DIAG) {
        const double2 uu = *reinterpret_cast<const double2*>(A.u + gi);
        if (A.diag) {
          const double dg = A.diag[gi >> 1];
          v.x = __dadd_rn(v.x, __dmul_rn(dg, uu.x));
          v.y = __dadd_rn(v.y, __dmul_rn(dg, uu.y));
        }
        if (A.sigma != 0.0) {
          v.x = __dsub_rn(v.x, __dmul_rn(A.sigma, uu.x));
          v.y = __dsub_rn(v.y, __dmul_rn(A.sigma, uu.y));
        }
      }
      *reinterpret_cast<double2*>(A.y + gi) = v;
    } else {
      double v = *sp;
      if (spectral) {
        const double ls = __dsub_rn(group_lambda<NF>(A, lam_low[qi], g), A.shift);
        v = A.epi == EPI_SPEC_MUL ? __dmul_rn(v, ls) : __ddiv_rn(v, ls);
      } else if (A.epi == EPI_AXPY_DIAG) {
        const double uu = A.u[gi];
        if (A.diag) v = __dadd_rn(v, __dmul_rn(A.diag[gi], uu));
        if (A.sigma != 0.0) v = __dsub_rn(v, __dmul_rn(A.sigma, uu));
      }
      A.y[gi] = v;
    }
  }
}

// CC > 0 (DFMA, isotropic three-axis group with C = CC and C Qt = 8): compile-time geometry
template <int NF, int K4, int NT, int DN, int CC = 0>
__global__ void __launch_bounds__(rt_threads<DN>(), rt_ctas<DN>()) fused_rot_kernel(const __grid_constant__ RotArgs A) {
  constexpr int THREADS = rt_threads<DN>();
  constexpr int RT_STAGES = rt_stages<DN>();
  constexpr int RT_TILE = rt_tile<DN>();
  constexpr int G = NT >= 3 ? 2 : (NT == 2 ? 2 : 4);  // 8 G NT independent DMMA chains per warp
  // DN > 0: DFMA path with n = DN on every group axis (matrices row-major, pitch DNP);
  // DN == 0: DMMA path (B fragments in fragment order)
  constexpr int DNP = (DN + 1) & ~1;
  constexpr int FRAG = DN > 0 ? DN * DNP : K4 * NT * 32;  // doubles per axis
  constexpr int GROUPS = DN > 0 ? 1 : KRONOP_DM_GROUPS;
  constexpr int GT = THREADS / GROUPS;  // threads per group
  extern __shared__ __align__(128) double sm[];
  double* stages = sm;                                   // RT_STAGES x RT_TILE
  double* frags = stages + RT_STAGES * RT_TILE;          // NF x FRAG
  double* lam_low2 = frags + NF * FRAG;  // 2 x 64 (Qt) per group (<= 4), double-buffered per tile
  uint64_t* full = reinterpret_cast<uint64_t*>(lam_low2 + 512);
  static_assert(GROUPS >= 1 && GROUPS <= 4 && THREADS % (32 * GROUPS) == 0, "warp groups");
  int* done = reinterpret_cast<int*>(full + RT_STAGES);  // per-stage count of warps finished
  // per-stage count of loads issued: with several warp groups a group can reach the next use of
  // a stage before the other group has consumed and refilled it, when the barrier would still
  // show the parity of the use before (phases two apart look alike) -- so a group first waits
  // until the load it needs has been issued
  int* issued = done + RT_STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = tid / GT, gtid = tid - grp * GT, gwarp = gtid >> 5;
  (void)warp;
  auto gsync = [&]() {
    if constexpr (GROUPS == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(GT) : "memory");
  };
  const int t = lane & 3;
  const bool spectral = A.epi == EPI_SPEC_MUL || A.epi == EPI_SPEC_DIV || A.epi == EPI_SPEC_PHASE;

  // B fragments of every group axis in fragment order: frag[j][(kk NT + nt) 32 + lane] =
  // M_j(8 nt + lane/4, k(lane%4, kk)); zero outside the n x n matrix.
  for (int j = 0; j < NF; ++j)
    for (int e = tid; e < FRAG; e += THREADS) {
      int i, k;
      if (DN > 0) {
        i = e / DNP;
        k = e - i * DNP;
      } else {
        const int ln = e & 31, rest = e >> 5, nt = rest % NT, kk = rest / NT;
        k = kidx(A.kpat[j], ln & 3, kk);
        i = 8 * nt + (ln >> 2);
      }
      const int m = A.n[j];
      frags[j * FRAG + e] =
          (k < m && i < m) ? A.a[j][i + static_cast<long long>(A.lda[j]) * k] : 0.0;
    }
  // per-thread k offsets per axis (k >= m reads the fiber's element 0: finite, times zero)
  int koff[NF][K4];
  {
    int S = A.C;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int kk = 0; kk < K4; ++kk) {
        const int k = kidx(A.kpat[j], t, kk);
        koff[j][kk] = k < A.n[j] ? k * S : 0;
      }
      S *= A.n[j];
    }
  }
  for (int e = tid; e < RT_STAGES * RT_TILE; e += THREADS) stages[e] = 0.0;  // finite padding
  if (tid == 0) {
    for (int s = 0; s < RT_STAGES; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0;
      issued[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < RT_STAGES; ++s) {
      const long long tile = blockIdx.x + static_cast<long long>(s) * gridDim.x;
      if (tile < A.ntiles) {
        issue_tile(A, tile, stages + s * RT_TILE, &full[s]);
        issued[s] = 1;
      }
    }

  const int tile_elems = A.Qt * A.C * A.F;
  double Mreg[DN > 0 ? DN : 1][DN > 0 ? DN : 1];  // DFMA path: the axis matrix in registers
  bool mloaded = false;
  for (int kt = 0;; ++kt) {
    const int it = kt * GROUPS + grp;  // this group's tiles: it = grp, grp + GROUPS, ...
    const long long tile = blockIdx.x + static_cast<long long>(it) * gridDim.x;
    if (tile >= A.ntiles) break;
    const int s = it % RT_STAGES;
    double* buf = stages + s * RT_TILE;
    const long long q0 = tile * A.Qt;
    const int qv = static_cast<int>(A.Q - q0 < A.Qt ? A.Q - q0 : A.Qt);
    // the group's warps may still store its previous tile
    double* lam_low = lam_low2 + 64 * (2 * grp + (kt & 1));
    if (spectral && gtid < A.Qt) {  // lambda of the axes below the group, axis order from 0.0
      long long q = q0 + gtid;
      double lam = 0.0;
      for (int j = 0; j < A.nq; ++j) {
        const long long e = A.qext[j];
        const long long idx = q % e;
        q /= e;
        lam = __dadd_rn(lam, A.lam_q[j][idx]);
      }
      lam_low[gtid] = lam;
    }
    if constexpr (GROUPS > 1) {
      if (lane == 0)
        while (*reinterpret_cast<volatile int*>(&issued[s]) <= it / RT_STAGES) {
        }
      __syncwarp();
    }
    mbar_wait(&full[s], (it / RT_STAGES) & 1);
    if constexpr (DN > 0 && CC > 0 && NF == 3) {
      if (!mloaded) load_matrix<DN>(Mreg, frags);
      mloaded = true;
      axis_dfma_ct<DN, THREADS, CC, 8 * DN * DN>(buf, Mreg, tid);
      __syncthreads();
      axis_dfma_ct<DN, THREADS, CC * DN, 8 * DN * DN>(buf, Mreg, tid);
      __syncthreads();
      axis_dfma_ct<DN, THREADS, CC * DN * DN, 8 * DN * DN>(buf, Mreg, tid);
      __syncthreads();
    } else {
    int S = A.C;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int m = A.n[j];
      if constexpr (DN > 0) {
        // one matrix for the whole group (isotropic grid): loaded once per CTA, below
        if (!A.uniform || !mloaded) load_matrix<DN>(Mreg, frags + j * FRAG);
        mloaded = true;
        axis_dfma<DN, THREADS>(buf, Mreg, S, tile_elems / DN, tid);
      } else
        axis_inplace<K4, NT, G, GT>(buf, frags + j * FRAG, koff[j], m, S, tile_elems / m,
                                    gwarp, lane);
      S *= m;
      gsync();
    }
    }
    store_tile<NF, GT>(A, buf, q0, qv, lam_low, gtid);
    // No CTA barrier here: a warp that has stored its share moves on to the next tile's first
    // axis (another stage) while the others finish storing. The last warp to finish with stage
    // s refills it.
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[s], 1) == GT / 32 - 1) {
        done[s] = 0;
        __threadfence_block();
        const long long next = tile + static_cast<long long>(RT_STAGES) * gridDim.x;
        if (next < A.ntiles) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue_tile(A, next, buf, &full[s]);
          __threadfence_block();
          atomicAdd(&issued[s], 1);
        }
      }
    }
  }
}

template <int NF, int K4, int NT, int DN>
constexpr size_t rot_smem_bytes() {
  constexpr int FRAG = DN > 0 ? DN * ((DN + 1) & ~1) : K4 * NT * 32;
  return (static_cast<size_t>(rt_stages<DN>()) * rt_tile<DN>() + NF * FRAG + 512) * sizeof(double) +
         rt_stages<DN>() * (2 * sizeof(uint64_t) + 2 * sizeof(int)) + 16;
}

template <int NF, int K4, int NT, int DN = 0, int CC = 0>
void launch_rot(cudaStream_t s, const RotArgs& a) {
  ensure_smem_attr(reinterpret_cast<const void*>(fused_rot_kernel<NF, K4, NT, DN, CC>),
                   rot_smem_bytes<NF, K4, NT, DN>());
  const int grid_cap = device_sm_count() * rt_ctas<DN>();
  const long long grid = a.ntiles < grid_cap ? a.ntiles : grid_cap;
  fused_rot_kernel<NF, K4, NT, DN, CC>
      <<<static_cast<unsigned>(grid), rt_threads<DN>(), rot_smem_bytes<NF, K4, NT, DN>(), s>>>(a);
  KCUDA(cudaGetLastError());
}

template <int NF>
void launch_rot_nf(cudaStream_t s, const RotArgs& a, int maxn) {
  switch ((maxn + 3) >> 2) {
    case 1: launch_rot<NF, 1, 1>(s, a); break;
    case 2: launch_rot<NF, 2, 1>(s, a); break;
    case 3: launch_rot<NF, 3, 2>(s, a); break;
    case 4: launch_rot<NF, 4, 2>(s, a); break;
    case 5: launch_rot<NF, 5, 3>(s, a); break;
    case 6: launch_rot<NF, 6, 3>(s, a); break;
    case 7: launch_rot<NF, 7, 4>(s, a); break;
    default: launch_rot<NF, 8, 4>(s, a); break;
  }
}

// Host model of the shared-memory bank wavefronts of one fragment load (first M-blocks of warp
// 0) for a k pattern; picks the pattern with fewer wavefronts.
int choose_kpat(int S, int m, int K4, bool last, int C, int F, int lcq) {
  int best = 0, best_w = 1 << 30;
  for (int pat = 0; pat < 2; ++pat) {
    if (pat == 1 && (K4 & 1)) continue;
    int waves = 0;
    for (int kk = 0; kk < K4; ++kk)
      for (int half = 0; half < 2; ++half) {
        int used[16] = {0};
        int w = 0;
        for (int l = 16 * half; l < 16 * half + 16; ++l) {
          const int g = l >> 2, t = l & 3;
          int base;
          if (last) {
            const int cq = g & ((1 << lcq) - 1);
            const int qi = cq / C, c = cq - qi * C;
            base = c + C * F * qi;
          } else {
            base = g % S + (g / S) * S * m;
          }
          const int k = pat == 0 ? 4 * kk + t : 8 * (kk >> 1) + 2 * t + (kk & 1);
          const int addr = base + (k < m ? k : 0) * S;
          w = w > ++used[addr & 15] ? w : used[addr & 15];
        }
        waves += w;
      }
    if (waves < best_w) {
      best_w = waves;
      best = pat;
    }
  }
  return best;
}

// Standalone spectral pass over a field in the original axis order (what the last forward group
// launch leaves behind), used when the contraction runs on the epilogue-free kernels: the
// per-element epilogue (one sincos per pair for the phase) then runs at full occupancy instead of
// on the 16 warps of the contraction kernel. lambda is the direct sum in axis order from 0.0 and
// every operation matches store_tile, so the result is bit-identical to the fused epilogue.
// Layout: a row = the first m axes (L = prod n[0..m) <= SP_LMAX entries, lambda prefix sums in
// shared memory); a block handles rows_per_block consecutive rows, the hi-axis eigenvalues of each row
// staged once in shared memory.
constexpr int SP_LMAX = 2048;
constexpr int SP_THREADS = 256;
struct SpecArgs {
  double* y;
  int C, d, m, L, rows_per_block, kind;
  float inv_L;  // 1 / L (fast_div)
  long long rows;
  int n[KRONOP_MAX_DIM];
  const double* lam[KRONOP_MAX_DIM];
  double shift, dt;
};

__global__ void __launch_bounds__(SP_THREADS) spectral_pass_kernel(const __grid_constant__ SpecArgs A) {
  __shared__ double lam_lo[SP_LMAX];
  extern __shared__ double hv[];  // rows_per_block x (d - m)
  const int tid = threadIdx.x;
  for (int lo = tid; lo < A.L; lo += SP_THREADS) {
    int r = lo;
    double lam = 0.0;
    for (int a = 0; a < A.m; ++a) {
      const int q = r / A.n[a];
      lam = __dadd_rn(lam, A.lam[a][r - q * A.n[a]]);
      r = q;
    }
    lam_lo[lo] = lam;
  }
  const int nh = A.d - A.m;
  const int RB = A.rows_per_block;
  const long long nchunks = (A.rows + RB - 1) / RB;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long r0 = ch * RB;
    const int rv = static_cast<int>(A.rows - r0 < RB ? A.rows - r0 : RB);
    __syncthreads();  // lam_lo ready / previous chunk's hv consumed
    for (int t = tid; t < rv * nh; t += SP_THREADS) {
      const int ri = t / nh, j = t - ri * nh;
      long long r = r0 + ri;
      for (int a = A.m; a < A.m + j; ++a) r /= A.n[a];
      const int a = A.m + j;
      hv[ri * nh + j] = A.lam[a][r % A.n[a]];
    }
    __syncthreads();
    const int units = rv * A.L;
    double* base = A.y + static_cast<long long>(A.C) * A.L * r0;
    // 4 units per thread per round: loads issued before the (latency-bound) sincos chains
    for (int u0 = tid; u0 < units; u0 += 4 * SP_THREADS) {
      double2 v[4];
      double ls[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int u = u0 + k * SP_THREADS;
        if (u < units) {
          const int ri = fast_div(u, A.L, A.inv_L), lo = u - ri * A.L;
          if (A.C == 2) {
            v[k] = reinterpret_cast<const double2*>(base)[u];
          } else {
            v[k].x = base[u];
            v[k].y = 0.0;
          }
          double lam = lam_lo[lo];
          for (int j = 0; j < nh; ++j) lam = __dadd_rn(lam, hv[ri * nh + j]);
          ls[k] = __dsub_rn(lam, A.shift);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int u = u0 + k * SP_THREADS;
        if (u >= units) break;
        if (A.C == 2) {
          double2 w = v[k];
          if (A.kind == EPI_SPEC_MUL) {
            w.x = __dmul_rn(w.x, ls[k]);
            w.y = __dmul_rn(w.y, ls[k]);
          } else if (A.kind == EPI_SPEC_DIV) {
            w.x = __ddiv_rn(w.x, ls[k]);
            w.y = __ddiv_rn(w.y, ls[k]);
          } else {  // operators.cpp:68-71
            const double phase = __dmul_rn(-ls[k], A.dt);
            double sn, cs;
            sincos(phase, &sn, &cs);
            w.x = __dsub_rn(__dmul_rn(v[k].x, cs), __dmul_rn(v[k].y, sn));
            w.y = __dadd_rn(__dmul_rn(v[k].x, sn), __dmul_rn(v[k].y, cs));
          }
          reinterpret_cast<double2*>(base)[u] = w;
        } else {
          base[u] = A.kind == EPI_SPEC_MUL ? __dmul_rn(v[k].x, ls[k]) : __ddiv_rn(v[k].x, ls[k]);
        }
      }
    }
  }
}

void launch_spectral_pass(cudaStream_t s, double* y, int C, int d, const int* n,
                          const double* const* lam, long long N, int kind, double shift,
                          double dt) {
  SpecArgs a{};
  a.y = y;
  a.C = C;
  a.d = d;
  a.kind = kind;
  a.shift = shift;
  a.dt = dt;
  a.m = 0;
  a.L = 1;
  for (int j = 0; j < d; ++j) {
    a.n[j] = n[j];
    a.lam[j] = lam[j];
  }
  while (a.m < d && a.L * n[a.m] <= SP_LMAX) a.L *= n[a.m++];
  param_check(a.m >= 1, "spectral pass: leading extent too large");
  a.inv_L = 1.0f / static_cast<float>(a.L);
  a.rows = N / a.L;
  a.rows_per_block = 1;
  while (a.rows_per_block * 2 * a.L <= 4096) a.rows_per_block *= 2;
  const int nh = d - a.m;
  const size_t smem = sizeof(double) * static_cast<size_t>(a.rows_per_block * (nh > 0 ? nh : 1));
  const long long nchunks = (a.rows + a.rows_per_block - 1) / a.rows_per_block;
  const long long grid = nchunks < 148LL * 8 ? nchunks : 148LL * 8;
  spectral_pass_kernel<<<static_cast<unsigned>(grid), SP_THREADS, smem, s>>>(a);
  KCUDA(cudaGetLastError());
}

}  // namespace

void prime_fused_rot_kernels() {}

bool fused_rot_eligible(const double* x) { return (reinterpret_cast<uintptr_t>(x) & 15u) == 0; }

int launch_fused_rot(cudaStream_t s, const double* x, double* y, int cplx, int f, const int* n,
                     long long N, const double* const* mats, const int* lda, const RotEpi& epi) {
  param_check(f >= 1 && f <= RT_MAXF, "fused_rot: group size");
  RotArgs a{};
  a.x = x;
  a.y = y;
  a.C = cplx ? 2 : 1;
  a.f = f;
  a.F = 1;
  int maxn = 1;
  for (int j = 0; j < f; ++j) {
    a.n[j] = n[j];
    a.F *= n[j];
    a.a[j] = mats[j];
    a.lda[j] = lda[j];
    maxn = n[j] > maxn ? n[j] : maxn;
  }
  param_check(maxn <= 32 && a.F <= 1024 && (f < 3 || maxn <= 12), "fused_rot: group too large");
  a.Q = N / a.F;
  bool same = true;
  for (int j = 1; j < f; ++j) same = same && n[j] == n[0];
  static const bool no_dfma = [] {
    const char* e = getenv("KRONOP_ROT_NO_DFMA");  // A/B switch: DMMA for every extent
    return e && e[0] == '1';
  }();
  const bool dfma_ok = same && maxn >= 2 && maxn <= 10 && !no_dfma;
  // A/B switch for the phase (last forward) launch: 0 = epilogue fused into the 16-warp DMMA
  // kernel; 1 = contraction on the epilogue-free kernels + the standalone spectral pass when the
  // DFMA kernel serves the group; 2 (default) = that split for every extent (9D n = 9 propagate
  // 29.7 -> 26.7 ms, 6D n = 29 51.7 -> 50.8 ms, bit-identical; tools/microbench/spec_split.py). The divide / multiply
  // epilogues stay fused (measured: splitting them costs the extra field round trip)
  static const int spec_split = [] {
    const char* e = getenv("KRONOP_ROT_SPEC_SPLIT");
    return e && e[0] >= '0' && e[0] <= '2' ? e[0] - '0' : 2;
  }();
  const bool spectral = epi.kind == EPI_SPEC_MUL || epi.kind == EPI_SPEC_DIV ||
                        epi.kind == EPI_SPEC_PHASE;
  const bool split = epi.kind == EPI_SPEC_PHASE && (spec_split == 2 || (spec_split == 1 && dfma_ok));
  // every (f, n) has an instantiation; the group must fit a DFMA stage (C Qt >= 8)
  const bool use_dfma = dfma_ok && (!spectral || split) && 8 * a.F <= KRONOP_DF_TILE;
  // C * Qt: the largest power of two >= 8 with C * Qt * F <= the stage size of the path
  const int tile_doubles = use_dfma ? KRONOP_DF_TILE : KRONOP_DM_TILE;
  int cqt = 8;
  while (cqt * 2 * a.F <= tile_doubles && cqt < 64) cqt *= 2;
  param_check(cqt * a.F <= tile_doubles, "fused_rot: group too large for a stage");
  a.lcq = 0;
  while ((1 << a.lcq) < cqt) ++a.lcq;
  a.Qt = cqt / a.C;
  a.ntiles = (a.Q + a.Qt - 1) / a.Qt;
  const int K4 = (maxn + 3) / 4;
  int S = a.C;
  for (int j = 0; j < f; ++j) {
    a.kpat[j] = choose_kpat(S, n[j], K4, false, a.C, a.F, a.lcq);
    S *= n[j];
  }
  for (int j = 0; j < f; ++j) a.inv_n[j] = 1.0f / static_cast<float>(n[j]);
  a.uniform = 1;
  for (int j = 1; j < f; ++j) a.uniform &= (mats[j] == mats[0] && lda[j] == lda[0]) ? 1 : 0;
  a.epi = epi.kind;
  a.shift = epi.shift;
  a.dt = epi.dt;
  a.sigma = epi.sigma;
  a.diag = epi.diag;
  a.u = epi.u;
  for (int j = 0; j < f; ++j) a.lam_g[j] = epi.lam_g[j];
  a.nq = epi.nq;
  for (int j = 0; j < epi.nq; ++j) {
    a.qext[j] = epi.qext[j];
    a.lam_q[j] = epi.lam_q[j];
  }
  if (split) a.epi = EPI_STORE;
  // fused epilogue: the spectral launch keeps the 16-warp DMMA kernel (its store pass, one sincos
  // per pair, is latency bound and needs the warps more than the contraction needs DFMA)
  bool launched = false;
  static const bool no_ct = [] {
    const char* e = getenv("KRONOP_ROT_CT");  // A/B switch: 0 = runtime-geometry DFMA kernel
    return e && e[0] == '0';
  }();
  // the config-5 9D group of a real field: compile-time geometry (9D solve 15.7 -> 14.5 ms); for
  // complex fields it measured slower (9D propagate 25.8 -> 30.2 ms), so they keep the runtime
  // kernel (profiles/r02_rot_variants.json)
  if (use_dfma && f == 3 && maxn == 9 && a.uniform && cqt == 8 && a.C == 1 && !no_ct) {
    launched = true;
    launch_rot<3, 1, 1, 9, 1>(s, a);
  }
  if (use_dfma && !launched) {
    launched = true;
    switch (f * 16 + maxn) {
#define RT_DF(F, N) \
  case F * 16 + N: launch_rot<F, 1, 1, N>(s, a); break;
      RT_DF(1, 2) RT_DF(1, 3) RT_DF(1, 4) RT_DF(1, 5) RT_DF(1, 6) RT_DF(1, 7) RT_DF(1, 8)
      RT_DF(1, 9) RT_DF(1, 10)
      RT_DF(2, 2) RT_DF(2, 3) RT_DF(2, 4) RT_DF(2, 5) RT_DF(2, 6) RT_DF(2, 7) RT_DF(2, 8)
      RT_DF(2, 9) RT_DF(2, 10)
      RT_DF(3, 2) RT_DF(3, 3) RT_DF(3, 4) RT_DF(3, 5) RT_DF(3, 6) RT_DF(3, 7) RT_DF(3, 8)
      RT_DF(3, 9) RT_DF(3, 10)
#undef RT_DF
      default: launched = false; break;
    }
  }
  if (!launched) {
    if (f == 1)
      launch_rot_nf<1>(s, a, maxn);
    else if (f == 2)
      launch_rot_nf<2>(s, a, maxn);
    else if (maxn <= 4)  // F <= 1024 -> n <= 10 for three axes
      launch_rot<3, 1, 1>(s, a);
    else if (maxn <= 8)
      launch_rot<3, 2, 1>(s, a);
    else
      launch_rot<3, 3, 2>(s, a);
  }
  if (!split) return 1;
  // the output is back in the original axis order: the axes below the group, then the group
  int dims[KRONOP_MAX_DIM];
  const double* lams[KRONOP_MAX_DIM];
  for (int j = 0; j < epi.nq; ++j) {
    dims[j] = static_cast<int>(epi.qext[j]);
    lams[j] = epi.lam_q[j];
  }
  for (int j = 0; j < f; ++j) {
    dims[epi.nq + j] = n[j];
    lams[epi.nq + j] = epi.lam_g[j];
  }
  launch_spectral_pass(s, y, a.C, epi.nq + f, dims, lams, N, epi.kind, epi.shift, epi.dt);
  return 2;
}

}  // namespace kronop_dev
