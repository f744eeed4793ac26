// Small-extent, high-dimensional transforms (SURVEY.md §7 hard part 5; BASELINE config 5: 6D
// n = 29, 9D n = 9): several consecutive axes are contracted per HBM round trip.
//
// At n <= 32 a single mode-product pass has arithmetic intensity n/8 flop/B (<= 4): HBM-bound, and
// the 8x8x4 DMMA tiles of the large-n kernels would be >= 50% padding. Here one CTA stages a tile
// [Qt q][n_a x ... x n_{a+f-1}][P p] of the real view (p = the axes below the group, q = the axes
// above it) in shared memory, applies the f per-axis matrices one after the other in place (each
// thread owns whole fibers: it reads its n inputs, forms the n outputs with DFMA against the
// matrix held in shared memory, and writes them back to the same fiber), runs the fused
// epilogue, and stores the tile. f axes cost one read + one write of the field instead of f, so a
// 6-axis propagate moves 2 x 3 (not 2 x 6) fields for n = 29 and 2 x 3 (not 2 x 9) for 9D n = 9.
// Same contraction as proj/src/tensor.cpp:105-145 per axis, same epilogues as operators.cpp.
#include <cuda_runtime.h>

#include <cstdint>

#include "epilogue.cuh"
#include "kronop_internal.cuh"

namespace kronop_dev {

namespace {

constexpr int FS_THREADS = 256;
constexpr int FS_MAXF = 3;

struct FSArgs {
  const double* __restrict__ x;
  double* __restrict__ y;
  long long pre, post;  // real-view extents below / above the group
  int f;                // number of fused axes
  int n[FS_MAXF];       // their extents
  int F;                // product of n
  const double* a[FS_MAXF];
  int lda[FS_MAXF];
  int P, Qt;            // tile: P consecutive p, Qt consecutive q (Qt > 1 only if P == pre)
  int Pp;               // padded row length in shared memory (4 mod 16 doubles)
  long long tiles_p;    // ceil(pre / P)
  EpiParams ep;         // ep.axis = real-view axis of the group's FIRST axis
  int spectral_last;    // apply the spectral epilogue (group ends at the last axis, forward)
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 8 : 0));
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// One axis of the group on the staged tile, in place, on the FP64 tensor cores: each warp takes
// 8 x G fibers at a time (G DMMA M-blocks), k = the fiber index (K = 4*K4), n = the output index
// (N = 8*NT). K4/NT are compile-time (chosen per axis from m) so the DMMA stream carries no
// predicates; the matrix fragments live in registers for the whole tile, shared memory carries
// only the fiber reads and writes (row strides are 4 mod 16 doubles: conflict free); the G * NT
// accumulator chains hide the DMMA latency.
template <int MAXN, int K4, int NT>
__device__ __forceinline__ void axis_dmma(double* tile, const double* am, int m, int S, int nfib,
                                          int warp, int lane) {
  constexpr int G = NT >= 4 ? 2 : 4;
  const int g = lane >> 2, t = lane & 3;
  double bf[K4][NT];
#pragma unroll
  for (int kk = 0; kk < K4; ++kk)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int k = 4 * kk + t, n = 8 * nt + g;
      bf[kk][nt] = (k < m && n < m) ? am[n + MAXN * k] : 0.0;
    }
  const float invS = 1.0f / static_cast<float>(S);
  const int Sm = S * m;
  for (int f0 = warp * 8 * G; f0 < nfib; f0 += 8 * G * (FS_THREADS / 32)) {
    int base[G];
    bool fok[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const int fib = f0 + 8 * gg + g;
      fok[gg] = fib < nfib;
      const int fb = fok[gg] ? fib : f0;
      // fb / S through a float reciprocal, corrected to the exact quotient (fb < 2^22)
      int o = __float2int_rz(static_cast<float>(fb) * invS);
      o -= (o * S > fb);
      o += ((o + 1) * S <= fb);
      base[gg] = fb + o * (Sm - S);
    }
    double acc[G][NT][2];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[gg][nt][0] = acc[gg][nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < K4; ++kk) {
      const int k = 4 * kk + t;
      double a[G];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) a[gg] = k < m ? tile[base[gg] + k * S] : 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int gg = 0; gg < G; ++gg) dmma884(acc[gg][nt], a[gg], bf[kk][nt]);
    }
    __syncwarp();
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int n = 8 * nt + 2 * t + v;
          if (fok[gg] && n < m) tile[base[gg] + n * S] = acc[gg][nt][v];
        }
  }
}

template <int MAXN>
__device__ __forceinline__ void axis_dispatch(double* tile, const double* am, int m, int S,
                                              int nfib, int warp, int lane) {
  switch ((m + 3) >> 2) {
    case 1: axis_dmma<MAXN, 1, 1>(tile, am, m, S, nfib, warp, lane); break;
    case 2: axis_dmma<MAXN, 2, 1>(tile, am, m, S, nfib, warp, lane); break;
    case 3: if (MAXN >= 16) axis_dmma<MAXN, (MAXN >= 16 ? 3 : 1), (MAXN >= 16 ? 2 : 1)>(tile, am, m, S, nfib, warp, lane); break;
    case 4: if (MAXN >= 16) axis_dmma<MAXN, (MAXN >= 16 ? 4 : 1), (MAXN >= 16 ? 2 : 1)>(tile, am, m, S, nfib, warp, lane); break;
    case 5: if (MAXN >= 32) axis_dmma<MAXN, (MAXN >= 32 ? 5 : 1), (MAXN >= 32 ? 3 : 1)>(tile, am, m, S, nfib, warp, lane); break;
    case 6: if (MAXN >= 32) axis_dmma<MAXN, (MAXN >= 32 ? 6 : 1), (MAXN >= 32 ? 3 : 1)>(tile, am, m, S, nfib, warp, lane); break;
    case 7: if (MAXN >= 32) axis_dmma<MAXN, (MAXN >= 32 ? 7 : 1), (MAXN >= 32 ? 4 : 1)>(tile, am, m, S, nfib, warp, lane); break;
    default: if (MAXN >= 32) axis_dmma<MAXN, (MAXN >= 32 ? 8 : 1), (MAXN >= 32 ? 4 : 1)>(tile, am, m, S, nfib, warp, lane); break;
  }
}

template <int MAXN>
__global__ void __launch_bounds__(FS_THREADS, 2) fused_small_kernel(const __grid_constant__ FSArgs args) {
  extern __shared__ __align__(16) double sm[];
  const int P = args.P, F = args.F, Qt = args.Qt, Pp = args.Pp;
  double* amat = sm;                                // FS_MAXF x MAXN x MAXN
  double* lam_low = sm + FS_MAXF * MAXN * MAXN;     // P (spectral epilogue), even-padded
  double* tile = lam_low + ((P + 1) & ~1);          // element (p, r) at p + Pp * r, r = (f, q)
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const long long pre = args.pre;
  const long long tp = blockIdx.x % args.tiles_p;
  const long long tq = blockIdx.x / args.tiles_p;
  const long long p0 = tp * P;
  const long long q0 = tq * Qt;
  const int Pv = static_cast<int>(pre - p0 < P ? pre - p0 : P);                 // valid p
  const int Qv = static_cast<int>(args.post - q0 < Qt ? args.post - q0 : Qt);  // valid q
  const int R = F * Qt;    // rows (f, q) of the tile
  const int Rv = F * Qv;   // valid rows
  const long long gbase = p0 + pre * static_cast<long long>(F) * q0;  // element (p, r) at gbase + p + pre * r

  for (int j = 0; j < args.f; ++j)
    for (int e = tid; e < MAXN * MAXN; e += FS_THREADS) {
      const int i = e % MAXN, k = e / MAXN;
      amat[j * MAXN * MAXN + e] = (i < args.n[j] && k < args.n[j])
                                      ? args.a[j][i + static_cast<long long>(args.lda[j]) * k]
                                      : 0.0;
    }
  // tile load (LDGSTS, zero-fill outside the field and in the padding columns). Lanes walk
  // (row, p) pairs with per-thread constant offsets: no per-element integer division.
  const int RW = P <= 32 ? 32 / P : 1;                 // rows per warp iteration
  const int lr = P <= 32 ? lane / P : 0;               // this lane's row within the iteration
  const int lp = P <= 32 ? lane - lr * P : lane;       // this lane's p
  const bool lane_on = P <= 32 ? lr < RW : true;
  for (int r0 = warp * RW; r0 < R; r0 += RW * (FS_THREADS / 32)) {
    const int r = r0 + lr;
    if (!lane_on || r >= R) continue;
    for (int p = lp; p < Pp; p += 32) {
      const bool ok = p < Pv && r < Rv;
      cp_async8(tile + p + Pp * r, args.x + (ok ? gbase + p + pre * r : 0), ok);
      if (P <= 32 && p + 32 >= Pp) break;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();

  const int PR = Pp * R;
  int S = Pp;
  for (int j = 0; j < args.f; ++j) {
    const int m = args.n[j];
    axis_dispatch<MAXN>(tile, amat + j * MAXN * MAXN, m, S, PR / m, warp, lane);
    S *= m;
    __syncthreads();
  }

  // epilogue + store (same division-free (row, p) walk). The spectral factor needs the global
  // multi-index: the axes below the group depend only on p (lam_low, computed once per tile in
  // axis order from 0.0 exactly like direct_sum_grid), the group indices only on the row (packed
  // per row once per tile); the spectral group always contains the last axis.
  const EpiParams& ep = args.ep;
  const bool spectral = args.spectral_last != 0;
  int* rowidx = reinterpret_cast<int*>(amat);  // the matrices are no longer needed
  if (spectral) {
    for (int pl = tid; pl < P; pl += FS_THREADS)
      lam_low[pl] = lambda_partial_low_ext(ep, p0 + pl, ep.axis);
    for (int fr = tid; fr < F; fr += FS_THREADS) {
      int rem = fr, packed = 0;
      for (int j = 0; j < args.f; ++j) {
        packed |= (rem % args.n[j]) << (10 * j);
        rem /= args.n[j];
      }
      rowidx[fr] = packed;
    }
    __syncthreads();
  }
  const bool plain = !spectral && ep.kind != EPI_AXPY_DIAG;
  const double* l0 = spectral ? ep.lam[ep.axis] : nullptr;
  const double* l1 = spectral && args.f > 1 ? ep.lam[ep.axis + 1] : nullptr;
  const double* l2 = spectral && args.f > 2 ? ep.lam[ep.axis + 2] : nullptr;
  for (int r0 = warp * RW; r0 < Rv; r0 += RW * (FS_THREADS / 32)) {
    const int r = r0 + lr;
    if (!lane_on || r >= Rv) continue;
    int packed = 0;
    if (spectral) {
      const int q = r / F;
      packed = rowidx[r - q * F];
    }
    for (int p = lp; p < Pv; p += 32) {
      const long long gi = gbase + p + pre * r;
      const int si = p + Pp * r;
      double val = tile[si];
      if (plain) {
        args.y[gi] = val;
      } else if (spectral) {
        double lam = lam_low[p];
        if (l0) lam = __dadd_rn(lam, l0[packed & 1023]);
        if (l1) lam = __dadd_rn(lam, l1[(packed >> 10) & 1023]);
        if (l2) lam = __dadd_rn(lam, l2[(packed >> 20) & 1023]);
        const double ls = __dsub_rn(lam, ep.shift);
        if (ep.kind == EPI_SPEC_MUL) {
          val = __dmul_rn(val, ls);
        } else if (ep.kind == EPI_SPEC_DIV) {
          val = __ddiv_rn(val, ls);
        } else {  // phase: the re/im partner is the neighbouring p (leading re/im axis)
          const bool is_im = ((p0 + p) & 1) != 0;
          const double other = tile[is_im ? si - 1 : si + 1];
          const double phase = __dmul_rn(-ls, ep.dt);
          double sn, cs;
          sincos(phase, &sn, &cs);
          const double re = is_im ? other : val;
          const double im = is_im ? val : other;
          val = is_im ? __dadd_rn(__dmul_rn(re, sn), __dmul_rn(im, cs))
                      : __dsub_rn(__dmul_rn(re, cs), __dmul_rn(im, sn));
        }
        args.y[gi] = val;
      } else {  // EPI_AXPY_DIAG
        const double uu = ep.u[gi];
        if (ep.diag) val = __dadd_rn(val, __dmul_rn(ep.diag[ep.cplx ? (gi >> 1) : gi], uu));
        if (ep.sigma != 0.0) val = __dsub_rn(val, __dmul_rn(ep.sigma, uu));
        args.y[gi] = val;
      }
      if (P <= 32) break;
    }
  }
}

template <int MAXN>
void launch_fs(cudaStream_t s, const FSArgs& a, size_t smem) {
  static bool attr = false;
  if (!attr) {
    KCUDA(cudaFuncSetAttribute(fused_small_kernel<MAXN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               232448 - 1024));
    attr = true;
  }
  const long long tiles = a.tiles_p * ((a.post + a.Qt - 1) / a.Qt);
  fused_small_kernel<MAXN><<<static_cast<unsigned>(tiles), FS_THREADS, smem, s>>>(a);
  KCUDA(cudaGetLastError());
}

}  // namespace

void prime_fused_small_kernels() {
  KCUDA(cudaFuncSetAttribute(fused_small_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             232448 - 1024));
  KCUDA(cudaFuncSetAttribute(fused_small_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             232448 - 1024));
  KCUDA(cudaFuncSetAttribute(fused_small_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             232448 - 1024));
}

int fused_small_max_extent() { return 32; }

// Plan + launch one fused group of `f` consecutive real-view axes starting at `axis` of the view
// (ext[] = current real-view extents). mats[j] / lda[j]: square n_j x n_j padded matrices.
void launch_fused_small(cudaStream_t s, const double* x, double* y, int nd, const long long* ext,
                        int axis, int f, const double* const* mats, const int* lda,
                        const EpiParams& ep, bool spectral_last) {
  param_check(f >= 1 && f <= FS_MAXF, "fused_small: group size");
  FSArgs a{};
  a.x = x;
  a.y = y;
  a.pre = 1;
  for (int i = 0; i < axis; ++i) a.pre *= ext[i];
  a.post = 1;
  for (int i = axis + f; i < nd; ++i) a.post *= ext[i];
  a.f = f;
  a.F = 1;
  int maxn = 1;
  for (int j = 0; j < f; ++j) {
    a.n[j] = static_cast<int>(ext[axis + j]);
    a.F *= a.n[j];
    a.a[j] = mats[j];
    a.lda[j] = lda[j];
    maxn = a.n[j] > maxn ? a.n[j] : maxn;
  }
  param_check(maxn <= 32, "fused_small: extent > 32");
  const int MAXN = maxn <= 8 ? 8 : maxn <= 16 ? 16 : 32;
  // tile: <= ~110 KB of shared memory so two CTAs share an SM (one loads while the other
  // computes); rows are padded to Pp = 4 mod 16 doubles (conflict-free fragment access).
  auto padp = [](long long P) { return P + ((4 - P) % 16 + 16) % 16; };
  const long long budget = 14080 - FS_MAXF * MAXN * MAXN - 64 - 512;  // doubles
  if (padp(a.pre) * a.F <= budget) {
    a.P = static_cast<int>(a.pre);
    long long qt = budget / (padp(a.pre) * a.F);
    if (qt > a.post) qt = a.post;
    a.Qt = static_cast<int>(qt < 1 ? 1 : qt);
  } else {
    long long P = 16;
    while (P + 16 <= 64 && padp(P + 16) * a.F <= budget) P += 16;
    if (padp(P) * a.F > budget) P = 4;
    param_check(padp(P) * a.F <= budget, "fused_small: tile does not fit");
    a.P = static_cast<int>(P);
    a.Qt = 1;
  }
  a.Pp = static_cast<int>(padp(a.P));
  a.tiles_p = (a.pre + a.P - 1) / a.P;
  a.ep = ep;
  a.ep.axis = axis;
  a.spectral_last = spectral_last ? 1 : 0;
  if (spectral_last && ep.kind == EPI_SPEC_PHASE)
    param_check(a.P % 2 == 0 || a.P == a.pre, "fused_small: phase needs re/im pairs in a tile");
  const size_t smem = (static_cast<size_t>(FS_MAXF) * MAXN * MAXN + ((a.P + 1) & ~1) +
                       static_cast<size_t>(a.Pp) * a.F * a.Qt) *
                      sizeof(double);
  if (MAXN == 8)
    launch_fs<8>(s, a, smem);
  else if (MAXN == 16)
    launch_fs<16>(s, a, smem);
  else
    launch_fs<32>(s, a, smem);
}

}  // namespace kronop_dev
