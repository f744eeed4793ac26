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
  const double* x;
  double* y;
  long long pre, post;  // real-view extents below / above the group
  int f;                // number of fused axes
  int n[FS_MAXF];       // their extents
  int F;                // product of n
  const double* a[FS_MAXF];
  int lda[FS_MAXF];
  int P, Qt;            // tile: P consecutive p, Qt consecutive q (Qt > 1 only if P == pre)
  long long tiles_p;    // ceil(pre / P)
  EpiParams ep;         // ep.axis = real-view axis of the group's FIRST axis
  int spectral_last;    // apply the spectral epilogue (group ends at the last axis, forward)
};

// One fiber per thread: its m inputs live in registers (so the transform is in place), the m
// outputs are formed 8 at a time (8 independent DFMA chains), and the 8 matrix entries of each
// step are one pair of 128-bit shared loads broadcast to the whole warp (the warp walks the same
// output block in lockstep).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 16 : 0));
}

template <int MAXN>
__device__ __forceinline__ void fiber_one(double* tile, const double* am, int m, int stride,
                                          int base) {
  double xin[MAXN];
#pragma unroll
  for (int k = 0; k < MAXN; ++k) xin[k] = k < m ? tile[base + k * stride] : 0.0;
#pragma unroll
  for (int i0 = 0; i0 < MAXN; i0 += 8) {
    if (i0 < m) {
      double acc[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r] = 0.0;
#pragma unroll
      for (int k = 0; k < MAXN; ++k) {
        if (k < m) {
          const double2* col = reinterpret_cast<const double2*>(am + i0 + MAXN * k);
          const double2 c0 = col[0], c1 = col[1], c2 = col[2], c3 = col[3];
          acc[0] = __fma_rn(c0.x, xin[k], acc[0]);
          acc[1] = __fma_rn(c0.y, xin[k], acc[1]);
          acc[2] = __fma_rn(c1.x, xin[k], acc[2]);
          acc[3] = __fma_rn(c1.y, xin[k], acc[3]);
          acc[4] = __fma_rn(c2.x, xin[k], acc[4]);
          acc[5] = __fma_rn(c2.y, xin[k], acc[5]);
          acc[6] = __fma_rn(c3.x, xin[k], acc[6]);
          acc[7] = __fma_rn(c3.y, xin[k], acc[7]);
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (i0 + r < m) tile[base + (i0 + r) * stride] = acc[r];
    }
  }
}

template <int MAXN>
__global__ void __launch_bounds__(FS_THREADS, 2) fused_small_kernel(const FSArgs args) {
  extern __shared__ __align__(16) double sm[];
  double* amat = sm;                                      // FS_MAXF x MAXN x MAXN
  double* lam_low = sm + FS_MAXF * MAXN * MAXN;           // P (spectral epilogue), even-padded
  double* tile = lam_low + ((args.P + 1) & ~1);           // [Qt][F][P]
  const int tid = threadIdx.x;
  const long long pre = args.pre;
  const int P = args.P, F = args.F, Qt = args.Qt;
  const long long tp = blockIdx.x % args.tiles_p;
  const long long tq = blockIdx.x / args.tiles_p;
  const long long p0 = tp * P;
  const long long q0 = tq * Qt;
  const int Pv = static_cast<int>(pre - p0 < P ? pre - p0 : P);                 // valid p
  const int Qv = static_cast<int>(args.post - q0 < Qt ? args.post - q0 : Qt);  // valid q

  // matrices (column-major, zero-padded to MAXN x MAXN)
  for (int j = 0; j < args.f; ++j)
    for (int e = tid; e < MAXN * MAXN; e += FS_THREADS) {
      const int i = e % MAXN, k = e / MAXN;
      amat[j * MAXN * MAXN + e] =
          (i < args.n[j] && k < args.n[j]) ? args.a[j][i + static_cast<long long>(args.lda[j]) * k] : 0.0;
    }
  // tile load: element (p, f, q) at x[p0 + p + pre * (f + F * (q0 + q))]
  const long long E = static_cast<long long>(P) * F * Qt;
  const long long gbase = p0 + pre * static_cast<long long>(F) * q0;
  // asynchronous copies (LDGSTS): thousands of loads in flight per CTA, zero-fill outside
  if (P == pre) {  // the whole tile is one contiguous run
    const long long Ev = static_cast<long long>(P) * F * Qv;
    const int Ei = static_cast<int>(E);
    const bool vec = ((gbase & 1) == 0) && ((reinterpret_cast<uintptr_t>(args.x) & 15) == 0);
    if (vec) {
      for (int e = 2 * tid; e < Ei; e += 2 * FS_THREADS) {
        const bool ok = e < Ev;  // Ev is even when P*F is even; else fall back below
        if (ok && e + 1 < Ev)
          cp_async16(tile + e, args.x + gbase + e, true);
        else {
          cp_async8(tile + e, args.x + gbase + (ok ? e : 0), ok);
          cp_async8(tile + e + 1, args.x + gbase + (e + 1 < Ev ? e + 1 : 0), e + 1 < Ev);
        }
      }
    } else {
      for (int e = tid; e < Ei; e += FS_THREADS)
        cp_async8(tile + e, args.x + gbase + (e < Ev ? e : 0), e < Ev);
    }
  } else {
    const int Ei = static_cast<int>(E);
    for (int e = tid; e < Ei; e += FS_THREADS) {
      const int r = e / P;  // (f, q) with Qt == 1
      const int p = e - r * P;
      cp_async8(tile + e, args.x + gbase + (p < Pv ? p + pre * r : 0), p < Pv);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();

  // the fused axes, one after the other, in place
  int stride = P;
  for (int j = 0; j < args.f; ++j) {
    const int m = args.n[j];
    const int nfib = static_cast<int>(E / m);
    for (int fib = tid; fib < nfib; fib += FS_THREADS) {
      const int inner = fib % stride;
      const int outer = fib / stride;
      fiber_one<MAXN>(tile, amat + j * MAXN * MAXN, m, stride, inner + outer * stride * m);
    }
    stride *= m;
    __syncthreads();
  }

  // epilogue + store. The spectral factor needs the global multi-index: the part from the axes
  // below the group depends only on p (precomputed once per tile, in axis order from 0.0 exactly
  // like direct_sum_grid), the group part is added axis by axis; the spectral group always
  // contains the last axis, so nothing lies above it.
  const EpiParams& ep = args.ep;
  const bool spectral = args.spectral_last != 0;
  const bool contiguous = P == pre;
  const int Ei = static_cast<int>(E);
  if (spectral) {
    for (int pl = tid; pl < P; pl += FS_THREADS)
      lam_low[pl] = lambda_partial_low_ext(ep, p0 + pl, ep.axis);
    __syncthreads();
  }
  if (!spectral && ep.kind != EPI_AXPY_DIAG) {
    if (contiguous) {
      const long long Ev = static_cast<long long>(P) * F * Qv;
#pragma unroll 4
      for (int e = tid; e < Ei; e += FS_THREADS)
        if (e < Ev) args.y[gbase + e] = tile[e];
    } else {
#pragma unroll 4
      for (int e = tid; e < Ei; e += FS_THREADS) {
        const int r = e / P;
        const int p = e - r * P;
        if (p < Pv) args.y[gbase + p + pre * r] = tile[e];
      }
    }
    return;
  }
  for (int e = tid; e < Ei; e += FS_THREADS) {
    const int r = e / P;
    const int p = e - r * P;
    const int q = r / F;
    const int fidx = r - q * F;
    if (p >= Pv || q >= Qv) continue;
    const long long gi = gbase + p + pre * (fidx + static_cast<long long>(F) * q);
    double val = tile[e];
    if (spectral) {
      double lam = lam_low[p];
      int rem = fidx;
      for (int j = 0; j < args.f; ++j) {
        const int idx = rem % args.n[j];
        rem /= args.n[j];
        if (ep.lam[ep.axis + j]) lam = __dadd_rn(lam, ep.lam[ep.axis + j][idx]);
      }
      const double ls = __dsub_rn(lam, ep.shift);
      if (ep.kind == EPI_SPEC_MUL) {
        val = __dmul_rn(val, ls);
      } else if (ep.kind == EPI_SPEC_DIV) {
        val = __ddiv_rn(val, ls);
      } else {  // phase: the re/im partner is the neighbouring p (leading re/im axis)
        const bool is_im = ((p0 + p) & 1) != 0;
        const double other = tile[is_im ? e - 1 : e + 1];
        const double phase = __dmul_rn(-ls, ep.dt);
        double sn, cs;
        sincos(phase, &sn, &cs);
        const double re = is_im ? other : val;
        const double im = is_im ? val : other;
        val = is_im ? __dadd_rn(__dmul_rn(re, sn), __dmul_rn(im, cs))
                    : __dsub_rn(__dmul_rn(re, cs), __dmul_rn(im, sn));
      }
    } else {  // EPI_AXPY_DIAG
      const double uu = ep.u[gi];
      if (ep.diag) val = __dadd_rn(val, __dmul_rn(ep.diag[ep.cplx ? (gi >> 1) : gi], uu));
      if (ep.sigma != 0.0) val = __dsub_rn(val, __dmul_rn(ep.sigma, uu));
    }
    args.y[gi] = val;
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
  // tile: ~96 KB of doubles so two CTAs share an SM (one loads while the other computes); when
  // that leaves runs of < 16 contiguous p (poor coalescing), use ~200 KB and one CTA per SM.
  long long budget = 14080 - FS_MAXF * MAXN * MAXN;  // doubles: <= 110 KB per CTA, 2 per SM
  if (a.pre * a.F > budget && budget / a.F < 8) budget = 27648 - FS_MAXF * MAXN * MAXN;
  if (a.pre * a.F <= budget) {
    a.P = static_cast<int>(a.pre);
    long long qt = budget / (a.pre * a.F);
    if (qt > a.post) qt = a.post;
    a.Qt = static_cast<int>(qt < 1 ? 1 : qt);
  } else {
    long long P = budget / a.F;
    if (P > 64) P = 64;
    if (a.pre % 2 == 0 && P > 1) P &= ~1LL;  // keep re/im pairs (leading re/im axis) together
    param_check(P >= 1, "fused_small: tile does not fit");
    a.P = static_cast<int>(P);
    a.Qt = 1;
  }
  a.tiles_p = (a.pre + a.P - 1) / a.P;
  a.ep = ep;
  a.ep.axis = axis;
  a.spectral_last = spectral_last ? 1 : 0;
  if (spectral_last && ep.kind == EPI_SPEC_PHASE)
    param_check(a.P % 2 == 0 || a.P == a.pre, "fused_small: phase needs re/im pairs in a tile");
  const size_t smem = (static_cast<size_t>(FS_MAXF) * MAXN * MAXN + ((a.P + 1) & ~1) +
                       static_cast<size_t>(a.P) * a.F * a.Qt) *
                      sizeof(double);
  if (MAXN == 8)
    launch_fs<8>(s, a, smem);
  else if (MAXN == 16)
    launch_fs<16>(s, a, smem);
  else
    launch_fs<32>(s, a, smem);
}

}  // namespace kronop_dev
