// HBM-bound vector kernels of the hot path: deterministic reductions (plain and mass-weighted dot
// products), the PCG updates with device-resident scalars, the split-step B-phase, and the
// index-decomposed field generators (mass grid, eigenvalue grid, rank-one ground state, SplitMix64).
//
// Reference loops restated: inner / norm / mass_field / direct_sum_grid (proj/src/tensor.cpp:
// 147-209), PCG vector algebra (proj/src/pcg.cpp:15-71), weighted dots (ground_state.cpp:42-45,
// gpe.cpp:12-17,24-26,71-73), pointwise_phase (splitting.cpp:44-51), ground_state
// (operators.cpp:77-91), SplitMix64 (rng.hpp:16-35).
//
// All reductions use a fixed grid (kRedBlocks blocks x 256 threads, grid-stride) writing one
// partial per block, then one block summing the partials in a fixed tree: results are bitwise
// reproducible run to run (acceptance.cpp:647-687 determinism), with no floating-point atomics.
// Elementwise kernels use 16-byte vector loads where the layout allows and a grid of
// 148 SMs x 8 blocks (persistent grid-stride), which saturates HBM on B200.
#include "vector_ops.cuh"
#include "epilogue.cuh"

namespace kronop_dev {

constexpr int kThreads = 256;

// ----------------------------------------------------------------- index helpers --
struct IndexGeom {
  int d;
  long long n[kMaxDims];
};

__device__ __forceinline__ double mass_weight(const IndexGeom& g, const double* const* mass,
                                              long long i) {
  // w = 1.0; w *= mass[a][i_a] in axis order (tensor.cpp:160-163 / :188-191)
  double w = 1.0;
  for (int a = 0; a < g.d; ++a) {
    const long long e = g.n[a];
    const long long idx = i % e;
    i /= e;
    w = __dmul_rn(w, mass[a][idx]);
  }
  return w;
}

// ------------------------------------------------------------------- reductions --
template <int NS>
__device__ __forceinline__ void block_reduce_store(double (&v)[NS], double* out_partials,
                                                   int stride) {
  __shared__ double sh[NS][kThreads];
#pragma unroll
  for (int s = 0; s < NS; ++s) sh[s][threadIdx.x] = v[s];
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
#pragma unroll
      for (int s = 0; s < NS; ++s) sh[s][threadIdx.x] += sh[s][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) out_partials[s * stride + blockIdx.x] = sh[s][0];
  }
}

// mode 0: sum a*b ; mode 1 (complex interleaved, n = complex count): sum conj(a)*b -> (re, im)
// wmode: multiply by the mass weight (index geometry per complex element / real element)
struct DotArgs {
  const double* a;
  const double* b;
  long long n;  // number of scalars (real) or complex elements
  int cplx;
  int weighted;
  IndexGeom geom;
  const double* mass[KRONOP_MAX_DIM];
};

__global__ void __launch_bounds__(kThreads) k_dot_partial(DotArgs args, double* partials) {
  double acc[2] = {0.0, 0.0};
  const long long stride = static_cast<long long>(gridDim.x) * kThreads;
  for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < args.n;
       i += stride) {
    const double w = args.weighted ? mass_weight(args.geom, args.mass, i) : 1.0;
    if (!args.cplx) {
      const double t = args.weighted ? __dmul_rn(w, args.a[i]) : args.a[i];
      acc[0] = __dadd_rn(acc[0], __dmul_rn(t, args.b[i]));
    } else {
      const double ar = args.a[2 * i], ai = args.a[2 * i + 1];
      const double br = args.b[2 * i], bi = args.b[2 * i + 1];
      // conj(a) * b = (ar br + ai bi) + i (ar bi - ai br)
      double re = __dadd_rn(__dmul_rn(ar, br), __dmul_rn(ai, bi));
      double im = __dsub_rn(__dmul_rn(ar, bi), __dmul_rn(ai, br));
      if (args.weighted) {
        re = __dmul_rn(w, re);
        im = __dmul_rn(w, im);
      }
      acc[0] = __dadd_rn(acc[0], re);
      acc[1] = __dadd_rn(acc[1], im);
    }
  }
  block_reduce_store<2>(acc, partials, gridDim.x);
}

// Sums nsum groups of `count` partials (group s at partials + s*count) into out[s], optionally
// applying a finaliser (sqrt) — one block, fixed tree.
__global__ void __launch_bounds__(1024) k_reduce_final(const double* partials, int count, int nsum,
                                                       double* out) {
  __shared__ double sh[1024];
  for (int s = 0; s < nsum; ++s) {
    double v = 0.0;
    for (int i = threadIdx.x; i < count; i += 1024) v = __dadd_rn(v, partials[s * count + i]);
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
      if (threadIdx.x < w) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) out[s] = sh[0];
    __syncthreads();
  }
}

void launch_dot(cudaStream_t s, Workspace& ws, const double* a, const double* b, long long n,
                int cplx, const IndexGeomHost* wgeom, double* out_dev) {
  DotArgs args{};
  args.a = a;
  args.b = b;
  args.n = n;
  args.cplx = cplx;
  args.weighted = wgeom != nullptr;
  if (wgeom) {
    args.geom.d = wgeom->d;
    for (int i = 0; i < wgeom->d; ++i) {
      args.geom.n[i] = wgeom->n[i];
      args.mass[i] = wgeom->mass[i];
    }
  }
  k_dot_partial<<<kRedBlocks, kThreads, 0, s>>>(args, ws.partials);
  k_reduce_final<<<1, 1024, 0, s>>>(ws.partials, kRedBlocks, cplx ? 2 : 1, out_dev);
  ws.launches += 2;
  KCUDA(cudaGetLastError());
}

// ------------------------------------------------------------ PCG vector updates --
// x += alpha p ; r -= alpha q ; partial sums of r.r (pcg.cpp:56-57, :15 norm)
__global__ void __launch_bounds__(kThreads) k_pcg_update_xr(double* __restrict__ x,
                                                          double* __restrict__ r,
                                                          const double* __restrict__ p,
                                                          const double* __restrict__ q,
                                                          const PcgScalars* sc, long long n,
                                                          double* partials) {
  double acc[1] = {0.0};
  if (sc->active) {
    const double alpha = sc->alpha;
    const long long stride = static_cast<long long>(gridDim.x) * kThreads;
    for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < n;
         i += stride) {
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      const double rn = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
      r[i] = rn;
      acc[0] = __dadd_rn(acc[0], __dmul_rn(rn, rn));
    }
  }
  block_reduce_store<1>(acc, partials, gridDim.x);
}

// p = z + beta p (pcg.cpp:60)
__global__ void __launch_bounds__(kThreads) k_pcg_update_p(double* __restrict__ p,
                                                         const double* __restrict__ z,
                                                         const PcgScalars* sc, long long n) {
  if (!sc->active) return;
  const double beta = sc->beta;
  const long long stride = static_cast<long long>(gridDim.x) * kThreads;
  for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < n;
       i += stride)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

void launch_pcg_update_xr(cudaStream_t s, Workspace& ws, double* x, double* r, const double* p,
                          const double* q, const PcgScalars* sc, long long n, double* out_rr) {
  k_pcg_update_xr<<<kRedBlocks, kThreads, 0, s>>>(x, r, p, q, sc, n, ws.partials);
  k_reduce_final<<<1, 1024, 0, s>>>(ws.partials, kRedBlocks, 1, out_rr);
  ws.launches += 2;
  KCUDA(cudaGetLastError());
}

void launch_pcg_update_p(cudaStream_t s, Workspace& ws, double* p, const double* z,
                         const PcgScalars* sc, long long n) {
  k_pcg_update_p<<<kEltBlocks, kThreads, 0, s>>>(p, z, sc, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// ------------------------------------------------------------------- elementwise --
__global__ void k_copy_if(double* __restrict__ dst, const double* __restrict__ src, long long n,
                          const int* flag) {
  if (flag && !*flag) return;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    dst[i] = src[i];
}

void launch_copy_if(cudaStream_t s, Workspace& ws, double* dst, const double* src, long long n,
                    const int* flag) {
  k_copy_if<<<kEltBlocks, kThreads, 0, s>>>(dst, src, n, flag);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// y = a * x  (a from device scalar pointer if ap != null, else immediate);  y may alias x
__global__ void k_scale(double* y, const double* x, long long n, double a, const double* ap,
                        int ap_mode) {
  double s = a;
  if (ap) s = ap_mode == 1 ? 1.0 / sqrt(*ap) : *ap;  // ap_mode 1: scale by 1/sqrt(*ap)
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    y[i] = __dmul_rn(x[i], s);
}

void launch_scale(cudaStream_t s, Workspace& ws, double* y, const double* x, long long n, double a,
                  const double* ap, int ap_mode) {
  k_scale<<<kEltBlocks, kThreads, 0, s>>>(y, x, n, a, ap, ap_mode);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

__global__ void k_fill(double* y, double v, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    y[i] = v;
}

void launch_fill(cudaStream_t s, Workspace& ws, double* y, double v, long long n) {
  k_fill<<<kEltBlocks, kThreads, 0, s>>>(y, v, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// y = x / *nrm (division, as in u.flat() /= sqrt(...) ground_state.cpp:63,84)
__global__ void k_div_by(double* y, const double* x, long long n, const double* nrm, int sq) {
  const double dnm = sq ? sqrt(*nrm) : *nrm;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    y[i] = __ddiv_rn(x[i], dnm);
}

void launch_div_by(cudaStream_t s, Workspace& ws, double* y, const double* x, long long n,
                   const double* nrm_dev, int take_sqrt) {
  k_div_by<<<kEltBlocks, kThreads, 0, s>>>(y, x, n, nrm_dev, take_sqrt);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// y = x .* d (real d, x real or complex interleaved)
__global__ void k_mul_diag(double* y, const double* x, const double* dg, long long n, int cplx) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long total = cplx ? 2 * n : n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += stride)
    y[i] = __dmul_rn(x[i], dg[cplx ? (i >> 1) : i]);
}

void launch_mul_diag(cudaStream_t s, Workspace& ws, double* y, const double* x, const double* d,
                     long long n, int cplx) {
  k_mul_diag<<<kEltBlocks, kThreads, 0, s>>>(y, x, d, n, cplx);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// psi *= exp(-i factor b)  (pointwise_phase, splitting.cpp:44-51)
__global__ void k_phase(double* psi, const double* b, double factor, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double phase = b ? __dmul_rn(-factor, b[i]) : -factor;  // b = nullptr: b = 1
    double sn, cs;
    sincos(phase, &sn, &cs);
    const double re = psi[2 * i], im = psi[2 * i + 1];
    psi[2 * i] = __dsub_rn(__dmul_rn(re, cs), __dmul_rn(im, sn));
    psi[2 * i + 1] = __dadd_rn(__dmul_rn(re, sn), __dmul_rn(im, cs));
  }
}

void launch_phase(cudaStream_t s, Workspace& ws, double* psi, const double* b, double factor,
                  long long n) {
  k_phase<<<kEltBlocks, kThreads, 0, s>>>(psi, b, factor, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// (cos, sin) of the B phase -factor * b[i] with k_phase's operations: the table a Kronecker
// propagate reads to apply the preceding B step to its input (bit-identical to k_phase).
__global__ void k_phase_table(double* tab, const double* b, double factor, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double phase = b ? __dmul_rn(-factor, b[i]) : -factor;
    double sn, cs;
    sincos(phase, &sn, &cs);
    reinterpret_cast<double2*>(tab)[i] = make_double2(cs, sn);
  }
}

void launch_phase_table(cudaStream_t s, Workspace& ws, double* tab, const double* b,
                        double factor, long long n) {
  k_phase_table<<<kEltBlocks, kThreads, 0, s>>>(tab, b, factor, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// out[i] = generator(multi-index of i): 0 = mass product, 1 = direct sum (from 0.0), 2 = product
struct GenArgs {
  IndexGeom geom;
  const double* v[KRONOP_MAX_DIM];
  int mode;
};
__global__ void k_generate(double* out, long long n, GenArgs args) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    long long r = i;
    double acc = args.mode == 1 ? 0.0 : 1.0;
    for (int a = 0; a < args.geom.d; ++a) {
      const long long e = args.geom.n[a];
      const long long idx = r % e;
      r /= e;
      acc = args.mode == 1 ? __dadd_rn(acc, args.v[a][idx]) : __dmul_rn(acc, args.v[a][idx]);
    }
    out[i] = acc;
  }
}

void launch_generate(cudaStream_t s, Workspace& ws, double* out, const IndexGeomHost& g,
                     const double* const* vecs, int mode) {
  GenArgs args{};
  args.geom.d = g.d;
  long long n = 1;
  for (int a = 0; a < g.d; ++a) {
    args.geom.n[a] = g.n[a];
    args.v[a] = vecs[a];
    n *= g.n[a];
  }
  args.mode = mode;
  k_generate<<<kEltBlocks, kThreads, 0, s>>>(out, n, args);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

__global__ void k_splitmix(double* out, unsigned long long seed, unsigned long long start,
                           long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    unsigned long long z = seed + (start + static_cast<unsigned long long>(i) + 1ull) *
                                      0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    out[i] = static_cast<double>(z >> 11) * 0x1.0p-52 - 1.0;
  }
}

void launch_splitmix(cudaStream_t s, Workspace& ws, double* out, unsigned long long seed,
                     unsigned long long start, long long n) {
  k_splitmix<<<kEltBlocks, kThreads, 0, s>>>(out, seed, start, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// Self-test of the batched division fast path used by the TMA divide epilogue: out[i] = 1 where
// div_rn_fast (with the __ddiv_rn fallback) differs from __ddiv_rn bit for bit, else 0.
__global__ void k_div_selftest(const double* a, const double* b, unsigned long long* bad,
                               long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  unsigned long long cnt = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    bool ok;
    double q = kronop_dev::div_rn_fast(a[i], b[i], ok);
    const double ref = __ddiv_rn(a[i], b[i]);
    if (!ok) q = __ddiv_rn(a[i], b[i]);
    if (__double_as_longlong(q) != __double_as_longlong(ref)) ++cnt;
  }
  if (cnt) atomicAdd(bad, cnt);
}

void launch_div_selftest(cudaStream_t s, Workspace& ws, const double* a, const double* b,
                         unsigned long long* bad, long long n) {
  k_div_selftest<<<kEltBlocks, kThreads, 0, s>>>(a, b, bad, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// interleaved complex from a real field (psi0[i] = real[i]) and axpy helpers
__global__ void k_axpby(double* y, const double* x, double a, double b, long long n) {
  // y = a x + b y   (used for r = b - A x and diff = psi - ref)
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    y[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
}

void launch_axpby(cudaStream_t s, Workspace& ws, double* y, const double* x, double a, double b,
                  long long n) {
  k_axpby<<<kEltBlocks, kThreads, 0, s>>>(y, x, a, b, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// y = x - b  (plain difference, no scaling: r = b - Ax written as r = b; r -= ax in pcg.cpp:21-24)
__global__ void k_sub(double* y, const double* x, const double* b, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    y[i] = __dsub_rn(x[i], b[i]);
}

void launch_sub(cudaStream_t s, Workspace& ws, double* y, const double* x, const double* b,
                long long n) {
  k_sub<<<kEltBlocks, kThreads, 0, s>>>(y, x, b, n);
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

// --------------------------------------------------------------- even/odd folding --
// Element (p, i, q) at p + pre * (i + n * q). Rows (i, q) are walked by blocks when pre is wide
// (threads over p, coalesced); for pre < 32 a block walks whole q-slabs of pre * n contiguous
// doubles (i = e / pre with a small divisor).
__device__ __forceinline__ double fold_value(const double* x, long long base, long long pre, int n,
                                             int i) {
  const int no = n / 2, ne = n - no;
  if (i < no) return __dadd_rn(x[base + pre * i], x[base + pre * (n - 1 - i)]);
  if (i < ne) return x[base + pre * i];  // middle node (n odd)
  const int j = i - ne;
  return __dsub_rn(x[base + pre * j], x[base + pre * (n - 1 - j)]);
}
__device__ __forceinline__ double unfold_value(const double* z, long long base, long long pre,
                                               int n, int i) {
  const int no = n / 2, ne = n - no;
  if (i < no) return __dadd_rn(z[base + pre * i], z[base + pre * (ne + i)]);
  const int j = n - 1 - i;
  if (j < no) return __dsub_rn(z[base + pre * j], z[base + pre * (ne + j)]);
  return z[base + pre * no];  // middle node
}

// one (i, mirror) pair per row: both outputs from the same two loads (each input read once)
__device__ __forceinline__ double fold_axpy(double v, long long yi, const double* diag,
                                            const double* u, double sigma, int cplx) {
  const double uu = u[yi];
  if (diag) v = __dadd_rn(v, __dmul_rn(diag[cplx ? (yi >> 1) : yi], uu));
  if (sigma != 0.0) v = __dsub_rn(v, __dmul_rn(sigma, uu));
  return v;
}
template <bool UNFOLD>
__global__ void k_fold_wide(const double* __restrict__ x, double* __restrict__ y, long long pre,
                            int n, long long post, const double* diag, const double* u,
                            double sigma, int cplx) {
  const int no = n / 2, ne = n - no;
  const long long rows = static_cast<long long>(ne) * post;
  const bool axpy = UNFOLD && (diag || sigma != 0.0);
  // work items = (pair row, chunk of the pre range): enough blocks in flight even when there
  // are few pair rows (the slowest axis of a 1024^3 field: 512 rows of 1 M elements)
  constexpr long long kChunk = 16384;
  const long long nch = (pre + kChunk - 1) / kChunk;
  for (long long w = blockIdx.x; w < rows * nch; w += gridDim.x) {
    const long long row = w / nch;
    const long long p0 = (w - row * nch) * kChunk;
    const long long p1 = p0 + kChunk < pre ? p0 + kChunk : pre;
    const long long q = row / ne;
    const int i = static_cast<int>(row - q * ne);
    const long long base = pre * n * q;
    // fold: (x_i, x_{n-1-i}) -> (y_i, y_{ne+i});  unfold: (z_i, z_{ne+i}) -> (y_i, y_{n-1-i})
    const long long s0 = base + pre * i;
    const long long s1 = base + pre * (UNFOLD ? ne + i : n - 1 - i);
    const long long d0 = base + pre * i;
    const long long d1 = base + pre * (UNFOLD ? n - 1 - i : ne + i);
    const bool mid = i >= no;  // middle node (n odd): a copy
    for (long long p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
      const double a = x[s0 + p];
      if (mid) {
        y[d0 + p] = axpy ? fold_axpy(a, d0 + p, diag, u, sigma, cplx) : a;
        continue;
      }
      const double b = x[s1 + p];
      double v0 = __dadd_rn(a, b), v1 = __dsub_rn(a, b);
      if (axpy) {
        v0 = fold_axpy(v0, d0 + p, diag, u, sigma, cplx);
        v1 = fold_axpy(v1, d1 + p, diag, u, sigma, cplx);
      }
      y[d0 + p] = v0;
      y[d1 + p] = v1;
    }
  }
}

template <bool UNFOLD>
__global__ void k_fold_narrow(const double* __restrict__ x, double* __restrict__ y, int pre, int n,
                              long long post, const double* diag, const double* u, double sigma,
                              int cplx) {
  const int span = pre * n;
  for (long long q = blockIdx.x; q < post; q += gridDim.x) {
    const long long base = static_cast<long long>(span) * q;
    for (int e = threadIdx.x; e < span; e += blockDim.x) {
      const int i = pre == 1 ? e : pre == 2 ? (e >> 1) : e / pre;
      const int p = e - i * pre;
      double v = UNFOLD ? unfold_value(x, base + p, pre, n, i) : fold_value(x, base + p, pre, n, i);
      const long long yi = base + e;
      if (UNFOLD && (diag || sigma != 0.0)) {
        const double uu = u[yi];
        if (diag) v = __dadd_rn(v, __dmul_rn(diag[cplx ? (yi >> 1) : yi], uu));
        if (sigma != 0.0) v = __dsub_rn(v, __dmul_rn(sigma, uu));
      }
      y[yi] = v;
    }
  }
}

static void launch_fold_impl(cudaStream_t s, Workspace& ws, const double* x, double* y,
                             long long pre, int n, long long post, const double* diag,
                             const double* u, double sigma, int cplx, bool unfold) {
  if (pre >= 32) {
    const long long rows = static_cast<long long>(n - n / 2) * post * ((pre + 16383) / 16384);
    const unsigned grid = static_cast<unsigned>(rows < 1184 * 4 ? rows : 1184 * 4);
    const int thr = pre >= 256 ? 256 : 128;
    if (unfold)
      k_fold_wide<true><<<grid, thr, 0, s>>>(x, y, pre, n, post, diag, u, sigma, cplx);
    else
      k_fold_wide<false><<<grid, thr, 0, s>>>(x, y, pre, n, post, diag, u, sigma, cplx);
  } else {
    const unsigned grid = static_cast<unsigned>(post < 1184 * 4 ? post : 1184 * 4);
    if (unfold)
      k_fold_narrow<true><<<grid, 256, 0, s>>>(x, y, static_cast<int>(pre), n, post, diag, u,
                                               sigma, cplx);
    else
      k_fold_narrow<false><<<grid, 256, 0, s>>>(x, y, static_cast<int>(pre), n, post, diag, u,
                                                sigma, cplx);
  }
  ws.launches += 1;
  KCUDA(cudaGetLastError());
}

void launch_fold(cudaStream_t s, Workspace& ws, const double* x, double* y, long long pre, int n,
                 long long post) {
  launch_fold_impl(s, ws, x, y, pre, n, post, nullptr, nullptr, 0.0, 0, false);
}

void launch_unfold(cudaStream_t s, Workspace& ws, const double* z, double* y, long long pre, int n,
                   long long post, const double* diag, const double* u, double sigma, int cplx) {
  launch_fold_impl(s, ws, z, y, pre, n, post, diag, u, sigma, cplx, true);
}

}  // namespace kronop_dev
