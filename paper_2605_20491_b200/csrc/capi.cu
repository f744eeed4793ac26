// extern "C" boundary (include/kronop_cuda.h): context, operators, tensor ops and the host setup
// entry points. Drivers (pcg / inverse iteration / gpe / splitting) are in drivers.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "context.cuh"
#include "host_setup.hpp"

namespace kronop_dev {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

template <class F>
int guard(F&& f) {
  try {
    f();
    return KRONOP_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return KRONOP_ECAPABILITY;
  } catch (const std::exception& e) {
    set_error(e.what());
    return KRONOP_ERUNTIME;
  }
}

View make_view(int d, const int* shape, int cplx) {
  param_check(d >= 1 && d <= KRONOP_MAX_DIM, "TensorField: dimension must be in [1, 9]");
  View v;
  v.cplx = cplx ? 1 : 0;
  v.nd = d + v.cplx;
  if (v.cplx) v.ext[0] = 2;
  for (int a = 0; a < d; ++a) {
    param_check(shape[a] >= 1, "TensorField: extents must be positive");
    v.ext[a + v.cplx] = shape[a];
  }
  return v;
}

void ensure_scratch(kronop_ctx& ctx, size_t doubles) {
  if (doubles <= ctx.scratch_cap) return;
  for (auto& p : ctx.scratch) {
    if (p) KCUDA(cudaFreeAsync(p, ctx.stream));
    p = nullptr;
  }
  ctx.scratch_cap = 0;
  for (auto& p : ctx.scratch) KCUDA(cudaMallocAsync(&p, doubles * sizeof(double), ctx.stream));
  ctx.scratch_cap = doubles;
}

double* pool_get(kronop_ctx& ctx, size_t n) {
  kronop_ctx::Block* best = nullptr;
  for (auto& b : ctx.pool)
    if (!b.used && b.cap >= n && (!best || b.cap < best->cap)) best = &b;
  if (best) {
    best->used = true;
    return best->p;
  }
  double* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(double)) != cudaSuccess) {
    (void)cudaGetLastError();
    pool_trim(ctx);  // give the idle blocks back and retry once
    KCUDA(cudaMalloc(&p, n * sizeof(double)));
  }
  ctx.pool.push_back({p, n, true});
  return p;
}

void pool_trim(kronop_ctx& ctx) {
  KCUDA(cudaStreamSynchronize(ctx.stream));
  std::vector<kronop_ctx::Block> keep;
  for (auto& b : ctx.pool) {
    if (b.used)
      keep.push_back(b);
    else
      KCUDA(cudaFree(b.p));
  }
  ctx.pool.swap(keep);
}

void pool_put(kronop_ctx& ctx, double* p) {
  for (auto& b : ctx.pool)
    if (b.p == p) {
      b.used = false;
      return;
    }
}

double* ensure_tmp(kronop_ctx& ctx, size_t doubles) {
  if (doubles > ctx.tmp_cap) {
    if (ctx.tmp) KCUDA(cudaFreeAsync(ctx.tmp, ctx.stream));
    ctx.tmp = nullptr;
    KCUDA(cudaMallocAsync(&ctx.tmp, doubles * sizeof(double), ctx.stream));
    ctx.tmp_cap = doubles;
  }
  return ctx.tmp;
}

void run_pass(kronop_ctx& ctx, const double* x, double* y, View& v, int raxis, const double* a,
              int lda, int m, const EpiParams& ep) {
  PassShape ps;
  for (int i = 0; i < raxis; ++i) ps.pre *= v.ext[i];
  for (int i = raxis + 1; i < v.nd; ++i) ps.post *= v.ext[i];
  ps.nk = static_cast<int>(v.ext[raxis]);
  ps.m = m;
  launch_mode_product(ctx.stream, x, y, a, lda, ps, ep);
  ctx.ws.launches += 1;
  v.ext[raxis] = m;
}

// Small-extent path: consecutive axes fused per HBM round trip (fused_rot.cu).
static bool use_fused_small(const kronop_op& op) {
  static const bool disabled = [] {
    const char* e = getenv("KRONOP_DISABLE_FUSED_SMALL");  // A/B switch for profiling
    return e && e[0] == '1';
  }();
  if (disabled) return false;
  for (int a = 0; a < op.d; ++a)
    if (op.n[a] > 32) return false;
  return true;
}

// Even/odd folded operator (kronop_op_create_folded): per axis, fold into [u | v] halves, two
// half-size DMMA passes on the sub-ranges (PassShape ldx/ldy = the full axis stride), and on the
// way back two half-size passes then unfold. Half the flops of the dense pass per axis at the
// cost of one extra HBM round trip (fold/unfold) per axis and direction.
static void sep_transform_folded(kronop_ctx& ctx, const kronop_op& op, const double* in,
                                 double* out, int cplx, SepKind kind, double shift, double dt,
                                 const double* diag, double sigma) {
  View v = make_view(op.d, op.n, cplx);
  ensure_scratch(ctx, static_cast<size_t>(v.total()));
  double* s0 = ctx.scratch[0];
  double* s1 = ctx.scratch[1];
  const int d = op.d;
  auto geom = [&](int a, long long& pre, long long& post) {
    const int ra = a + v.cplx;
    pre = 1;
    post = 1;
    for (int i = 0; i < ra; ++i) pre *= v.ext[i];
    for (int i = ra + 1; i < v.nd; ++i) post *= v.ext[i];
  };
  auto halves = [&](int a, const double* x, double* y, bool forward, const EpiParams& ep0) {
    long long pre, post;
    geom(a, pre, post);
    const int n = op.n[a];
    for (int h = 0; h < 2; ++h) {
      const int m = h == 0 ? op.ne[a] : op.no[a];
      if (m == 0) continue;
      const long long off = h == 0 ? 0 : pre * op.ne[a];
      PassShape ps;
      ps.pre = pre;
      ps.post = post;
      ps.nk = m;
      ps.m = m;
      ps.ldx = pre * n;
      ps.ldy = pre * n;
      EpiParams ep = ep0;
      if (ep.kind != EPI_STORE) ep.lam[a + v.cplx] = op.lam[a] + (h == 0 ? 0 : op.ne[a]);
      const double* mat = forward ? (h == 0 ? op.fe[a] : op.fo[a]) : (h == 0 ? op.be[a] : op.bo[a]);
      const int lda = h == 0 ? op.lda_e[a] : op.lda_o[a];
      launch_mode_product(ctx.stream, x + off, y + off, mat, lda, ps, ep);
      ctx.ws.launches += 1;
    }
  };
  const double* cur = in;
  for (int a = 0; a < d; ++a) {
    long long pre, post;
    geom(a, pre, post);
    launch_fold(ctx.stream, ctx.ws, cur, s0, pre, op.n[a], post);
    EpiParams ep;
    if (a == d - 1) {
      ep.kind = kind == SEP_APPLY ? EPI_SPEC_MUL : kind == SEP_SOLVE ? EPI_SPEC_DIV : EPI_SPEC_PHASE;
      ep.axis = a + v.cplx;
      ep.ndims = v.nd;
      for (int i = 0; i < v.nd; ++i) ep.ext[i] = v.ext[i];
      for (int b = 0; b < d; ++b) ep.lam[b + v.cplx] = op.lam[b];
      ep.shift = shift;
      ep.dt = dt;
      ep.cplx = v.cplx;
    }
    halves(a, s0, s1, true, ep);
    cur = s1;
  }
  for (int a = 0; a < d; ++a) {
    long long pre, post;
    geom(a, pre, post);
    halves(a, s1, s0, false, EpiParams{});
    const bool last = a == d - 1;
    launch_unfold(ctx.stream, ctx.ws, s0, last ? out : s1, pre, op.n[a], post,
                  last ? diag : nullptr, last ? in : nullptr, last ? sigma : 0.0, v.cplx);
  }
}

// Kronecker-factored propagate (kron_prop.cu) for complex fields whose axes all have n <= 10:
// e^{-i (lambda - shift) dt} applied as e^{i shift dt} (x)_a E_a with
// E_a = T_a diag(e^{-i lambda_a dt}) T_a^{-1} (operators.cpp:63-75 re-associated: the exponential
// of a Kronecker sum is the Kronecker product of the exponentials). E_a is formed here in extended
// precision from the host copies of T, T^{-1}, lambda; the shift's phase goes into the first
// axis. Row-major [i][k] complex (re, im), as the kernel reads it.
static void kron_prop_matrix(const kronop_op& op, int a, double dt, double shift_phase,
                             double* E) {
  const int n = op.n[a];
  const std::vector<double>& T = op.hT[a];
  const std::vector<double>& Ti = op.hTinv[a];
  std::vector<long double> cr(n), ci(n);
  for (int m = 0; m < n; ++m) {
    const long double ph = -static_cast<long double>(op.hlam[a][m]) * dt;
    cr[m] = std::cos(ph);
    ci[m] = std::sin(ph);
  }
  const long double gr = std::cos(static_cast<long double>(shift_phase));
  const long double gi = std::sin(static_cast<long double>(shift_phase));
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      long double sr = 0.0L, si = 0.0L;
      for (int m = 0; m < n; ++m) {
        const long double t = static_cast<long double>(T[i + static_cast<size_t>(n) * m]) *
                              Ti[m + static_cast<size_t>(n) * k];
        sr += t * cr[m];
        si += t * ci[m];
      }
      E[2 * (i * n + k)] = static_cast<double>(sr * gr - si * gi);
      E[2 * (i * n + k) + 1] = static_cast<double>(sr * gi + si * gr);
    }
}

// Parity symmetry of an axis propagator: R E R = E (R: i -> n-1-i) to rounding (64 ulp of the
// largest entry). Exact for a symmetric box with an even potential; E's asymmetry is then only
// the rounding of T, T^{-1}.
static bool kron_fold_symmetric(const double* E, int n) {
  double emax = 0.0, dmax = 0.0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const double* a = E + 2 * (i * n + k);
      const double* b = E + 2 * ((n - 1 - i) * n + (n - 1 - k));
      emax = std::max(emax, std::max(std::abs(a[0]), std::abs(a[1])));
      dmax = std::max(dmax, std::max(std::abs(a[0] - b[0]), std::abs(a[1] - b[1])));
    }
  return n >= 2 && dmax <= 64.0 * 2.220446049250313e-16 * emax;
}

// E (n x n complex, row-major) -> its parity blocks in place: Ae ((M+c) x (M+c)) then Ao (M x M),
// M = n / 2, c = n % 2 (the layout kr_contract reads with FOLD).
static void kron_fold_blocks(double* E, int n) {
  const int M = n / 2, ME = M + n % 2;
  std::vector<double> out(static_cast<size_t>(n) * n * 2, 0.0);
  auto at = [&](int i, int k, int c) { return E[2 * (i * n + k) + c]; };
  for (int i = 0; i < ME; ++i)
    for (int k = 0; k < ME; ++k)
      for (int c = 0; c < 2; ++c)
        out[2 * (i * ME + k) + c] = k < M ? 0.5 * (at(i, k, c) + at(i, n - 1 - k, c)) : at(i, k, c);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < M; ++k)
      for (int c = 0; c < 2; ++c)
        out[2 * (ME * ME + i * M + k) + c] = 0.5 * (at(i, k, c) - at(i, n - 1 - k, c));
  std::copy(out.begin(), out.end(), E);
}

// Groups for the Kronecker propagate: up to three consecutive axes of the same extent n <= 10
// (DFMA kernel), or up to two of the same extent 11..32 with n^2 <= 1024 (DMMA kernel, parity-
// symmetric axes only); empty when some axis is outside that range or the host copies are
// missing.
static std::vector<std::pair<int, int>> kron_groups(const kronop_op& op) {
  std::vector<std::pair<int, int>> groups;
  static const bool off = [] {
    const char* e = getenv("KRONOP_KRON_PROP");  // A/B switch: 0 = transform / phase / transform
    return e && e[0] == '0';
  }();
  if (off || op.folded || op.exec_prec != KRONOP_PREC_FP64) return groups;
  for (int a = 0; a < op.d; ++a)
    if (op.hT[a].empty() || !kron_group_supported(op.n[a], 1)) return groups;
  for (int a = 0; a < op.d;) {
    const int fmax = op.n[a] <= 10 ? 3 : 2;
    int f = 1;
    while (a + f < op.d && f < fmax && op.n[a + f] == op.n[a]) ++f;
    groups.emplace_back(a, f);
    a += f;
  }
  return groups;
}

static bool sep_propagate_kron(kronop_ctx& ctx, const kronop_op& op, const double* in, double* out,
                               double shift, double dt, bool bphase, const double* bfield,
                               double bfactor, const double* pre = nullptr) {
  const std::vector<std::pair<int, int>> groups = kron_groups(op);
  if (groups.empty() || !fused_rot_eligible(in) || !fused_rot_eligible(out)) return false;
  static const bool no_fold = [] {
    const char* e = getenv("KRONOP_KRON_FOLD");  // A/B switch: 0 = dense E_a even when symmetric
    return e && e[0] == '0';
  }();
  const int ng = static_cast<int>(groups.size());
  // every group's matrices first: a group the kernels cannot take (an extent > 10 whose axis is
  // not parity symmetric) sends the whole propagate to the transform / phase / transform path
  constexpr size_t kSlot = 3 * 32 * 32 * 2;
  std::vector<double> E(kSlot * ng);
  std::vector<char> fold(ng);
  for (int g = 0; g < ng; ++g) {
    const int a0 = groups[g].first, f = groups[g].second, n = op.n[a0];
    bool fl = !no_fold || kron_group_needs_fold(n);
    for (int j = 0; j < f; ++j) {
      double* e = E.data() + kSlot * g + static_cast<size_t>(j) * n * n * 2;
      kron_prop_matrix(op, a0 + j, dt, (g == 0 && j == 0) ? shift * dt : 0.0, e);
      fl = fl && kron_fold_symmetric(e, n);
    }
    if (!fl && kron_group_needs_fold(n)) return false;
    if (fl)
      for (int j = 0; j < f; ++j)
        kron_fold_blocks(E.data() + kSlot * g + static_cast<size_t>(j) * n * n * 2, n);
    fold[g] = fl;
  }
  const size_t nd = static_cast<size_t>(op.N) * 2;
  ensure_scratch(ctx, nd);
  const double* src = in;
  for (int g = 0; g < ng; ++g) {
    const int a0 = groups[g].first, f = groups[g].second, n = op.n[a0];
    const bool last = g == ng - 1;
    // a launch must not write its own input (other CTAs still read the tiles it overwrites)
    double* dst = (last && src != out) ? out
                  : src == ctx.scratch[0]  ? ctx.scratch[1]
                                           : ctx.scratch[0];
    launch_kron_group(ctx.stream, src, dst, n, f, fold[g] != 0, op.N, E.data() + kSlot * g,
                      last && bphase ? bfield : nullptr, bfactor, last && bphase ? 1 : 0,
                      g == 0 ? pre : nullptr);
    ctx.ws.launches += 1;
    src = dst;
  }
  if (src != out)
    KCUDA(cudaMemcpyAsync(out, src, nd * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
  return true;
}

// psi <- e^{-i(A - shift) dt} (e^{-i factor B} psi) in place: the split-step's B phase followed
// by its next A propagation, with the phase applied by the Kronecker kernel's first group as it
// reads psi (pre_tab = the (cos, sin) table of k_phase's operations; bit-identical to the phase
// pass followed by the propagate). Returns false when the propagate does not take the Kronecker
// path (the caller then runs the phase pass and the propagate).
bool kron_path_likely(const kronop_op& op) {
  return op.exec_prec == KRONOP_PREC_FP64 && !op.folded && use_fused_small(op) &&
         !kron_groups(op).empty();
}

bool sep_propagate_prephased(kronop_ctx& ctx, const kronop_op& op, double* psi, double shift,
                             double dt, const double* pre_tab) {
  if (op.exec_prec != KRONOP_PREC_FP64 || op.folded || !use_fused_small(op)) return false;
  return sep_propagate_kron(ctx, op, psi, psi, shift, dt, false, nullptr, 0.0, pre_tab);
}

// Real fields whose axes all have n <= 10 (the config-5 9D solves / applies of inverse
// iteration): the transform form on kron_real_kernel (kron_prop.cu) -- the real axis matrices as
// kernel parameters, 1 CTA x 3 stages over contiguous tile ranges; the same operations and
// order as fused_rot's DFMA path (identical results, KRONOP_KRON_REAL=0 selects fused_rot).
static bool sep_transform_real_kron(kronop_ctx& ctx, const kronop_op& op, const double* in,
                                    double* out, SepKind kind, double shift, const double* diag,
                                    double sigma) {
  static const bool off = [] {
    const char* e = getenv("KRONOP_KRON_REAL");
    return e && e[0] == '0';
  }();
  if (off || op.folded || op.exec_prec != KRONOP_PREC_FP64 || kind == SEP_PROPAGATE) return false;
  if (!fused_rot_eligible(in)) return false;
  for (int a = 0; a < op.d; ++a)
    if (op.hT[a].empty() || !kron_real_supported(op.n[a], 1)) return false;
  std::vector<std::pair<int, int>> groups;
  for (int a = 0; a < op.d;) {
    int f = 1;
    while (a + f < op.d && f < 3 && op.n[a + f] == op.n[a]) ++f;
    groups.emplace_back(a, f);
    a += f;
  }
  const size_t nd = static_cast<size_t>(op.N);
  ensure_scratch(ctx, nd);
  const int ng = static_cast<int>(groups.size());
  std::vector<double> M(3 * 10 * 10);
  const double* src = in;
  int k = 0;
  for (int dir = 0; dir < 2; ++dir)
    for (int g = 0; g < ng; ++g, ++k) {
      const int a0 = groups[g].first, f = groups[g].second, n = op.n[a0];
      const bool last = dir == 1 && g == ng - 1;
      for (int j = 0; j < f; ++j) {
        const std::vector<double>& T = dir == 0 ? op.hTinv[a0 + j] : op.hT[a0 + j];
        for (int i = 0; i < n; ++i)
          for (int kk = 0; kk < n; ++kk)
            M[(j * n + i) * n + kk] = T[i + static_cast<size_t>(n) * kk];  // column-major
      }
      KronRealLaunch L;
      L.x = src;
      L.y = last ? out : ctx.scratch[k % 2];
      L.Ntot = op.N;
      L.n = n;
      L.f = f;
      L.M = M.data();
      if (dir == 0 && g == ng - 1) {
        L.epi = kind == SEP_SOLVE ? 1 : 2;
        L.shift = shift;
        for (int j = 0; j < f; ++j) L.lam_g[j] = op.lam[a0 + j];
        L.nq = a0;
        for (int j = 0; j < a0; ++j) {
          L.qext[j] = op.n[j];
          L.lam_q[j] = op.lam[j];
        }
      } else if (last && (diag != nullptr || sigma != 0.0)) {
        L.epi = 3;
        L.diag = diag;
        L.u = in;
        L.sigma = sigma;
      }
      launch_kron_real_group(ctx.stream, L);
      ctx.ws.launches += 1;
      src = L.y;
    }
  return true;
}

// Small-extent path, rotating layout (fused_rot.cu): groups of up to 3 consecutive axes (fused
// extent <= 1024), forward groups then backward groups; each launch moves its group to the slow
// end, so after each direction the layout is the caller's again.
static void sep_transform_rot(kronop_ctx& ctx, const kronop_op& op, const double* in, double* out,
                              int cplx, SepKind kind, double shift, double dt, const double* diag,
                              double sigma, bool bphase, const double* bfield, double bfactor) {
  if (kind == SEP_PROPAGATE && cplx && diag == nullptr && sigma == 0.0 &&
      sep_propagate_kron(ctx, op, in, out, shift, dt, bphase, bfield, bfactor))
    return;
  if (!cplx && sep_transform_real_kron(ctx, op, in, out, kind, shift, diag, sigma)) return;
  const size_t nd = static_cast<size_t>(op.N) * (cplx ? 2 : 1);
  ensure_scratch(ctx, nd);
  std::vector<std::pair<int, int>> groups;
  for (int a = 0; a < op.d;) {
    int f = 1, F = op.n[a];
    // three-axis groups only for extents <= 12 (the kernels' K/N instantiations for f = 3)
    while (a + f < op.d && F * op.n[a + f] <= 1024 &&
           (f < 2 || (f == 2 && op.n[a] <= 12 && op.n[a + 1] <= 12 && op.n[a + 2] <= 12)))
      F *= op.n[a + f++];
    groups.emplace_back(a, f);
    a += f;
  }
  const double* src = in;
  if (!fused_rot_eligible(in)) {  // bulk copies need 16-byte aligned tiles
    double* t = ensure_tmp(ctx, nd);
    KCUDA(cudaMemcpyAsync(t, in, nd * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
    src = t;
  }
  const int ng = static_cast<int>(groups.size());
  int k = 0;
  for (int dir = 0; dir < 2; ++dir)
    for (int g = 0; g < ng; ++g, ++k) {
      const int a0 = groups[g].first, f = groups[g].second;
      const bool last = dir == 1 && g == ng - 1;
      double* dst = last ? out : ctx.scratch[k % 2];
      const double* mats[3];
      int lda[3], n[3];
      for (int j = 0; j < f; ++j) {
        mats[j] = dir == 0 ? op.fwd[a0 + j] : op.bwd[a0 + j];
        lda[j] = op.lda[a0 + j];
        n[j] = op.n[a0 + j];
      }
      RotEpi e;
      if (dir == 0 && g == ng - 1) {
        e.kind = kind == SEP_APPLY ? EPI_SPEC_MUL : kind == SEP_SOLVE ? EPI_SPEC_DIV : EPI_SPEC_PHASE;
        e.shift = shift;
        e.dt = dt;
        for (int j = 0; j < f; ++j) e.lam_g[j] = op.lam[a0 + j];
        e.nq = a0;
        for (int j = 0; j < a0; ++j) {
          e.qext[j] = op.n[j];
          e.lam_q[j] = op.lam[j];
        }
      } else if (last && (diag != nullptr || sigma != 0.0)) {
        e.kind = EPI_AXPY_DIAG;
        e.diag = diag;
        e.u = in;
        e.sigma = sigma;
      } else if (last && bphase) {
        e.kind = EPI_BPHASE;
        e.diag = bfield;
        e.dt = bfactor;
      }
      ctx.ws.launches += launch_fused_rot(ctx.stream, src, dst, cplx, f, n, op.N, mats, lda, e);
      src = dst;
    }
}

// Rotated pass sequence for the large-extent path: every pass contracts the fastest axis after
// the re/im axis and writes its output axis to the SLOWEST end (y = r + R i), so the next axis is
// the fastest again and after d passes the layout is the original one. Every pass then reads
// through the CONTIG (real) / CPLX0 (complex) TMA loader -- the STRIDED loader the passes on axes
// 1..d-1 used ran at 89-90% of the DMMA pipe vs ~95% (profiles/r02_pass_a1.json; cuBLAS on the
// same shapes, profiles/r02_cublas_passes.json: 61.1 / 61.5 / 61.9 ms vs 62.5 / 66.6 / 66.2 ms).
// The last forward pass's rows enumerate axes 0..d-2 in order (the same rows as the unrotated
// last-axis pass), so the fused spectral epilogue sums the eigenvalues exactly as before
// (PassShape::rot); the last backward pass writes the original layout, so the FullOperator AXPY
// and the B phase index u / V2 as before. The contraction order over k inside the DMMA differs
// between the loaders' k permutations, so results agree with the axis-order passes to rounding
// (KRONOP_ROTATE_PASSES=0 selects those; tests/test_gpu_switches.py).
static bool rotated_passes_ok(const kronop_ctx& ctx, const kronop_op& op, const double* in,
                              const double* out, const View& v) {
  static const bool off = [] {
    const char* e = getenv("KRONOP_ROTATE_PASSES");  // A/B switch: 0 = axis-order passes
    return e && e[0] == '0';
  }();
  if (off || op.d < 2 || !mode_product_tma_enabled()) return false;
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!aligned(in) || !aligned(out) || !aligned(ctx.scratch[0]) || !aligned(ctx.scratch[1]))
    return false;
  for (int a = 0; a < op.d; ++a) {
    if ((!v.cplx && op.n[a] % 2 != 0) || op.n[a] < 2) return false;  // CONTIG rows of even length
    if (v.total() / op.n[a] > 0x7fffffffLL) return false;  // rows: TMA coordinates are 32-bit
  }
  return true;
}

static void sep_transform_rotated(kronop_ctx& ctx, const kronop_op& op, const double* in,
                                  double* out, const View& v, SepKind kind, double shift,
                                  double dt, const double* diag, double sigma, bool bphase,
                                  const double* bfield, double bfactor) {
  const int d = op.d;
  const long long c = v.cplx ? 2 : 1;
  const long long total = v.total();
  const double* cur = in;
  for (int k = 0; k < 2 * d; ++k) {
    const bool forward = k < d;
    const int axis = forward ? k : k - d;
    double* dst = (k == 2 * d - 1) ? out : ctx.scratch[k % 2];
    PassShape ps;
    ps.pre = c;
    ps.nk = op.n[axis];
    ps.m = op.n[axis];
    ps.post = total / (c * op.n[axis]);
    ps.ldy = c;                   // ybase = r
    ps.ycol = total / op.n[axis];  // output axis at the slow end
    ps.rot = 1;
    EpiParams ep;
    if (k == d - 1) {  // the spectral epilogue, rows = axes 0..d-2 in order (as the unrotated pass)
      ep.kind = kind == SEP_APPLY ? EPI_SPEC_MUL : kind == SEP_SOLVE ? EPI_SPEC_DIV : EPI_SPEC_PHASE;
      ep.axis = d - 1 + v.cplx;
      ep.ndims = v.nd;
      for (int i = 0; i < v.nd; ++i) ep.ext[i] = v.ext[i];
      for (int a = 0; a < d; ++a) ep.lam[a + v.cplx] = op.lam[a];
      ep.shift = shift;
      ep.dt = dt;
      ep.cplx = v.cplx;
    }
    if (k == 2 * d - 1 && (diag != nullptr || sigma != 0.0)) {
      ep.kind = EPI_AXPY_DIAG;
      ep.diag = diag;
      ep.u = in;
      ep.sigma = sigma;
      ep.cplx = v.cplx;
    } else if (k == 2 * d - 1 && bphase) {
      ep.kind = EPI_BPHASE;
      ep.diag = bfield;
      ep.dt = bfactor;
      ep.cplx = v.cplx;
    }
    launch_mode_product(ctx.stream, cur, dst, forward ? op.fwd[axis] : op.bwd[axis],
                        op.lda[axis], ps, ep);
    ctx.ws.launches += 1;
    cur = dst;
  }
}

void sep_transform(kronop_ctx& ctx, const kronop_op& op, const double* in, double* out, int cplx,
                   SepKind kind, double shift, double dt, const double* diag, double sigma,
                   bool bphase, const double* bfield, double bfactor) {
  param_check(!bphase || (kind == SEP_PROPAGATE && cplx), "B phase: complex propagate only");
  if (bphase && (op.folded || op.exec_prec >= KRONOP_PREC_FP64_OZAKI)) {
    // paths without the fused epilogue: the phase as its own pass (k_phase)
    sep_transform(ctx, op, in, out, cplx, kind, shift, dt, diag, sigma);
    launch_phase(ctx.stream, ctx.ws, out, bfield, bfactor, op.N);
    return;
  }
  if (op.exec_prec >= KRONOP_PREC_FP64_OZAKI && (kind != SEP_PROPAGATE || cplx)) {
    // kronop_op_set_precision: every transform of this operator on the INT8 path (ozaki.cu)
    const int epi = kind == SEP_SOLVE ? 1 : kind == SEP_APPLY ? 2 : 3;
    sep_ozaki(ctx, const_cast<kronop_op&>(op), in, out, cplx, epi, shift, dt, diag, sigma,
              7 - (op.exec_prec - KRONOP_PREC_FP64_OZAKI));
    return;
  }
  if (op.folded) {
    sep_transform_folded(ctx, op, in, out, cplx, kind, shift, dt, diag, sigma);
    return;
  }
  if (use_fused_small(op)) {
    sep_transform_rot(ctx, op, in, out, cplx, kind, shift, dt, diag, sigma, bphase, bfield,
                      bfactor);
    return;
  }
  View v = make_view(op.d, op.n, cplx);
  ensure_scratch(ctx, static_cast<size_t>(v.total()));
  const int d = op.d;
  const double* cur = in;
  if (rotated_passes_ok(ctx, op, in, out, v)) {
    sep_transform_rotated(ctx, op, in, out, v, kind, shift, dt, diag, sigma, bphase, bfield,
                          bfactor);
    return;
  }
  for (int k = 0; k < 2 * d; ++k) {
    const bool forward = k < d;
    const int axis = forward ? k : k - d;
    double* dst = (k == 2 * d - 1) ? out : ctx.scratch[k % 2];
    EpiParams ep;
    if (k == d - 1) {
      ep.kind = kind == SEP_APPLY ? EPI_SPEC_MUL : kind == SEP_SOLVE ? EPI_SPEC_DIV : EPI_SPEC_PHASE;
      ep.axis = axis + v.cplx;
      ep.ndims = v.nd;
      for (int i = 0; i < v.nd; ++i) ep.ext[i] = v.ext[i];
      for (int a = 0; a < d; ++a) ep.lam[a + v.cplx] = op.lam[a];
      ep.shift = shift;
      ep.dt = dt;
      ep.cplx = v.cplx;
    }
    if (k == 2 * d - 1 && (diag != nullptr || sigma != 0.0)) {
      ep.kind = EPI_AXPY_DIAG;
      ep.diag = diag;
      ep.u = in;
      ep.sigma = sigma;
      ep.cplx = v.cplx;
    } else if (k == 2 * d - 1 && bphase) {
      ep.kind = EPI_BPHASE;
      ep.diag = bfield;
      ep.dt = bfactor;
      ep.cplx = v.cplx;
    }
    run_pass(ctx, cur, dst, v, axis + v.cplx, forward ? op.fwd[axis] : op.bwd[axis], op.lda[axis],
             op.n[axis], ep);
    cur = dst;
  }
}

// min |lambda - shift| over the direct-sum grid (device, deterministic min-reduction)
struct GapArgs {
  int d;
  long long n[KRONOP_MAX_DIM];
  const double* lam[KRONOP_MAX_DIM];
  double shift;
  long long total;
};
__global__ void k_gap_partial(GapArgs a, double* partials) {
  __shared__ double sh[256];
  double best = INFINITY;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < a.total;
       i += stride) {
    long long r = i;
    double s = 0.0;
    for (int ax = 0; ax < a.d; ++ax) {
      const long long idx = r % a.n[ax];
      r /= a.n[ax];
      s = __dadd_rn(s, a.lam[ax][idx]);
    }
    best = fmin(best, fabs(__dsub_rn(s, a.shift)));
  }
  sh[threadIdx.x] = best;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = fmin(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

void check_solve_shift(kronop_ctx& ctx, const kronop_op& op, double shift) {
  const double floor = 1e-14 * std::max(std::abs(op.lmin), std::abs(op.lmax));
  double closest = std::min(std::abs(op.lmin - shift), std::abs(op.lmax - shift));
  if (shift > op.lmin && shift < op.lmax) {
    GapArgs a{};
    a.d = op.d;
    for (int i = 0; i < op.d; ++i) {
      a.n[i] = op.n[i];
      a.lam[i] = op.lam[i];
    }
    a.shift = shift;
    a.total = op.N;
    k_gap_partial<<<kRedBlocks, 256, 0, ctx.stream>>>(a, ctx.ws.partials);
    KCUDA(cudaGetLastError());
    ctx.ws.launches += 1;
    std::vector<double> part(kRedBlocks);
    KCUDA(cudaMemcpyAsync(part.data(), ctx.ws.partials, kRedBlocks * sizeof(double),
                          cudaMemcpyDeviceToHost, ctx.stream));
    KCUDA(cudaStreamSynchronize(ctx.stream));
    closest = *std::min_element(part.begin(), part.end());
  }
  if (closest < floor)
    fail(KRONOP_ENUMERICAL, "SeparableOperator::solve: shift coincides with an eigenvalue");
}

IndexGeomHost mass_geom(const kronop_op& op) {
  param_check(op.has_mass, "inner: field has no mass weights attached");
  IndexGeomHost g;
  g.d = op.d;
  for (int a = 0; a < op.d; ++a) {
    g.n[a] = op.n[a];
    g.mass[a] = op.mass[a];
  }
  return g;
}

// Upload a host column-major m x k matrix into a zero-padded device copy (lda = pad(m,128),
// pad(k,16) columns). Returns lda.
static int upload_padded(kronop_ctx& ctx, const double* host, int m, int k, double** dev,
                         bool allocate) {
  const int lda = pad_up(m, kMatPadM), kp = pad_up(k, kMatPadK);
  std::vector<double> hp(static_cast<size_t>(lda) * kp, 0.0);
  for (int j = 0; j < k; ++j)
    std::memcpy(&hp[static_cast<size_t>(lda) * j], host + static_cast<size_t>(m) * j,
                sizeof(double) * m);
  if (allocate) KCUDA(cudaMalloc(dev, hp.size() * sizeof(double)));
  KCUDA(cudaMemcpyAsync(*dev, hp.data(), hp.size() * sizeof(double), cudaMemcpyHostToDevice,
                        ctx.stream));
  KCUDA(cudaStreamSynchronize(ctx.stream));  // hp is a stack temporary
  return lda;
}

static void generic_kron(kronop_ctx& ctx, const double* x, int d, const int* shape, int cplx,
                         const double* const* mats, const int* ms, double* out) {
  View v = make_view(d, shape, cplx);
  // plan: sizes of every intermediate
  size_t maxsz = static_cast<size_t>(v.total());
  {
    View w = v;
    for (int a = 0; a < d; ++a) {
      if (!mats[a]) continue;
      param_check(ms[a] >= 1, "kron_apply: matrix rows must be positive");
      w.ext[a + w.cplx] = ms[a];
      maxsz = std::max(maxsz, static_cast<size_t>(w.total()));
    }
  }
  int nmat = 0, last = -1;
  size_t matsz = 0;
  for (int a = 0; a < d; ++a)
    if (mats[a]) {
      ++nmat;
      last = a;
      matsz += static_cast<size_t>(pad_up(ms[a], kMatPadM)) * pad_up(shape[a], kMatPadK);
    }
  if (nmat == 0) {
    if (out != x)
      KCUDA(cudaMemcpyAsync(out, x, v.total() * sizeof(double), cudaMemcpyDeviceToDevice,
                            ctx.stream));
    return;
  }
  ensure_scratch(ctx, maxsz);
  double* mbuf = ensure_tmp(ctx, matsz);
  std::vector<double*> dm(d, nullptr);
  std::vector<int> lda(d, 0);
  size_t off = 0;
  for (int a = 0; a < d; ++a) {
    if (!mats[a]) continue;
    dm[a] = mbuf + off;
    lda[a] = upload_padded(ctx, mats[a], ms[a], shape[a], &dm[a], false);
    off += static_cast<size_t>(lda[a]) * pad_up(shape[a], kMatPadK);
  }
  const double* cur = x;
  int k = 0;
  for (int a = 0; a < d; ++a) {
    if (!mats[a]) continue;
    double* dst = (a == last) ? out : ctx.scratch[k % 2];
    EpiParams ep;
    run_pass(ctx, cur, dst, v, a + v.cplx, dm[a], lda[a], ms[a], ep);
    cur = dst;
    ++k;
  }
}

}  // namespace kronop_dev

using namespace kronop_dev;

extern "C" {

const char* kronop_last_error(void) { return g_last_error.c_str(); }
const char* kronop_version(void) { return "kronop-b200 0.1.0 (sm_100a, FP64 DMMA)"; }

int kronop_ctx_create(int device, void* stream, kronop_ctx** out) {
  return guard([&] {
    param_check(out != nullptr, "kronop_ctx_create: null out");
    auto* c = new kronop_ctx();
    try {
      c->device = device;
      KCUDA(cudaSetDevice(device));
      if (stream) {
        c->stream = static_cast<cudaStream_t>(stream);
      } else {
        KCUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
      }
      KCUDA(cudaMalloc(&c->ws.partials, kRedBlocks * 4 * sizeof(double)));
      KCUDA(cudaMalloc(&c->dscal, kScalarSlots * sizeof(double)));
      KCUDA(cudaMemset(c->dscal, 0, kScalarSlots * sizeof(double)));
      KCUDA(cudaMallocHost(&c->hscal, kScalarSlots * sizeof(double)));
      prime_mode_product_kernels();
      prime_mode_product_tma_kernels();
      prime_fused_rot_kernels();
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int kronop_ctx_destroy(kronop_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto p : ctx->scratch) if (p) cudaFree(p);
    for (auto p : ctx->io) if (p) cudaFree(p);
    for (auto p : ctx->bio) if (p) cudaFree(p);
    for (int p = 0; p < 2; ++p) {
      if (ctx->ev_up[p]) cudaEventDestroy(ctx->ev_up[p]);
      if (ctx->ev_comp[p]) cudaEventDestroy(ctx->ev_comp[p]);
      if (ctx->ev_down[p]) cudaEventDestroy(ctx->ev_down[p]);
    }
    for (auto& b : ctx->pool) cudaFree(b.p);
    if (ctx->tmp) cudaFree(ctx->tmp);
    if (ctx->ws.partials) cudaFree(ctx->ws.partials);
    if (ctx->dscal) cudaFree(ctx->dscal);
    if (ctx->hscal) cudaFreeHost(ctx->hscal);
    for (auto st : ctx->copy_stream) if (st) cudaStreamDestroy(st);
    for (int i = 0; i < kronop_ctx::kMaxChunks; ++i) {
      if (ctx->ev_in[i]) cudaEventDestroy(ctx->ev_in[i]);
      if (ctx->ev_out[i]) cudaEventDestroy(ctx->ev_out[i]);
    }
    if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int kronop_ctx_trim(kronop_ctx* ctx) {
  return guard([&] {
    param_check(ctx != nullptr, "ctx_trim: null context");
    pool_trim(*ctx);  // synchronises the stream
    // the host-path staging (single and batched entry points) is re-made on the next call
    for (auto& p : ctx->io) {
      if (p) KCUDA(cudaFree(p));
      p = nullptr;
    }
    ctx->io_cap = 0;
    for (auto& b : ctx->bio) {
      if (b) KCUDA(cudaFree(b));
      b = nullptr;
    }
    ctx->bio_cap = 0;
  });
}

int kronop_ctx_synchronize(kronop_ctx* ctx) {
  return guard([&] { KCUDA(cudaStreamSynchronize(ctx->stream)); });
}

int kronop_ctx_workspace_bytes(kronop_ctx* ctx, size_t* bytes) {
  return guard([&] {
    *bytes = (2 * ctx->scratch_cap + ctx->tmp_cap + 2 * ctx->io_cap) * sizeof(double);
  });
}

int kronop_ctx_launch_count(kronop_ctx* ctx, uint64_t* count) {
  return guard([&] { *count = ctx->ws.launches; });
}

int kronop_field_alloc(kronop_ctx* ctx, size_t doubles, double** out) {
  return guard([&] {
    param_check(ctx && out, "field_alloc: null argument");
    KCUDA(cudaMalloc(out, std::max<size_t>(doubles, 1) * sizeof(double)));
  });
}

int kronop_field_free(kronop_ctx* ctx, double* p) {
  return guard([&] {
    if (ctx) KCUDA(cudaStreamSynchronize(ctx->stream));
    if (p) KCUDA(cudaFree(p));
  });
}

int kronop_field_upload(kronop_ctx* ctx, double* dst, const double* host, size_t doubles) {
  return guard([&] {
    KCUDA(cudaMemcpyAsync(dst, host, doubles * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
    KCUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int kronop_field_download(kronop_ctx* ctx, double* host, const double* src, size_t doubles) {
  return guard([&] {
    KCUDA(cudaMemcpyAsync(host, src, doubles * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
    KCUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int kronop_mode_product(kronop_ctx* ctx, const double* x, int d, const int* shape, int is_complex,
                        const double* a, int m, int axis, double* out) {
  return guard([&] {
    param_check(ctx && x && out && shape && a, "mode_product: null argument");
    param_check(axis >= 0 && axis < d, "mode_product: axis out of range");
    param_check(m >= 1, "mode_product: matrix rows must be positive");
    param_check(out != x, "mode_product: out must not alias x");
    std::vector<const double*> mats(d, nullptr);
    std::vector<int> ms(d, 0);
    mats[axis] = a;
    ms[axis] = m;
    generic_kron(*ctx, x, d, shape, is_complex, mats.data(), ms.data(), out);
  });
}

int kronop_kron_apply(kronop_ctx* ctx, const double* x, int d, const int* shape, int is_complex,
                      const double* const* mats, const int* m, double* out) {
  return guard([&] {
    param_check(ctx && x && out && shape && mats && m, "kron_apply: null argument");
    make_view(d, shape, is_complex);
    generic_kron(*ctx, x, d, shape, is_complex, mats, m, out);
  });
}

int kronop_inner(kronop_ctx* ctx, const double* u, const double* v, int d, const int* shape,
                 int is_complex, const double* const* mass, double* result) {
  return guard([&] {
    param_check(ctx && u && v && shape && result, "inner: null argument");
    View vw = make_view(d, shape, 0);
    const long long n = vw.total();
    IndexGeomHost g;
    IndexGeomHost* gp = nullptr;
    if (mass) {
      size_t tot = 0;
      for (int a = 0; a < d; ++a) tot += shape[a];
      double* mb = ensure_tmp(*ctx, tot);
      g.d = d;
      size_t off = 0;
      for (int a = 0; a < d; ++a) {
        KCUDA(cudaMemcpyAsync(mb + off, mass[a], shape[a] * sizeof(double), cudaMemcpyHostToDevice,
                              ctx->stream));
        g.n[a] = shape[a];
        g.mass[a] = mb + off;
        off += shape[a];
      }
      gp = &g;
    }
    launch_dot(ctx->stream, ctx->ws, u, v, n, is_complex, gp, ctx->dscal);
    KCUDA(cudaMemcpyAsync(ctx->hscal, ctx->dscal, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
    KCUDA(cudaStreamSynchronize(ctx->stream));
    result[0] = ctx->hscal[0];
    if (is_complex) result[1] = ctx->hscal[1];
  });
}

static void generate_from_host(kronop_ctx* ctx, int d, const int* shape,
                               const double* const* vecs, int mode, double* out) {
  View vw = make_view(d, shape, 0);
  size_t tot = 0;
  for (int a = 0; a < d; ++a) tot += shape[a];
  double* mb = ensure_tmp(*ctx, tot);
  IndexGeomHost g;
  g.d = d;
  std::vector<const double*> dv(d);
  size_t off = 0;
  for (int a = 0; a < d; ++a) {
    param_check(vecs[a] != nullptr, "per-axis vector missing");
    KCUDA(cudaMemcpyAsync(mb + off, vecs[a], shape[a] * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
    g.n[a] = shape[a];
    dv[a] = mb + off;
    off += shape[a];
  }
  (void)vw;
  launch_generate(ctx->stream, ctx->ws, out, g, dv.data(), mode);
}

int kronop_mass_field(kronop_ctx* ctx, int d, const int* shape, const double* const* mass,
                      double* out) {
  return guard([&] { generate_from_host(ctx, d, shape, mass, 0, out); });
}

int kronop_direct_sum_grid(kronop_ctx* ctx, int d, const int* shape, const double* const* values,
                           double* out) {
  return guard([&] { generate_from_host(ctx, d, shape, values, 1, out); });
}

int kronop_op_create(kronop_ctx* ctx, int d, const int* n, const double* const* T,
                     const double* const* Tinv, const double* const* lambda,
                     const double* const* mass, double shift, kronop_op** out) {
  return guard([&] {
    param_check(ctx && n && T && Tinv && lambda && out, "SeparableOperator: null argument");
    param_check(d >= 1 && d <= KRONOP_MAX_DIM, "SeparableOperator: need at least one axis");
    auto* op = new kronop_op();
    try {
      op->ctx = ctx;
      op->d = d;
      op->N = 1;
      op->shift = shift;
      op->has_mass = mass != nullptr;
      double lmin = 0.0, lmax = 0.0;
      for (int a = 0; a < d; ++a) {
        param_check(n[a] >= 1 && T[a] && Tinv[a] && lambda[a], "SeparableOperator: bad axis");
        op->n[a] = n[a];
        op->N *= n[a];
        op->hlam[a].assign(lambda[a], lambda[a] + n[a]);
        if (n[a] <= 32) {
          op->hT[a].assign(T[a], T[a] + static_cast<size_t>(n[a]) * n[a]);
          op->hTinv[a].assign(Tinv[a], Tinv[a] + static_cast<size_t>(n[a]) * n[a]);
        }
        // an axis identical to an earlier one (isotropic grids) shares its device transforms:
        // less memory, and the small-extent kernel can keep one matrix in registers for a group
        int same = -1;
        const size_t nn = static_cast<size_t>(n[a]) * n[a];
        for (int b = 0; b < a && same < 0; ++b)
          if (n[b] == n[a] && !std::memcmp(T[a], T[b], nn * sizeof(double)) &&
              !std::memcmp(Tinv[a], Tinv[b], nn * sizeof(double)))
            same = b;
        if (same >= 0) {
          op->fwd[a] = op->fwd[same];
          op->bwd[a] = op->bwd[same];
          op->lda[a] = op->lda[same];
          op->shared_axis[a] = true;
        } else {
          op->lda[a] = upload_padded(*ctx, Tinv[a], n[a], n[a], &op->fwd[a], true);
          upload_padded(*ctx, T[a], n[a], n[a], &op->bwd[a], true);
        }
        KCUDA(cudaMalloc(&op->lam[a], n[a] * sizeof(double)));
        KCUDA(cudaMemcpy(op->lam[a], lambda[a], n[a] * sizeof(double), cudaMemcpyHostToDevice));
        // direct-sum extremes in axis order from 0.0 (operators.cpp:13-15; rounding is
        // monotone so the grid min/max sit at the per-axis min/max entries)
        lmin += *std::min_element(lambda[a], lambda[a] + n[a]);
        lmax += *std::max_element(lambda[a], lambda[a] + n[a]);
        if (mass) {
          param_check(mass[a] != nullptr, "SeparableOperator: mass vector missing");
          op->hmass[a].assign(mass[a], mass[a] + n[a]);
          KCUDA(cudaMalloc(&op->mass[a], n[a] * sizeof(double)));
          KCUDA(cudaMemcpy(op->mass[a], mass[a], n[a] * sizeof(double), cudaMemcpyHostToDevice));
        }
      }
      op->lmin = lmin;
      op->lmax = lmax;
    } catch (...) {
      kronop_op_destroy(op);
      throw;
    }
    *out = op;
  });
}

int kronop_op_create_folded(kronop_ctx* ctx, int d, const int* n, const double* const* fe,
                            const double* const* fo, const double* const* be,
                            const double* const* bo, const double* const* lambda_even,
                            const double* const* lambda_odd, const double* const* ground,
                            const double* const* mass, double shift, kronop_op** out) {
  return guard([&] {
    param_check(ctx && n && fe && fo && be && bo && lambda_even && lambda_odd && ground && out,
                "SeparableOperator(folded): null argument");
    param_check(d >= 1 && d <= KRONOP_MAX_DIM, "SeparableOperator: need at least one axis");
    auto* op = new kronop_op();
    try {
      op->ctx = ctx;
      op->d = d;
      op->N = 1;
      op->shift = shift;
      op->has_mass = mass != nullptr;
      op->folded = true;
      double lmin = 0.0, lmax = 0.0;
      for (int a = 0; a < d; ++a) {
        const int na = n[a], ne = na - na / 2, no = na / 2;
        param_check(na >= 1 && fe[a] && be[a] && lambda_even[a] && lambda_odd[a] && ground[a] &&
                        (no == 0 || (fo[a] && bo[a])),
                    "SeparableOperator(folded): bad axis");
        op->n[a] = na;
        op->ne[a] = ne;
        op->no[a] = no;
        op->N *= na;
        // eigenvalues in folded order [even | odd], matching the transformed layout
        op->hlam[a].assign(lambda_even[a], lambda_even[a] + ne);
        op->hlam[a].insert(op->hlam[a].end(), lambda_odd[a], lambda_odd[a] + no);
        op->lda_e[a] = upload_padded(*ctx, fe[a], ne, ne, &op->fe[a], true);
        upload_padded(*ctx, be[a], ne, ne, &op->be[a], true);
        if (no) {
          op->lda_o[a] = upload_padded(*ctx, fo[a], no, no, &op->fo[a], true);
          upload_padded(*ctx, bo[a], no, no, &op->bo[a], true);
        }
        KCUDA(cudaMalloc(&op->lam[a], na * sizeof(double)));
        KCUDA(cudaMemcpy(op->lam[a], op->hlam[a].data(), na * sizeof(double),
                         cudaMemcpyHostToDevice));
        KCUDA(cudaMalloc(&op->bwd[a], na * sizeof(double)));  // ground-state column only
        KCUDA(cudaMemcpy(op->bwd[a], ground[a], na * sizeof(double), cudaMemcpyHostToDevice));
        lmin += *std::min_element(op->hlam[a].begin(), op->hlam[a].end());
        lmax += *std::max_element(op->hlam[a].begin(), op->hlam[a].end());
        if (mass) {
          param_check(mass[a] != nullptr, "SeparableOperator: mass vector missing");
          op->hmass[a].assign(mass[a], mass[a] + na);
          KCUDA(cudaMalloc(&op->mass[a], na * sizeof(double)));
          KCUDA(cudaMemcpy(op->mass[a], mass[a], na * sizeof(double), cudaMemcpyHostToDevice));
        }
      }
      op->lmin = lmin;
      op->lmax = lmax;
    } catch (...) {
      kronop_op_destroy(op);
      throw;
    }
    *out = op;
  });
}

int kronop_op_destroy(kronop_op* op) {
  return guard([&] {
    if (!op) return;
    if (op->ctx) cudaStreamSynchronize(op->ctx->stream);
    for (int a = 0; a < KRONOP_MAX_DIM; ++a) {
      for (double* p : {op->fe[a], op->fo[a], op->be[a], op->bo[a]})
        if (p) cudaFree(p);
      for (void* p : {op->lp_fwd[a], op->lp_bwd[a], op->tf_fwd[a], op->tf_bwd[a], op->f3_fwd[a],
                      op->f3_bwd[a], op->oz_fwd[a], op->oz_bwd[a], op->oz_fo[a], op->oz_bo[a]})
        if (p) cudaFree(p);
      if (!op->shared_axis[a]) {
        if (op->fwd[a]) cudaFree(op->fwd[a]);
        if (op->bwd[a]) cudaFree(op->bwd[a]);
      }
      if (op->lam[a]) cudaFree(op->lam[a]);
      if (op->mass[a]) cudaFree(op->mass[a]);
    }
    delete op;
  });
}

int kronop_op_set_shift(kronop_op* op, double shift) {
  return guard([&] { op->shift = shift; });
}

int kronop_op_info(const kronop_op* op, double* shift, double* lambda_min, double* lambda_max,
                   size_t* size) {
  return guard([&] {
    if (shift) *shift = op->shift;
    if (lambda_min) *lambda_min = op->lmin;
    if (lambda_max) *lambda_max = op->lmax;
    if (size) *size = static_cast<size_t>(op->N);
  });
}

int kronop_op_eigenvalue_grid(kronop_ctx* ctx, const kronop_op* op, double* out) {
  return guard([&] {
    IndexGeomHost g;
    g.d = op->d;
    for (int a = 0; a < op->d; ++a) g.n[a] = op->n[a];
    launch_generate(ctx->stream, ctx->ws, out, g, op->lam, 1);
  });
}

int kronop_op_ground_state(kronop_ctx* ctx, const kronop_op* op, double* out) {
  return guard([&] {
    IndexGeomHost g;
    g.d = op->d;
    for (int a = 0; a < op->d; ++a) g.n[a] = op->n[a];
    // column 0 of each padded T is its first n entries (operators.cpp:77-91)
    launch_generate(ctx->stream, ctx->ws, out, g, op->bwd, 2);
  });
}

int kronop_sep_apply(kronop_ctx* ctx, const kronop_op* op, const double* u, int is_complex,
                     double* out) {
  return guard([&] {
    param_check(ctx && op && u && out, "apply: null argument");
    sep_transform(*ctx, *op, u, out, is_complex, SEP_APPLY, op->shift, 0.0, nullptr, 0.0);
  });
}

int kronop_sep_solve(kronop_ctx* ctx, const kronop_op* op, const double* b, int is_complex,
                     double* out) {
  return guard([&] {
    param_check(ctx && op && b && out, "solve: null argument");
    check_solve_shift(*ctx, *op, op->shift);
    sep_transform(*ctx, *op, b, out, is_complex, SEP_SOLVE, op->shift, 0.0, nullptr, 0.0);
  });
}

int kronop_sep_propagate(kronop_ctx* ctx, const kronop_op* op, const double* psi, double dt,
                         double* out) {
  return guard([&] {
    param_check(ctx && op && psi && out, "propagate: null argument");
    if (dt == 0.0) {  // operators.cpp:64
      if (out != psi)
        KCUDA(cudaMemcpyAsync(out, psi, 2 * op->N * sizeof(double), cudaMemcpyDeviceToDevice,
                              ctx->stream));
      return;
    }
    sep_transform(*ctx, *op, psi, out, 1, SEP_PROPAGATE, op->shift, dt, nullptr, 0.0);
  });
}

int kronop_sep_solve_lowp(kronop_ctx* ctx, kronop_op* op, const double* b, int precision,
                          double* out) {
  return guard([&] {
    param_check(ctx && op && b && out && b != out, "solve_lowp: bad argument");
    param_check(precision >= KRONOP_PREC_BF16 && precision <= KRONOP_PREC_FP64_OZAKI5,
                "solve_lowp: unsupported precision");
    check_solve_shift(*ctx, *op, op->shift);
    if (precision >= KRONOP_PREC_FP64_OZAKI)
      sep_solve_ozaki(*ctx, *op, b, out, 7 - (precision - KRONOP_PREC_FP64_OZAKI));
    else
      sep_solve_lowp(*ctx, *op, b, out, precision);
  });
}

int kronop_op_set_precision(kronop_ctx* ctx, kronop_op* op, int precision) {
  return guard([&] {
    param_check(ctx && op, "op_set_precision: null argument");
    param_check(precision == KRONOP_PREC_FP64 ||
                    (precision >= KRONOP_PREC_FP64_OZAKI && precision <= KRONOP_PREC_FP64_OZAKI5),
                "op_set_precision: unsupported precision");
    if (precision != KRONOP_PREC_FP64) {
      for (int a = 0; a < op->d; ++a)
        param_check(op->n[a] <= 3200, "op_set_precision: Ozaki mode needs extents <= 3200");
      ozaki_prepare(*ctx, *op, 7 - (precision - KRONOP_PREC_FP64_OZAKI));
    }
    op->exec_prec = precision;
  });
}

int kronop_sep_propagate_lowp(kronop_ctx* ctx, kronop_op* op, const double* psi, double dt,
                              int precision, double* out) {
  return guard([&] {
    param_check(ctx && op && psi && out && psi != out, "propagate_lowp: bad argument");
    param_check(precision >= KRONOP_PREC_FP64_OZAKI && precision <= KRONOP_PREC_FP64_OZAKI5,
                "propagate_lowp: unsupported precision");
    sep_propagate_ozaki(*ctx, *op, psi, dt, out, 7 - (precision - KRONOP_PREC_FP64_OZAKI));
  });
}

int kronop_full_apply(kronop_ctx* ctx, const kronop_op* op, const double* diag, double sigma,
                      const double* u, int is_complex, double* out) {
  return guard([&] {
    param_check(ctx && op && u && out, "FullOperator::apply: null argument");
    sep_transform(*ctx, *op, u, out, is_complex, SEP_APPLY, op->shift, 0.0, diag, sigma);
  });
}

int kronop_op_pass(kronop_ctx* ctx, const kronop_op* op, int axis, int forward, const double* in,
                   int is_complex, double* out) {
  return guard([&] {
    param_check(ctx && op && in && out && in != out, "op_pass: bad argument");
    param_check(axis >= 0 && axis < op->d, "op_pass: axis out of range");
    param_check(!op->folded, "op_pass: not available on a folded operator");
    View v = make_view(op->d, op->n, is_complex);
    EpiParams ep;
    run_pass(*ctx, in, out, v, axis + v.cplx, forward ? op->fwd[axis] : op->bwd[axis],
             op->lda[axis], op->n[axis], ep);
  });
}

int kronop_op_pass_ex(kronop_ctx* ctx, const kronop_op* op, int axis, int forward,
                      const double* in, int is_complex, double* out, int epilogue, double dt,
                      const double* diag, double sigma, const double* u) {
  return guard([&] {
    param_check(ctx && op && in && out && in != out, "op_pass: bad argument");
    param_check(axis >= 0 && axis < op->d, "op_pass: axis out of range");
    param_check(!op->folded, "op_pass: not available on a folded operator");
    param_check(epilogue >= KRONOP_EPI_STORE && epilogue <= KRONOP_EPI_AXPY_DIAG,
                "op_pass: bad epilogue");
    View v = make_view(op->d, op->n, is_complex);
    EpiParams ep;
    ep.kind = epilogue;
    ep.axis = axis + v.cplx;
    ep.ndims = v.nd;
    for (int i = 0; i < v.nd; ++i) ep.ext[i] = v.ext[i];
    for (int a = 0; a < op->d; ++a) ep.lam[a + v.cplx] = op->lam[a];
    ep.shift = op->shift;
    ep.dt = dt;
    ep.cplx = v.cplx;
    ep.diag = diag;
    ep.sigma = sigma;
    ep.u = u;
    if (epilogue == KRONOP_EPI_AXPY_DIAG) param_check(u != nullptr, "op_pass: AXPY needs u");
    run_pass(*ctx, in, out, v, axis + v.cplx, forward ? op->fwd[axis] : op->bwd[axis],
             op->lda[axis], op->n[axis], ep);
  });
}

// End-to-end path for host buffers (what a CPU caller of the reference API hands over). The
// field is streamed in and out in slabs of the slowest axis on two copy streams so the PCIe
// transfers overlap the transform: the forward passes on axes 0..d-2 of slab c run while slab
// c+1 is still in flight; the last axis (forward, fused spectral op, backward) needs the whole
// field; the backward passes on axes 0..d-2 of slab c run while slab c-1 is being copied out.
// (Backward axis d-1 runs before axes 0..d-2 here: the Kronecker factors commute, results agree
// with sep_transform to rounding.)
static void ensure_io(kronop_ctx* ctx, size_t nd) {
  if (nd <= ctx->io_cap) return;
  for (auto& p : ctx->io) {
    if (p) KCUDA(cudaFree(p));
    p = nullptr;
  }
  ctx->io_cap = 0;
  for (auto& p : ctx->io) KCUDA(cudaMalloc(&p, nd * sizeof(double)));
  ctx->io_cap = nd;
}

static void ensure_copy_engines(kronop_ctx* ctx) {
  if (ctx->copy_stream[0]) return;
  for (auto& st : ctx->copy_stream) KCUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int i = 0; i < kronop_ctx::kMaxChunks; ++i) {
    KCUDA(cudaEventCreateWithFlags(&ctx->ev_in[i], cudaEventDisableTiming));
    KCUDA(cudaEventCreateWithFlags(&ctx->ev_out[i], cudaEventDisableTiming));
  }
  KCUDA(cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming));
}

static void host_roundtrip(kronop_ctx* ctx, const kronop_op* op, const double* in_host, int cplx,
                           double* out_host, SepKind kind, double dt) {
  const size_t nd = static_cast<size_t>(op->N) * (cplx ? 2 : 1);
  ensure_io(ctx, nd);
  if (kind == SEP_SOLVE) check_solve_shift(*ctx, *op, op->shift);
  const int d = op->d;
  const int nz = op->n[d - 1];
  // the pipelined path below runs the FP64 DMMA passes itself; operators switched to another
  // execution precision (kronop_op_set_precision) or folded ones take their own transform
  if (d < 2 || nz < 2 || op->folded || op->exec_prec != KRONOP_PREC_FP64) {
    KCUDA(cudaMemcpyAsync(ctx->io[0], in_host, nd * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
    sep_transform(*ctx, *op, ctx->io[0], ctx->io[1], cplx, kind, op->shift, dt, nullptr, 0.0);
    KCUDA(cudaMemcpyAsync(out_host, ctx->io[1], nd * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
    KCUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  ensure_copy_engines(ctx);
  ensure_scratch(*ctx, nd);
  cudaStream_t sc = ctx->stream, sin = ctx->copy_stream[0], sout = ctx->copy_stream[1];
  const int chunks = std::min(nz, kronop_ctx::kMaxChunks);
  const size_t plane = nd / nz;  // doubles per plane of the slowest axis
  std::vector<int> zc(chunks), z0(chunks);
  for (int c = 0, acc = 0; c < chunks; ++c) {
    zc[c] = nz / chunks + (c < nz % chunks ? 1 : 0);
    z0[c] = acc;
    acc += zc[c];
  }
  // the copy streams must not start before earlier work on the compute stream is done
  KCUDA(cudaEventRecord(ctx->ev_ready, sc));
  KCUDA(cudaStreamWaitEvent(sin, ctx->ev_ready, 0));
  KCUDA(cudaStreamWaitEvent(sout, ctx->ev_ready, 0));
  double* io0 = ctx->io[0];
  double* io1 = ctx->io[1];
  double* s0 = ctx->scratch[0];
  double* s1 = ctx->scratch[1];
  // forward passes on axes 0..d-2, slab by slab, as the slabs arrive: io0 -> s0/s1 ping-pong
  double* fwd_local = nullptr;
  for (int c = 0; c < chunks; ++c) {
    const size_t off = plane * z0[c], cnt = plane * zc[c];
    KCUDA(cudaMemcpyAsync(io0 + off, in_host + off, cnt * sizeof(double), cudaMemcpyHostToDevice,
                          sin));
    KCUDA(cudaEventRecord(ctx->ev_in[c], sin));
    KCUDA(cudaStreamWaitEvent(sc, ctx->ev_in[c], 0));
    std::vector<int> shp(op->n, op->n + d);
    shp[d - 1] = zc[c];
    View v = make_view(d, shp.data(), cplx);
    const double* cur = io0 + off;
    for (int a = 0; a < d - 1; ++a) {
      double* dst = (a % 2 == 0 ? s0 : s1) + off;
      EpiParams ep;
      run_pass(*ctx, cur, dst, v, a + v.cplx, op->fwd[a], op->lda[a], op->n[a], ep);
      cur = dst;
    }
    fwd_local = ((d - 2) % 2 == 0) ? s0 : s1;
  }
  // last axis on the whole field: forward + fused spectral op, then backward
  double* other = (fwd_local == s0) ? s1 : s0;
  {
    View v = make_view(d, op->n, cplx);
    EpiParams ep;
    ep.kind = kind == SEP_APPLY ? EPI_SPEC_MUL : kind == SEP_SOLVE ? EPI_SPEC_DIV : EPI_SPEC_PHASE;
    ep.axis = d - 1 + v.cplx;
    ep.ndims = v.nd;
    for (int i = 0; i < v.nd; ++i) ep.ext[i] = v.ext[i];
    for (int a = 0; a < d; ++a) ep.lam[a + v.cplx] = op->lam[a];
    ep.shift = op->shift;
    ep.dt = dt;
    ep.cplx = v.cplx;
    run_pass(*ctx, fwd_local, other, v, d - 1 + v.cplx, op->fwd[d - 1], op->lda[d - 1],
             op->n[d - 1], ep);
    View v2 = make_view(d, op->n, cplx);
    EpiParams plain;
    run_pass(*ctx, other, io0, v2, d - 1 + v2.cplx, op->bwd[d - 1], op->lda[d - 1],
             op->n[d - 1], plain);
  }
  // backward passes on axes 0..d-2 slab by slab, each slab copied out as soon as it is done
  for (int c = 0; c < chunks; ++c) {
    const size_t off = plane * z0[c], cnt = plane * zc[c];
    std::vector<int> shp(op->n, op->n + d);
    shp[d - 1] = zc[c];
    View v = make_view(d, shp.data(), cplx);
    const double* cur = io0 + off;
    for (int a = 0; a < d - 1; ++a) {
      double* dst = (a == d - 2) ? io1 + off : ((a % 2 == 0 ? s0 : s1) + off);
      EpiParams ep;
      run_pass(*ctx, cur, dst, v, a + v.cplx, op->bwd[a], op->lda[a], op->n[a], ep);
      cur = dst;
    }
    KCUDA(cudaEventRecord(ctx->ev_out[c], sc));
    KCUDA(cudaStreamWaitEvent(sout, ctx->ev_out[c], 0));
    KCUDA(cudaMemcpyAsync(out_host + off, io1 + off, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                          sout));
  }
  KCUDA(cudaStreamSynchronize(sout));
  KCUDA(cudaStreamSynchronize(sc));
}

// Batched host path: items alternate between two device (in, out) pairs; per item the upload
// (copy stream 0) waits for the compute that last read its input buffer, the transform (compute
// stream, the device path's own pass sequence) waits for the upload and for the download that
// last read its output buffer, and the download (copy stream 1) waits for the transform.
static void host_batch(kronop_ctx* ctx, const kronop_op* op, int count, const double* const* in,
                       int cplx, double* const* out, SepKind kind, double dt) {
  param_check(count >= 0 && (count == 0 || (in && out)), "host batch: bad arguments");
  for (int i = 0; i < count; ++i) param_check(in[i] && out[i], "host batch: null field");
  if (count == 0) return;
  if (count == 1) {
    host_roundtrip(ctx, op, in[0], cplx, out[0], kind, dt);
    return;
  }
  const size_t nd = static_cast<size_t>(op->N) * (cplx ? 2 : 1);
  if (kind == SEP_SOLVE) check_solve_shift(*ctx, *op, op->shift);
  ensure_copy_engines(ctx);
  if (!ctx->ev_up[0])
    for (int p = 0; p < 2; ++p) {
      KCUDA(cudaEventCreateWithFlags(&ctx->ev_up[p], cudaEventDisableTiming));
      KCUDA(cudaEventCreateWithFlags(&ctx->ev_comp[p], cudaEventDisableTiming));
      KCUDA(cudaEventCreateWithFlags(&ctx->ev_down[p], cudaEventDisableTiming));
    }
  if (nd > ctx->bio_cap) {
    KCUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& b : ctx->bio) {
      if (b) KCUDA(cudaFree(b));
      b = nullptr;
    }
    ctx->bio_cap = 0;
    for (auto& b : ctx->bio) KCUDA(cudaMalloc(&b, nd * sizeof(double)));
    ctx->bio_cap = nd;
  }
  ensure_scratch(*ctx, nd);
  cudaStream_t sc = ctx->stream, sin = ctx->copy_stream[0], sout = ctx->copy_stream[1];
  KCUDA(cudaEventRecord(ctx->ev_ready, sc));
  KCUDA(cudaStreamWaitEvent(sin, ctx->ev_ready, 0));
  KCUDA(cudaStreamWaitEvent(sout, ctx->ev_ready, 0));
  const SepKind k = kind;
  for (int i = 0; i < count; ++i) {
    const int p = i & 1;
    double* din = ctx->bio[p];
    double* dout = ctx->bio[2 + p];
    if (i >= 2) KCUDA(cudaStreamWaitEvent(sin, ctx->ev_comp[p], 0));  // item i-2 read din
    KCUDA(cudaMemcpyAsync(din, in[i], nd * sizeof(double), cudaMemcpyHostToDevice, sin));
    KCUDA(cudaEventRecord(ctx->ev_up[p], sin));
    KCUDA(cudaStreamWaitEvent(sc, ctx->ev_up[p], 0));
    if (i >= 2) KCUDA(cudaStreamWaitEvent(sc, ctx->ev_down[p], 0));  // item i-2 left dout
    if (k == SEP_PROPAGATE && dt == 0.0)  // operators.cpp:64
      KCUDA(cudaMemcpyAsync(dout, din, nd * sizeof(double), cudaMemcpyDeviceToDevice, sc));
    else
      sep_transform(*ctx, *op, din, dout, cplx, k, op->shift, dt, nullptr, 0.0);
    KCUDA(cudaEventRecord(ctx->ev_comp[p], sc));
    KCUDA(cudaStreamWaitEvent(sout, ctx->ev_comp[p], 0));
    KCUDA(cudaMemcpyAsync(out[i], dout, nd * sizeof(double), cudaMemcpyDeviceToHost, sout));
    KCUDA(cudaEventRecord(ctx->ev_down[p], sout));
  }
  KCUDA(cudaStreamSynchronize(sout));
  KCUDA(cudaStreamSynchronize(sin));
  KCUDA(cudaStreamSynchronize(sc));
}

int kronop_sep_solve_host_batch(kronop_ctx* ctx, const kronop_op* op, int count,
                                const double* const* b_hosts, int is_complex,
                                double* const* out_hosts) {
  return guard([&] {
    param_check(ctx && op, "solve: null argument");
    host_batch(ctx, op, count, b_hosts, is_complex, out_hosts, SEP_SOLVE, 0.0);
  });
}

int kronop_sep_propagate_host_batch(kronop_ctx* ctx, const kronop_op* op, int count,
                                    const double* const* psi_hosts, double dt,
                                    double* const* out_hosts) {
  return guard([&] {
    param_check(ctx && op, "propagate: null argument");
    host_batch(ctx, op, count, psi_hosts, 1, out_hosts, SEP_PROPAGATE, dt);
  });
}

int kronop_sep_solve_host(kronop_ctx* ctx, const kronop_op* op, const double* b_host,
                          int is_complex, double* out_host) {
  return guard([&] { host_roundtrip(ctx, op, b_host, is_complex, out_host, SEP_SOLVE, 0.0); });
}

int kronop_sep_apply_host(kronop_ctx* ctx, const kronop_op* op, const double* u_host,
                          int is_complex, double* out_host) {
  return guard([&] { host_roundtrip(ctx, op, u_host, is_complex, out_host, SEP_APPLY, 0.0); });
}

int kronop_sep_propagate_host(kronop_ctx* ctx, const kronop_op* op, const double* psi_host,
                              double dt, double* out_host) {
  return guard([&] {
    if (dt == 0.0) {
      std::memcpy(out_host, psi_host, 2 * op->N * sizeof(double));
      return;
    }
    host_roundtrip(ctx, op, psi_host, 1, out_host, SEP_PROPAGATE, dt);
  });
}

int kronop_splitmix_uniform(kronop_ctx* ctx, uint64_t seed, uint64_t start, size_t count,
                            double* out) {
  return guard([&] {
    launch_splitmix(ctx->stream, ctx->ws, out, seed, start, static_cast<long long>(count));
  });
}

int kronop_selftest_division(kronop_ctx* ctx, const double* a, const double* b, size_t n,
                             unsigned long long* mismatches) {
  return guard([&] {
    unsigned long long* d = nullptr;
    KCUDA(cudaMallocAsync(&d, sizeof(unsigned long long), ctx->stream));
    KCUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), ctx->stream));
    launch_div_selftest(ctx->stream, ctx->ws, a, b, d, static_cast<long long>(n));
    KCUDA(cudaMemcpyAsync(mismatches, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ctx->stream));
    KCUDA(cudaFreeAsync(d, ctx->stream));
    KCUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ------------------------------------------------------------------------ host setup --
int kronop_host_gll_rule(int degree, double* nodes, double* weights, double* diff) {
  return guard([&] {
    const kronop_host::GllRule r = kronop_host::gll_rule(degree);
    std::copy(r.nodes.begin(), r.nodes.end(), nodes);
    std::copy(r.weights.begin(), r.weights.end(), weights);
    if (diff) std::copy(r.diff.begin(), r.diff.end(), diff);
  });
}

int kronop_host_gauss_legendre(int points, double* nodes, double* weights) {
  return guard([&] {
    std::vector<double> x, w;
    kronop_host::gauss_legendre(points, x, w);
    std::copy(x.begin(), x.end(), nodes);
    std::copy(w.begin(), w.end(), weights);
  });
}

int kronop_host_assemble_sem(double half_width, int cell_count, int degree, double* nodes,
                             double* mass, double* stiffness) {
  return guard([&] {
    const kronop_host::SemBasis b = kronop_host::assemble_sem(half_width, cell_count, degree);
    std::copy(b.nodes.begin(), b.nodes.end(), nodes);
    std::copy(b.mass.begin(), b.mass.end(), mass);
    if (stiffness) std::copy(b.stiffness.begin(), b.stiffness.end(), stiffness);
  });
}

int kronop_host_interp_matrix(double half_width, int coarse_cells, int coarse_degree,
                              int fine_cells, int fine_degree, double* p) {
  return guard([&] {
    const auto c = kronop_host::assemble_sem(half_width, coarse_cells, coarse_degree);
    const auto f = kronop_host::assemble_sem(half_width, fine_cells, fine_degree);
    const auto m = kronop_host::interp_matrix(c, f);
    std::copy(m.begin(), m.end(), p);
  });
}

int kronop_host_sym_eig(int n, const double* a, double* eigenvalues, double* q) {
  return guard([&] {
    std::vector<double> lam, qq;
    kronop_host::sym_eig(n, a, lam, qq);
    std::copy(lam.begin(), lam.end(), eigenvalues);
    std::copy(qq.begin(), qq.end(), q);
  });
}

int kronop_host_eval_weights(double half_width, int cell_count, int degree, const double* x,
                             int count, double* out) {
  return guard([&] {
    const auto b = kronop_host::assemble_sem(half_width, cell_count, degree);
    const int n = b.size();
    for (int t = 0; t < count; ++t) {
      const auto row = kronop_host::eval_weights_row(b, x[t]);
      std::copy(row.begin(), row.end(), out + static_cast<size_t>(n) * t);
    }
  });
}

int kronop_host_hermite_basis(int n, double* nodes, double* psi_last, double* mass, double* diff) {
  return guard([&] {
    const auto b = kronop_host::hermite_basis(n);
    std::copy(b.nodes.begin(), b.nodes.end(), nodes);
    std::copy(b.psi_last.begin(), b.psi_last.end(), psi_last);
    std::copy(b.mass.begin(), b.mass.end(), mass);
    if (diff) std::copy(b.diff.begin(), b.diff.end(), diff);
  });
}

int kronop_host_build_hermite_axis(int n, const double* fvals, double* lambda, double* T,
                                   double* Tinv) {
  return guard([&] {
    const auto b = kronop_host::hermite_basis(n);
    const auto f = kronop_host::build_hermite_axis(b, fvals);
    std::copy(f.eigenvalues.begin(), f.eigenvalues.end(), lambda);
    std::copy(f.transform.begin(), f.transform.end(), T);
    std::copy(f.inverse_transform.begin(), f.inverse_transform.end(), Tinv);
  });
}

int kronop_host_build_sem_axis_folded(double half_width, int cell_count, int degree,
                                      const double* fvals, double* lambda_even,
                                      double* lambda_odd, double* fe, double* fo, double* be,
                                      double* bo, double* ground) {
  return guard([&] {
    const auto b = kronop_host::assemble_sem(half_width, cell_count, degree);
    const auto f = kronop_host::build_sem_axis_folded(b, fvals);
    std::copy(f.lam_e.begin(), f.lam_e.end(), lambda_even);
    std::copy(f.lam_o.begin(), f.lam_o.end(), lambda_odd);
    std::copy(f.fe.begin(), f.fe.end(), fe);
    std::copy(f.be.begin(), f.be.end(), be);
    if (fo) std::copy(f.fo.begin(), f.fo.end(), fo);
    if (bo) std::copy(f.bo.begin(), f.bo.end(), bo);
    std::copy(f.g0.begin(), f.g0.end(), ground);
  });
}

int kronop_host_build_sem_axis(double half_width, int cell_count, int degree, const double* fvals,
                               double* lambda, double* T, double* Tinv) {
  return guard([&] {
    const auto b = kronop_host::assemble_sem(half_width, cell_count, degree);
    const auto f = kronop_host::build_sem_axis(b, fvals);
    std::copy(f.eigenvalues.begin(), f.eigenvalues.end(), lambda);
    std::copy(f.transform.begin(), f.transform.end(), T);
    std::copy(f.inverse_transform.begin(), f.inverse_transform.end(), Tinv);
  });
}

}  // extern "C"
