// CPU ORACLE (C++ restatement) — test infrastructure and the timed CPU reference arm only; never
// the product. Only tests/, bench.py's cpu_baseline / --impl reference legs and smoke() load it.
//
// An Eigen-free C++20 restatement of the reference's CPU hot path (/root/reference/proj, "kronop")
// with the reference's own execution structure, so that timing it on the host cores measures what
// the reference does:
//   * fields are std::vector<double> that are zero-filled on construction (tensor.hpp:31-32), and
//     kron_apply copies its input and allocates a new field per mode product (tensor.cpp:116,
//     136-145), exactly like TensorField;
//   * mode products are OpenMP static partitions of GEMMs (tensor.cpp:31-84): contract_first_axis
//     chunks the columns, contract_inner_axis chunks the rows (one slab) or parallelises over the
//     slabs; each chunk is one single-threaded GEMM. Eigen's GEMM is replaced by OpenBLAS
//     (numpy's bundled libscipy_openblas64_, dlopen'd, 1 BLAS thread), which is at least as fast
//     as Eigen compiled without -march (proj/CMakeLists.txt:9): the baseline errs in the
//     reference's favour;
//   * the spectral divide / multiply / phase loops, FullOperator's diagonal AXPY and the PCG
//     vector algebra are serial loops, as in operators.cpp:31-105 and pcg.cpp:8-81 (Eigen
//     vector expressions outside an OpenMP region run on one thread);
//   * the eigenvalue grid is materialised by the constructor (operators.cpp:12, tensor.cpp:196-209).
// Build: oracle/cpu/build.sh (g++ -O3 -fopenmp, no -march, as proj/CMakeLists.txt:9).
#include <dlfcn.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using cplx = std::complex<double>;
using blasint = int64_t;
// cblas enums (cblas.h): CblasColMajor = 102, CblasNoTrans = 111, CblasTrans = 112.
using dgemm_fn = void (*)(int, int, int, blasint, blasint, blasint, double, const double*, blasint,
                          const double*, blasint, double, double*, blasint);
using setthreads_fn = void (*)(int);
dgemm_fn g_dgemm = nullptr;
thread_local std::string g_err;
int g_threads = 0;

int effective_threads() { return g_threads > 0 ? g_threads : omp_get_max_threads(); }

// C = A(m x k, lda) * B(k x n, ldb), column-major; transb selects B^T.
void gemm(bool transb, blasint m, blasint n, blasint k, const double* a, blasint lda,
          const double* b, blasint ldb, double* c, blasint ldc) {
  g_dgemm(102, 111, transb ? 112 : 111, m, n, k, 1.0, a, lda, b, ldb, 0.0, c, ldc);
}

struct Matrix {  // column-major n_rows x n_cols (Eigen::MatrixXd's layout)
  int rows = 0, cols = 0;
  std::vector<double> v;
};

template <typename S>
struct Field {  // TensorField<S> (tensor.hpp:27-70): zero-filled on construction
  std::vector<int> shape;
  std::vector<S> values;
  explicit Field(std::vector<int> s) : shape(std::move(s)) {
    size_t n = 1;
    for (int e : shape) n *= (size_t)e;
    values.assign(n, S(0));
  }
};

// tensor.cpp:31-55. Complex data: the reference maps re / im with inner stride 2 and multiplies
// each; BLAS needs unit stride, so each chunk is de-interleaved through a thread-local buffer.
void contract_first_axis(const double* in, double* out, const Matrix& a, int64_t n0, int64_t m,
                         int64_t cols, bool complex_data) {
  const int nth = effective_threads();
  const int64_t chunk = (cols + nth - 1) / nth;
#pragma omp parallel for schedule(static) num_threads(nth)
  for (int t = 0; t < nth; ++t) {
    const int64_t c0 = t * chunk;
    const int64_t nc = std::min(chunk, cols - c0);
    if (nc <= 0) continue;
    if (!complex_data) {
      gemm(false, m, nc, n0, a.v.data(), a.rows, in + c0 * n0, n0, out + c0 * m, m);
    } else {
      std::vector<double> xs(2 * n0 * nc), rs(2 * m * nc);
      for (int64_t c = 0; c < nc; ++c)
        for (int64_t i = 0; i < n0; ++i) {
          xs[c * n0 + i] = in[2 * ((c0 + c) * n0 + i)];
          xs[(nc + c) * n0 + i] = in[2 * ((c0 + c) * n0 + i) + 1];
        }
      gemm(false, m, 2 * nc, n0, a.v.data(), a.rows, xs.data(), n0, rs.data(), m);
      for (int64_t c = 0; c < nc; ++c)
        for (int64_t i = 0; i < m; ++i) {
          out[2 * ((c0 + c) * m + i)] = rs[c * m + i];
          out[2 * ((c0 + c) * m + i) + 1] = rs[(nc + c) * m + i];
        }
    }
  }
}

// tensor.cpp:60-84: R_q = X_q A^T per slab q of shape (pre x nk).
void contract_inner_axis(const double* in, double* out, const Matrix& a, int64_t pre, int64_t nk,
                         int64_t m, int64_t slabs) {
  const int nth = effective_threads();
  if (slabs == 1) {
    const int64_t chunk = (pre + nth - 1) / nth;
#pragma omp parallel for schedule(static) num_threads(nth)
    for (int t = 0; t < nth; ++t) {
      const int64_t r0 = t * chunk;
      const int64_t nr = std::min(chunk, pre - r0);
      if (nr <= 0) continue;
      gemm(true, nr, m, nk, in + r0, pre, a.v.data(), a.rows, out + r0, pre);
    }
    return;
  }
#pragma omp parallel for schedule(static) num_threads(nth)
  for (int64_t q = 0; q < slabs; ++q)
    gemm(true, pre, m, nk, in + q * pre * nk, pre, a.v.data(), a.rows, out + q * pre * m, pre);
}

// tensor.cpp:105-134
template <typename S>
Field<S> mode_product(const Field<S>& x, const Matrix& a, int axis) {
  const auto& shape = x.shape;
  const int d = (int)shape.size();
  if (axis < 0 || axis >= d) throw std::invalid_argument("mode_product: axis out of range");
  if (a.cols != shape[axis])
    throw std::invalid_argument("mode_product: matrix columns do not match axis extent");
  const int m = a.rows;
  std::vector<int> os = shape;
  os[axis] = m;
  Field<S> out(os);
  constexpr bool is_complex = !std::is_same_v<S, double>;
  const double* ip = reinterpret_cast<const double*>(x.values.data());
  double* op = reinterpret_cast<double*>(out.values.data());
  int64_t pre = 1, post = 1;
  for (int i = 0; i < axis; ++i) pre *= shape[i];
  for (int i = axis + 1; i < d; ++i) post *= shape[i];
  if (axis == 0) {
    contract_first_axis(ip, op, a, shape[0], m, post, is_complex);
  } else {
    const int64_t width = is_complex ? 2 * pre : pre;
    contract_inner_axis(ip, op, a, width, shape[axis], m, post);
  }
  return out;
}

// tensor.cpp:136-145 (null = identity)
template <typename S>
Field<S> kron_apply(const Field<S>& x, const std::vector<const Matrix*>& mats) {
  Field<S> out = x;
  for (int axis = 0; axis < (int)x.shape.size(); ++axis)
    if (mats[axis] != nullptr) out = mode_product(out, *mats[axis], axis);
  return out;
}

struct Op {  // SeparableOperator (operators.hpp:15-53, operators.cpp:7-22)
  std::vector<int> shape;
  std::vector<Matrix> T, Tinv;
  Field<double> lambda{std::vector<int>{1}};
  double lambda_min = 0, lambda_max = 0, shift = 0;
  std::vector<const Matrix*> forward, backward;
};

// tensor.cpp:196-209: summed in axis order from 0.0, IndexWalker order (axis 0 fastest)
Field<double> direct_sum_grid(const std::vector<std::vector<double>>& vals) {
  std::vector<int> shape;
  for (const auto& v : vals) shape.push_back((int)v.size());
  Field<double> out(shape);
  const int d = (int)shape.size();
  std::vector<int> idx(d, 0);
  for (size_t i = 0; i < out.values.size(); ++i) {
    double s = 0.0;
    for (int a = 0; a < d; ++a) s += vals[a][idx[a]];
    out.values[i] = s;
    for (int a = 0; a < d; ++a) {
      if (++idx[a] < shape[a]) break;
      idx[a] = 0;
    }
  }
  return out;
}

// operators.cpp:31-40
template <typename S>
Field<S> sep_apply(const Op& op, const Field<S>& u) {
  Field<S> w = kron_apply(u, op.forward);
  const double* lam = op.lambda.values.data();
  for (size_t i = 0; i < w.values.size(); ++i) w.values[i] *= lam[i] - op.shift;
  return kron_apply(w, op.backward);
}

// operators.cpp:42-61
template <typename S>
Field<S> sep_solve(const Op& op, const Field<S>& b) {
  const double floor = 1e-14 * std::max(std::abs(op.lambda_min), std::abs(op.lambda_max));
  double closest = std::min(std::abs(op.lambda_min - op.shift), std::abs(op.lambda_max - op.shift));
  if (op.shift > op.lambda_min && op.shift < op.lambda_max) {
    closest = INFINITY;
    for (double l : op.lambda.values) closest = std::min(closest, std::abs(l - op.shift));
  }
  if (closest < floor)
    throw std::domain_error("SeparableOperator::solve: shift coincides with an eigenvalue");
  Field<S> w = kron_apply(b, op.forward);
  const double* lam = op.lambda.values.data();
  for (size_t i = 0; i < w.values.size(); ++i) w.values[i] /= lam[i] - op.shift;
  return kron_apply(w, op.backward);
}

// operators.cpp:63-75
Field<cplx> sep_propagate(const Op& op, const Field<cplx>& psi, double dt) {
  if (dt == 0.0) return psi;
  Field<cplx> w = kron_apply(psi, op.forward);
  const double* lam = op.lambda.values.data();
  for (size_t i = 0; i < w.values.size(); ++i) {
    const double phase = -(lam[i] - op.shift) * dt;
    w.values[i] *= cplx(std::cos(phase), std::sin(phase));
  }
  return kron_apply(w, op.backward);
}

// operators.cpp:93-105
Field<double> full_apply(const Op& op, const Field<double>* diag, const Field<double>& u) {
  Field<double> out = sep_apply(op, u);
  if (diag)
    for (size_t i = 0; i < out.values.size(); ++i) out.values[i] += diag->values[i] * u.values[i];
  return out;
}

double dot(const Field<double>& a, const Field<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.values.size(); ++i) s += a.values[i] * b.values[i];
  return s;
}

int fail(const char* what) {
  g_err = what;
  return 2;
}

template <typename F>
int guarded(F&& f) {
  if (!g_dgemm) return fail("kcpu: BLAS not loaded (call kcpu_init)");
  try {
    f();
    return 0;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

template <typename S>
Field<S> from_host(const Op& op, const double* p) {
  Field<S> f(op.shape);
  std::memcpy(static_cast<void*>(f.values.data()), p, f.values.size() * sizeof(S));
  return f;
}

template <typename S>
void to_host(const Field<S>& f, double* p) {
  std::memcpy(p, f.values.data(), f.values.size() * sizeof(S));
}

}  // namespace

extern "C" {

const char* kcpu_last_error(void) { return g_err.c_str(); }

// Loads the BLAS (path to numpy's libscipy_openblas64_) and pins it to one thread per call, so
// each OpenMP chunk runs one single-threaded GEMM (Eigen-in-OpenMP, tensor.cpp:36-54).
int kcpu_init(const char* blas_path, int omp_threads) {
  void* h = dlopen(blas_path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return fail(dlerror());
  g_dgemm = (dgemm_fn)dlsym(h, "scipy_cblas_dgemm64_");
  auto st = (setthreads_fn)dlsym(h, "scipy_openblas_set_num_threads64_");
  if (!g_dgemm || !st) return fail("kcpu_init: OpenBLAS symbols not found");
  st(1);
  g_threads = omp_threads;
  return 0;
}

int kcpu_threads(void) { return effective_threads(); }

// SeparableOperator(axes, shift) (operators.cpp:7-22). T / Tinv: n x n column-major.
int kcpu_op_create(int d, const int* n, const double* const* T, const double* const* Tinv,
                   const double* const* lambda, double shift, void** out) {
  return guarded([&] {
    auto op = std::make_unique<Op>();
    std::vector<std::vector<double>> lams;
    for (int a = 0; a < d; ++a) {
      op->shape.push_back(n[a]);
      Matrix t{n[a], n[a], std::vector<double>(T[a], T[a] + (size_t)n[a] * n[a])};
      Matrix ti{n[a], n[a], std::vector<double>(Tinv[a], Tinv[a] + (size_t)n[a] * n[a])};
      op->T.push_back(std::move(t));
      op->Tinv.push_back(std::move(ti));
      lams.emplace_back(lambda[a], lambda[a] + n[a]);
    }
    op->lambda = direct_sum_grid(lams);
    op->lambda_min = *std::min_element(op->lambda.values.begin(), op->lambda.values.end());
    op->lambda_max = *std::max_element(op->lambda.values.begin(), op->lambda.values.end());
    op->shift = shift;
    for (int a = 0; a < d; ++a) {
      op->forward.push_back(&op->Tinv[a]);
      op->backward.push_back(&op->T[a]);
    }
    *out = op.release();
  });
}

int kcpu_op_destroy(void* op) {
  delete static_cast<Op*>(op);
  return 0;
}

int kcpu_op_set_shift(void* op, double shift) {
  static_cast<Op*>(op)->shift = shift;
  return 0;
}

// in / out are host arrays (interleaved complex when is_complex); the timed work is the
// reference's: field construction from the input, kron_apply, the serial spectral loop, kron_apply.
int kcpu_sep_solve(void* opv, const double* b, int is_complex, double* out) {
  const Op& op = *static_cast<Op*>(opv);
  return guarded([&] {
    if (is_complex)
      to_host(sep_solve(op, from_host<cplx>(op, b)), out);
    else
      to_host(sep_solve(op, from_host<double>(op, b)), out);
  });
}

int kcpu_sep_apply(void* opv, const double* u, int is_complex, double* out) {
  const Op& op = *static_cast<Op*>(opv);
  return guarded([&] {
    if (is_complex)
      to_host(sep_apply(op, from_host<cplx>(op, u)), out);
    else
      to_host(sep_apply(op, from_host<double>(op, u)), out);
  });
}

int kcpu_sep_propagate(void* opv, const double* psi, double dt, double* out) {
  const Op& op = *static_cast<Op*>(opv);
  return guarded([&] { to_host(sep_propagate(op, from_host<cplx>(op, psi), dt), out); });
}

int kcpu_full_apply(void* opv, const double* diag, const double* u, double* out) {
  const Op& op = *static_cast<Op*>(opv);
  return guarded([&] {
    std::unique_ptr<Field<double>> dg;
    if (diag) dg = std::make_unique<Field<double>>(from_host<double>(op, diag));
    to_host(full_apply(op, dg.get(), from_host<double>(op, u)), out);
  });
}

// pcg (pcg.cpp:8-81) with apply_a = FullOperator{a_op, diag}.apply and precond = p_op.solve
// (the `pcg-bench` pairing, harness.cpp:515-556). x is in/out; history (capacity max_iter + 1)
// receives the relative residuals. iterations / converged / final_residual are returned.
int kcpu_pcg(void* a_opv, const double* diag, void* p_opv, const double* b, double* x,
             double rel_tol, int max_iter, int stagnation_window, int preconditioned_norm,
             int* iterations, int* converged, double* final_residual, double* history,
             int* history_len) {
  const Op& aop = *static_cast<Op*>(a_opv);
  const Op& pop = *static_cast<Op*>(p_opv);
  return guarded([&] {
    std::unique_ptr<Field<double>> dg;
    if (diag) dg = std::make_unique<Field<double>>(from_host<double>(aop, diag));
    auto apply_a = [&](const Field<double>& v) { return full_apply(aop, dg.get(), v); };
    auto precond = [&](const Field<double>& v) { return sep_solve(pop, v); };
    Field<double> bf = from_host<double>(aop, b);
    Field<double> xf = from_host<double>(aop, x);
    int its = 0, conv = 0, hl = 0;
    const double norm_b = std::sqrt(dot(bf, bf));
    if (norm_b == 0.0) {
      std::fill(xf.values.begin(), xf.values.end(), 0.0);
      conv = 1;
      *final_residual = 0.0;
    } else {
      Field<double> r = bf;
      if (std::sqrt(dot(xf, xf)) != 0.0) {
        const Field<double> ax = apply_a(xf);
        for (size_t i = 0; i < r.values.size(); ++i) r.values[i] -= ax.values[i];
      }
      Field<double> z = precond(r);
      Field<double> p = z;
      double rz = dot(r, z);
      const double pnorm0 = std::sqrt(std::abs(rz));
      auto rel_res = [&](const Field<double>& res, double rzc) {
        return preconditioned_norm ? std::sqrt(std::abs(rzc)) / pnorm0
                                   : std::sqrt(dot(res, res)) / norm_b;
      };
      double rel = rel_res(r, rz);
      history[hl++] = rel;
      double best_rel = rel;
      Field<double> best_x = xf;
      int since = 0;
      Field<double> q(bf.shape);
      for (int it = 0; it < max_iter; ++it) {
        if (rel <= rel_tol) {
          conv = 1;
          break;
        }
        if (stagnation_window > 0 && since >= stagnation_window) break;
        q = apply_a(p);
        const double pq = dot(p, q);
        if (pq <= 0.0)
          throw std::domain_error("pcg: indefinite direction at iteration " +
                                  std::to_string(it + 1));
        const double alpha = rz / pq;
        for (size_t i = 0; i < xf.values.size(); ++i) xf.values[i] += alpha * p.values[i];
        for (size_t i = 0; i < r.values.size(); ++i) r.values[i] -= alpha * q.values[i];
        z = precond(r);
        const double rz_next = dot(r, z);
        const double beta = rz_next / rz;
        for (size_t i = 0; i < p.values.size(); ++i) p.values[i] = z.values[i] + beta * p.values[i];
        rz = rz_next;
        ++its;
        rel = rel_res(r, rz);
        history[hl++] = rel;
        if (rel < 0.99 * best_rel) {
          best_rel = rel;
          best_x = xf;
          since = 0;
        } else {
          ++since;
        }
      }
      if (rel <= rel_tol) {
        conv = 1;
      } else if (best_rel < rel) {
        xf = best_x;
        rel = best_rel;
      }
      *final_residual = rel;
    }
    to_host(xf, x);
    *iterations = its;
    *converged = conv;
    *history_len = hl;
  });
}

// Timed repetitions of one operator call on a field built once outside the timed region (the
// reference's caller already holds a TensorField): kind 0 = solve, 1 = apply, 2 = propagate
// (complex only). seconds[r] = wall time of repetition r; out = the last result.
int kcpu_time_op(void* opv, int kind, const double* in, int is_complex, double dt, int reps,
                 double* out, double* seconds) {
  const Op& op = *static_cast<Op*>(opv);
  return guarded([&] {
    auto run = [&](auto tag) {
      using S = decltype(tag);
      const Field<S> x = from_host<S>(op, in);
      for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        Field<S> y = kind == 0 ? sep_solve(op, x) : kind == 1 ? sep_apply(op, x) : [&] {
          if constexpr (std::is_same_v<S, cplx>)
            return sep_propagate(op, x, dt);
          else
            throw std::invalid_argument("kcpu_time_op: propagate needs a complex field");
          return x;
        }();
        seconds[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (r + 1 == reps) to_host(y, out);
      }
    };
    if (is_complex)
      run(cplx{});
    else
      run(0.0);
  });
}

// random_field (harness.cpp:184-189) with SplitMix64::uniform_pm1 (rng.hpp:16-31): out[i] = the
// (start + i + 1)-th output of SplitMix64(seed) mapped to [-1, 1). Counter-based, so OpenMP chunks
// produce exactly the sequential stream.
int kcpu_uniform_pm1(uint64_t seed, uint64_t start, int64_t count, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    uint64_t z = seed + (start + (uint64_t)i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    out[i] = (double)(z >> 11) * 0x1.0p-52 - 1.0;
  }
  return 0;
}

}  // extern "C"
