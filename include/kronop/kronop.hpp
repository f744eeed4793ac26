// kronop/kronop.hpp — header-only C++20 mirror of the reference's solver/operator API
// (proj/include/kronop/{errors,tensor,axis,basis1d,operators,pcg,splitting,ground_state,gpe}.hpp)
// over the C-ABI in kronop_cuda.h. Same names, same argument meaning, same exceptions; Eigen is
// replaced by std::vector (column-major n x n for matrices) because Eigen is not a dependency.
//
// Two field types:
//   TensorField<S>  host values with the reference's value semantics (tensor.hpp:27-70); every
//                   operator call on a host field uploads, runs on the GPU and downloads.
//   DeviceField<S>  resident on the GPU (the production path: drivers keep everything there).
#pragma once

#include <complex>
#include <cstddef>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "../kronop_cuda.h"

namespace kronop {

// ------------------------------------------------------------------ errors.hpp:9-30 --
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ParameterError : public Error {
 public:
  using Error::Error;
};
class NumericalError : public Error {
 public:
  using Error::Error;
};
class CapabilityError : public Error {
 public:
  using Error::Error;
};

inline void check(int rc) {
  if (rc == KRONOP_OK) return;
  const std::string msg = kronop_last_error();
  if (rc == KRONOP_EPARAM) throw ParameterError(msg);
  if (rc == KRONOP_ENUMERICAL) throw NumericalError(msg);
  if (rc == KRONOP_ECAPABILITY) throw CapabilityError(msg);
  throw Error(msg);
}

using Shape = std::vector<int>;  // tensor.hpp:14
inline std::size_t shape_size(const Shape& s) {
  std::size_t t = 1;
  for (int n : s) t *= static_cast<std::size_t>(n);
  return t;
}
using MassWeights = std::vector<std::vector<double>>;  // tensor.hpp:22

template <typename S>
constexpr int is_complex_v = std::is_same_v<S, std::complex<double>> ? 1 : 0;

// ------------------------------------------------------------------------ context --
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    check(kronop_ctx_create(device, stream, &h_));
  }
  ~Context() { kronop_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  kronop_ctx* get() const { return h_; }
  void synchronize() const { check(kronop_ctx_synchronize(h_)); }

 private:
  kronop_ctx* h_ = nullptr;
};

// ------------------------------------------------------------------ tensor.hpp:27-70 --
template <typename S>
class TensorField {
 public:
  TensorField() = default;
  explicit TensorField(Shape shape) : shape_(std::move(shape)), values_(shape_size(shape_), S(0)) {
    if (shape_.empty() || shape_.size() > 9)
      throw ParameterError("TensorField: dimension must be in [1, 9]");
    for (int n : shape_)
      if (n < 1) throw ParameterError("TensorField: extents must be positive");
  }
  static TensorField constant(Shape shape, S value) {
    TensorField f(std::move(shape));
    std::fill(f.values_.begin(), f.values_.end(), value);
    return f;
  }
  const Shape& shape() const { return shape_; }
  int dim() const { return static_cast<int>(shape_.size()); }
  std::size_t size() const { return values_.size(); }
  S* data() { return values_.data(); }
  const S* data() const { return values_.data(); }
  S& operator[](std::size_t i) { return values_[i]; }
  const S& operator[](std::size_t i) const { return values_[i]; }
  void set_mass(std::shared_ptr<const MassWeights> m) { mass_ = std::move(m); }
  const std::shared_ptr<const MassWeights>& mass() const { return mass_; }

 private:
  Shape shape_;
  std::vector<S> values_;
  std::shared_ptr<const MassWeights> mass_;
};
using RealField = TensorField<double>;
using ComplexField = TensorField<std::complex<double>>;

template <typename S>
class DeviceField {
 public:
  DeviceField() = default;
  DeviceField(Context& ctx, Shape shape) : ctx_(&ctx), shape_(std::move(shape)), n_(shape_size(shape_)) {
    check(kronop_field_alloc(ctx_->get(), doubles(), &p_));
  }
  DeviceField(Context& ctx, const TensorField<S>& host) : DeviceField(ctx, host.shape()) {
    upload(host);
  }
  ~DeviceField() {
    if (p_) kronop_field_free(ctx_->get(), p_);
  }
  DeviceField(DeviceField&& o) noexcept : ctx_(o.ctx_), shape_(std::move(o.shape_)), n_(o.n_), p_(o.p_) {
    o.p_ = nullptr;
  }
  DeviceField& operator=(DeviceField&& o) noexcept {
    std::swap(ctx_, o.ctx_);
    std::swap(shape_, o.shape_);
    std::swap(n_, o.n_);
    std::swap(p_, o.p_);
    return *this;
  }
  DeviceField(const DeviceField&) = delete;
  void upload(const TensorField<S>& h) {
    check(kronop_field_upload(ctx_->get(), p_, reinterpret_cast<const double*>(h.data()), doubles()));
  }
  TensorField<S> download() const {
    TensorField<S> h(shape_);
    check(kronop_field_download(ctx_->get(), reinterpret_cast<double*>(h.data()), p_, doubles()));
    return h;
  }
  const Shape& shape() const { return shape_; }
  std::size_t size() const { return n_; }
  double* data() { return p_; }
  const double* data() const { return p_; }
  std::size_t doubles() const { return n_ * (is_complex_v<S> ? 2 : 1); }

 private:
  Context* ctx_ = nullptr;
  Shape shape_;
  std::size_t n_ = 0;
  double* p_ = nullptr;
};

// ------------------------------------------------------------- fieldio.hpp:10-16 --
template <typename S>
void dump_field(const std::string& path, const TensorField<S>& field) {
  std::vector<int> shp(field.shape().begin(), field.shape().end());
  check(kronop_field_dump_host(path.c_str(), field.dim(), shp.data(), is_complex_v<S>,
                               reinterpret_cast<const double*>(field.data())));
}
// Device fields stream through pinned staging chunks (no full host copy).
template <typename S>
void dump_field(const std::string& path, Context& ctx, const DeviceField<S>& field) {
  std::vector<int> shp(field.shape().begin(), field.shape().end());
  check(kronop_field_dump(ctx.get(), path.c_str(), static_cast<int>(shp.size()), shp.data(),
                          is_complex_v<S>, field.data()));
}
using LoadedField = std::variant<RealField, ComplexField>;
inline LoadedField load_field(const std::string& path) {
  int d = 0, cplx = 0, shp[9] = {};
  check(kronop_field_load_header(path.c_str(), &d, shp, &cplx));
  const Shape shape(shp, shp + d);
  auto load = [&](auto f) -> LoadedField {
    check(kronop_field_load_host(path.c_str(), reinterpret_cast<double*>(f.data()),
                                 f.size() * (cplx ? 2 : 1)));
    return f;
  };
  return cplx ? load(ComplexField(shape)) : load(RealField(shape));
}
template <typename S>
DeviceField<S> load_field(const std::string& path, Context& ctx) {
  int d = 0, cplx = 0, shp[9] = {};
  check(kronop_field_load_header(path.c_str(), &d, shp, &cplx));
  if (cplx != is_complex_v<S>) throw ParameterError("load_field: scalar kind mismatch");
  DeviceField<S> f(ctx, Shape(shp, shp + d));
  check(kronop_field_load(ctx.get(), path.c_str(), f.data(), f.doubles()));
  return f;
}

// -------------------------------------------------------- axis.hpp / basis1d.hpp (host) --
struct Basis1D {  // basis1d.hpp:17-29
  double half_width = 0.0;
  int cell_count = 0, degree = 0;
  std::vector<double> nodes, mass, stiffness;  // stiffness n x n column-major
  int size() const { return static_cast<int>(nodes.size()); }
};
inline Basis1D assemble_sem(double half_width, int cell_count, int degree) {  // basis1d.hpp:30
  Basis1D b{half_width, cell_count, degree, {}, {}, {}};
  const int n = cell_count * degree - 1;
  if (n < 1) throw ParameterError("assemble_sem: no interior nodes");
  b.nodes.resize(n);
  b.mass.resize(n);
  b.stiffness.resize(static_cast<std::size_t>(n) * n);
  check(kronop_host_assemble_sem(half_width, cell_count, degree, b.nodes.data(), b.mass.data(),
                                 b.stiffness.data()));
  return b;
}

struct AxisEigens {  // axis.hpp:23-29
  std::vector<double> eigenvalues;        // ascending
  std::vector<double> transform;          // T, column-major
  std::vector<double> inverse_transform;  // T^{-1}
  int size() const { return static_cast<int>(eigenvalues.size()); }
};
template <class F>
AxisEigens build_axis(const Basis1D& basis, F&& f) {  // axis.hpp:37
  const int n = basis.size();
  std::vector<double> fv(n);
  for (int i = 0; i < n; ++i) fv[i] = f(basis.nodes[i]);
  AxisEigens a;
  a.eigenvalues.resize(n);
  a.transform.resize(static_cast<std::size_t>(n) * n);
  a.inverse_transform.resize(static_cast<std::size_t>(n) * n);
  check(kronop_host_build_sem_axis(basis.half_width, basis.cell_count, basis.degree, fv.data(),
                                   a.eigenvalues.data(), a.transform.data(),
                                   a.inverse_transform.data()));
  return a;
}

struct HermiteBasis {  // hermite.hpp:13-19
  int size = 0;
  std::vector<double> nodes, psi_last, mass;
  std::vector<double> diff;  // n x n column-major
};
inline HermiteBasis hermite_basis(int n) {  // hermite.hpp:29
  if (n < 2) throw ParameterError("hermite_basis: need n >= 2");
  HermiteBasis b;
  b.size = n;
  b.nodes.resize(n);
  b.psi_last.resize(n);
  b.mass.resize(n);
  b.diff.resize(static_cast<std::size_t>(n) * n);
  check(kronop_host_hermite_basis(n, b.nodes.data(), b.psi_last.data(), b.mass.data(),
                                  b.diff.data()));
  return b;
}
template <class F>
AxisEigens build_axis(const HermiteBasis& basis, F&& f) {  // axis.hpp:39
  const int n = basis.size;
  std::vector<double> fv(n);
  for (int i = 0; i < n; ++i) fv[i] = f(basis.nodes[i]);
  AxisEigens a;
  a.eigenvalues.resize(n);
  a.transform.resize(static_cast<std::size_t>(n) * n);
  a.inverse_transform.resize(static_cast<std::size_t>(n) * n);
  check(kronop_host_build_hermite_axis(n, fv.data(), a.eigenvalues.data(), a.transform.data(),
                                       a.inverse_transform.data()));
  return a;
}

// ------------------------------------------------------------- operators.hpp:15-62 --
class SeparableOperator {
 public:
  SeparableOperator(Context& ctx, std::vector<AxisEigens> axes, double shift = 0.0,
                    std::shared_ptr<const MassWeights> mass = nullptr)
      : ctx_(&ctx), axes_(std::move(axes)) {
    const int d = static_cast<int>(axes_.size());
    if (d < 1) throw ParameterError("SeparableOperator: need at least one axis");
    std::vector<int> n(d);
    std::vector<const double*> T(d), Ti(d), L(d), M(d);
    for (int a = 0; a < d; ++a) {
      n[a] = axes_[a].size();
      T[a] = axes_[a].transform.data();
      Ti[a] = axes_[a].inverse_transform.data();
      L[a] = axes_[a].eigenvalues.data();
      if (mass) M[a] = (*mass)[a].data();
    }
    kronop_op* h = nullptr;
    check(kronop_op_create(ctx.get(), d, n.data(), T.data(), Ti.data(), L.data(),
                           mass ? M.data() : nullptr, shift, &h));
    op_.reset(h, [](kronop_op* p) { kronop_op_destroy(p); });
    mass_ = std::move(mass);
  }
  int dim() const { return static_cast<int>(axes_.size()); }
  Shape shape() const {
    Shape s;
    for (const auto& a : axes_) s.push_back(a.size());
    return s;
  }
  const std::vector<AxisEigens>& axes() const { return axes_; }
  double shift() const {
    double s;
    check(kronop_op_info(op_.get(), &s, nullptr, nullptr, nullptr));
    return s;
  }
  void set_shift(double s) { check(kronop_op_set_shift(op_.get(), s)); }
  double min_eigenvalue() const {
    double v;
    check(kronop_op_info(op_.get(), nullptr, &v, nullptr, nullptr));
    return v;
  }
  double max_eigenvalue() const {
    double v;
    check(kronop_op_info(op_.get(), nullptr, nullptr, &v, nullptr));
    return v;
  }
  // device-resident forms
  template <typename S>
  void apply(const DeviceField<S>& u, DeviceField<S>& out) const {
    check(kronop_sep_apply(ctx_->get(), op_.get(), u.data(), is_complex_v<S>, out.data()));
  }
  template <typename S>
  void solve(const DeviceField<S>& b, DeviceField<S>& out) const {
    check(kronop_sep_solve(ctx_->get(), op_.get(), b.data(), is_complex_v<S>, out.data()));
  }
  void propagate(const DeviceField<std::complex<double>>& psi, double dt,
                 DeviceField<std::complex<double>>& out) const {
    check(kronop_sep_propagate(ctx_->get(), op_.get(), psi.data(), dt, out.data()));
  }
  // Separately reported solve variants on the tcgen05 tensor cores (real fields):
  // KRONOP_PREC_BF16 / _TF32 / _FP32X3 (the paper's reduced-precision rows) and
  // KRONOP_PREC_FP64_OZAKI (FP64 emulated on the INT8 tensor cores; _OZAKI6 / _OZAKI5 fewer slices)
  void solve_variant(const DeviceField<double>& b, int precision, DeviceField<double>& out) const {
    check(kronop_sep_solve_lowp(ctx_->get(), op_.get(), b.data(), precision, out.data()));
  }
  // value-semantics forms of the reference (operators.hpp:32-46)
  template <typename S>
  TensorField<S> apply(const TensorField<S>& u) const {
    TensorField<S> out(u.shape());
    check(kronop_sep_apply_host(ctx_->get(), op_.get(), reinterpret_cast<const double*>(u.data()),
                                is_complex_v<S>, reinterpret_cast<double*>(out.data())));
    out.set_mass(u.mass());
    return out;
  }
  template <typename S>
  TensorField<S> solve(const TensorField<S>& b) const {
    TensorField<S> out(b.shape());
    check(kronop_sep_solve_host(ctx_->get(), op_.get(), reinterpret_cast<const double*>(b.data()),
                                is_complex_v<S>, reinterpret_cast<double*>(out.data())));
    out.set_mass(b.mass());
    return out;
  }
  // a caller's loop of solve() over host fields as one call (kronop_sep_solve_host_batch): the
  // copies of neighbouring right-hand sides overlap each one's transform
  template <typename S>
  std::vector<TensorField<S>> solve(const std::vector<TensorField<S>>& bs) const {
    std::vector<TensorField<S>> outs;
    outs.reserve(bs.size());
    std::vector<const double*> in;
    std::vector<double*> out;
    for (const auto& b : bs) {
      outs.emplace_back(b.shape());
      outs.back().set_mass(b.mass());
      in.push_back(reinterpret_cast<const double*>(b.data()));
      out.push_back(reinterpret_cast<double*>(outs.back().data()));
    }
    check(kronop_sep_solve_host_batch(ctx_->get(), op_.get(), static_cast<int>(bs.size()),
                                      in.data(), is_complex_v<S>, out.data()));
    return outs;
  }
  ComplexField propagate(const ComplexField& psi, double dt) const {
    ComplexField out(psi.shape());
    check(kronop_sep_propagate_host(ctx_->get(), op_.get(),
                                    reinterpret_cast<const double*>(psi.data()), dt,
                                    reinterpret_cast<double*>(out.data())));
    out.set_mass(psi.mass());
    return out;
  }
  RealField ground_state() const {
    DeviceField<double> d(*ctx_, shape());
    check(kronop_op_ground_state(ctx_->get(), op_.get(), d.data()));
    return d.download();
  }
  kronop_op* handle() const { return op_.get(); }
  Context& context() const { return *ctx_; }
  const std::shared_ptr<const MassWeights>& mass() const { return mass_; }

 private:
  Context* ctx_;
  std::vector<AxisEigens> axes_;
  std::shared_ptr<kronop_op> op_;
  std::shared_ptr<const MassWeights> mass_;
};

struct FullOperator {  // operators.hpp:56-62 (diagonal resident on the device)
  const SeparableOperator* sep = nullptr;
  const DeviceField<double>* diagonal = nullptr;

  template <typename S>
  void apply(const DeviceField<S>& u, DeviceField<S>& out, double sigma = 0.0) const {
    check(kronop_full_apply(sep->context().get(), sep->handle(),
                            diagonal ? diagonal->data() : nullptr, sigma, u.data(),
                            is_complex_v<S>, out.data()));
  }
};

// -------------------------------------------------------------------- pcg.hpp:10-37 --
struct PcgConfig {
  double rel_tol = 1e-12;
  int max_iter = 500;
  bool record_history = false;
  bool preconditioned_norm = false;
  int stagnation_window = 0;
  kronop_pcg_config c() const {
    return {rel_tol, max_iter, record_history ? 1 : 0, preconditioned_norm ? 1 : 0,
            stagnation_window};
  }
};
struct PcgReport {
  int iterations = 0;
  double final_residual = 0.0;
  bool converged = false;
  std::vector<double> history;
};
// The reference's LinearMap callbacks (pcg.hpp:29) are the two device-map shapes every caller
// uses (see kronop_linear_map in kronop_cuda.h).
struct LinearMap {
  kronop_linear_map m;
  static LinearMap apply(const SeparableOperator& op, const DeviceField<double>* diag = nullptr,
                         double sigma = 0.0) {
    return {{op.handle(), KRONOP_MAP_APPLY, diag ? diag->data() : nullptr, sigma, nullptr}};
  }
  static LinearMap solve(const SeparableOperator& op, const DeviceField<double>* scale = nullptr) {
    return {{op.handle(), KRONOP_MAP_SOLVE, nullptr, 0.0, scale ? scale->data() : nullptr}};
  }
};
inline PcgReport pcg(Context& ctx, const LinearMap& apply_a, const LinearMap& precond,
                     const DeviceField<double>& b, DeviceField<double>& x,
                     const PcgConfig& config = {}) {
  kronop_pcg_config cfg = config.c();
  kronop_pcg_report rep{};
  std::vector<double> hist(config.record_history ? config.max_iter + 2 : 0);
  check(kronop_pcg(ctx.get(), &apply_a.m, &precond.m, b.data(), x.data(), &cfg, &rep,
                   config.record_history ? hist.data() : nullptr));
  PcgReport out{rep.iterations, rep.final_residual, rep.converged != 0, {}};
  if (config.record_history) out.history.assign(hist.begin(), hist.begin() + rep.history_len);
  return out;
}

// -------------------------------------------------------- splitting.hpp:17-69 --
struct YoshidaCoeffs {
  double gamma1, gamma2;
};
inline YoshidaCoeffs yoshida_coeffs() {
  YoshidaCoeffs c;
  check(kronop_yoshida_coeffs(&c.gamma1, &c.gamma2));
  return c;
}
enum class Composition { Single, Yoshida };
struct SplitSpec {
  int quad_points = 1;
  Composition composition = Composition::Single;
  double dt = 0.0, total_time = 0.0;
  bool merge_across_steps = false, mass_weighted_error = false;
};
struct EvolveResult {
  double error = 0.0;
  int steps = 0;
};
inline EvolveResult evolve(const SplitSpec& spec, const SeparableOperator& a,
                           const DeviceField<double>& b_diag,
                           const DeviceField<std::complex<double>>& psi0,
                           DeviceField<std::complex<double>>& state,
                           const SeparableOperator* exact, double stationary_eigenvalue = 0.0) {
  kronop_split_spec s{spec.quad_points,
                      spec.composition == Composition::Single ? KRONOP_COMPOSITION_SINGLE
                                                              : KRONOP_COMPOSITION_YOSHIDA,
                      spec.dt, spec.total_time, spec.merge_across_steps ? 1 : 0,
                      spec.mass_weighted_error ? 1 : 0};
  EvolveResult r;
  check(kronop_evolve(a.context().get(), &s, a.handle(), b_diag.data(), psi0.data(),
                      exact ? exact->handle() : nullptr, stationary_eigenvalue, state.data(),
                      &r.error, &r.steps));
  return r;
}

// -------------------------------------------------------- ground_state.hpp:17-56 --
enum class ShiftMode { FractionOfMin, OffsetBelowMin, Zero };
struct InverseIterationConfig {
  ShiftMode shift_mode = ShiftMode::FractionOfMin;
  double shift_fraction = 0.9, shift_offset = 1e-4, eig_rel_tol = 1e-12;
  int max_outer = 60;
  PcgConfig inner{.stagnation_window = 100};
};
struct EigenpairResult {
  double eigenvalue = 0.0;
  int outer_iterations = 0, total_inner_iterations = 0;
  std::vector<int> inner_per_outer;
  bool converged = false;
};
inline EigenpairResult inverse_iteration(const FullOperator& op,
                                         const InverseIterationConfig& config,
                                         const DeviceField<double>& initial,
                                         DeviceField<double>& eigenvector) {
  kronop_inverse_iteration_config c{static_cast<int>(config.shift_mode), config.shift_fraction,
                                    config.shift_offset, config.eig_rel_tol, config.max_outer,
                                    config.inner.c()};
  kronop_eigenpair_result r{};
  std::vector<int> per(config.max_outer > 0 ? config.max_outer : 1);
  check(kronop_inverse_iteration(op.sep->context().get(), op.sep->handle(),
                                 op.diagonal ? op.diagonal->data() : nullptr, &c, initial.data(),
                                 eigenvector.data(), &r, per.data()));
  EigenpairResult out{r.eigenvalue, r.outer_iterations, r.total_inner_iterations, {},
                      r.converged != 0};
  if (op.diagonal) out.inner_per_outer.assign(per.begin(), per.begin() + r.outer_iterations);
  return out;
}

// ------------------------------------------------------------------- tensor.hpp:79-106 --
template <typename S>
void mode_product(Context& ctx, const DeviceField<S>& x, const std::vector<double>& a, int m,
                  int axis, DeviceField<S>& out) {  // a: column-major m x shape[axis]
  check(kronop_mode_product(ctx.get(), x.data(), static_cast<int>(x.shape().size()),
                            x.shape().data(), is_complex_v<S>, a.data(), m, axis, out.data()));
}
template <typename S>
void kron_apply(Context& ctx, const DeviceField<S>& x,
                const std::vector<const std::vector<double>*>& mats, const std::vector<int>& rows,
                DeviceField<S>& out) {  // null entries = identity
  std::vector<const double*> p(mats.size(), nullptr);
  for (std::size_t a = 0; a < mats.size(); ++a) p[a] = mats[a] ? mats[a]->data() : nullptr;
  check(kronop_kron_apply(ctx.get(), x.data(), static_cast<int>(x.shape().size()),
                          x.shape().data(), is_complex_v<S>, p.data(), rows.data(), out.data()));
}
inline double inner(Context& ctx, const DeviceField<double>& u, const DeviceField<double>& v,
                    const MassWeights* mass = nullptr) {  // Weighting::Plain / Mass
  double r[2] = {0, 0};
  std::vector<const double*> m;
  if (mass)
    for (const auto& w : *mass) m.push_back(w.data());
  check(kronop_inner(ctx.get(), u.data(), v.data(), static_cast<int>(u.shape().size()),
                     u.shape().data(), 0, mass ? m.data() : nullptr, r));
  return r[0];
}

// ------------------------------------------------------------- splitting.hpp:46-52 --
inline void qhop_step(const SeparableOperator& a, const DeviceField<double>& b_diag,
                      const DeviceField<std::complex<double>>& psi, double h, int quad_points,
                      DeviceField<std::complex<double>>& out) {
  check(kronop_qhop_step(a.context().get(), a.handle(), b_diag.data(), psi.data(), h, quad_points,
                         out.data()));
}
inline void yoshida_step(const SeparableOperator& a, const DeviceField<double>& b_diag,
                         const DeviceField<std::complex<double>>& psi, double h, int quad_points,
                         DeviceField<std::complex<double>>& out) {
  check(kronop_yoshida_step(a.context().get(), a.handle(), b_diag.data(), psi.data(), h,
                            quad_points, out.data()));
}

// -------------------------------------------------------------------- gpe.hpp:17-74 --
enum class GpeFlowKind { ModifiedH1, AdaptiveMetric };
enum class GpeInit { Constant, Eigenfunction, Supplied };
struct GpeFlowConfig {
  GpeFlowKind kind = GpeFlowKind::ModifiedH1;
  double step = 0.1, metric_shift = 20.0, energy_rel_tol = 1e-12;
  int max_iterations = 20000;
  PcgConfig inner{.stagnation_window = 100};
  GpeInit init = GpeInit::Eigenfunction;
  bool record_history = false;
};
struct GpeHistoryRow {
  int iteration = 0;
  double energy = 0.0, rel_change = 0.0;
  long linear_solves = 0;
  double seconds = 0.0;
};
struct GpeResult {
  double energy = 0.0, eigenvalue = 0.0;
  int iterations = 0;
  long linear_solves = 0;
  bool converged = false;
  std::vector<GpeHistoryRow> history;
};
struct GpeProblem {  // gpe.hpp:17-22 (mass weights travel with the operator)
  FullOperator hamiltonian;
  const SeparableOperator* laplacian = nullptr;
  double beta = 0.0;
};
inline double gpe_energy(const GpeProblem& p, const DeviceField<double>& u) {
  double e = 0.0;
  check(kronop_gpe_energy(p.hamiltonian.sep->context().get(), p.hamiltonian.sep->handle(),
                          p.hamiltonian.diagonal ? p.hamiltonian.diagonal->data() : nullptr,
                          p.beta, u.data(), &e));
  return e;
}
inline GpeResult gpe_gradient_flow(const GpeProblem& p, const GpeFlowConfig& config,
                                   DeviceField<double>& state,
                                   const DeviceField<double>* initial = nullptr) {
  kronop_gpe_config c{config.kind == GpeFlowKind::ModifiedH1 ? KRONOP_GPE_H1 : KRONOP_GPE_AU,
                      config.step, config.metric_shift, config.energy_rel_tol,
                      config.max_iterations, config.inner.c(),
                      config.init == GpeInit::Constant        ? KRONOP_GPE_INIT_CONSTANT
                      : config.init == GpeInit::Eigenfunction ? KRONOP_GPE_INIT_EIGENFUNCTION
                                                              : KRONOP_GPE_INIT_SUPPLIED,
                      config.record_history ? 1 : 0};
  kronop_gpe_result r{};
  std::vector<double> hist(config.record_history ? 5 * static_cast<size_t>(config.max_iterations) : 0);
  check(kronop_gpe_gradient_flow(p.hamiltonian.sep->context().get(), p.hamiltonian.sep->handle(),
                                 p.hamiltonian.diagonal ? p.hamiltonian.diagonal->data() : nullptr,
                                 p.laplacian->handle(), p.beta, &c,
                                 initial ? initial->data() : nullptr, state.data(), &r,
                                 config.record_history ? hist.data() : nullptr));
  GpeResult out{r.energy, r.eigenvalue, r.iterations, static_cast<long>(r.linear_solves),
                r.converged != 0, {}};
  for (int i = 0; i < r.history_len; ++i)
    out.history.push_back({static_cast<int>(hist[5 * i]), hist[5 * i + 1], hist[5 * i + 2],
                           static_cast<long>(hist[5 * i + 3]), hist[5 * i + 4]});
  return out;
}

// ------------------------------------------ slab decomposition (kronop_slab_*, multi-GPU) --
// SeparableOperator / FullOperator / pcg on fields cut into slabs of the slowest axis across the
// GPUs of `devices` (one process; a repeated device gives virtual slabs on one GPU). Host fields
// keep the reference's value semantics: scattered to the parts, transformed, gathered back.
class SlabOperator {
 public:
  SlabOperator(const std::vector<int>& devices, std::vector<AxisEigens> axes, double shift = 0.0,
               std::shared_ptr<const MassWeights> mass = nullptr)
      : axes_(std::move(axes)) {
    const int d = static_cast<int>(axes_.size());
    std::vector<int> n(d);
    std::vector<const double*> T(d), Ti(d), L(d), M(d);
    for (int a = 0; a < d; ++a) {
      n[a] = axes_[a].size();
      T[a] = axes_[a].transform.data();
      Ti[a] = axes_[a].inverse_transform.data();
      L[a] = axes_[a].eigenvalues.data();
      if (mass) M[a] = (*mass)[a].data();
    }
    kronop_slab* h = nullptr;
    check(kronop_slab_create(static_cast<int>(devices.size()), devices.data(), d, n.data(),
                             T.data(), Ti.data(), L.data(), mass ? M.data() : nullptr, shift, &h));
    slab_.reset(h, [](kronop_slab* p) { kronop_slab_destroy(p); });
    int nl = 0;
    check(kronop_slab_info(h, nullptr, &nl, nullptr));
    elems_.resize(nl);
    for (int i = 0; i < nl; ++i)
      check(kronop_slab_part(h, i, nullptr, nullptr, nullptr, nullptr, &elems_[i]));
  }
  int parts() const { return static_cast<int>(elems_.size()); }
  void set_shift(double s) { check(kronop_slab_set_shift(slab_.get(), s)); }

  template <typename S>
  TensorField<S> apply(const TensorField<S>& u) const {  // operators.cpp:31-40
    return run(u, [&](double* const* in, double* const* out) {
      check(kronop_slab_apply(slab_.get(), in, is_complex_v<S>, nullptr, 0.0, out));
    });
  }
  template <typename S>
  TensorField<S> solve(const TensorField<S>& b) const {  // operators.cpp:42-61
    return run(b, [&](double* const* in, double* const* out) {
      check(kronop_slab_solve(slab_.get(), in, is_complex_v<S>, out));
    });
  }
  ComplexField propagate(const ComplexField& psi, double dt) const {  // operators.cpp:63-75
    return run(psi, [&](double* const* in, double* const* out) {
      check(kronop_slab_propagate(slab_.get(), in, dt, out));
    });
  }
  // pcg(FullOperator{this, diagonal}.apply, this.solve, b, x&) (pcg.cpp:8-81); x in/out
  // gpe_gradient_flow, a_u flow (gpe.cpp:55-165) on the Hamiltonian this + diagonal (V2 or
  // null); config.kind must be AdaptiveMetric, init Constant (or Supplied with `initial`).
  // `state` receives the final state (host, value semantics).
  GpeResult gpe_au(const RealField* diagonal, double beta, const GpeFlowConfig& config,
                   RealField& state, const RealField* initial = nullptr) const {
    Parts dd(*this, 1), di(*this, 1), ds(*this, 1);
    if (diagonal)
      check(kronop_slab_scatter(slab_.get(), diagonal->data(), 0, dd.p.data()));
    if (initial)
      check(kronop_slab_scatter(slab_.get(), initial->data(), 0, di.p.data()));
    kronop_gpe_config c{KRONOP_GPE_AU, config.step, config.metric_shift, config.energy_rel_tol,
                        config.max_iterations, config.inner.c(),
                        config.init == GpeInit::Supplied ? KRONOP_GPE_INIT_SUPPLIED
                                                         : KRONOP_GPE_INIT_CONSTANT,
                        config.record_history ? 1 : 0};
    kronop_gpe_result r{};
    std::vector<double> hist(config.record_history ? 5 * static_cast<size_t>(config.max_iterations)
                                                   : 0);
    check(kronop_slab_gpe_au(slab_.get(), diagonal ? dd.p.data() : nullptr, beta, &c,
                             initial ? di.p.data() : nullptr, ds.p.data(), &r,
                             config.record_history ? hist.data() : nullptr));
    check(kronop_slab_gather(slab_.get(), ds.p.data(), 0, state.data()));
    GpeResult out{r.energy, r.eigenvalue, r.iterations, static_cast<long>(r.linear_solves),
                  r.converged != 0, {}};
    for (int i = 0; i < r.history_len; ++i)
      out.history.push_back({static_cast<int>(hist[5 * i]), hist[5 * i + 1], hist[5 * i + 2],
                             static_cast<long>(hist[5 * i + 3]), hist[5 * i + 4]});
    return out;
  }

  PcgReport pcg(const RealField* diagonal, const RealField& b, RealField& x,
                const PcgConfig& cfg) const {
    Parts db(*this, 1), dx(*this, 1), dd(*this, 1);
    check(kronop_slab_scatter(slab_.get(), reinterpret_cast<const double*>(b.data()), 0, db.p.data()));
    check(kronop_slab_scatter(slab_.get(), reinterpret_cast<const double*>(x.data()), 0, dx.p.data()));
    if (diagonal)
      check(kronop_slab_scatter(slab_.get(), diagonal->data(), 0, dd.p.data()));
    kronop_pcg_config c{cfg.rel_tol, cfg.max_iter, cfg.record_history ? 1 : 0,
                        cfg.preconditioned_norm ? 1 : 0, cfg.stagnation_window};
    kronop_pcg_report r{};
    std::vector<double> hist(static_cast<size_t>(cfg.max_iter) + 1);
    check(kronop_slab_pcg(slab_.get(), diagonal ? dd.p.data() : nullptr, 0.0, db.p.data(),
                          dx.p.data(), &c, &r, hist.data()));
    check(kronop_slab_gather(slab_.get(), dx.p.data(), 0, x.data()));
    PcgReport rep;
    rep.iterations = r.iterations;
    rep.final_residual = r.final_residual;
    rep.converged = r.converged != 0;
    if (cfg.record_history) rep.history.assign(hist.begin(), hist.begin() + r.history_len);
    return rep;
  }

 private:
  struct Parts {  // one device buffer per local part
    const SlabOperator* o;
    std::vector<double*> p;
    Parts(const SlabOperator& op, int c) : o(&op), p(op.elems_.size(), nullptr) {
      for (size_t i = 0; i < p.size(); ++i)
        check(kronop_slab_field_alloc(op.slab_.get(), static_cast<int>(i),
                                      static_cast<size_t>(op.elems_[i]) * c, &p[i]));
    }
    ~Parts() {
      for (size_t i = 0; i < p.size(); ++i) kronop_slab_field_free(o->slab_.get(), static_cast<int>(i), p[i]);
    }
  };
  template <typename S, class F>
  TensorField<S> run(const TensorField<S>& in, F&& f) const {
    constexpr int c = is_complex_v<S> ? 2 : 1;
    Parts a(*this, c), b(*this, c);
    check(kronop_slab_scatter(slab_.get(), reinterpret_cast<const double*>(in.data()),
                              is_complex_v<S>, a.p.data()));
    f(a.p.data(), b.p.data());
    TensorField<S> out(in.shape());
    check(kronop_slab_gather(slab_.get(), b.p.data(), is_complex_v<S>,
                             reinterpret_cast<double*>(out.data())));
    out.set_mass(in.mass());
    return out;
  }
  std::vector<AxisEigens> axes_;
  std::shared_ptr<kronop_slab> slab_;
  std::vector<long long> elems_;
};

}  // namespace kronop
