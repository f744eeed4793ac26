// The reference's C++ API (include/kronop/kronop.hpp) used the way the reference's own unit tests
// use theirs (proj/tests/test_operators.cpp, test_pcg.cpp, test_splitting.cpp, test_ground_state.cpp).
// Built and run by tests/test_cpp_api.py on the GPU box; prints one line per check, exits non-zero
// on the first failure.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>

#include "kronop/kronop.hpp"

using namespace kronop;

static int g_checks = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      std::exit(1);                                                      \
    }                                                                    \
  } while (0)

static double uniform(std::uint64_t& state) {  // SplitMix64::uniform_pm1 (rng.hpp:16-31)
  state += 0x9E3779B97F4A7C15ULL;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return static_cast<double>((z ^ (z >> 31)) >> 11) * 0x1.0p-52 - 1.0;
}

int main() {
  Context ctx(0);
  const auto osc = [](double x) { return x * x; };

  // test_operators.cpp:30-46 — apply reproduces eigenvectors of the Kronecker sum
  {
    const Basis1D b = assemble_sem(2.0, 3, 4);
    std::vector<AxisEigens> axes = {build_axis(b, osc), build_axis(b, osc)};
    SeparableOperator op(ctx, axes, 0.5);
    const int n = axes[0].size();
    RealField u({n, n});
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        u[i + n * j] = axes[0].transform[i + n * 2] * axes[1].transform[j + n * 0];
    const double lam = axes[0].eigenvalues[2] + axes[1].eigenvalues[0];
    const RealField hu = op.apply(u);
    double err = 0.0, umax = 0.0;
    for (std::size_t k = 0; k < u.size(); ++k) {
      err = std::max(err, std::abs(hu[k] - (lam - 0.5) * u[k]));
      umax = std::max(umax, std::abs(u[k]));
    }
    CHECK(err < 1e-9 * std::abs(lam) * umax);
    std::printf("ok apply-eigenvector err %.3e\n", err);
  }

  // test_operators.cpp:60-93 — solve inverts apply; singular shift refused (:95-102)
  {
    const Basis1D b = assemble_sem(1.0, 4, 3);
    std::vector<AxisEigens> axes = {build_axis(b, osc), build_axis(b, osc)};
    SeparableOperator op(ctx, axes, 0.0);
    const int n = b.size();
    RealField rhs({n, n});
    std::uint64_t s = 3;
    for (std::size_t k = 0; k < rhs.size(); ++k) rhs[k] = uniform(s);
    const RealField x = op.solve(rhs);
    const RealField back = op.apply(x);
    double num = 0, den = 0;
    for (std::size_t k = 0; k < rhs.size(); ++k) {
      num += (back[k] - rhs[k]) * (back[k] - rhs[k]);
      den += rhs[k] * rhs[k];
    }
    CHECK(std::sqrt(num / den) < 1e-12);
    // the batched form (kronop_sep_solve_host_batch) equals solve() item by item
    {
      std::vector<RealField> bs;
      for (int i = 0; i < 3; ++i) {
        RealField r({n, n});
        for (std::size_t k = 0; k < r.size(); ++k) r[k] = uniform(s);
        bs.push_back(r);
      }
      const std::vector<RealField> xs = op.solve(bs);
      CHECK(xs.size() == 3);
      for (int i = 0; i < 3; ++i) {
        const RealField xi = op.solve(bs[i]);
        double dn = 0, dd = 0;
        for (std::size_t k = 0; k < xi.size(); ++k) {
          dn += (xs[i][k] - xi[k]) * (xs[i][k] - xi[k]);
          dd += xi[k] * xi[k];
        }
        CHECK(std::sqrt(dn / dd) < 1e-15);
      }
    }
    op.set_shift(axes[0].eigenvalues[1] + axes[1].eigenvalues[3]);
    bool threw = false;
    try {
      op.solve(rhs);
    } catch (const NumericalError&) {
      threw = true;
    }
    CHECK(threw);
    std::printf("ok solve residual %.3e, singular shift -> NumericalError\n", std::sqrt(num / den));
  }

  // test_operators.cpp:104-137 — propagation is unitary in the mass norm and reversible
  {
    const Basis1D b = assemble_sem(8.0, 4, 7);
    auto mass = std::make_shared<MassWeights>(MassWeights{b.mass, b.mass, b.mass});
    std::vector<AxisEigens> axes(3, build_axis(b, osc));
    SeparableOperator op(ctx, axes, 0.0, mass);
    const int n = b.size();
    ComplexField psi({n, n, n});
    std::uint64_t s = 9;
    for (std::size_t k = 0; k < psi.size(); ++k) psi[k] = {uniform(s), uniform(s)};
    const ComplexField fwd = op.propagate(psi, 0.37);
    const ComplexField back = op.propagate(fwd, -0.37);
    double err = 0, nrm = 0, m0 = 0, m1 = 0;
    for (int k2 = 0; k2 < n; ++k2)
      for (int k1 = 0; k1 < n; ++k1)
        for (int k0 = 0; k0 < n; ++k0) {
          const std::size_t k = k0 + n * (k1 + static_cast<std::size_t>(n) * k2);
          const double w = b.mass[k0] * b.mass[k1] * b.mass[k2];
          err += std::norm(back[k] - psi[k]);
          nrm += std::norm(psi[k]);
          m0 += w * std::norm(psi[k]);
          m1 += w * std::norm(fwd[k]);
        }
    CHECK(std::sqrt(err / nrm) < 1e-11);
    CHECK(std::abs(m1 - m0) < 1e-11 * m0);
    std::printf("ok propagate reversible %.3e, mass-norm drift %.3e\n", std::sqrt(err / nrm),
                std::abs(m1 - m0) / m0);
  }

  // test_pcg.cpp:36-69 — the exact preconditioner converges in one iteration (device-resident)
  {
    const Basis1D b = assemble_sem(2.0, 3, 4);
    std::vector<AxisEigens> axes(3, build_axis(b, osc));
    SeparableOperator op(ctx, axes, 0.0);
    const int n = b.size();
    RealField rhs({n, n, n});
    std::uint64_t s = 5;
    for (std::size_t k = 0; k < rhs.size(); ++k) rhs[k] = uniform(s);
    DeviceField<double> db(ctx, rhs), dx(ctx, RealField({n, n, n}));
    PcgConfig cfg;
    cfg.rel_tol = 1e-10;
    cfg.record_history = true;
    const PcgReport rep = pcg(ctx, LinearMap::apply(op), LinearMap::solve(op), db, dx, cfg);
    CHECK(rep.converged && rep.iterations == 1);
    CHECK(rep.history.size() == 2 && rep.history[1] <= 1e-10);
    std::printf("ok pcg exact preconditioner: %d iteration(s), residual %.3e\n", rep.iterations,
                rep.final_residual);
    // FP64 emulated on the INT8 tensor cores: the same solve to FP64 level
    DeviceField<double> d64(ctx, RealField({n, n, n})), doz(ctx, RealField({n, n, n}));
    op.solve(db, d64);
    op.solve_variant(db, KRONOP_PREC_FP64_OZAKI, doz);
    const RealField h64 = d64.download(), hoz = doz.download();
    double e2 = 0.0, n2 = 0.0;
    for (std::size_t k = 0; k < h64.size(); ++k) {
      e2 += (hoz[k] - h64[k]) * (hoz[k] - h64[k]);
      n2 += h64[k] * h64[k];
    }
    CHECK(std::sqrt(e2 / n2) < 1e-12);
    std::printf("ok ozaki solve variant rel diff %.3e\n", std::sqrt(e2 / n2));
  }

  // test_splitting.cpp:29-35 — Yoshida coefficients
  {
    const YoshidaCoeffs c = yoshida_coeffs();
    CHECK(std::abs(2.0 * c.gamma1 + c.gamma2 - 1.0) < 1e-15);
    CHECK(std::abs(2.0 * std::pow(c.gamma1, 3) + std::pow(c.gamma2, 3)) < 1e-14);
    std::printf("ok yoshida %.15f %.15f\n", c.gamma1, c.gamma2);
  }

  // test_ground_state.cpp — separable inverse iteration matches the sum of axis minima
  {
    const Basis1D b = assemble_sem(8.0, 4, 8);
    auto mass = std::make_shared<MassWeights>(MassWeights{b.mass, b.mass, b.mass});
    const auto f = [](double x) { return x * x + 100.0 * std::pow(std::sin(M_PI * x / 4.0), 2); };
    std::vector<AxisEigens> axes(3, build_axis(b, f));
    SeparableOperator sep(ctx, axes, 0.0, mass);
    const int n = b.size();
    DeviceField<double> init(ctx, RealField::constant({n, n, n}, 1.0)), vec(ctx, Shape{n, n, n});
    FullOperator op{&sep, nullptr};
    const EigenpairResult r = inverse_iteration(op, InverseIterationConfig{}, init, vec);
    const double exact = 3.0 * axes[0].eigenvalues[0];
    CHECK(r.converged);
    CHECK(std::abs(r.eigenvalue - exact) < 1e-11 * exact);
    std::printf("ok inverse iteration lambda %.12f (exact %.12f) in %d outer\n", r.eigenvalue,
                exact, r.outer_iterations);
  }

  // test_gpe.cpp — H1 and a_u flows agree (acceptance.cpp:397-401 criterion 8c, small grid)
  {
    const Basis1D b = assemble_sem(8.0, 2, 12);
    auto mass = std::make_shared<MassWeights>(MassWeights{b.mass, b.mass, b.mass});
    const auto f = [](double x) { return x * x + 100.0 * std::pow(std::sin(M_PI * x / 4.0), 2); };
    std::vector<AxisEigens> axes(3, build_axis(b, f));
    std::vector<AxisEigens> lap_axes(3, build_axis(b, [](double) { return 0.0; }));
    SeparableOperator sep(ctx, axes, 0.0, mass), lap(ctx, lap_axes, 0.0, mass);
    const int n = b.size();
    GpeProblem prob{FullOperator{&sep, nullptr}, &lap, 10.0};
    GpeFlowConfig cfg;
    cfg.energy_rel_tol = 1e-13;
    DeviceField<double> s1(ctx, Shape{n, n, n}), s2(ctx, Shape{n, n, n});
    const GpeResult h1 = gpe_gradient_flow(prob, cfg, s1);
    cfg.kind = GpeFlowKind::AdaptiveMetric;
    cfg.step = 1.0;
    const GpeResult au = gpe_gradient_flow(prob, cfg, s2);
    CHECK(h1.converged && au.converged);
    CHECK(std::abs(h1.energy - au.energy) <= 1e-10 * std::abs(h1.energy));
    CHECK(std::abs(gpe_energy(prob, s1) - h1.energy) <= 1e-12 * std::abs(h1.energy));
    std::printf("ok gpe h1 E=%.12f (%d its), a_u E=%.12f (%d its)\n", h1.energy, h1.iterations,
                au.energy, au.iterations);
  }

  // test_axis_eigen.cpp:130-140 — Hermite axis oscillator levels
  {
    const HermiteBasis hb = hermite_basis(60);
    const AxisEigens ax = build_axis(hb, osc);
    for (int j = 0; j < 4; ++j) CHECK(std::abs(ax.eigenvalues[j] - (2.0 * j + 1.0)) < 1e-9);
    std::printf("ok hermite levels %.12f %.12f\n", ax.eigenvalues[0], ax.eigenvalues[3]);
  }

  // fieldio.cpp:28-73 — host and device checkpoints round-trip bit for bit
  {
    ComplexField psi({7, 5, 3});
    std::uint64_t s = 11;
    for (std::size_t k = 0; k < psi.size(); ++k) psi[k] = {uniform(s), uniform(s)};
    dump_field("/tmp/kronop_cpp_io.kf", psi);
    const LoadedField back = load_field("/tmp/kronop_cpp_io.kf");
    const ComplexField& b2 = std::get<ComplexField>(back);
    for (std::size_t k = 0; k < psi.size(); ++k) CHECK(b2[k] == psi[k]);
    DeviceField<std::complex<double>> dpsi(ctx, psi);
    dump_field("/tmp/kronop_cpp_io2.kf", ctx, dpsi);
    const auto d2 = load_field<std::complex<double>>("/tmp/kronop_cpp_io2.kf", ctx).download();
    for (std::size_t k = 0; k < psi.size(); ++k) CHECK(d2[k] == psi[k]);
    std::printf("ok field io round trips\n");
  }

  // errors.hpp: ParameterError on bad input through the C-ABI
  {
    bool threw = false;
    try {
      assemble_sem(-1.0, 3, 2);
    } catch (const ParameterError&) {
      threw = true;
    }
    CHECK(threw);
  }
  // slab decomposition behind the C-ABI from C++ (kronop::SlabOperator, virtual slabs on device
  // 0): solve / apply / propagate equal the single-device operator, pcg equals pcg
  {
    const Basis1D b = assemble_sem(8.0, 5, 5);  // 24^3
    std::vector<AxisEigens> axes = {build_axis(b, osc), build_axis(b, osc), build_axis(b, osc)};
    SeparableOperator op(ctx, axes, -0.3);
    const int n = axes[0].size();
    RealField f({n, n, n});
    std::uint64_t st = 5;
    for (std::size_t k = 0; k < f.size(); ++k) f[k] = uniform(st);
    ComplexField psi({n, n, n});
    for (std::size_t k = 0; k < psi.size(); ++k) psi[k] = {uniform(st), uniform(st)};
    for (int P : {2, 3}) {
      SlabOperator so(std::vector<int>(P, 0), axes, -0.3);
      CHECK(so.parts() == P);
      auto relerr = [](const auto& x, const auto& y) {
        double num = 0.0, den = 0.0;
        for (std::size_t k = 0; k < x.size(); ++k) {
          num += std::norm(std::complex<double>(x[k]) - std::complex<double>(y[k]));
          den += std::norm(std::complex<double>(y[k]));
        }
        return std::sqrt(num / den);
      };
      const double es = relerr(so.solve(f), op.solve(f));
      const double ea = relerr(so.apply(f), op.apply(f));
      const double ep = relerr(so.propagate(psi, 0.02), op.propagate(psi, 0.02));
      CHECK(es < 1e-13 && ea < 1e-13 && ep < 1e-13);
      std::printf("ok slab P=%d solve %.2e apply %.2e propagate %.2e\n", P, es, ea, ep);
    }
    // a_u GPE flow on 3 virtual slabs equals the single-device flow (gpe.cpp:118-157)
    auto mass = std::make_shared<const MassWeights>(MassWeights{b.mass, b.mass, b.mass});
    SeparableOperator ham(ctx, axes, 0.0, mass);
    SeparableOperator lap(ctx, {build_axis(b, [](double) { return 0.0; }),
                                build_axis(b, [](double) { return 0.0; }),
                                build_axis(b, [](double) { return 0.0; })}, 0.0, mass);
    GpeProblem prob{FullOperator{&ham, nullptr}, &lap, 10.0};
    GpeFlowConfig cfg;
    cfg.kind = GpeFlowKind::AdaptiveMetric;
    cfg.step = 1.0;
    cfg.energy_rel_tol = 1e-30;
    cfg.max_iterations = 6;
    cfg.init = GpeInit::Constant;
    DeviceField<double> gst(ctx, Shape{n, n, n});
    const GpeResult g1 = gpe_gradient_flow(prob, cfg, gst);
    SlabOperator so(std::vector<int>(3, 0), axes, 0.0, mass);
    RealField sst({n, n, n});
    const GpeResult g3 = so.gpe_au(nullptr, 10.0, cfg, sst);
    CHECK(g3.iterations == g1.iterations && g3.linear_solves == g1.linear_solves);
    CHECK(std::abs(g3.energy - g1.energy) <= 1e-11 * std::abs(g1.energy));
    std::printf("ok slab gpe_au E %.12f vs %.12f, %ld solves\n", g3.energy, g1.energy,
                g3.linear_solves);
  }

  std::printf("all %d checks passed\n", g_checks);
  return 0;
}
