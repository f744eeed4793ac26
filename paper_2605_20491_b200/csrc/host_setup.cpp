// Host prerequisites of the hot path: GLL / Gauss-Legendre rules, Q^k SEM
// assembly, linear prolongation, the Eigen-free symmetric eigensolver and the per-axis
// factorisation T = M^{-1/2} Q, T^{-1} = Q^T M^{1/2}. These run once per operator on the CPU (O(n^3)
// per axis); everything per-application runs on the GPU.
//
// Restated from proj/src/quadrature.cpp, basis1d.cpp and axis.cpp (cited per function). The
// reference's eigensolver is Eigen's SelfAdjointEigenSolver (axis.cpp:36); Eigen is not available,
// so sym_eig here is a Householder tridiagonalisation followed by implicit-shift QL, which is the
// same algorithm family (tridiagonal reduction + implicit symmetric QR/QL) and is held to the
// reference's own tolerances (proj/tests/test_axis_eigen.cpp:75-112).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/kronop_cuda.h"
#include "host_setup.hpp"

namespace kronop_host {

// ------------------------------------------------------------------ quadrature.cpp --
void legendre_pair(int k, double x, double& p, double& dp) {  // quadrature.cpp:12-26
  double p0 = 1.0, p1 = x;
  if (k == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int m = 2; m <= k; ++m) {
    const double p2 = ((2 * m - 1) * x * p1 - (m - 1) * p0) / m;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  dp = k * (x * p1 - p0) / (x * x - 1.0);
}

static std::vector<double> barycentric_weights(const std::vector<double>& nodes) {  // :28-39
  const int n = static_cast<int>(nodes.size());
  std::vector<double> w(n, 1.0);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j)
      if (j != i) w[i] *= nodes[i] - nodes[j];
    w[i] = 1.0 / w[i];
  }
  return w;
}

void gauss_legendre(int m, std::vector<double>& nodes, std::vector<double>& weights) {  // :41-87
  if (m < 1 || m > 16) throw Error(KRONOP_EPARAM, "gauss_legendre: points must be in [1, 16]");
  nodes.assign(m, 0.0);
  weights.assign(m, 0.0);
  if (m == 1) {
    weights[0] = 2.0;
    return;
  }
  for (int i = 0; i < m; ++i) {
    double x = -std::cos(M_PI * (4.0 * i + 3.0) / (4.0 * m + 2.0));
    double p, dp;
    bool done = false;
    for (int it = 0; it < 100; ++it) {
      legendre_pair(m, x, p, dp);
      const double dx = p / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) {
        done = true;
        break;
      }
    }
    if (!done) throw Error(KRONOP_ENUMERICAL, "gauss_legendre: Newton failed to converge");
    legendre_pair(m, x, p, dp);
    nodes[i] = x;
    weights[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  for (int i = 0; i < m / 2; ++i) {
    const int j = m - 1 - i;
    const double xm = 0.5 * (nodes[j] - nodes[i]);
    nodes[i] = -xm;
    nodes[j] = xm;
    const double wm = 0.5 * (weights[i] + weights[j]);
    weights[i] = weights[j] = wm;
  }
  if (m % 2 == 1) nodes[m / 2] = 0.0;
}

static std::vector<double> lagrange_diff_matrix(const std::vector<double>& nodes) {  // :95-110
  const int n = static_cast<int>(nodes.size());
  const std::vector<double> b = barycentric_weights(nodes);
  std::vector<double> d(static_cast<size_t>(n) * n, 0.0);  // col-major
  for (int i = 0; i < n; ++i) {
    double diag = 0.0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const double v = (b[j] / b[i]) / (nodes[i] - nodes[j]);
      d[i + static_cast<size_t>(n) * j] = v;
      diag -= v;
    }
    d[i + static_cast<size_t>(n) * i] = diag;
  }
  return d;
}

GllRule gll_rule(int degree) {  // quadrature.cpp:124-187
  if (degree < 1 || degree > 40) throw Error(KRONOP_EPARAM, "gll_rule: degree must be in [1, 40]");
  const int k = degree;
  GllRule rule;
  rule.degree = k;
  rule.nodes.assign(k + 1, 0.0);
  rule.weights.assign(k + 1, 0.0);
  rule.nodes[0] = -1.0;
  rule.nodes[k] = 1.0;
  for (int i = 1; i < k; ++i) {
    double x = -std::cos(M_PI * i / k);
    double lo = -std::cos(M_PI * (i - 0.5) / k);
    double hi = -std::cos(M_PI * (i + 0.5) / k);
    bool done = (k == 2 && i == 1);
    if (done) x = 0.0;
    for (int it = 0; !done && it < 100; ++it) {
      double p, dp;
      legendre_pair(k, x, p, dp);
      const double ddp = (2.0 * x * dp - k * (k + 1.0) * p) / (1.0 - x * x);
      const double dx = dp / ddp;
      x -= dx;
      if (x <= lo || x >= hi) break;
      if (std::abs(dx) < 1e-14) done = true;
    }
    if (!done) {
      double plo, dplo, tmp;
      legendre_pair(k, lo, tmp, dplo);
      plo = dplo;
      for (int it = 0; it < 200; ++it) {
        x = 0.5 * (lo + hi);
        double p, dp;
        legendre_pair(k, x, p, dp);
        if ((dp > 0) == (plo > 0)) {
          lo = x;
          plo = dp;
        } else {
          hi = x;
        }
        if (hi - lo < 1e-15) break;
      }
    }
    rule.nodes[i] = x;
  }
  for (int i = 0; i <= k / 2; ++i) {
    const int j = k - i;
    const double xm = 0.5 * (rule.nodes[j] - rule.nodes[i]);
    rule.nodes[i] = -xm;
    rule.nodes[j] = xm;
  }
  if (k % 2 == 0) rule.nodes[k / 2] = 0.0;
  for (int i = 0; i <= k; ++i) {
    double p, dp;
    legendre_pair(k, rule.nodes[i], p, dp);
    rule.weights[i] = 2.0 / (k * (k + 1.0) * p * p);
  }
  rule.diff = lagrange_diff_matrix(rule.nodes);
  return rule;
}

// --------------------------------------------------------------------- basis1d.cpp --
SemBasis assemble_sem(double half_width, int cell_count, int degree) {  // basis1d.cpp:10-60
  if (half_width <= 0.0) throw Error(KRONOP_EPARAM, "assemble_sem: half_width must be positive");
  if (cell_count < 1) throw Error(KRONOP_EPARAM, "assemble_sem: cell_count must be >= 1");
  if (degree < 1) throw Error(KRONOP_EPARAM, "assemble_sem: degree must be >= 1");
  SemBasis basis;
  basis.half_width = half_width;
  basis.cell_count = cell_count;
  basis.degree = degree;
  basis.rule = gll_rule(degree);
  const int k = degree;
  const double h = 2.0 * half_width / cell_count;
  const int ng = cell_count * k + 1;
  std::vector<double> xg(ng);
  for (int c = 0; c < cell_count; ++c) {
    const double left = -half_width + c * h;
    for (int j = 0; j <= k; ++j) xg[c * k + j] = left + (basis.rule.nodes[j] + 1.0) * h / 2.0;
  }
  xg.front() = -half_width;
  xg.back() = half_width;
  const std::vector<double>& w = basis.rule.weights;
  const std::vector<double>& d = basis.rule.diff;  // col-major (k+1)^2
  const int kk = k + 1;
  std::vector<double> sloc(static_cast<size_t>(kk) * kk);
  for (int i = 0; i <= k; ++i)
    for (int j = 0; j <= k; ++j) {
      double acc = 0.0;
      for (int q = 0; q <= k; ++q) acc += w[q] * d[q + kk * i] * d[q + kk * j];
      sloc[i + kk * j] = (2.0 / h) * acc;
    }
  const int n = ng - 2;
  basis.nodes.assign(xg.begin() + 1, xg.end() - 1);
  std::vector<double> mg(ng, 0.0);
  // Global stiffness restricted to the interior (Dirichlet trim), assembled directly in
  // col-major n x n; contributions to the same entry accumulate in cell order as in :52-57.
  basis.stiffness.assign(static_cast<size_t>(n) * n, 0.0);
  for (int c = 0; c < cell_count; ++c) {
    const int base = c * k;
    for (int i = 0; i <= k; ++i) {
      mg[base + i] += w[i] * h / 2.0;
      const int gi = base + i - 1;
      if (gi < 0 || gi >= n) continue;
      for (int j = 0; j <= k; ++j) {
        const int gj = base + j - 1;
        if (gj < 0 || gj >= n) continue;
        basis.stiffness[gi + static_cast<size_t>(n) * gj] += sloc[i + kk * j];
      }
    }
  }
  basis.mass.assign(mg.begin() + 1, mg.end() - 1);
  return basis;
}

std::vector<double> interp_matrix(const SemBasis& coarse, const SemBasis& fine) {  // :62-88
  if (coarse.half_width != fine.half_width)
    throw Error(KRONOP_EPARAM, "interp_matrix: bases must share the same domain");
  if (fine.size() < coarse.size())
    throw Error(KRONOP_EPARAM, "interp_matrix: fine basis must not be smaller than the coarse one");
  const int nc = coarse.size(), nf = fine.size();
  const double l = coarse.half_width;
  std::vector<double> xe;
  xe.reserve(nc + 2);
  xe.push_back(-l);
  xe.insert(xe.end(), coarse.nodes.begin(), coarse.nodes.end());
  xe.push_back(l);
  std::vector<double> p(static_cast<size_t>(nf) * nc, 0.0);
  for (int i = 0; i < nf; ++i) {
    const double t = fine.nodes[i];
    auto it = std::upper_bound(xe.begin(), xe.end(), t);
    int j = static_cast<int>(it - xe.begin()) - 1;
    j = std::clamp(j, 0, nc);
    const double w1 = (t - xe[j]) / (xe[j + 1] - xe[j]);
    if (j - 1 >= 0 && j - 1 < nc) p[i + static_cast<size_t>(nf) * (j - 1)] = 1.0 - w1;
    if (j < nc) p[i + static_cast<size_t>(nf) * j] = w1;
  }
  return p;
}

// ------------------------------------------------------------------------ axis.cpp --
// Householder tridiagonalisation (accumulating the orthogonal transform) followed by the
// implicit-shift QL iteration on the tridiagonal matrix (the classic EISPACK tred2/tql2 pair).
// V(r, c) = v[r + n*c] is column-major, so every inner loop (over r) walks a contiguous column and
// the eigenvectors end up in the columns of v.
static void tridiagonalize(int n, std::vector<double>& v, std::vector<double>& d,
                           std::vector<double>& e) {
  auto V = [&](int r, int c) -> double& { return v[r + static_cast<size_t>(n) * c]; };
  for (int j = 0; j < n; ++j) d[j] = V(n - 1, j);
  for (int i = n - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
    for (int k = 0; k < i; ++k) scale += std::abs(d[k]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
      for (int j = 0; j < i; ++j) {
        d[j] = V(i - 1, j);
        V(i, j) = 0.0;
        V(j, i) = 0.0;
      }
    } else {
      for (int k = 0; k < i; ++k) {
        d[k] /= scale;
        h += d[k] * d[k];
      }
      double f = d[i - 1];
      double g = std::sqrt(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h = h - f * g;
      d[i - 1] = f - g;
      for (int j = 0; j < i; ++j) e[j] = 0.0;
      for (int j = 0; j < i; ++j) {
        f = d[j];
        V(j, i) = f;
        g = e[j] + V(j, j) * f;
        const double* cj = &V(0, j);
        for (int k = j + 1; k <= i - 1; ++k) {
          g += cj[k] * d[k];
          e[k] += cj[k] * f;
        }
        e[j] = g;
      }
      f = 0.0;
      for (int j = 0; j < i; ++j) {
        e[j] /= h;
        f += e[j] * d[j];
      }
      const double hh = f / (h + h);
      for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
      for (int j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
        double* cj = &V(0, j);
        for (int k = j; k <= i - 1; ++k) cj[k] -= (f * e[k] + g * d[k]);
        d[j] = V(i - 1, j);
        V(i, j) = 0.0;
      }
    }
    d[i] = h;
  }
  for (int i = 0; i < n - 1; ++i) {
    V(n - 1, i) = V(i, i);
    V(i, i) = 1.0;
    const double h = d[i + 1];
    const double* ci1 = &V(0, i + 1);
    if (h != 0.0) {
      for (int k = 0; k <= i; ++k) d[k] = ci1[k] / h;
#pragma omp parallel for schedule(static) if (i > 256)
      for (int j = 0; j <= i; ++j) {
        double* cj = &V(0, j);
        double g = 0.0;
        for (int k = 0; k <= i; ++k) g += ci1[k] * cj[k];
        for (int k = 0; k <= i; ++k) cj[k] -= g * d[k];
      }
    }
    double* cw = &V(0, i + 1);
    for (int k = 0; k <= i; ++k) cw[k] = 0.0;
  }
  for (int j = 0; j < n; ++j) {
    d[j] = V(n - 1, j);
    V(n - 1, j) = 0.0;
  }
  V(n - 1, n - 1) = 1.0;
  e[0] = 0.0;
}

static void tridiagonal_ql(int n, std::vector<double>& v, std::vector<double>& d,
                           std::vector<double>& e) {
  // Rotations act on the contiguous columns i and i+1 of the column-major eigenvector matrix.
  auto col = [&](int j) { return v.data() + static_cast<size_t>(n) * j; };
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = std::ldexp(1.0, -52);
  for (int l = 0; l < n; ++l) {
    tst1 = std::max(tst1, std::abs(d[l]) + std::abs(e[l]));
    int m = l;
    while (m < n) {
      if (std::abs(e[m]) <= eps * tst1) break;
      ++m;
    }
    if (m > l) {
      int iter = 0;
      do {
        if (++iter > 200) throw Error(KRONOP_ENUMERICAL, "sym_eig: eigenvalue iteration did not converge");
        double g = d[l];
        double p = (d[l + 1] - g) / (2.0 * e[l]);
        double r = std::hypot(p, 1.0);
        if (p < 0) r = -r;
        d[l] = e[l] / (p + r);
        d[l + 1] = e[l] * (p + r);
        const double dl1 = d[l + 1];
        double h = g - d[l];
        for (int i = l + 2; i < n; ++i) d[i] -= h;
        f += h;
        p = d[m];
        double c = 1.0, c2 = c, c3 = c;
        const double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
        for (int i = m - 1; i >= l; --i) {
          c3 = c2;
          c2 = c;
          s2 = s;
          g = c * e[i];
          h = c * p;
          r = std::hypot(p, e[i]);
          e[i + 1] = s * r;
          s = e[i] / r;
          c = p / r;
          p = c * d[i] - s * g;
          d[i + 1] = h + s * (c * g + s * d[i]);
          double* vi = col(i);
          double* vi1 = col(i + 1);
          for (int k = 0; k < n; ++k) {
            const double hk = vi1[k];
            vi1[k] = s * vi[k] + c * hk;
            vi[k] = c * vi[k] - s * hk;
          }
        }
        p = -s * s2 * c3 * el1 * e[l] / dl1;
        e[l] = s * p;
        d[l] = c * p;
      } while (std::abs(e[l]) > eps * tst1);
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
}

void sym_eig(int n, const double* a, std::vector<double>& lam, std::vector<double>& q) {  // axis.cpp:29-53
  if (n < 1) throw Error(KRONOP_EPARAM, "sym_eig: matrix must be square");
  double amax = 0.0, asym = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      amax = std::max(amax, std::abs(a[i + static_cast<size_t>(n) * j]));
      asym = std::max(asym, std::abs(a[i + static_cast<size_t>(n) * j] -
                                     a[j + static_cast<size_t>(n) * i]));
    }
  if (amax > 0.0 && asym > 1e-8 * amax) throw Error(KRONOP_EPARAM, "sym_eig: input not symmetric");
  std::vector<double> v(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      v[i + static_cast<size_t>(n) * j] =
          0.5 * (a[i + static_cast<size_t>(n) * j] + a[j + static_cast<size_t>(n) * i]);
  std::vector<double> d(n), e(n);
  if (n == 1) {
    d[0] = v[0];
    v[0] = 1.0;
  } else {
    tridiagonalize(n, v, d, e);
    tridiagonal_ql(n, v, d, e);
  }
  // ascending order
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return d[x] < d[y]; });
  lam.resize(n);
  q.resize(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j) {
    lam[j] = d[order[j]];
    const double* src = v.data() + static_cast<size_t>(n) * order[j];
    double* dst = q.data() + static_cast<size_t>(n) * j;
    std::copy(src, src + n, dst);
    // Sign convention (axis.cpp:44-52): first |q_i| >= (1 - 1e-8) max|q| made positive.
    double max_abs = 0.0;
    for (int i = 0; i < n; ++i) max_abs = std::max(max_abs, std::abs(dst[i]));
    for (int i = 0; i < n; ++i) {
      if (std::abs(dst[i]) >= (1.0 - 1e-8) * max_abs) {
        if (dst[i] < 0.0)
          for (int k = 0; k < n; ++k) dst[k] = -dst[k];
        break;
      }
    }
  }
}

AxisFactor build_sem_axis(const SemBasis& basis, const double* fvals) {  // axis.cpp:55-74
  const int n = basis.size();
  std::vector<double> sqrt_m(n), inv_sqrt_m(n);
  for (int i = 0; i < n; ++i) {
    sqrt_m[i] = std::sqrt(basis.mass[i]);
    inv_sqrt_m[i] = 1.0 / sqrt_m[i];
  }
  std::vector<double> a(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      a[i + static_cast<size_t>(n) * j] =
          inv_sqrt_m[i] * basis.stiffness[i + static_cast<size_t>(n) * j] * inv_sqrt_m[j];
  for (int i = 0; i < n; ++i) {
    if (!std::isfinite(fvals[i])) throw Error(KRONOP_EPARAM, "build_axis: f not finite at a node");
    a[i + static_cast<size_t>(n) * i] += fvals[i];
  }
  AxisFactor out;
  std::vector<double> q;
  sym_eig(n, a.data(), out.eigenvalues, q);
  out.transform.resize(static_cast<size_t>(n) * n);
  out.inverse_transform.resize(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      out.transform[i + static_cast<size_t>(n) * j] = inv_sqrt_m[i] * q[i + static_cast<size_t>(n) * j];
      out.inverse_transform[i + static_cast<size_t>(n) * j] =
          q[j + static_cast<size_t>(n) * i] * sqrt_m[j];
    }
  return out;
}

// ---------------------------------------------------------------- even/odd folding --
FoldedAxis build_sem_axis_folded(const SemBasis& basis, const double* fvals) {
  const int n = basis.size();
  const double L = basis.half_width;
  auto S = [&](int i, int j) { return basis.stiffness[i + static_cast<size_t>(n) * j]; };
  double smax = 0.0, fmax = 0.0, mmax = 0.0;
  for (int i = 0; i < n; ++i) {
    fmax = std::max(fmax, std::abs(fvals[i]));
    mmax = std::max(mmax, basis.mass[i]);
    for (int j = 0; j < n; ++j) smax = std::max(smax, std::abs(S(i, j)));
  }
  for (int i = 0; i < n; ++i) {
    const int r = n - 1 - i;
    if (std::abs(basis.nodes[i] + basis.nodes[r]) > 1e-12 * L ||
        std::abs(basis.mass[i] - basis.mass[r]) > 1e-12 * mmax ||
        std::abs(fvals[i] - fvals[r]) > 1e-12 * std::max(fmax, 1e-300))
      throw Error(KRONOP_EPARAM, "build_sem_axis_folded: axis is not mirror symmetric");
    for (int j = 0; j < n; ++j)
      if (std::abs(S(i, j) - S(r, n - 1 - j)) > 1e-12 * smax)
        throw Error(KRONOP_EPARAM, "build_sem_axis_folded: stiffness is not persymmetric");
  }
  // symmetrised axis operator A = M^{-1/2} S M^{-1/2} + diag(f) (axis.cpp:55-66)
  std::vector<double> sq(n), isq(n);
  for (int i = 0; i < n; ++i) {
    sq[i] = std::sqrt(basis.mass[i]);
    isq[i] = 1.0 / sq[i];
  }
  auto A = [&](int i, int j) {
    double a = isq[i] * S(i, j) * isq[j];
    if (i == j) a += fvals[i];
    return a;
  };
  FoldedAxis fa;
  fa.n = n;
  fa.no = n / 2;
  fa.ne = n - fa.no;
  const int no = fa.no, ne = fa.ne;
  const bool odd_n = (n % 2) == 1;
  const int mid = no;  // index of the middle node when n is odd
  const double r2 = std::sqrt(2.0), ir2 = 1.0 / std::sqrt(2.0);
  // blocks in the orthonormal bases (e_i +- e_{n-1-i})/sqrt2 (+ e_mid)
  std::vector<double> ae(static_cast<size_t>(ne) * ne), ao(static_cast<size_t>(no) * no);
  for (int j = 0; j < no; ++j)
    for (int i = 0; i < no; ++i) {
      const double a = A(i, j), b = A(i, n - 1 - j);
      ae[i + static_cast<size_t>(ne) * j] = a + b;
      ao[i + static_cast<size_t>(no) * j] = a - b;
    }
  if (odd_n) {
    for (int i = 0; i < no; ++i) {
      ae[i + static_cast<size_t>(ne) * (ne - 1)] = r2 * A(i, mid);
      ae[(ne - 1) + static_cast<size_t>(ne) * i] = r2 * A(mid, i);
    }
    ae[(ne - 1) + static_cast<size_t>(ne) * (ne - 1)] = A(mid, mid);
  }
  // symmetrise exactly (rounding of a + b vs b + a is already symmetric; guard anyway)
  for (int j = 0; j < ne; ++j)
    for (int i = 0; i < j; ++i) {
      const double v = 0.5 * (ae[i + static_cast<size_t>(ne) * j] + ae[j + static_cast<size_t>(ne) * i]);
      ae[i + static_cast<size_t>(ne) * j] = ae[j + static_cast<size_t>(ne) * i] = v;
    }
  std::vector<double> y, z;
  sym_eig(ne, ae.data(), fa.lam_e, y);
  if (no > 0) sym_eig(no, ao.data(), fa.lam_o, z);
  // full-length eigenvector components of block row i (i < no: mirrored pair, i == mid)
  auto ye = [&](int i, int k) { return y[i + static_cast<size_t>(ne) * k]; };
  auto zo = [&](int i, int k) { return z[i + static_cast<size_t>(no) * k]; };
  // sign rule on the full vector (axis.cpp:44-52): first |q_i| >= (1-1e-8) max|q| is positive.
  // For an even/odd vector the first such index lies in the first half (or is the middle node).
  for (int k = 0; k < ne; ++k) {
    double mx = 0.0;
    for (int i = 0; i < no; ++i) mx = std::max(mx, std::abs(ye(i, k)) * ir2);
    if (odd_n) mx = std::max(mx, std::abs(ye(mid, k)));
    double first = 0.0;
    for (int i = 0; i < no && first == 0.0; ++i)
      if (std::abs(ye(i, k)) * ir2 >= (1.0 - 1e-8) * mx) first = ye(i, k);
    if (first == 0.0 && odd_n) first = ye(mid, k);
    if (first < 0.0)
      for (int i = 0; i < ne; ++i) y[i + static_cast<size_t>(ne) * k] = -y[i + static_cast<size_t>(ne) * k];
  }
  for (int k = 0; k < no; ++k) {
    double mx = 0.0;
    for (int i = 0; i < no; ++i) mx = std::max(mx, std::abs(zo(i, k)));
    for (int i = 0; i < no; ++i)
      if (std::abs(zo(i, k)) >= (1.0 - 1e-8) * mx) {
        if (zo(i, k) < 0.0)
          for (int t = 0; t < no; ++t) z[t + static_cast<size_t>(no) * k] = -z[t + static_cast<size_t>(no) * k];
        break;
      }
  }
  // forward: w_k = sum_i q_k(i) sqrt(m_i) x_i  ->  Fe[k][i] (on u), Fo[k][i] (on v), column-major
  fa.fe.assign(static_cast<size_t>(ne) * ne, 0.0);
  fa.be.assign(static_cast<size_t>(ne) * ne, 0.0);
  for (int k = 0; k < ne; ++k) {
    for (int i = 0; i < no; ++i) {
      fa.fe[k + static_cast<size_t>(ne) * i] = ye(i, k) * ir2 * sq[i];
      fa.be[i + static_cast<size_t>(ne) * k] = ye(i, k) * ir2 * isq[i];
    }
    if (odd_n) {
      fa.fe[k + static_cast<size_t>(ne) * mid] = ye(mid, k) * sq[mid];
      fa.be[mid + static_cast<size_t>(ne) * k] = ye(mid, k) * isq[mid];
    }
  }
  fa.fo.assign(static_cast<size_t>(no) * no, 0.0);
  fa.bo.assign(static_cast<size_t>(no) * no, 0.0);
  for (int k = 0; k < no; ++k)
    for (int i = 0; i < no; ++i) {
      fa.fo[k + static_cast<size_t>(no) * i] = zo(i, k) * ir2 * sq[i];
      fa.bo[i + static_cast<size_t>(no) * k] = zo(i, k) * ir2 * isq[i];
    }
  // ground state column of T: the lowest even mode (the global minimum of a symmetric problem)
  fa.g0.assign(n, 0.0);
  for (int i = 0; i < no; ++i) fa.g0[i] = fa.g0[n - 1 - i] = ye(i, 0) * ir2 * isq[i];
  if (odd_n) fa.g0[mid] = ye(mid, 0) * isq[mid];
  return fa;
}

// ------------------------------------------------------- point evaluation (slices) --
static std::vector<double> lagrange_eval_weights(const std::vector<double>& nodes, double x) {
  // quadrature.cpp:105-122
  const int n = static_cast<int>(nodes.size());
  std::vector<double> w(n, 0.0);
  for (int j = 0; j < n; ++j)
    if (x == nodes[j]) {
      w[j] = 1.0;
      return w;
    }
  const std::vector<double> b = barycentric_weights(nodes);
  double denom = 0.0;
  for (int j = 0; j < n; ++j) {
    w[j] = b[j] / (x - nodes[j]);
    denom += w[j];
  }
  for (int j = 0; j < n; ++j) w[j] /= denom;
  return w;
}

std::vector<double> eval_weights_row(const SemBasis& basis, double x) {  // basis1d.cpp:90-115
  const double l = basis.half_width;
  if (x < -l || x > l) throw Error(KRONOP_EPARAM, "eval_cellwise: target outside [-L, L]");
  const int n = basis.size();
  std::vector<double> row(n, 0.0);
  const auto hit = std::lower_bound(basis.nodes.begin(), basis.nodes.end(), x);
  if (hit != basis.nodes.end() && *hit == x) {
    row[hit - basis.nodes.begin()] = 1.0;
    return row;
  }
  const int k = basis.degree;
  const double h = 2.0 * l / basis.cell_count;
  int c = static_cast<int>(std::floor((x + l) / h));
  c = std::clamp(c, 0, basis.cell_count - 1);
  const double left = -l + c * h;
  const double xi = 2.0 * (x - left) / h - 1.0;
  const std::vector<double> wloc = lagrange_eval_weights(basis.rule.nodes, xi);
  for (int j = 0; j <= k; ++j) {
    const int g = c * k + j;
    if (g == 0 || g == basis.cell_count * k) continue;  // boundary value is zero
    row[g - 1] += wloc[j];
  }
  return row;
}

// ------------------------------------------------------------------ Hermite axes --
HermiteAxis hermite_basis(int n) {  // hermite.cpp:10-66
  if (n < 2) throw Error(KRONOP_EPARAM, "hermite_basis: need n >= 2");
  if (n > 745)
    throw Error(KRONOP_ECAPABILITY,
                "hermite_basis: n > 745 underflows the Hermite recurrence in FP64");
  HermiteAxis b;
  b.n = n;
  // nodes = eigenvalues of the Jacobi matrix (zero diagonal, off-diagonal sqrt(k/2))
  std::vector<double> v(static_cast<size_t>(n) * n, 0.0), d(n, 0.0), e(n, 0.0);
  for (int i = 0; i < n; ++i) v[i + static_cast<size_t>(n) * i] = 1.0;
  for (int k = 1; k < n; ++k) e[k] = std::sqrt(k / 2.0);  // e[i]: coupling of rows i-1 and i
  tridiagonal_ql(n, v, d, e);
  std::sort(d.begin(), d.end());
  b.nodes = d;
  for (int i = 0; i < n / 2; ++i) {  // symmetrise exactly
    const int j = n - 1 - i;
    const double xm = 0.5 * (b.nodes[j] - b.nodes[i]);
    b.nodes[i] = -xm;
    b.nodes[j] = xm;
  }
  if (n % 2 == 1) b.nodes[n / 2] = 0.0;
  b.psi_last.resize(n);
  const double c0 = std::pow(M_PI, -0.25);
  for (int j = 0; j < n; ++j) {
    const double x = b.nodes[j];
    double pk = c0 * std::exp(-x * x / 2.0), pkm1 = 0.0;
    for (int k = 0; k < n - 1; ++k) {
      const double pk1 = x * std::sqrt(2.0 / (k + 1)) * pk - std::sqrt(k / (k + 1.0)) * pkm1;
      pkm1 = pk;
      pk = pk1;
    }
    if (pk == 0.0) throw Error(KRONOP_ECAPABILITY, "hermite_basis: psi_{n-1} underflowed at a node");
    b.psi_last[j] = pk;
  }
  b.diff.assign(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (i != j)
        b.diff[i + static_cast<size_t>(n) * j] =
            b.psi_last[i] / (b.psi_last[j] * (b.nodes[i] - b.nodes[j]));
  b.mass.resize(n);
  for (int j = 0; j < n; ++j) b.mass[j] = 1.0 / (n * b.psi_last[j] * b.psi_last[j]);
  return b;
}

AxisFactor build_hermite_axis(const HermiteAxis& basis, const double* fvals) {
  const int n = basis.n;
  // a = -(W D W^-1)^2 + diag(f), W D W^-1 = [1 / (x_i - x_j)] (hermite.cpp:75-86)
  std::vector<double> w(static_cast<size_t>(n) * n, 0.0), a(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (i != j) w[i + static_cast<size_t>(n) * j] = 1.0 / (basis.nodes[i] - basis.nodes[j]);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k)
        acc += w[i + static_cast<size_t>(n) * k] * w[k + static_cast<size_t>(n) * j];
      a[i + static_cast<size_t>(n) * j] = -acc;
    }
  for (int j = 0; j < n; ++j) {
    if (!std::isfinite(fvals[j]))
      throw Error(KRONOP_EPARAM, "hermite_operator: f not finite at a node");
    a[j + static_cast<size_t>(n) * j] += fvals[j];
  }
  double amax = 0.0, asym = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      amax = std::max(amax, std::abs(a[i + static_cast<size_t>(n) * j]));
      asym = std::max(asym, std::abs(a[i + static_cast<size_t>(n) * j] -
                                     a[j + static_cast<size_t>(n) * i]));
    }
  if (asym > 1e-8 * amax)
    throw Error(KRONOP_ENUMERICAL,
                "hermite_operator: symmetrization degraded at n = " + std::to_string(n));
  AxisFactor out;
  std::vector<double> q;
  sym_eig(n, a.data(), out.eigenvalues, q);  // symmetrises 0.5 (a + a^T) itself
  out.transform.resize(static_cast<size_t>(n) * n);
  out.inverse_transform.resize(static_cast<size_t>(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      // T = diag(psi) Q, T^{-1} = Q^T diag(1/psi) (axis.cpp:80-81)
      out.transform[i + static_cast<size_t>(n) * j] =
          basis.psi_last[i] * q[i + static_cast<size_t>(n) * j];
      out.inverse_transform[i + static_cast<size_t>(n) * j] =
          q[j + static_cast<size_t>(n) * i] * (1.0 / basis.psi_last[j]);
    }
  return out;
}

}  // namespace kronop_host
