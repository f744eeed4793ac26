// Host-side setup (quadrature, SEM basis, Eigen-free sym_eig, per-axis factorisation).
// See host_setup.cpp; these mirror proj/include/kronop/{quadrature,basis1d,axis}.hpp without Eigen.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

namespace kronop_host {

// Carries a kronop status code (KRONOP_EPARAM / ENUMERICAL / ECAPABILITY / ERUNTIME) to the C-ABI
// shim, which turns it into a return code + kronop_last_error() text (errors.hpp:9-30).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct GllRule {  // quadrature.hpp:13-18
  int degree = 0;
  std::vector<double> nodes, weights;
  std::vector<double> diff;  // (k+1)^2 column-major, diff(i,j) = l_j'(x_i)
};

struct SemBasis {  // basis1d.hpp:17-29 (Basis1D)
  double half_width = 0.0;
  int cell_count = 0;
  int degree = 0;
  GllRule rule;
  std::vector<double> nodes, mass;
  std::vector<double> stiffness;  // n x n column-major
  int size() const { return static_cast<int>(nodes.size()); }
};

struct AxisFactor {  // axis.hpp:23-29 (AxisEigens)
  std::vector<double> eigenvalues;        // ascending
  std::vector<double> transform;          // T, n x n column-major
  std::vector<double> inverse_transform;  // T^{-1}
};

// Even/odd folding of a mirror-symmetric axis (symmetric nodes and mass, persymmetric stiffness,
// even potential): the axis operator commutes with the reversal J, so its eigenvectors are even
// or odd and each transform splits into two half-size blocks acting on
//   u_i = x_i + x_{n-1-i} (i < no), u_mid = x_mid (n odd)   and   v_i = x_i - x_{n-1-i}.
// Folded layout along the axis: [u (ne entries) | v (no entries)], ne = ceil(n/2), no = floor(n/2).
struct FoldedAxis {
  int n = 0, ne = 0, no = 0;
  std::vector<double> lam_e, lam_o;  // eigenvalues of the even / odd modes (ascending each)
  std::vector<double> fe, fo;        // forward blocks: w_e = Fe u (ne x ne), w_o = Fo v (no x no)
  std::vector<double> be, bo;        // backward blocks: e = Be w_e, o = Bo w_o; x = unfold(e, o)
  std::vector<double> g0;            // full-length lowest eigenvector column of T (ground state)
};
// Throws KRONOP_EPARAM when the axis is not mirror symmetric to 1e-12 (relative).
FoldedAxis build_sem_axis_folded(const SemBasis& basis, const double* fvals);

// Hermite-function collocation axis on the real line (hermite.hpp:13-19, hermite.cpp:10-66).
struct HermiteAxis {
  int n = 0;
  std::vector<double> nodes;     // ascending, exactly symmetric about 0
  std::vector<double> psi_last;  // psi_{n-1}(x_j)
  std::vector<double> mass;      // 1 / (n psi_{n-1}(x_j)^2)
  std::vector<double> diff;      // n x n column-major, D(i,j) = psi_i / (psi_j (x_i - x_j))
};
HermiteAxis hermite_basis(int n);
// eval_weights_row(basis, x) (basis1d.cpp:90-115): the row r with r . u = u_h(x).
std::vector<double> eval_weights_row(const SemBasis& basis, double x);
// build_axis(HermiteBasis, f) (axis.cpp:76-84 over hermite_operator, hermite.cpp:68-95).
AxisFactor build_hermite_axis(const HermiteAxis& basis, const double* fvals);

void legendre_pair(int k, double x, double& p, double& dp);
void gauss_legendre(int m, std::vector<double>& nodes, std::vector<double>& weights);
GllRule gll_rule(int degree);
SemBasis assemble_sem(double half_width, int cell_count, int degree);
std::vector<double> interp_matrix(const SemBasis& coarse, const SemBasis& fine);
void sym_eig(int n, const double* a, std::vector<double>& lam, std::vector<double>& q);
AxisFactor build_sem_axis(const SemBasis& basis, const double* fvals);

}  // namespace kronop_host
