// Launchers for the HBM-bound vector kernels (vector_ops.cu).
#pragma once

#include "kronop_internal.cuh"

namespace kronop_dev {

struct IndexGeomHost {
  int d = 0;
  long long n[kMaxDims] = {};
  const double* mass[KRONOP_MAX_DIM] = {};  // device per-axis mass vectors (weighted dots)
};

// Device-resident PCG state (proj/src/pcg.cpp:8-81 locals). Lives in device memory for the whole
// solve; the host reads it once after the loop.
struct PcgScalars {
  double rz, rz_next, pq, alpha, beta, rr, rel, best_rel, pnorm0, norm_b;
  double rel_tol;
  int max_iter, stagnation_window, preconditioned_norm, record_history;
  int active;      // 1 while the loop runs (body kernels are no-ops otherwise)
  int iterations;  // completed iterations
  int since;       // iterations since the best residual improved by 1%
  int converged;
  int breakdown;   // p.q <= 0 seen (NumericalError)
  int improved;    // this iteration set a new best iterate -> copy x to best_x
  int history_len;
  int pad_;
};

void launch_dot(cudaStream_t s, Workspace& ws, const double* a, const double* b, long long n,
                int cplx, const IndexGeomHost* wgeom, double* out_dev);
void launch_pcg_update_xr(cudaStream_t s, Workspace& ws, double* x, double* r, const double* p,
                          const double* q, const PcgScalars* sc, long long n, double* out_rr);
void launch_pcg_update_p(cudaStream_t s, Workspace& ws, double* p, const double* z,
                         const PcgScalars* sc, long long n);
void launch_copy_if(cudaStream_t s, Workspace& ws, double* dst, const double* src, long long n,
                    const int* flag);
void launch_scale(cudaStream_t s, Workspace& ws, double* y, const double* x, long long n, double a,
                  const double* ap, int ap_mode);
void launch_fill(cudaStream_t s, Workspace& ws, double* y, double v, long long n);
void launch_div_by(cudaStream_t s, Workspace& ws, double* y, const double* x, long long n,
                   const double* nrm_dev, int take_sqrt);
void launch_mul_diag(cudaStream_t s, Workspace& ws, double* y, const double* x, const double* d,
                     long long n, int cplx);
void launch_phase_table(cudaStream_t s, Workspace& ws, double* tab, const double* b,
                        double factor, long long n);
void launch_phase(cudaStream_t s, Workspace& ws, double* psi, const double* b, double factor,
                  long long n);
void launch_generate(cudaStream_t s, Workspace& ws, double* out, const IndexGeomHost& g,
                     const double* const* vecs, int mode);
void launch_div_selftest(cudaStream_t s, Workspace& ws, const double* a, const double* b,
                         unsigned long long* bad, long long n);
void launch_splitmix(cudaStream_t s, Workspace& ws, double* out, unsigned long long seed,
                     unsigned long long start, long long n);
void launch_axpby(cudaStream_t s, Workspace& ws, double* y, const double* x, double a, double b,
                  long long n);
void launch_sub(cudaStream_t s, Workspace& ws, double* y, const double* x, const double* b,
                long long n);
// Even/odd fold / unfold along one real-view axis of extent n (pre below, post above):
// fold: [u_i = x_i + x_{n-1-i}, u_mid = x_mid | v_i = x_i - x_{n-1-i}];
// unfold: x_i = e_i + o_i, x_{n-1-i} = e_i - o_i, x_mid = e_mid, then optionally
// y = (y + diag .* u) - sigma u (FullOperator / shifted map epilogue).
void launch_fold(cudaStream_t s, Workspace& ws, const double* x, double* y, long long pre, int n,
                 long long post);
void launch_unfold(cudaStream_t s, Workspace& ws, const double* z, double* y, long long pre, int n,
                   long long post, const double* diag, const double* u, double sigma, int cplx);

}  // namespace kronop_dev
