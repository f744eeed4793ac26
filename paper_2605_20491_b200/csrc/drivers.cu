// Device-resident drivers on top of the transform passes: PCG, shifted inverse iteration, the GPE
// gradient flows and the split-step propagators (proj/src/pcg.cpp, ground_state.cpp, gpe.cpp,
// splitting.cpp).
//
// PCG runs as ONE CUDA graph: a conditional WHILE node whose body is the whole iteration
// (A p -> p.q -> alpha -> x, r update (+ r.r) -> M r -> r.z -> beta -> p update -> bookkeeping ->
// best-iterate copy). All scalars (alpha, beta, rz, residuals, best/stagnation counters) live in
// device memory and the loop condition is set on the device with cudaGraphSetConditional, so the
// host does not touch the loop between launch and the final report (north-star item 3).
// Split-step marches enqueue every propagation / phase of the schedule without host syncs.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "context.cuh"

namespace kronop_dev {

template <class F>
int guard2(F&& f) {
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

// ------------------------------------------------------------------------ linear maps --
static void apply_map(kronop_ctx& ctx, const kronop_linear_map& m, const double* in, double* out,
                      double* tmp, long long n) {
  if (m.mode == KRONOP_MAP_APPLY) {
    sep_transform(ctx, *m.op, in, out, 0, SEP_APPLY, m.op->shift, 0.0, m.diag, m.sigma);
  } else {
    if (m.scale) {  // t = r .* s; t = solve(t); t .* s  (harness.cpp:533-538)
      launch_mul_diag(ctx.stream, ctx.ws, tmp, in, m.scale, n, 0);
      sep_transform(ctx, *m.op, tmp, out, 0, SEP_SOLVE, m.op->shift, 0.0, nullptr, 0.0);
      launch_mul_diag(ctx.stream, ctx.ws, out, out, m.scale, n, 0);
    } else {
      sep_transform(ctx, *m.op, in, out, 0, SEP_SOLVE, m.op->shift, 0.0, nullptr, 0.0);
    }
  }
}

static void check_map(kronop_ctx& ctx, const kronop_linear_map* m, long long n) {
  param_check(m && m->op, "pcg: linear map needs an operator");
  param_check(m->mode == KRONOP_MAP_APPLY || m->mode == KRONOP_MAP_SOLVE, "pcg: bad map mode");
  param_check(m->op->N == n, "pcg: operator size mismatch");
  if (m->mode == KRONOP_MAP_SOLVE) check_solve_shift(ctx, *m->op, m->op->shift);
}

// ----------------------------------------------------------------------- PCG scalars --
__global__ void k_pcg_init(PcgScalars* sc, const double* rz, const double* rr, double norm_b,
                           double* history) {
  sc->rz = *rz;
  sc->pnorm0 = sqrt(fabs(sc->rz));
  sc->norm_b = norm_b;
  sc->rr = *rr;
  sc->rel = sc->preconditioned_norm ? sqrt(fabs(sc->rz)) / sc->pnorm0 : sqrt(sc->rr) / norm_b;
  if (sc->record_history) history[0] = sc->rel;
  sc->history_len = 1;
  sc->best_rel = sc->rel;
  sc->since = 0;
  sc->iterations = 0;
  sc->converged = sc->rel <= sc->rel_tol;
  sc->breakdown = 0;
  sc->improved = 0;
  sc->active = !sc->converged && sc->max_iter > 0 &&
               !(sc->stagnation_window > 0 && sc->since >= sc->stagnation_window);
}

__global__ void k_set_cond_from(cudaGraphConditionalHandle h, const PcgScalars* sc) {
  cudaGraphSetConditional(h, sc->active ? 1u : 0u);
}

__global__ void k_pcg_alpha(PcgScalars* sc) {  // pcg.cpp:51-55
  sc->improved = 0;
  if (!sc->active) return;
  if (sc->pq <= 0.0) {
    sc->breakdown = 1;
    sc->active = 0;
    return;
  }
  sc->alpha = sc->rz / sc->pq;
}

__global__ void k_pcg_beta(PcgScalars* sc) {  // pcg.cpp:60
  if (!sc->active) return;
  sc->beta = sc->rz_next / sc->rz;
}

// pcg.cpp:61-71 and the loop-top tests of the next iteration (pcg.cpp:45-50)
__device__ void pcg_finish_body(PcgScalars* sc, double* history) {
  if (!sc->active) return;
  sc->rz = sc->rz_next;
  sc->iterations += 1;
  sc->rel = sc->preconditioned_norm ? sqrt(fabs(sc->rz)) / sc->pnorm0 : sqrt(sc->rr) / sc->norm_b;
  if (sc->record_history) history[sc->history_len] = sc->rel;
  sc->history_len += 1;
  if (sc->rel < 0.99 * sc->best_rel) {
    sc->best_rel = sc->rel;
    sc->since = 0;
    sc->improved = 1;
  } else {
    sc->since += 1;
  }
  if (sc->rel <= sc->rel_tol) {
    sc->converged = 1;
    sc->active = 0;
  } else if (sc->iterations >= sc->max_iter ||
             (sc->stagnation_window > 0 && sc->since >= sc->stagnation_window)) {
    sc->active = 0;
  }
}

__global__ void k_pcg_finish(PcgScalars* sc, double* history, cudaGraphConditionalHandle h) {
  pcg_finish_body(sc, history);
  cudaGraphSetConditional(h, sc->active ? 1u : 0u);
}

__global__ void k_pcg_finish_plain(PcgScalars* sc, double* history) {
  pcg_finish_body(sc, history);
}

// Launchers of the PCG scalar / GPE kernels for the host-enqueued drivers of other translation
// units (the slab-decomposed drivers, slab.cu).
void launch_pcg_init(cudaStream_t s, Workspace& ws, PcgScalars* sc, const double* rz,
                     const double* rr, double norm_b, double* history) {
  k_pcg_init<<<1, 1, 0, s>>>(sc, rz, rr, norm_b, history);
  KCUDA(cudaGetLastError());
  ws.launches += 1;
}
void launch_pcg_alpha(cudaStream_t s, Workspace& ws, PcgScalars* sc) {
  k_pcg_alpha<<<1, 1, 0, s>>>(sc);
  KCUDA(cudaGetLastError());
  ws.launches += 1;
}
void launch_pcg_beta(cudaStream_t s, Workspace& ws, PcgScalars* sc) {
  k_pcg_beta<<<1, 1, 0, s>>>(sc);
  KCUDA(cudaGetLastError());
  ws.launches += 1;
}
void launch_pcg_finish(cudaStream_t s, Workspace& ws, PcgScalars* sc, double* history) {
  k_pcg_finish_plain<<<1, 1, 0, s>>>(sc, history);
  KCUDA(cudaGetLastError());
  ws.launches += 1;
}

struct PcgWork {
  DBuf r, z, p, q, best, tmp, hist;
  DBuf scal;  // PcgScalars + slots
  PcgWork(kronop_ctx& c, long long n, int max_iter)
      : r(c, n), z(c, n), p(c, n), q(c, n), best(c, n), tmp(c, n), hist(c, max_iter + 2),
        scal(c, 64) {}
  PcgScalars* sc() { return reinterpret_cast<PcgScalars*>(scal.p); }
  double* slot(int i) { return scal.p + 32 + i; }
};

// Runs the PCG loop; returns report. Throws NumericalError on breakdown.
static void pcg_run(kronop_ctx& ctx, const kronop_linear_map& A, const kronop_linear_map& M,
                    const double* b, double* x, long long n, const kronop_pcg_config& cfg,
                    kronop_pcg_report& rep, double* history_host, PcgWork& w) {
  param_check(cfg.rel_tol > 0.0, "pcg: rel_tol must be positive");
  param_check(cfg.max_iter >= 1, "pcg: max_iter must be >= 1");
  cudaStream_t s = ctx.stream;
  ensure_scratch(ctx, static_cast<size_t>(n));
  rep = kronop_pcg_report{};
  // ||b|| and ||x0|| (setup, pcg.cpp:15-26)
  launch_dot(s, ctx.ws, b, b, n, 0, nullptr, w.slot(0));
  launch_dot(s, ctx.ws, x, x, n, 0, nullptr, w.slot(1));
  double hb[2];
  KCUDA(cudaMemcpyAsync(hb, w.slot(0), 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  KCUDA(cudaStreamSynchronize(s));
  const double norm_b = std::sqrt(hb[0]);
  if (norm_b == 0.0) {
    KCUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    KCUDA(cudaStreamSynchronize(s));
    rep.converged = 1;
    return;
  }
  // r = b - A x (only for a nonzero warm start)
  if (std::sqrt(hb[1]) != 0.0) {
    apply_map(ctx, A, x, w.q.p, w.tmp.p, n);
    launch_sub(s, ctx.ws, w.r.p, b, w.q.p, n);
  } else {
    KCUDA(cudaMemcpyAsync(w.r.p, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  apply_map(ctx, M, w.r.p, w.z.p, w.tmp.p, n);
  KCUDA(cudaMemcpyAsync(w.p.p, w.z.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  launch_dot(s, ctx.ws, w.r.p, w.z.p, n, 0, nullptr, w.slot(2));
  launch_dot(s, ctx.ws, w.r.p, w.r.p, n, 0, nullptr, w.slot(3));
  KCUDA(cudaMemcpyAsync(w.best.p, x, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  PcgScalars init{};
  init.rel_tol = cfg.rel_tol;
  init.max_iter = cfg.max_iter;
  init.stagnation_window = cfg.stagnation_window;
  init.preconditioned_norm = cfg.preconditioned_norm;
  init.record_history = history_host != nullptr || cfg.record_history;
  KCUDA(cudaMemcpyAsync(w.sc(), &init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_pcg_init<<<1, 1, 0, s>>>(w.sc(), w.slot(2), w.slot(3), norm_b, w.hist.p);
  KCUDA(cudaGetLastError());
  ctx.ws.launches += 1;
  KCUDA(cudaStreamSynchronize(s));  // init copy above reads a host stack struct

  // ---- the loop: one graph, conditional WHILE, body = one PCG iteration ----
  cudaGraph_t graph;
  KCUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle handle;
  KCUDA(cudaGraphConditionalHandleCreate(&handle, graph, 0, 0));
  cudaGraphNode_t init_node;
  {
    cudaKernelNodeParams kp{};
    PcgScalars* scp = w.sc();
    void* args[] = {&handle, &scp};
    kp.func = reinterpret_cast<void*>(k_set_cond_from);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    KCUDA(cudaGraphAddKernelNode(&init_node, graph, nullptr, 0, &kp));
  }
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond_node;
  KCUDA(cudaGraphAddNode(&cond_node, graph, &init_node, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const unsigned long long launches_before = ctx.ws.launches;
  KCUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal));
  try {
    apply_map(ctx, A, w.p.p, w.q.p, w.tmp.p, n);                                     // q = A p
    launch_dot(s, ctx.ws, w.p.p, w.q.p, n, 0, nullptr, &w.sc()->pq);                  // p.q
    k_pcg_alpha<<<1, 1, 0, s>>>(w.sc());                                              // alpha
    launch_pcg_update_xr(s, ctx.ws, x, w.r.p, w.p.p, w.q.p, w.sc(), n, &w.sc()->rr);  // x, r, r.r
    apply_map(ctx, M, w.r.p, w.z.p, w.tmp.p, n);                                     // z = M r
    launch_dot(s, ctx.ws, w.r.p, w.z.p, n, 0, nullptr, &w.sc()->rz_next);             // r.z
    k_pcg_beta<<<1, 1, 0, s>>>(w.sc());
    launch_pcg_update_p(s, ctx.ws, w.p.p, w.z.p, w.sc(), n);                          // p
    k_pcg_finish<<<1, 1, 0, s>>>(w.sc(), w.hist.p, handle);
    launch_copy_if(s, ctx.ws, w.best.p, x, n, &w.sc()->improved);                     // best x
    KCUDA(cudaGetLastError());
  } catch (...) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(s, &dummy);
    cudaGraphDestroy(graph);
    throw;
  }
  KCUDA(cudaStreamEndCapture(s, &body));
  const unsigned long long body_launches = ctx.ws.launches - launches_before + 3;
  ctx.ws.launches = launches_before;
  cudaGraphExec_t exec;
  KCUDA(cudaGraphInstantiate(&exec, graph, 0));
  KCUDA(cudaGraphLaunch(exec, s));
  PcgScalars fin{};
  KCUDA(cudaMemcpyAsync(&fin, w.sc(), sizeof(fin), cudaMemcpyDeviceToHost, s));
  KCUDA(cudaStreamSynchronize(s));
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  ctx.ws.launches += 1 + body_launches * static_cast<unsigned long long>(fin.iterations +
                                                                          (fin.breakdown ? 1 : 0));
  if (fin.breakdown)
    fail(KRONOP_ENUMERICAL,
         "pcg: indefinite direction at iteration " + std::to_string(fin.iterations + 1));
  double rel = fin.rel;
  if (rel <= cfg.rel_tol) {  // pcg.cpp:73-79
    rep.converged = 1;
  } else if (fin.best_rel < rel) {
    KCUDA(cudaMemcpyAsync(x, w.best.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    rel = fin.best_rel;
  }
  rep.iterations = fin.iterations;
  rep.final_residual = rel;
  rep.history_len = fin.record_history ? fin.history_len : 0;
  if (history_host && rep.history_len > 0)
    KCUDA(cudaMemcpyAsync(history_host, w.hist.p, rep.history_len * sizeof(double),
                          cudaMemcpyDeviceToHost, s));
  KCUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- small helpers --
static double read_slot(kronop_ctx& ctx, const double* dev) {
  double v;
  KCUDA(cudaMemcpyAsync(&v, dev, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  KCUDA(cudaStreamSynchronize(ctx.stream));
  return v;
}

static double wdot(kronop_ctx& ctx, const kronop_op& op, const double* a, const double* b,
                   double* slot) {
  const IndexGeomHost g = mass_geom(op);
  launch_dot(ctx.stream, ctx.ws, a, b, op.N, 0, &g, slot);
  return read_slot(ctx, slot);
}

// first index of max |u| (Eigen maxCoeff) -> negate if that entry is negative
__global__ void k_argmax_abs_partial(const double* u, long long n, double* pv, long long* pi) {
  __shared__ double sv[256];
  __shared__ long long si[256];
  double best = -1.0;
  long long bi = 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double a = fabs(u[i]);
    if (a > best) {
      best = a;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double ov = sv[threadIdx.x + w];
      const long long oi = si[threadIdx.x + w];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = sv[0];
    pi[blockIdx.x] = si[0];
  }
}

static void fix_sign(kronop_ctx& ctx, double* u, long long n) {  // ground_state.cpp:23-27
  DBuf pv(ctx, kRedBlocks), pi(ctx, kRedBlocks);
  k_argmax_abs_partial<<<kRedBlocks, 256, 0, ctx.stream>>>(u, n, pv.p,
                                                           reinterpret_cast<long long*>(pi.p));
  KCUDA(cudaGetLastError());
  ctx.ws.launches += 1;
  std::vector<double> hv(kRedBlocks);
  std::vector<long long> hi(kRedBlocks);
  KCUDA(cudaMemcpyAsync(hv.data(), pv.p, kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost,
                        ctx.stream));
  KCUDA(cudaMemcpyAsync(hi.data(), pi.p, kRedBlocks * sizeof(long long), cudaMemcpyDeviceToHost,
                        ctx.stream));
  KCUDA(cudaStreamSynchronize(ctx.stream));
  double best = -1.0;
  long long bi = 0;
  for (int b = 0; b < kRedBlocks; ++b)
    if (hv[b] > best || (hv[b] == best && hi[b] < bi)) {
      best = hv[b];
      bi = hi[b];
    }
  const double val = read_slot(ctx, u + bi);
  if (val < 0.0) launch_scale(ctx.stream, ctx.ws, u, u, n, -1.0, nullptr, 0);
}

}  // namespace kronop_dev

using namespace kronop_dev;

extern "C" {

int kronop_pcg(kronop_ctx* ctx, const kronop_linear_map* apply_a, const kronop_linear_map* precond,
               const double* b, double* x, const kronop_pcg_config* config,
               kronop_pcg_report* report, double* history) {
  return guard2([&] {
    param_check(ctx && apply_a && precond && b && x && config && report, "pcg: null argument");
    const long long n = apply_a->op ? apply_a->op->N : 0;
    check_map(*ctx, apply_a, n);
    check_map(*ctx, precond, n);
    PcgWork w(*ctx, n, config->max_iter);
    pcg_run(*ctx, *apply_a, *precond, b, x, n, *config, *report, history, w);
  });
}

// ---------------------------------------------------------------- inverse iteration --
int kronop_inverse_iteration(kronop_ctx* ctx, const kronop_op* op, const double* diag,
                             const kronop_inverse_iteration_config* cfg, const double* initial,
                             double* eigenvector, kronop_eigenpair_result* result,
                             int* inner_per_outer) {
  return guard2([&] {
    param_check(ctx && op && cfg && initial && eigenvector && result,
                "inverse_iteration: null argument");
    param_check(cfg->eig_rel_tol > 0.0, "inverse_iteration: tolerance must be positive");
    param_check(op->has_mass, "inverse_iteration: initial guess needs mass weights");
    kronop_ctx& c = *ctx;
    const long long n = op->N;
    const bool separable = diag == nullptr;
    // shift_value (ground_state.cpp:11-21)
    double sigma = 0.0;
    if (cfg->shift_mode == KRONOP_SHIFT_FRACTION) sigma = cfg->shift_fraction * op->lmin;
    else if (cfg->shift_mode == KRONOP_SHIFT_OFFSET) sigma = op->lmin - cfg->shift_offset;
    ensure_scratch(c, static_cast<size_t>(n));
    DBuf u(c, n), hu(c, n), w(c, n), slots(c, 8);
    auto rayleigh = [&](const double* v) {  // ground_state.cpp:46-49
      sep_transform(c, *op, v, hu.p, 0, SEP_APPLY, op->shift, 0.0, diag, 0.0);
      const double num = wdot(c, *op, v, hu.p, slots.p);
      const double den = wdot(c, *op, v, v, slots.p + 1);
      return num / den;
    };
    *result = kronop_eigenpair_result{};
    const double nrm0 = wdot(c, *op, initial, initial, slots.p);
    (void)nrm0;
    // u = initial / sqrt(<initial, initial>_M)  (ground_state.cpp:63)
    launch_div_by(c.stream, c.ws, u.p, initial, n, slots.p, 1);
    double lambda = rayleigh(u.p);
    if (sigma >= lambda)
      fail(KRONOP_EPARAM, "inverse_iteration: shift is not below the Rayleigh estimate");
    KCUDA(cudaMemsetAsync(w.p, 0, n * sizeof(double), c.stream));
    if (separable) check_solve_shift(c, *op, sigma);
    kronop_linear_map A{op, KRONOP_MAP_APPLY, diag, sigma, nullptr};
    kronop_linear_map M{op, KRONOP_MAP_SOLVE, nullptr, 0.0, nullptr};
    if (!separable) check_solve_shift(c, *op, op->shift);
    std::unique_ptr<PcgWork> pw;
    if (!separable) pw.reset(new PcgWork(c, n, cfg->inner.max_iter));
    for (int outer = 0; outer < cfg->max_outer; ++outer) {
      if (separable) {
        sep_transform(c, *op, u.p, w.p, 0, SEP_SOLVE, sigma, 0.0, nullptr, 0.0);
      } else {
        kronop_pcg_report rep;
        pcg_run(c, A, M, u.p, w.p, n, cfg->inner, rep, nullptr, *pw);
        if (inner_per_outer) inner_per_outer[outer] = rep.iterations;
        result->total_inner_iterations += rep.iterations;
      }
      const double nn = wdot(c, *op, w.p, w.p, slots.p);
      (void)nn;
      launch_div_by(c.stream, c.ws, u.p, w.p, n, slots.p, 1);  // next = w / sqrt(<w,w>_M)
      const double lambda_next = rayleigh(u.p);
      result->outer_iterations += 1;
      const bool done = std::abs(lambda_next - lambda) < cfg->eig_rel_tol * std::abs(lambda_next);
      lambda = lambda_next;
      if (done) {
        result->converged = 1;
        break;
      }
    }
    fix_sign(c, u.p, n);
    result->eigenvalue = lambda;
    KCUDA(cudaMemcpyAsync(eigenvector, u.p, n * sizeof(double), cudaMemcpyDeviceToDevice,
                          c.stream));
    KCUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"

// ----------------------------------------------------------------------------- GPE --
namespace kronop_dev {

// r = hu + beta u^3 ; energy terms
__global__ void k_add_beta_cube(double* r, const double* u, double beta, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double x = u[i];
    r[i] = __dadd_rn(r[i], __dmul_rn(beta, __dmul_rn(__dmul_rn(x, x), x)));  // gpe.cpp:111
  }
}
__global__ void k_beta_square(double* dg, const double* u, double beta, const double* v2,
                              long long n) {  // gpe.cpp:120-122
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    double v = __dmul_rn(beta, __dmul_rn(u[i], u[i]));
    if (v2) v = __dadd_rn(v, v2[i]);
    dg[i] = v;
  }
}
// g = a - c * b   (grad = rt - proj ut ; grad = u - proj w)
__global__ void k_sub_scaled(double* g, const double* a, const double* b, double c, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    g[i] = __dsub_rn(a[i], __dmul_rn(c, b[i]));
}
// sq[i] = u^2 * u^2 (for the quartic term, gpe.cpp:16)
__global__ void k_square2(double* sq, const double* u, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double s = __dmul_rn(u[i], u[i]);
    sq[i] = s;
  }
}

static double gpe_energy_dev(kronop_ctx& c, const kronop_op& h, const double* diag, double beta,
                             const double* u, double* hu, double* sq, double* slots) {
  sep_transform(c, h, u, hu, 0, SEP_APPLY, h.shift, 0.0, diag, 0.0);
  const double quad = wdot(c, h, u, hu, slots);
  k_square2<<<kEltBlocks, 256, 0, c.stream>>>(sq, u, h.N);
  KCUDA(cudaGetLastError());
  c.ws.launches += 1;
  const double quartic = wdot(c, h, sq, sq, slots + 1);
  return 0.5 * quad + 0.25 * beta * quartic;
}

void launch_beta_square(cudaStream_t s, Workspace& ws, double* dg, const double* u, double beta,
                        const double* v2, long long n) {
  k_beta_square<<<kEltBlocks, 256, 0, s>>>(dg, u, beta, v2, n);
  KCUDA(cudaGetLastError());
  ws.launches += 1;
}
void launch_sub_scaled(cudaStream_t s, Workspace& ws, double* g, const double* a, const double* b,
                       double c, long long n) {
  k_sub_scaled<<<kEltBlocks, 256, 0, s>>>(g, a, b, c, n);
  KCUDA(cudaGetLastError());
  ws.launches += 1;
}
void launch_square2(cudaStream_t s, Workspace& ws, double* sq, const double* u, long long n) {
  k_square2<<<kEltBlocks, 256, 0, s>>>(sq, u, n);
  KCUDA(cudaGetLastError());
  ws.launches += 1;
}

}  // namespace kronop_dev

extern "C" {

int kronop_gpe_energy(kronop_ctx* ctx, const kronop_op* hamiltonian, const double* diag,
                      double beta, const double* u, double* energy) {
  return guard2([&] {
    param_check(ctx && hamiltonian && u && energy, "gpe_energy: null argument");
    param_check(hamiltonian->has_mass, "gpe_energy: field needs mass weights");
    DBuf hu(*ctx, hamiltonian->N), sq(*ctx, hamiltonian->N), slots(*ctx, 4);
    *energy = gpe_energy_dev(*ctx, *hamiltonian, diag, beta, u, hu.p, sq.p, slots.p);
  });
}

int kronop_gpe_gradient_flow(kronop_ctx* ctx, const kronop_op* ham, const double* diag,
                             const kronop_op* lap, double beta, const kronop_gpe_config* cfg,
                             const double* initial, double* state, kronop_gpe_result* result,
                             double* history) {
  return guard2([&] {
    param_check(ctx && ham && lap && cfg && state && result, "gpe_gradient_flow: null argument");
    param_check(beta >= 0.0, "gpe_gradient_flow: beta must be >= 0");
    param_check(cfg->step > 0.0, "gpe_gradient_flow: step must be positive");
    param_check(cfg->metric_shift > 0.0, "gpe_gradient_flow: metric shift must be positive");
    param_check(ham->has_mass, "gpe_gradient_flow: problem needs mass weights");
    param_check(!(cfg->init == KRONOP_GPE_INIT_SUPPLIED && !initial),
                "gpe_gradient_flow: init = Supplied but no initial state given");
    param_check(ham->N == lap->N, "gpe_gradient_flow: operator size mismatch");
    kronop_ctx& c = *ctx;
    const long long n = ham->N;
    const auto t0 = std::chrono::steady_clock::now();
    ensure_scratch(c, static_cast<size_t>(n));
    DBuf u(c, n), w(c, n), grad(c, n), r(c, n), rt(c, n), ut(c, n), dg(c, n), sq(c, n),
        slots(c, 8);
    // initial state (gpe.cpp:76-92)
    if (cfg->init == KRONOP_GPE_INIT_SUPPLIED) {
      KCUDA(cudaMemcpyAsync(u.p, initial, n * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    } else if (cfg->init == KRONOP_GPE_INIT_CONSTANT) {
      launch_fill(c.stream, c.ws, u.p, 1.0, n);
    } else {
      KCUDA(cudaMemsetAsync(u.p, 0, n * sizeof(double), c.stream));
      IndexGeomHost g;
      g.d = ham->d;
      for (int a = 0; a < ham->d; ++a) g.n[a] = ham->n[a];
      launch_generate(c.stream, c.ws, u.p, g, ham->bwd, 2);
      if (diag) {
        kronop_inverse_iteration_config ic{};
        ic.shift_mode = KRONOP_SHIFT_FRACTION;
        ic.shift_fraction = 0.9;
        ic.shift_offset = 1e-4;
        ic.eig_rel_tol = 1e-12;
        ic.max_outer = 60;
        ic.inner = {1e-12, 500, 0, 0, 100};
        kronop_eigenpair_result er;
        const int rc = kronop_inverse_iteration(ctx, ham, diag, &ic, u.p, u.p, &er, nullptr);
        if (rc != KRONOP_OK) fail(rc, kronop_last_error());
      }
    }
    wdot(c, *ham, u.p, u.p, slots.p);
    launch_div_by(c.stream, c.ws, u.p, u.p, n, slots.p, 1);
    *result = kronop_gpe_result{};
    double e_old = gpe_energy_dev(c, *ham, diag, beta, u.p, r.p, sq.p, slots.p + 2);
    int increases = 0;
    KCUDA(cudaMemsetAsync(w.p, 0, n * sizeof(double), c.stream));
    const double alpha = -cfg->metric_shift;  // h1 metric = laplacian with shift -alpha
    if (cfg->kind == KRONOP_GPE_H1) check_solve_shift(c, *lap, alpha);
    else check_solve_shift(c, *ham, ham->shift);
    std::unique_ptr<PcgWork> pw;
    if (cfg->kind == KRONOP_GPE_AU) pw.reset(new PcgWork(c, n, cfg->inner.max_iter));
    for (int it = 0; it < cfg->max_iterations; ++it) {
      if (cfg->kind == KRONOP_GPE_H1) {  // gpe.cpp:108-117
        sep_transform(c, *ham, u.p, r.p, 0, SEP_APPLY, ham->shift, 0.0, diag, 0.0);
        k_add_beta_cube<<<kEltBlocks, 256, 0, c.stream>>>(r.p, u.p, beta, n);
        KCUDA(cudaGetLastError());
        c.ws.launches += 1;
        sep_transform(c, *lap, r.p, rt.p, 0, SEP_SOLVE, alpha, 0.0, nullptr, 0.0);
        sep_transform(c, *lap, u.p, ut.p, 0, SEP_SOLVE, alpha, 0.0, nullptr, 0.0);
        result->linear_solves += 2;
        const double proj = wdot(c, *ham, rt.p, u.p, slots.p) / wdot(c, *ham, ut.p, u.p, slots.p + 1);
        k_sub_scaled<<<kEltBlocks, 256, 0, c.stream>>>(grad.p, rt.p, ut.p, proj, n);
      } else {  // gpe.cpp:118-134
        k_beta_square<<<kEltBlocks, 256, 0, c.stream>>>(dg.p, u.p, beta, diag, n);
        KCUDA(cudaGetLastError());
        c.ws.launches += 1;
        kronop_linear_map A{ham, KRONOP_MAP_APPLY, dg.p, 0.0, nullptr};
        kronop_linear_map M{ham, KRONOP_MAP_SOLVE, nullptr, 0.0, nullptr};
        kronop_pcg_report rep;
        pcg_run(c, A, M, u.p, w.p, n, cfg->inner, rep, nullptr, *pw);
        result->linear_solves += rep.iterations;
        const double proj = wdot(c, *ham, u.p, u.p, slots.p) / wdot(c, *ham, w.p, u.p, slots.p + 1);
        k_sub_scaled<<<kEltBlocks, 256, 0, c.stream>>>(grad.p, u.p, w.p, proj, n);
      }
      KCUDA(cudaGetLastError());
      c.ws.launches += 1;
      // u -= tau grad ; u /= sqrt(<u,u>_M)   (gpe.cpp:136-137)
      k_sub_scaled<<<kEltBlocks, 256, 0, c.stream>>>(u.p, u.p, grad.p, cfg->step, n);
      KCUDA(cudaGetLastError());
      c.ws.launches += 1;
      wdot(c, *ham, u.p, u.p, slots.p);
      launch_div_by(c.stream, c.ws, u.p, u.p, n, slots.p, 1);
      const double energy = gpe_energy_dev(c, *ham, diag, beta, u.p, r.p, sq.p, slots.p + 2);
      const double rel = std::abs(energy - e_old) / std::abs(energy);
      result->iterations = it + 1;
      if (cfg->record_history && history) {
        const double secs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        double* row = history + 5 * static_cast<size_t>(result->history_len);
        row[0] = it + 1;
        row[1] = energy;
        row[2] = rel;
        row[3] = static_cast<double>(result->linear_solves);
        row[4] = secs;
        result->history_len += 1;
      }
      if (energy - e_old > 1e-13 * std::abs(energy)) {  // gpe.cpp:144-151
        if (++increases > 10)
          fail(KRONOP_ENUMERICAL,
               "gpe_gradient_flow: energy increased for more than 10 consecutive steps; reduce "
               "the step size");
      } else {
        increases = 0;
      }
      e_old = energy;
      if (rel < cfg->energy_rel_tol) {
        result->converged = 1;
        break;
      }
    }
    // eigenvalue = <u,Hu>_M + beta sum m u^4 (gpe.cpp:159-161)
    sep_transform(c, *ham, u.p, r.p, 0, SEP_APPLY, ham->shift, 0.0, diag, 0.0);
    const double quad = wdot(c, *ham, u.p, r.p, slots.p);
    k_square2<<<kEltBlocks, 256, 0, c.stream>>>(sq.p, u.p, n);
    KCUDA(cudaGetLastError());
    c.ws.launches += 1;
    const double quartic = wdot(c, *ham, sq.p, sq.p, slots.p + 1);
    result->eigenvalue = quad + beta * quartic;
    result->energy = e_old;
    KCUDA(cudaMemcpyAsync(state, u.p, n * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    KCUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"

// ------------------------------------------------------------------------ splitting --
namespace kronop_dev {

struct Schedule {  // StepSchedule (splitting.cpp:17-18)
  std::vector<double> a_times, b_factors;
};

static Schedule single_schedule(double h, int m) {  // splitting.cpp:20-34
  std::vector<double> nodes, weights;
  kronop_host::gauss_legendre(m, nodes, weights);
  Schedule s;
  s.a_times.resize(m + 1);
  s.b_factors.resize(m);
  double prev = 0.0;
  for (int k = 0; k < m; ++k) {
    const double sk = h * (1.0 + nodes[k]) / 2.0;
    s.a_times[k] = sk - prev;
    s.b_factors[k] = 0.5 * weights[k] * h;
    prev = sk;
  }
  s.a_times[m] = h - prev;
  return s;
}

static void yoshida(double& g1, double& g2) {  // splitting.cpp:86-90
  const double cbrt2 = std::cbrt(2.0);
  const double denom = 2.0 - cbrt2;
  g1 = 1.0 / denom;
  g2 = -cbrt2 / denom;
}

static std::vector<Schedule> step_schedules(int composition, int m, double h) {  // :36-42
  if (composition == KRONOP_COMPOSITION_SINGLE) return {single_schedule(h, m)};
  double g1, g2;
  yoshida(g1, g2);
  return {single_schedule(g1 * h, m), single_schedule(g2 * h, m), single_schedule(g1 * h, m)};
}

// run_schedules (splitting.cpp:53-82): psi is updated in place (device, complex interleaved).
static void run_schedules(kronop_ctx& c, const kronop_op& a, const double* b_diag,
                          const std::vector<Schedule>& schedules, double* psi, int steps,
                          bool merge) {
  // The A-propagation due before a B phase is deferred to it and fused: the phase runs in the
  // epilogue of the propagate's last pass (EPI_BPHASE), saving a field round trip per B step.
  // The operations and their order are those of splitting.cpp:53-82 (merge: A-times accumulate
  // and flush before each B or at the end; no merge: each A-time is flushed on its own).
  // B phase fused into the propagate's last pass (EPI_BPHASE) only on request
  // (KRONOP_BPHASE_FUSED=1): it is bit-identical, but measured slower on every config-5 grid
  // (Strang steps/s, tools/microbench/bphase_bench.py: 9D n = 9 25.4 vs 29.5, 6D n = 29 15.5 vs
  // 16.0, 3D 499^3 15.8 vs 16.8) -- the per-element sincos makes the latency-bound store phase
  // of the contraction longer than the HBM-bound standalone phase pass it saves.
  static const bool unfused = [] {
    const char* e = getenv("KRONOP_BPHASE_FUSED");
    return !(e && e[0] == '1');
  }();
  // Default on the Kronecker path (small extents, config 5): a B phase is deferred to the A
  // propagation that follows it and applied by that propagate's first group as it reads psi,
  // from a (cos, sin) table per distinct B factor (k_phase's operations, so bit-identical): one
  // field round trip and no per-element sincos per step. KRONOP_BPHASE_PRE=0 turns it off.
  static const bool pre_off = [] {
    const char* e = getenv("KRONOP_BPHASE_PRE");
    return e && e[0] == '0';
  }();
  std::vector<double> factors;
  for (const Schedule& sc : schedules)
    for (double f : sc.b_factors)
      if (std::find(factors.begin(), factors.end(), f) == factors.end()) factors.push_back(f);
  // worth it when the B phases outnumber the tables to make (one pass each): every run with more
  // than one step, and single qHOP / Yoshida steps with repeated factors
  long long nb = 0;
  for (const Schedule& sc : schedules) nb += static_cast<long long>(sc.b_factors.size());
  nb *= steps;
  bool use_pre = !pre_off && unfused && nb > static_cast<long long>(factors.size()) &&
                 kron_path_likely(a);
  if (use_pre) {  // the tables (2N doubles each) must leave room for the rest of the run
    size_t free_b = 0, total_b = 0;
    KCUDA(cudaMemGetInfo(&free_b, &total_b));
    use_pre = factors.size() * 2.0 * a.N * sizeof(double) <= 0.5 * static_cast<double>(free_b);
  }
  std::vector<std::unique_ptr<DBuf>> tables(factors.size());
  auto table_of = [&](double f) -> const double* {
    const size_t i = std::find(factors.begin(), factors.end(), f) - factors.begin();
    if (!tables[i]) {
      tables[i] = std::make_unique<DBuf>(c, static_cast<size_t>(2 * a.N));
      launch_phase_table(c.stream, c.ws, tables[i]->p, b_diag, f, a.N);
    }
    return tables[i]->p;
  };
  bool pending_b = false;
  double pending_bf = 0.0;
  auto apply_pending_b = [&]() {
    if (pending_b) launch_phase(c.stream, c.ws, psi, b_diag, pending_bf, a.N);
    pending_b = false;
  };
  double pending = 0.0;
  bool has_pending = false;
  auto flush = [&](bool with_b, double factor) {
    const double t = pending;
    const bool prop = has_pending && t != 0.0;  // propagate(psi, 0) is a copy (operators.cpp:64)
    pending = 0.0;
    has_pending = false;
    if (prop && pending_b &&
        sep_propagate_prephased(c, a, psi, a.shift, t, table_of(pending_bf))) {
      pending_b = false;  // B, then this A: done by the propagate
    } else {
      apply_pending_b();
      if (prop && with_b && !unfused) {
        sep_transform(c, a, psi, psi, 1, SEP_PROPAGATE, a.shift, t, nullptr, 0.0, true, b_diag,
                      factor);
        return;
      }
      if (prop) sep_transform(c, a, psi, psi, 1, SEP_PROPAGATE, a.shift, t, nullptr, 0.0);
    }
    if (with_b) {
      if (use_pre) {
        pending_b = true;
        pending_bf = factor;
      } else {
        launch_phase(c.stream, c.ws, psi, b_diag, factor, a.N);
      }
    }
  };
  auto propagate_a = [&](double t) {
    if (!merge && has_pending) flush(false, 0.0);
    pending += t;
    has_pending = true;
  };
  auto multiply_b = [&](double factor) { flush(true, factor); };
  for (int step = 0; step < steps; ++step)
    for (const Schedule& s : schedules) {
      const int m = static_cast<int>(s.b_factors.size());
      for (int k = 0; k < m; ++k) {
        propagate_a(s.a_times[k]);
        multiply_b(s.b_factors[k]);
      }
      propagate_a(s.a_times[m]);
    }
  flush(false, 0.0);
  apply_pending_b();
}

}  // namespace kronop_dev

extern "C" {

int kronop_yoshida_coeffs(double* gamma1, double* gamma2) {
  return guard2([&] { yoshida(*gamma1, *gamma2); });
}

int kronop_qhop_step(kronop_ctx* ctx, const kronop_op* a, const double* b_diag, const double* psi,
                     double h, int quad_points, double* out) {
  return guard2([&] {
    param_check(ctx && a && b_diag && psi && out, "qhop_step: null argument");
    ensure_scratch(*ctx, static_cast<size_t>(2 * a->N));
    if (out != psi)
      KCUDA(cudaMemcpyAsync(out, psi, 2 * a->N * sizeof(double), cudaMemcpyDeviceToDevice,
                            ctx->stream));
    run_schedules(*ctx, *a, b_diag, {single_schedule(h, quad_points)}, out, 1, false);
  });
}

int kronop_yoshida_step(kronop_ctx* ctx, const kronop_op* a, const double* b_diag,
                        const double* psi, double h, int quad_points, double* out) {
  return guard2([&] {
    param_check(ctx && a && b_diag && psi && out, "yoshida_step: null argument");
    ensure_scratch(*ctx, static_cast<size_t>(2 * a->N));
    if (out != psi)
      KCUDA(cudaMemcpyAsync(out, psi, 2 * a->N * sizeof(double), cudaMemcpyDeviceToDevice,
                            ctx->stream));
    run_schedules(*ctx, *a, b_diag, step_schedules(KRONOP_COMPOSITION_YOSHIDA, quad_points, h),
                  out, 1, false);
  });
}

int kronop_evolve(kronop_ctx* ctx, const kronop_split_spec* spec, const kronop_op* a,
                  const double* b_diag, const double* psi0, const kronop_op* exact,
                  double stationary_eigenvalue, double* state, double* error, int* steps_out) {
  return guard2([&] {
    param_check(ctx && spec && a && b_diag && psi0 && state && error, "evolve: null argument");
    param_check(spec->dt > 0.0 && spec->total_time > 0.0,
                "evolve: dt and total_time must be positive");
    const double ratio = spec->total_time / spec->dt;
    const long long steps = std::llround(ratio);
    param_check(steps >= 1 && std::abs(ratio - static_cast<double>(steps)) <= 1e-9,
                "evolve: total_time must be an integer multiple of dt");
    param_check(spec->composition == KRONOP_COMPOSITION_SINGLE ||
                    spec->composition == KRONOP_COMPOSITION_YOSHIDA,
                "evolve: bad composition");
    if (exact) param_check(exact->N == a->N, "evolve: exact reference size mismatch");
    kronop_ctx& c = *ctx;
    const long long n = a->N;
    ensure_scratch(c, static_cast<size_t>(2 * n));
    DBuf start(c, 2 * n), ref(c, 2 * n), slots(c, 4);
    // psi = psi0 / ||psi0||_2 (splitting.cpp:118-119)
    launch_dot(c.stream, c.ws, psi0, psi0, n, 1, nullptr, slots.p);
    launch_div_by(c.stream, c.ws, state, psi0, 2 * n, slots.p, 1);
    KCUDA(cudaMemcpyAsync(start.p, state, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice,
                          c.stream));
    run_schedules(c, *a, b_diag, step_schedules(spec->composition, spec->quad_points, spec->dt),
                  state, static_cast<int>(steps), spec->merge_across_steps != 0);
    if (exact) {  // splitting.cpp:125-134
      sep_transform(c, *exact, start.p, ref.p, 1, SEP_PROPAGATE, exact->shift, spec->total_time,
                    nullptr, 0.0);
    } else {
      const double phase = -stationary_eigenvalue * spec->total_time;
      KCUDA(cudaMemcpyAsync(ref.p, start.p, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice,
                            c.stream));
      // ref *= complex(cos, sin): the B-phase kernel with b = 1 (nullptr), factor = -phase
      launch_phase(c.stream, c.ws, ref.p, nullptr, -phase, n);
    }
    DBuf diff(c, 2 * n);
    launch_sub(c.stream, c.ws, diff.p, state, ref.p, 2 * n);
    if (spec->mass_weighted_error) {
      const IndexGeomHost g = mass_geom(*a);
      launch_dot(c.stream, c.ws, diff.p, diff.p, n, 1, &g, slots.p);
    } else {
      launch_dot(c.stream, c.ws, diff.p, diff.p, n, 1, nullptr, slots.p);
    }
    *error = std::sqrt(read_slot(c, slots.p));
    if (steps_out) *steps_out = static_cast<int>(steps);
  });
}

}  // extern "C"
