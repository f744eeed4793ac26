// Context / operator objects behind the opaque C handles, and the transform-chain helpers shared
// by the C-ABI entry points (capi.cu) and the device-resident drivers (drivers.cu).
#pragma once

#include <algorithm>
#include <string>
#include <vector>

#include "kronop_internal.cuh"
#include "vector_ops.cuh"

struct kronop_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  kronop_dev::Workspace ws;
  double* scratch[2] = {nullptr, nullptr};  // ping-pong transform buffers
  size_t scratch_cap = 0;                   // doubles each
  double* dscal = nullptr;                  // device scalar slots
  double* hscal = nullptr;                  // pinned host mirror
  double* tmp = nullptr;                    // temp device buffer (host matrices, mass vectors)
  size_t tmp_cap = 0;
  double* io[2] = {nullptr, nullptr};       // device staging for the *_host entry points
  size_t io_cap = 0;
  // copy engines for the pipelined host path (H2D / D2H overlap the slab-local passes)
  cudaStream_t copy_stream[2] = {nullptr, nullptr};
  static constexpr int kMaxChunks = 32;
  cudaEvent_t ev_in[kMaxChunks] = {};
  cudaEvent_t ev_out[kMaxChunks] = {};
  cudaEvent_t ev_ready = nullptr;
  // batched host path (kronop_sep_*_host_batch): ping-pong device in / out fields and the
  // upload / compute / download events of the two items in flight
  double* bio[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t bio_cap = 0;
  cudaEvent_t ev_up[2] = {}, ev_comp[2] = {}, ev_down[2] = {};
  // device block pool for driver vectors (stream-ordered reuse on `stream`; freed at destroy)
  struct Block {
    double* p;
    size_t cap;
    bool used;
  };
  std::vector<Block> pool;
};


constexpr int kScalarSlots = 256;

struct kronop_op {
  kronop_ctx* ctx = nullptr;
  int d = 0;
  int n[KRONOP_MAX_DIM] = {};
  long long N = 0;
  double* fwd[KRONOP_MAX_DIM] = {};  // T^{-1}, padded, lda[a]
  double* bwd[KRONOP_MAX_DIM] = {};  // T, padded
  int lda[KRONOP_MAX_DIM] = {};
  double* lam[KRONOP_MAX_DIM] = {};
  double* mass[KRONOP_MAX_DIM] = {};
  bool has_mass = false;
  std::vector<double> hlam[KRONOP_MAX_DIM];
  std::vector<double> hmass[KRONOP_MAX_DIM];
  // host copies of T and T^{-1} (column-major n x n) for axes with n <= 32: the Kronecker-factored
  // small-extent propagate forms E_a = T_a diag(e^{-i lambda_a dt}) T_a^{-1} from them per dt
  std::vector<double> hT[KRONOP_MAX_DIM], hTinv[KRONOP_MAX_DIM];
  double shift = 0.0, lmin = 0.0, lmax = 0.0;
  // even/odd folded operator (kronop_op_create_folded): per axis the half-size blocks; lam[a] is
  // in folded order [even modes | odd modes]; bwd[a] holds the ground-state column only.
  bool shared_axis[KRONOP_MAX_DIM] = {};  // fwd/bwd alias an earlier identical axis
  // reduced-precision copies of the transforms (tc_lowp.cu), made on first use
  void* lp_fwd[KRONOP_MAX_DIM] = {};  // BF16
  void* lp_bwd[KRONOP_MAX_DIM] = {};
  void* tf_fwd[KRONOP_MAX_DIM] = {};  // FP32 storage for TF32
  void* tf_bwd[KRONOP_MAX_DIM] = {};
  void* f3_fwd[KRONOP_MAX_DIM] = {};  // (hi, lo) TF32 pairs for the 3xTF32 FP32 mode
  void* f3_bwd[KRONOP_MAX_DIM] = {};
  void* oz_fwd[KRONOP_MAX_DIM] = {};  // tiled INT8 slices + row exponents (ozaki.cu)
  void* oz_bwd[KRONOP_MAX_DIM] = {};
  void* oz_fo[KRONOP_MAX_DIM] = {};  // folded operators: odd blocks (oz_fwd / oz_bwd: even)
  void* oz_bo[KRONOP_MAX_DIM] = {};
  int oz_slices = 0;
  int exec_prec = 0;  // kronop_op_set_precision: 0 = FP64 DMMA, KRONOP_PREC_FP64_OZAKI* = INT8
  bool folded = false;
  int ne[KRONOP_MAX_DIM] = {}, no[KRONOP_MAX_DIM] = {};
  double* fe[KRONOP_MAX_DIM] = {};
  double* fo[KRONOP_MAX_DIM] = {};
  double* be[KRONOP_MAX_DIM] = {};
  double* bo[KRONOP_MAX_DIM] = {};
  int lda_e[KRONOP_MAX_DIM] = {}, lda_o[KRONOP_MAX_DIM] = {};
};

namespace kronop_dev {
void sep_solve_lowp(kronop_ctx& ctx, kronop_op& op, const double* b, double* x, int precision);
void sep_solve_ozaki(kronop_ctx& ctx, kronop_op& op, const double* b, double* x, int slices);
void sep_propagate_ozaki(kronop_ctx& ctx, kronop_op& op, const double* psi, double dt, double* out,
                         int slices);
void sep_ozaki(kronop_ctx& ctx, kronop_op& op, const double* in, double* out, int cplx, int epi,
               double shift, double dt, const double* diag, double sigma, int slices);
void ozaki_prepare(kronop_ctx& ctx, kronop_op& op, int slices);
// Smallest free pool block with capacity >= n doubles, else a new cudaMalloc'd block.
double* pool_get(kronop_ctx& ctx, size_t n);
void pool_put(kronop_ctx& ctx, double* p);
void pool_trim(kronop_ctx& ctx);  // cudaFree every idle block

// RAII device buffer from the context's block pool (pool_get / pool_put, capi.cu): drivers that
// are called repeatedly (PCG, inverse iteration, GPE, evolve) reuse their vectors instead of a
// cudaMalloc / cudaFree pair (which synchronises the device) per call.
struct DBuf {
  kronop_ctx* c = nullptr;
  double* p = nullptr;
  DBuf() = default;
  DBuf(kronop_ctx& ctx, size_t n) : c(&ctx), p(pool_get(ctx, std::max<size_t>(n, 1))) {}
  ~DBuf() {
    if (p) pool_put(*c, p);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};


// Real view of a field: an optional leading re/im axis of extent 2, then the spatial axes.
struct View {
  int nd = 0;
  int cplx = 0;
  long long ext[kMaxDims] = {};
  long long total() const {
    long long t = 1;
    for (int i = 0; i < nd; ++i) t *= ext[i];
    return t;
  }
};
View make_view(int d, const int* shape, int cplx);

void ensure_scratch(kronop_ctx& ctx, size_t doubles);
double* ensure_tmp(kronop_ctx& ctx, size_t doubles);

// One pass on real-view axis `raxis` of `v` (updated to the output shape).
void run_pass(kronop_ctx& ctx, const double* x, double* y, View& v, int raxis, const double* a,
              int lda, int m, const EpiParams& ep);

enum SepKind { SEP_APPLY = 0, SEP_SOLVE = 1, SEP_PROPAGATE = 2 };
// out = T (f(lambda - shift) . (T^{-1} in)) [+ diag .* in - sigma in], f = x, / or exp(-i . dt).
// in may alias out. Uses ctx.scratch.
// bphase: complex propagate only -- the split-step B phase psi * exp(-i bfactor B) (B = bfield,
// NULL = 1) applied to the result, fused into the last pass where the path allows.
void sep_transform(kronop_ctx& ctx, const kronop_op& op, const double* in, double* out, int cplx,
                   SepKind kind, double shift, double dt, const double* diag, double sigma,
                   bool bphase = false, const double* bfield = nullptr, double bfactor = 0.0);
// psi <- propagate(pointwise_phase(psi)) in place with the phase ((cos, sin) table pre_tab)
// applied by the Kronecker propagate's first group as it reads psi; false (nothing enqueued)
// when the propagate does not take the Kronecker path.
bool sep_propagate_prephased(kronop_ctx& ctx, const kronop_op& op, double* psi, double shift,
                             double dt, const double* pre_tab);
// true when complex propagates of op take the Kronecker path (for steps whose E_a fold or are
// small; sep_propagate_prephased has the final say per dt)
bool kron_path_likely(const kronop_op& op);
// Singular-shift guard of SeparableOperator::solve (operators.cpp:44-52).
void check_solve_shift(kronop_ctx& ctx, const kronop_op& op, double shift);

IndexGeomHost mass_geom(const kronop_op& op);

// driver kernels (drivers.cu) for the host-enqueued slab drivers (slab.cu)
void launch_pcg_init(cudaStream_t s, Workspace& ws, PcgScalars* sc, const double* rz,
                     const double* rr, double norm_b, double* history);
void launch_pcg_alpha(cudaStream_t s, Workspace& ws, PcgScalars* sc);
void launch_pcg_beta(cudaStream_t s, Workspace& ws, PcgScalars* sc);
void launch_pcg_finish(cudaStream_t s, Workspace& ws, PcgScalars* sc, double* history);
void launch_beta_square(cudaStream_t s, Workspace& ws, double* dg, const double* u, double beta,
                        const double* v2, long long n);
void launch_sub_scaled(cudaStream_t s, Workspace& ws, double* g, const double* a, const double* b,
                       double c, long long n);
void launch_square2(cudaStream_t s, Workspace& ws, double* sq, const double* u, long long n);
void set_error(const std::string& msg);

}  // namespace kronop_dev
