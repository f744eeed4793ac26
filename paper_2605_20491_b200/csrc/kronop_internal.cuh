// Internal declarations shared by the kronop CUDA translation units.
// Not part of the public boundary (that is include/kronop_cuda.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/kronop_cuda.h"
#include "host_setup.hpp"

namespace kronop_dev {

// ---------------------------------------------------------------- errors --
// Mirrors the reference's exception hierarchy (proj/include/kronop/errors.hpp:9-30) as status
// codes at the C boundary; internally C++ exceptions carry the code to the extern "C" shim.
using Error = kronop_host::Error;
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void param_check(bool ok, const std::string& msg) {
  if (!ok) fail(KRONOP_EPARAM, msg);
}

#define KCUDA(expr)                                                                        \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      ::kronop_dev::fail(_e == cudaErrorMemoryAllocation ? KRONOP_ECAPABILITY : KRONOP_ERUNTIME, \
                         std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " +   \
                             __FILE__ + ":" + std::to_string(__LINE__));                   \
  } while (0)

// Opt-in dynamic shared memory is a per-device function attribute: set it once per (kernel,
// device), so a process with contexts on several GPUs (kronop_slab_create) launches everywhere.
inline void ensure_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, std::unordered_map<int, size_t>> done;
  int dev = 0;
  KCUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[fn][dev];
  if (have >= bytes) return;
  KCUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(bytes)));
  have = bytes;
}
inline int device_sm_count() {
  int dev = 0, v = 148;
  KCUDA(cudaGetDevice(&dev));
  KCUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  return v;
}

// ------------------------------------------------------------ mode product --
// One pass of the mode-k product on a field viewed as a real (pre x nk x post) array, axis 0
// fastest:  Y[p, i, q] = sum_j A[i, j] X[p, j, q]  (proj/src/tensor.cpp:105-134).
// Complex fields (interleaved re/im, the reference's std::complex layout) are the real view with a
// leading axis of extent 2, exactly as contract_inner_axis reinterprets them (tensor.cpp:124-131).
constexpr int kMatPadM = 128;  // row padding of device copies of per-axis matrices
constexpr int kMatPadK = 16;   // column (contraction) padding

inline int pad_up(int v, int p) { return (v + p - 1) / p * p; }

enum EpiKind : int {
  EPI_STORE = 0,       // y = acc
  EPI_SPEC_MUL = 1,    // y = acc * (lambda - shift)              operators.cpp:36
  EPI_SPEC_DIV = 2,    // y = acc / (lambda - shift)              operators.cpp:57
  EPI_SPEC_PHASE = 3,  // complex: y = acc * exp(-i (lambda - shift) dt)   operators.cpp:68-71
  EPI_AXPY_DIAG = 4,   // y = (acc + diag .* u) - sigma * u       operators.cpp:102, ground_state.cpp:70-72
  // complex: y = acc * exp(-i dt B) with B = diag (spatial, NULL = 1), the split-step B phase
  // (pointwise_phase, splitting.cpp:44-51) fused into the propagate's last backward pass
  EPI_BPHASE = 5,
};

constexpr int kMaxDims = 10;  // 9 spatial axes + the complex component axis

struct EpiParams {
  int kind = EPI_STORE;
  int axis = 0;                  // real-view axis this pass contracts
  // index decomposition of the real view (for lambda / diag indexing)
  int ndims = 0;                 // real-view dimensions
  long long ext[kMaxDims] = {};  // real-view extents (output shape of this pass)
  const double* lam[kMaxDims] = {};  // per real-view axis eigenvalues, null for the re/im axis
  double shift = 0.0;
  double dt = 0.0;
  const double* diag = nullptr;  // V2 / diag field (spatial index, real)
  const double* u = nullptr;     // the operator's input field (same layout as y)
  double sigma = 0.0;
  int cplx = 0;                  // real view has a leading re/im axis
  // optional device flag (a PcgScalars::active of a host-enqueued driver loop): the pass is
  // skipped when *active == 0, so speculatively enqueued iterations cost a launch, not a pass
  const int* active = nullptr;
};

// Exchange-fused output of a pass (slab decomposition, slab.cu): the output columns i are split
// into consecutive ranges [i0[k], i0[k+1]) owned by destination part k, and element (p, i, q)
// (p < pre, q < post) is stored at dst[k] + (i - i0[k]) * ccol[k] + p + q * cq[k] -- straight into
// the part's slab buffer (peer memory over NVLink, or the same device), so the pass that precedes
// a slab transpose IS the transpose.
constexpr int kMaxSplit = 8;
struct SplitDst {
  int parts = 0;
  int i0[kMaxSplit + 1] = {};
  double* dst[kMaxSplit] = {};
  long long ccol[kMaxSplit] = {};
  long long cq[kMaxSplit] = {};
};

struct PassShape {
  // exchange-fused store (TMA kernel, EPI_STORE only); null = the pass's own output y
  const SplitDst* split = nullptr;
  long long pre = 1, post = 1;
  int nk = 0, m = 0;
  // q-strides of X and Y (doubles). 0 = dense (pre * nk, pre * m); larger values address a
  // sub-range of a longer axis (the even/odd halves of a folded axis).
  long long ldx = 0, ldy = 0;
  // Rotated output (TMA kernel only): ycol = stride of the output index i (0 = pre), and rot = 1
  // when the spectral eigenvalue sum runs over the full row index r (the rows enumerate the other
  // axes in order: the layout of a pass that moves its contracted axis to the slowest end).
  long long ycol = 0;
  int rot = 0;
  long long ldx_eff() const { return ldx ? ldx : pre * nk; }
  long long ldy_eff() const { return ldy ? ldy : pre * m; }
};

// Launch one pass. a_pad: device matrix, column-major with leading dimension lda >= pad_up(m,128),
// zero padded to pad_up(nk,16) columns. x and y must not alias.
void prime_mode_product_kernels();
// TMA + mbarrier warp-specialised kernel (mode_product_tma.cu) for the STRIDED (pre % 128 == 0)
// and CONTIG (pre == 1, even nk) geometries; launch_mode_product dispatches to it when eligible.
void prime_mode_product_tma_kernels();
// Rotating-layout group transform (fused_rot.cu): contracts the f fastest axes after the re/im
// axis and writes them to the slowest end. Used when every axis has n <= 32.
struct RotEpi {
  int kind = EPI_STORE;  // EPI_STORE, EPI_SPEC_* (last forward group), EPI_AXPY_DIAG (last backward)
  double shift = 0.0, dt = 0.0, sigma = 0.0;
  const double* diag = nullptr;
  const double* u = nullptr;
  const double* lam_g[3] = {};               // eigenvalues of the group axes
  int nq = 0;                                // axes below the group (original order)
  long long qext[KRONOP_MAX_DIM] = {};
  const double* lam_q[KRONOP_MAX_DIM] = {};
};
void prime_fused_rot_kernels();
bool fused_rot_eligible(const double* x);
// returns the number of kernels launched (2 when the spectral epilogue runs as its own pass)
int launch_fused_rot(cudaStream_t s, const double* x, double* y, int cplx, int f, const int* n,
                     long long N, const double* const* mats, const int* lda, const RotEpi& epi);

// Kronecker-factored complex propagate (kron_prop.cu): one launch contracts a group of f <= 3
// consecutive axes of extent n (2..10) with the complex matrices E (f x n x n x (re, im), row i =
// output, k = input) and moves the group to the slowest end (the rotating layout of fused_rot.cu).
// bphase: the output is multiplied by exp(-i bfactor B) (B = bfield, null = 1). fold: E holds
// the parity blocks [Ae | Ao] of R-symmetric axis matrices instead (see kr_contract).
bool kron_group_supported(int n, int f);
bool kron_group_needs_fold(int n);  // extents > 10 (DMMA kernel): parity-symmetric axes only
// Real-field transform-form group launch (kron_prop.cu, kron_real_kernel): one group of f <= 3
// consecutive axes of extent n <= 10, real matrices M (f x n x n row-major: output i, input k),
// rotating layout; epi 0 store, 1 spectral divide, 2 spectral multiply (last forward group:
// lambda = the nq axes below the group (qext / lam_q) then the group axes lam_g, minus shift),
// 3 AXPY (+ diag u - sigma u, last backward group).
struct KronRealLaunch {
  const double* x = nullptr;
  double* y = nullptr;
  long long Ntot = 0;
  int n = 0, f = 0, epi = 0;
  const double* M = nullptr;
  double shift = 0.0, sigma = 0.0;
  const double* diag = nullptr;
  const double* u = nullptr;
  const double* lam_g[3] = {};
  int nq = 0;
  long long qext[KRONOP_MAX_DIM] = {};
  const double* lam_q[KRONOP_MAX_DIM] = {};
};
bool kron_real_supported(int n, int f);
void launch_kron_real_group(cudaStream_t s, const KronRealLaunch& L);
// pre: (cos, sin) table of the B phase that precedes this propagate (first group only; null =
// none), applied to the input as it is read.
void launch_kron_group(cudaStream_t s, const double* x, double* y, int n, int f, bool fold,
                       long long Ntot, const double* E, const double* bfield, double bfactor,
                       int bphase, const double* pre);

bool mode_product_tma_eligible(const double* x, const PassShape& ps);
bool mode_product_tma_enabled();  // false under KRONOP_DISABLE_TMA=1
void launch_mode_product_tma(cudaStream_t s, const double* x, double* y, const double* a_pad,
                             int lda, const PassShape& ps, const EpiParams& ep);
void launch_mode_product(cudaStream_t s, const double* x, double* y, const double* a_pad, int lda,
                         const PassShape& ps, const EpiParams& ep);

// ------------------------------------------------------------- workspace --
constexpr int kRedBlocks = 592;   // 4 x 148 SMs: reduction grid (fixed => deterministic)
constexpr int kEltBlocks = 1184;  // 8 x 148 SMs: elementwise grid-stride kernels

struct Workspace {
  double* partials = nullptr;  // kRedBlocks * 4 doubles
  unsigned long long launches = 0;
};

}  // namespace kronop_dev
