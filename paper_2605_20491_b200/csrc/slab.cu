// Slab decomposition of the tensor-product operators over several GPUs (SURVEY.md §8e,
// north-star item 4), behind the C-ABI (kronop_slab_*).
//
// A field of shape (n_0, ..., n_{d-1}) is cut into P contiguous slabs of its slowest axis:
// part p owns planes [z0_p, z0_p + nz_p) (uneven splits allowed). An operator application
//   forward passes on axes 0..d-2 (local, the part's z-slab)
//   z -> y exchange: every part sends the (nz_p, ny_q, R) block of its slab to part q, which
//                    stacks them into its y-slab (nz, ny_q, R) -- R = prod n_0..n_{d-3}
//   forward pass on axis d-1 with the fused spectral epilogue (global lambda via sliced pointers)
//   backward pass on axis d-1
//   y -> z exchange (the transpose back)
//   backward passes on axes 0..d-2, the last fusing + V2 u - sigma u (FullOperator::apply)
// equals T (f(lambda - shift) . T^{-1} x) of operators.cpp:31-75 up to the order of the commuting
// Kronecker factors. Two exchanges per application, two scalar all-gathers per PCG iteration.
//
// Two transports, one algorithm:
//   * in-process (kronop_slab_create): one process drives all P parts, one stream per part, on
//     the listed devices -- distinct GPUs (peer access over NVLink / NVSwitch: the exchange is
//     cudaMemcpy3DPeerAsync of each (p, q) block straight from the source slab into the
//     destination slab, no packing) or the same device repeated ("virtual slabs", the
//     single-GPU check of the decomposition); cross-part ordering by events;
//   * NCCL (kronop_slab_create_nccl): one process per GPU, part = rank; the exchange is one
//     grouped ncclSend / ncclRecv per (plane, peer), so neither side packs or stages; libnccl is
//     dlopen'd (the same libnccl.so.2 torch.distributed loaded, when present).
// Scalars (dot products) are all-gathered partial sums added in part order on every part, so all
// parts hold bit-identical scalars and take identical loop decisions without talking to the host.
//
// The drivers (PCG, the a_u GPE flow) are host-enqueued with a one-iteration lookahead: the
// convergence flag of iteration k-1 is read from pinned memory while iteration k is already
// queued, and every pass / vector kernel of an iteration is gated on the device-side `active` flag
// (EpiParams::active, PcgScalars::active), so the one speculative iteration after convergence
// costs kernel launches, not passes.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "context.cuh"

namespace kronop_dev {

int guard_slab_impl(const std::exception_ptr& ep);

template <class F>
int guard_slab(F&& f) {
  try {
    f();
    return KRONOP_OK;
  } catch (...) {
    return guard_slab_impl(std::current_exception());
  }
}

int guard_slab_impl(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
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
  return KRONOP_ERUNTIME;
}

// ------------------------------------------------------------------------------ NCCL --
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;

static void nccl_load(const char* path) {
  if (g_nccl.h) return;
  void* h = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) fail(KRONOP_ECAPABILITY, std::string("NCCL not available: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) fail(KRONOP_ECAPABILITY, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  NcclApi a;
  a.h = h;
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
  a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  g_nccl = a;
}

#define KNCCL(expr)                                                                     \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess)                                                              \
      ::kronop_dev::fail(KRONOP_ERUNTIME, std::string("NCCL error: ") +                 \
                                              g_nccl.GetErrorString(_r) + " at " +      \
                                              __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// -------------------------------------------------------------------- slab geometry --
// Contiguous, as-even-as-possible split of n planes into `parts` (the first n % parts get one more).
static void split_extent(int n, int parts, std::vector<int>& ext, std::vector<int>& off) {
  ext.assign(parts, n / parts);
  for (int p = 0; p < n % parts; ++p) ext[p] += 1;
  off.assign(parts, 0);
  for (int p = 1; p < parts; ++p) off[p] = off[p - 1] + ext[p - 1];
}

// sum_p src[p][j] for j < k, in part order (identical bits on every part)
__global__ void k_gather_sum(const double* const* src, int nparts, int k, double* dst) {
  const int j = threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s = __dadd_rn(s, src[p][j]);
  dst[j] = s;
}

// out[j] = a[j] / b[j] for the pair (num, den) slots -> (proj) etc. are done on the host side;
// device-side copy of one slot into a PcgScalars field
__global__ void k_copy_scalar(double* dst, const double* src) { *dst = *src; }

// all-gathered PCG scalars into the PcgScalars block: which = 0: p.q; 1: (r.r, r.z_next)
__global__ void k_pcg_take(PcgScalars* sc, const double* v, int which) {
  if (which == 0) {
    sc->pq = v[0];
  } else {
    sc->rr = v[0];
    sc->rz_next = v[1];
  }
}

}  // namespace kronop_dev

using namespace kronop_dev;

constexpr int kSlabSlots = 8;   // doubles per all-gather
constexpr int kSlabRing = 4;    // ring of partial-sum buffers (WAR safety across all-gathers)

struct SlabPart {
  kronop_ctx* ctx = nullptr;
  bool own_ctx = false;
  int p = 0;  // slab index
  double* fwd[KRONOP_MAX_DIM] = {};
  double* bwd[KRONOP_MAX_DIM] = {};
  int lda[KRONOP_MAX_DIM] = {};
  double* lam[KRONOP_MAX_DIM] = {};   // full per-axis eigenvalues
  double* mass[KRONOP_MAX_DIM] = {};  // full per-axis mass weights (or null)
  double* zx = nullptr;               // exchange buffer, z-slab layout
  size_t zx_cap = 0;
  double* yx = nullptr;               // receive buffer of the fused z -> y exchange, y-slab layout
  size_t yx_cap = 0;
  double* red = nullptr;              // partials ring [kSlabRing][kSlabSlots] + gathered
  double* gathered = nullptr;         // NCCL: [P][kSlabSlots]
  const double** srcs = nullptr;      // device array of P pointers (this ring slot's sources)
  std::vector<const double**> srcs_ring;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
};

struct kronop_slab {
  int P = 1;
  int d = 0;
  int n[KRONOP_MAX_DIM] = {};
  long long N = 0;
  long long R = 1;  // prod n_0..n_{d-3}
  double shift = 0.0, lmin = 0.0, lmax = 0.0;
  bool has_mass = false;
  std::vector<int> zs, z0, ys, y0;
  std::vector<SlabPart> parts;  // local parts
  bool nccl = false;
  ncclComm_t comm = nullptr;
  int ring = 0;  // next partials ring slot
  long long fused_transforms = 0;  // applications whose transposes were exchange-fused passes
  // NCCL transport: the peers' receive buffers mapped into this process (CUDA IPC), so the
  // exchange-fused passes store into them over NVLink. 0 = not set up yet, 1 = on, -1 = off
  // (IPC unavailable or the collective self-check failed: grouped send / recv instead)
  int ipc = 0;
  int ipc_c = 0;                           // field kind (1 real, 2 complex) the mapping was sized for
  std::vector<double*> peer_yx, peer_zx;  // [P], own buffers at this rank
  std::vector<void*> ipc_opened;
  double* bar = nullptr;                   // barrier all-gather buffer (1 + P doubles)
};

namespace kronop_dev {

static long long zslab_elems(const kronop_slab& s, int p) {
  long long e = s.zs[p];
  for (int a = 0; a < s.d - 1; ++a) e *= s.n[a];
  return e;
}
static long long yslab_elems(const kronop_slab& s, int q) {
  return s.R * s.ys[q] * s.n[s.d - 1];
}

static void part_device(const SlabPart& pt) { KCUDA(cudaSetDevice(pt.ctx->device)); }

// ---------------------------------------------------------------------- exchanges --
// 2-D copy of `height` rows of `width` doubles (pitches in doubles) between two parts' buffers,
// on the destination part's stream.
static void copy2d(const SlabPart& dst_part, double* dst, long long dpitch, const SlabPart& src_part,
                   const double* src, long long spitch, long long width, long long height) {
  if (width == 0 || height == 0) return;
  cudaStream_t st = dst_part.ctx->stream;
  if (dst_part.ctx->device == src_part.ctx->device) {
    KCUDA(cudaMemcpy2DAsync(dst, dpitch * 8, src, spitch * 8, width * 8, height,
                            cudaMemcpyDeviceToDevice, st));
  } else {
    cudaMemcpy3DPeerParms pr{};
    pr.srcPtr = make_cudaPitchedPtr(const_cast<double*>(src), spitch * 8, width * 8, height);
    pr.srcDevice = src_part.ctx->device;
    pr.dstPtr = make_cudaPitchedPtr(dst, dpitch * 8, width * 8, height);
    pr.dstDevice = dst_part.ctx->device;
    pr.extent = make_cudaExtent(width * 8, height, 1);
    KCUDA(cudaMemcpy3DPeerAsync(&pr, st));
  }
}

// all local parts: record ev_a (work so far done); every part waits for every other's ev_a
static void barrier_a(kronop_slab& s) {
  if (s.parts.size() < 2) return;
  for (auto& pt : s.parts) {
    part_device(pt);
    KCUDA(cudaEventRecord(pt.ev_a, pt.ctx->stream));
  }
  for (auto& q : s.parts) {
    part_device(q);
    for (auto& p : s.parts)
      if (&p != &q) KCUDA(cudaStreamWaitEvent(q.ctx->stream, p.ev_a, 0));
  }
}
static void barrier_b(kronop_slab& s) {
  if (s.parts.size() < 2) return;
  for (auto& pt : s.parts) {
    part_device(pt);
    KCUDA(cudaEventRecord(pt.ev_b, pt.ctx->stream));
  }
  for (auto& q : s.parts) {
    part_device(q);
    for (auto& p : s.parts)
      if (&p != &q) KCUDA(cudaStreamWaitEvent(q.ctx->stream, p.ev_b, 0));
  }
}

// z-slabs src[] (part layout (nz_p, ny, Rc)) -> y-slabs dst[] ((nz, ny_q, Rc)); c = 2 complex
static void exchange_z_to_y(kronop_slab& s, const std::vector<const double*>& src,
                            const std::vector<double*>& dst, int c) {
  const long long Rc = s.R * c;
  const int ny = s.n[s.d - 2];
  if (!s.nccl) {
    barrier_a(s);
    for (size_t qi = 0; qi < s.parts.size(); ++qi) {
      SlabPart& q = s.parts[qi];
      part_device(q);
      for (size_t pi = 0; pi < s.parts.size(); ++pi) {
        const SlabPart& p = s.parts[pi];
        copy2d(q, dst[qi] + static_cast<long long>(s.z0[p.p]) * s.ys[q.p] * Rc, s.ys[q.p] * Rc, p,
               src[pi] + static_cast<long long>(s.y0[q.p]) * Rc, ny * Rc, s.ys[q.p] * Rc,
               s.zs[p.p]);
      }
    }
    return;
  }
  SlabPart& me = s.parts[0];
  const int r = me.p;
  cudaStream_t st = me.ctx->stream;
  // own block: local copy
  copy2d(me, dst[0] + static_cast<long long>(s.z0[r]) * s.ys[r] * Rc, s.ys[r] * Rc, me,
         src[0] + static_cast<long long>(s.y0[r]) * Rc, ny * Rc, s.ys[r] * Rc, s.zs[r]);
  KNCCL(g_nccl.GroupStart());
  for (int q = 0; q < s.P; ++q) {
    if (q == r) continue;
    for (int z = 0; z < s.zs[r]; ++z)  // plane z of my slab, rows of q
      KNCCL(g_nccl.Send(src[0] + (static_cast<long long>(z) * ny + s.y0[q]) * Rc,
                        static_cast<size_t>(s.ys[q] * Rc), ncclDouble, q, s.comm, st));
    for (int z = 0; z < s.zs[q]; ++z)  // plane z of q's slab, my rows (contiguous destination)
      KNCCL(g_nccl.Recv(dst[0] + (static_cast<long long>(s.z0[q]) + z) * s.ys[r] * Rc,
                        static_cast<size_t>(s.ys[r] * Rc), ncclDouble, q, s.comm, st));
  }
  KNCCL(g_nccl.GroupEnd());
}

// y-slabs src[] ((nz, ny_q, Rc)) -> z-slabs dst[] ((nz_p, ny, Rc))
static void exchange_y_to_z(kronop_slab& s, const std::vector<const double*>& src,
                            const std::vector<double*>& dst, int c) {
  const long long Rc = s.R * c;
  const int ny = s.n[s.d - 2];
  if (!s.nccl) {
    barrier_a(s);
    for (size_t pi = 0; pi < s.parts.size(); ++pi) {
      SlabPart& p = s.parts[pi];
      part_device(p);
      for (size_t qi = 0; qi < s.parts.size(); ++qi) {
        const SlabPart& q = s.parts[qi];
        copy2d(p, dst[pi] + static_cast<long long>(s.y0[q.p]) * Rc, ny * Rc, q,
               src[qi] + static_cast<long long>(s.z0[p.p]) * s.ys[q.p] * Rc, s.ys[q.p] * Rc,
               s.ys[q.p] * Rc, s.zs[p.p]);
      }
    }
    barrier_b(s);  // sources (the y-slabs in scratch) are rewritten right after
    return;
  }
  SlabPart& me = s.parts[0];
  const int r = me.p;
  cudaStream_t st = me.ctx->stream;
  copy2d(me, dst[0] + static_cast<long long>(s.y0[r]) * Rc, ny * Rc, me,
         src[0] + static_cast<long long>(s.z0[r]) * s.ys[r] * Rc, s.ys[r] * Rc, s.ys[r] * Rc,
         s.zs[r]);
  KNCCL(g_nccl.GroupStart());
  for (int q = 0; q < s.P; ++q) {
    if (q == r) continue;
    for (int z = 0; z < s.zs[q]; ++z)  // q's planes of my y-rows (contiguous source)
      KNCCL(g_nccl.Send(src[0] + (static_cast<long long>(s.z0[q]) + z) * s.ys[r] * Rc,
                        static_cast<size_t>(s.ys[r] * Rc), ncclDouble, q, s.comm, st));
    for (int z = 0; z < s.zs[r]; ++z)  // my plane z, q's rows
      KNCCL(g_nccl.Recv(dst[0] + (static_cast<long long>(z) * ny + s.y0[q]) * Rc,
                        static_cast<size_t>(s.ys[q] * Rc), ncclDouble, q, s.comm, st));
  }
  KNCCL(g_nccl.GroupEnd());
}

// -------------------------------------------------------------------- the transform --
struct SlabEpi {
  int kind = EPI_SPEC_MUL;
  double shift = 0.0, dt = 0.0, sigma = 0.0;
  std::vector<const double*> diag;  // per local part, spatial z-slab (or empty)
  const int* const* active = nullptr;  // per local part device flag (or null)
};

static void ensure_part_buffers(kronop_slab& s, int c) {
  for (auto& pt : s.parts) {
    part_device(pt);
    const size_t need = static_cast<size_t>(std::max(zslab_elems(s, pt.p), yslab_elems(s, pt.p))) * c;
    ensure_scratch(*pt.ctx, need);
    const size_t zneed = static_cast<size_t>(zslab_elems(s, pt.p)) * c;
    if (zneed > pt.zx_cap) {
      if (pt.zx) KCUDA(cudaFree(pt.zx));
      pt.zx = nullptr;
      KCUDA(cudaMalloc(&pt.zx, zneed * sizeof(double)));
      pt.zx_cap = zneed;
    }
  }
}

// Exchange-fused transform (in-process transport): the pass before each slab transpose stores
// its output columns straight into the destination parts' slab buffers (SplitDst epilogue of the
// TMA pass kernel: NVLink peer stores for distinct GPUs, plain stores for virtual slabs), so the
// transposes cost no copy and no extra HBM round trip, and the transfer overlaps the pass's
// math tile by tile:
//   forward passes 0..d-3 (local) | barrier | pass d-2 -> every part's y-slab receive buffer (yx)
//   | barrier | pass d-1 forward + spectral (local) | pass d-1 backward -> every part's z-slab
//   buffer (zx) | barrier | backward passes 0..d-2 (local)
// Used when both transpose passes take the TMA kernel on every part (KRONOP_SLAB_FUSED=0: the
// copy exchange). The NCCL transport keeps grouped send / recv.
// stream-ordered barrier of the NCCL transport: an all-gather of one double per rank completes
// on a rank only when every rank's stream has reached it
static void nccl_barrier(kronop_slab& s) {
  SlabPart& me = s.parts[0];
  KNCCL(g_nccl.AllGather(s.bar, s.bar + 1, 1, ncclDouble, s.comm, me.ctx->stream));
}

__global__ void k_ipc_probe(double* const* dsts, int P, int rank) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < P) dsts[q][rank] = static_cast<double>(rank + 1);
}

// One-time, collective (every rank calls it at the same transform): allocate the receive
// buffers at complex size (they never move afterwards), exchange their CUDA IPC handles over
// NCCL, open the peers', and check the mapping end to end (every rank writes its id into every
// rank's buffer through the mapped pointers, all-gather barrier, every rank reads them back);
// all ranks then agree on the outcome, so a failure anywhere falls back everywhere.
// Grow a receive buffer to `need` doubles without losing the old one on failure (false: out of
// memory, old buffer kept -- the caller falls back to the copy / send-recv exchange).
static bool grow_buffer(double*& p, size_t& cap, size_t need) {
  if (cap >= need) return true;
  double* q = nullptr;
  if (cudaMalloc(&q, need * sizeof(double)) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  if (p) KCUDA(cudaFree(p));
  p = q;
  cap = need;
  return true;
}

// (Re)run for a field kind c larger than the mapped buffers were sized for (c = 2 after real
// transforms); every rank reaches it at the same transform, so it stays collective.
static void slab_ipc_setup(kronop_slab& s, int c) {
  SlabPart& me = s.parts[0];
  part_device(me);
  cudaStream_t st = me.ctx->stream;
  const int P = s.P, r = me.p;
  KCUDA(cudaStreamSynchronize(st));
  if (!s.bar) {
    KCUDA(cudaMalloc(&s.bar, (1 + P) * sizeof(double)));
    KCUDA(cudaMemsetAsync(s.bar, 0, (1 + P) * sizeof(double), st));
  }
  // a re-setup: every rank drops its mappings of the peers' buffers, and all have dropped them
  // before anyone frees a buffer it exported
  const bool had = !s.ipc_opened.empty() || s.ipc > 0;
  for (void* p : s.ipc_opened) cudaIpcCloseMemHandle(p);
  s.ipc_opened.clear();
  if (had) {
    nccl_barrier(s);
    KCUDA(cudaStreamSynchronize(st));
  }
  bool ok = true;
  try {
    const size_t zneed = static_cast<size_t>(zslab_elems(s, r)) * c;
    const size_t yneed = static_cast<size_t>(yslab_elems(s, r)) * c;
    ok = grow_buffer(me.zx, me.zx_cap, zneed) && grow_buffer(me.yx, me.yx_cap, yneed);
  } catch (...) {
    ok = false;
  }
  // handle exchange (every rank takes part, whatever its local outcome)
  struct Handles {
    cudaIpcMemHandle_t y, z;
    int ok;
  };
  Handles mine{};
  if (ok) {
    ok = cudaIpcGetMemHandle(&mine.y, me.yx) == cudaSuccess &&
         cudaIpcGetMemHandle(&mine.z, me.zx) == cudaSuccess;
    (void)cudaGetLastError();
  }
  mine.ok = ok ? 1 : 0;
  unsigned char* dh = nullptr;
  KCUDA(cudaMalloc(&dh, sizeof(Handles) * (1 + P)));
  KCUDA(cudaMemcpyAsync(dh, &mine, sizeof(Handles), cudaMemcpyHostToDevice, st));
  KNCCL(g_nccl.AllGather(dh, dh + sizeof(Handles), sizeof(Handles), ncclUint8, s.comm, st));
  std::vector<Handles> all(P);
  KCUDA(cudaMemcpyAsync(all.data(), dh + sizeof(Handles), sizeof(Handles) * P,
                        cudaMemcpyDeviceToHost, st));
  KCUDA(cudaStreamSynchronize(st));
  for (const Handles& h : all) ok = ok && h.ok;
  s.peer_yx.assign(P, nullptr);
  s.peer_zx.assign(P, nullptr);
  if (ok) {
    for (int q = 0; q < P && ok; ++q) {
      if (q == r) {
        s.peer_yx[q] = me.yx;
        s.peer_zx[q] = me.zx;
        continue;
      }
      void *py = nullptr, *pz = nullptr;
      ok = cudaIpcOpenMemHandle(&py, all[q].y, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (ok) s.ipc_opened.push_back(py);
      ok = ok && cudaIpcOpenMemHandle(&pz, all[q].z, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (pz) s.ipc_opened.push_back(pz);
      (void)cudaGetLastError();
      s.peer_yx[q] = static_cast<double*>(py);
      s.peer_zx[q] = static_cast<double*>(pz);
    }
  }
  // probe through the mapping: rank r writes r + 1 into slot r of every rank's y buffer
  double** dptrs = nullptr;
  KCUDA(cudaMalloc(&dptrs, P * sizeof(double*)));
  if (ok) {
    KCUDA(cudaMemcpyAsync(dptrs, s.peer_yx.data(), P * sizeof(double*), cudaMemcpyHostToDevice,
                          st));
    k_ipc_probe<<<1, 32 * ((P + 31) / 32), 0, st>>>(dptrs, P, r);
    ok = cudaGetLastError() == cudaSuccess;
  }
  nccl_barrier(s);
  std::vector<double> got(P, 0.0);
  if (ok) {
    KCUDA(cudaMemcpyAsync(got.data(), me.yx, P * sizeof(double), cudaMemcpyDeviceToHost, st));
    KCUDA(cudaStreamSynchronize(st));
    for (int q = 0; q < P; ++q) ok = ok && got[q] == static_cast<double>(q + 1);
  }
  // agreement: every rank's verdict
  Handles verdict{};
  verdict.ok = ok ? 1 : 0;
  KCUDA(cudaMemcpyAsync(dh, &verdict, sizeof(Handles), cudaMemcpyHostToDevice, st));
  KNCCL(g_nccl.AllGather(dh, dh + sizeof(Handles), sizeof(Handles), ncclUint8, s.comm, st));
  KCUDA(cudaMemcpyAsync(all.data(), dh + sizeof(Handles), sizeof(Handles) * P,
                        cudaMemcpyDeviceToHost, st));
  KCUDA(cudaStreamSynchronize(st));
  for (const Handles& h : all) ok = ok && h.ok;
  KCUDA(cudaFree(dh));
  KCUDA(cudaFree(dptrs));
  s.ipc = ok ? 1 : -1;
  s.ipc_c = c;
}

// Exchange-fused transform (in-process transport, or NCCL with the peers' buffers mapped by CUDA
// IPC): the pass before each slab transpose stores its output columns straight into the
// destination parts' slab buffers (SplitDst epilogue of the TMA pass kernel: NVLink peer stores
// for distinct GPUs, plain stores for virtual slabs), so the transposes cost no copy and no extra
// HBM round trip, and the transfer overlaps the pass's math tile by tile:
//   forward passes 0..d-3 (local) | barrier | pass d-2 -> every part's y-slab receive buffer (yx)
//   | barrier | pass d-1 forward + spectral (local) | pass d-1 backward -> every part's z-slab
//   buffer (zx) | barrier | backward passes 0..d-2 (local)
// (barriers: cross-stream events in process, a one-double NCCL all-gather across processes).
// Used when both transpose passes take the TMA kernel on every part -- decided from the global
// slab geometry, so all ranks decide alike (KRONOP_SLAB_FUSED=0: the copy / send-recv exchange).
static bool slab_fused_ok(kronop_slab& s, int c) {
  static const bool off = [] {
    const char* e = getenv("KRONOP_SLAB_FUSED");
    return e && e[0] == '0';
  }();
  if (off || s.d < 2 || s.P > kMaxSplit || !mode_product_tma_enabled()) return false;
  const int d = s.d;
  for (int p = 0; p < s.P; ++p) {  // every part's geometry (all fields are 16-byte aligned here)
    PassShape a;
    a.pre = s.R * c;
    a.nk = a.m = s.n[d - 2];
    a.post = s.zs[p];
    PassShape b;
    b.pre = s.R * c * s.ys[p];
    b.nk = b.m = s.n[d - 1];
    b.post = 1;
    const double* aligned = reinterpret_cast<const double*>(static_cast<uintptr_t>(256));
    if (!mode_product_tma_eligible(aligned, a) || !mode_product_tma_eligible(aligned, b))
      return false;
  }
  if (s.nccl) {
    if (s.ipc == 0 || (s.ipc > 0 && c > s.ipc_c)) slab_ipc_setup(s, c);
    return s.ipc > 0;
  }
  // in process: the y-slab receive buffers (one slab more than the copy exchange needs); out of
  // memory -> the copy exchange
  for (auto& pt : s.parts) {
    part_device(pt);
    const size_t yneed = static_cast<size_t>(yslab_elems(s, pt.p)) * c;
    if (pt.yx_cap < yneed) {
      KCUDA(cudaStreamSynchronize(pt.ctx->stream));
      if (!grow_buffer(pt.yx, pt.yx_cap, yneed)) return false;
    }
  }
  return true;
}

static void slab_transform_fused(kronop_slab& s, const std::vector<const double*>& in,
                                 const std::vector<double*>& out, int cplx, const SlabEpi& e) {
  const int c = cplx ? 2 : 1;
  const int d = s.d;
  const long long Rc = s.R * c;
  const int ny = s.n[d - 2];
  // destination buffers of every part (the local ones, or the IPC-mapped peers')
  std::vector<double*> yx(s.P, nullptr), zx(s.P, nullptr);
  if (s.nccl) {
    yx = s.peer_yx;
    zx = s.peer_zx;
  } else {
    for (auto& pt : s.parts) {
      yx[pt.p] = pt.yx;
      zx[pt.p] = pt.zx;
    }
  }
  auto barrier = [&]() {
    if (s.nccl)
      nccl_barrier(s);
    else
      barrier_a(s);
  };
  // forward passes on axes 0..d-3 (local)
  std::vector<const double*> cur(s.parts.size());
  for (size_t i = 0; i < s.parts.size(); ++i) {
    SlabPart& pt = s.parts[i];
    part_device(pt);
    kronop_ctx& ctx = *pt.ctx;
    int shp[KRONOP_MAX_DIM];
    for (int a = 0; a < d - 1; ++a) shp[a] = s.n[a];
    shp[d - 1] = s.zs[pt.p];
    View v = make_view(d, shp, cplx);
    cur[i] = in[i];
    if ((reinterpret_cast<uintptr_t>(cur[i]) & 15) != 0) {  // TMA needs 16-byte aligned rows
      double* t = ensure_tmp(ctx, static_cast<size_t>(zslab_elems(s, pt.p)) * c);
      KCUDA(cudaMemcpyAsync(t, cur[i], zslab_elems(s, pt.p) * c * sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx.stream));
      cur[i] = t;
    }
    for (int a = 0; a < d - 2; ++a) {
      double* dst = ctx.scratch[a % 2];
      EpiParams ep;
      ep.active = e.active ? e.active[i] : nullptr;
      run_pass(ctx, cur[i], dst, v, a + v.cplx, pt.fwd[a], pt.lda[a], s.n[a], ep);
      cur[i] = dst;
    }
  }
  barrier();  // every part's receive buffer is free (its last reader was the previous call)
  // pass d-2 = the z -> y transpose: column y of part p's output goes to part q = owner(y) at
  // yx_q[(z0_p + z) ys_q Rc + (y - y0_q) Rc + r]
  for (size_t i = 0; i < s.parts.size(); ++i) {
    SlabPart& pt = s.parts[i];
    part_device(pt);
    SplitDst sd;
    sd.parts = s.P;
    for (int q = 0; q < s.P; ++q) {
      sd.i0[q] = s.y0[q];
      sd.dst[q] = yx[q] + static_cast<long long>(s.z0[pt.p]) * s.ys[q] * Rc;
      sd.ccol[q] = Rc;
      sd.cq[q] = static_cast<long long>(s.ys[q]) * Rc;
    }
    sd.i0[s.P] = ny;
    PassShape ps;
    ps.pre = Rc;
    ps.nk = ps.m = ny;
    ps.post = s.zs[pt.p];
    ps.split = &sd;
    EpiParams ep;
    ep.active = e.active ? e.active[i] : nullptr;
    launch_mode_product(pt.ctx->stream, cur[i], pt.zx, pt.fwd[d - 2], pt.lda[d - 2], ps, ep);
    pt.ctx->ws.launches += 1;
  }
  barrier();  // every part's y-slab is complete
  // forward axis d-1 + spectral epilogue (local), then backward axis d-1 = the y -> z transpose:
  // column z of part q's output goes to part p = owner(z) at zx_p[(z - z0_p) ny Rc + y0_q Rc + r']
  for (size_t i = 0; i < s.parts.size(); ++i) {
    SlabPart& pt = s.parts[i];
    part_device(pt);
    kronop_ctx& ctx = *pt.ctx;
    int shp[KRONOP_MAX_DIM];
    for (int a = 0; a < d - 2; ++a) shp[a] = s.n[a];
    shp[d - 2] = s.ys[pt.p];
    shp[d - 1] = s.n[d - 1];
    View v = make_view(d, shp, cplx);
    EpiParams ep;
    ep.kind = e.kind;
    ep.axis = d - 1 + v.cplx;
    ep.ndims = v.nd;
    for (int k = 0; k < v.nd; ++k) ep.ext[k] = v.ext[k];
    for (int a = 0; a < d; ++a) ep.lam[a + v.cplx] = pt.lam[a];
    ep.lam[d - 2 + v.cplx] = pt.lam[d - 2] + s.y0[pt.p];  // this part's rows of axis d-2
    ep.shift = e.shift;
    ep.dt = e.dt;
    ep.cplx = v.cplx;
    ep.active = e.active ? e.active[i] : nullptr;
    run_pass(ctx, pt.yx, ctx.scratch[1], v, d - 1 + v.cplx, pt.fwd[d - 1], pt.lda[d - 1],
             s.n[d - 1], ep);
    SplitDst sd;
    sd.parts = s.P;
    for (int p = 0; p < s.P; ++p) {
      sd.i0[p] = s.z0[p];
      sd.dst[p] = zx[p] + static_cast<long long>(s.y0[pt.p]) * Rc;
      sd.ccol[p] = static_cast<long long>(ny) * Rc;
      sd.cq[p] = 0;
    }
    sd.i0[s.P] = s.n[d - 1];
    PassShape ps;
    ps.pre = Rc * s.ys[pt.p];
    ps.nk = ps.m = s.n[d - 1];
    ps.post = 1;
    ps.split = &sd;
    EpiParams st;
    st.active = ep.active;
    launch_mode_product(ctx.stream, ctx.scratch[1], ctx.scratch[0], pt.bwd[d - 1],
                        pt.lda[d - 1], ps, st);
    ctx.ws.launches += 1;
  }
  barrier();  // every part's z-slab is complete
  // backward passes on axes 0..d-2, the last with the FullOperator AXPY epilogue
  for (size_t i = 0; i < s.parts.size(); ++i) {
    SlabPart& pt = s.parts[i];
    part_device(pt);
    kronop_ctx& ctx = *pt.ctx;
    int shp[KRONOP_MAX_DIM];
    for (int a = 0; a < d - 1; ++a) shp[a] = s.n[a];
    shp[d - 1] = s.zs[pt.p];
    View v = make_view(d, shp, cplx);
    const double* src = pt.zx;
    for (int a = 0; a < d - 1; ++a) {
      const bool last = a == d - 2;
      double* dst = last ? out[i] : ctx.scratch[a % 2];
      EpiParams ep;
      ep.active = e.active ? e.active[i] : nullptr;
      const double* dg = e.diag.empty() ? nullptr : e.diag[i];
      if (last && (dg != nullptr || e.sigma != 0.0)) {
        ep.kind = EPI_AXPY_DIAG;
        ep.diag = dg;
        ep.u = in[i];
        ep.sigma = e.sigma;
        ep.cplx = v.cplx;
      }
      run_pass(ctx, src, dst, v, a + v.cplx, pt.bwd[a], pt.lda[a], s.n[a], ep);
      src = dst;
    }
  }
}

// out = T (f(lambda - shift) . T^{-1} in) [+ diag .* in - sigma in] on every local part's slab
static void slab_transform(kronop_slab& s, const std::vector<const double*>& in,
                           const std::vector<double*>& out, int cplx, const SlabEpi& e) {
  const int c = cplx ? 2 : 1;
  const int d = s.d;
  // the fused-exchange decision first: on the NCCL transport it may (collectively) re-map the
  // receive buffers, which must not be reallocated under the peers' mappings
  const bool fused = slab_fused_ok(s, c);
  ensure_part_buffers(s, c);
  if (fused) {
    slab_transform_fused(s, in, out, cplx, e);
    ++s.fused_transforms;
    return;
  }
  std::vector<const double*> zsrc(s.parts.size()), ysrc(s.parts.size());
  std::vector<double*> ydst(s.parts.size()), zdst(s.parts.size());
  // forward passes on axes 0..d-2 (z-slab), ending in zx
  for (size_t i = 0; i < s.parts.size(); ++i) {
    SlabPart& pt = s.parts[i];
    part_device(pt);
    kronop_ctx& ctx = *pt.ctx;
    int shp[KRONOP_MAX_DIM];
    for (int a = 0; a < d - 1; ++a) shp[a] = s.n[a];
    shp[d - 1] = s.zs[pt.p];
    View v = make_view(d, shp, cplx);
    const double* cur = in[i];
    for (int a = 0; a < d - 1; ++a) {
      double* dst = (a == d - 2) ? pt.zx : ctx.scratch[a % 2];
      EpiParams ep;
      ep.active = e.active ? e.active[i] : nullptr;
      run_pass(ctx, cur, dst, v, a + v.cplx, pt.fwd[a], pt.lda[a], s.n[a], ep);
      cur = dst;
    }
    zsrc[i] = pt.zx;
    ydst[i] = ctx.scratch[0];
  }
  exchange_z_to_y(s, zsrc, ydst, c);
  // forward axis d-1 with the spectral epilogue, backward axis d-1 (y-slab)
  for (size_t i = 0; i < s.parts.size(); ++i) {
    SlabPart& pt = s.parts[i];
    part_device(pt);
    kronop_ctx& ctx = *pt.ctx;
    int shp[KRONOP_MAX_DIM];
    for (int a = 0; a < d - 2; ++a) shp[a] = s.n[a];
    shp[d - 2] = s.ys[pt.p];
    shp[d - 1] = s.n[d - 1];
    View v = make_view(d, shp, cplx);
    EpiParams ep;
    ep.kind = e.kind;
    ep.axis = d - 1 + v.cplx;
    ep.ndims = v.nd;
    for (int k = 0; k < v.nd; ++k) ep.ext[k] = v.ext[k];
    for (int a = 0; a < d; ++a) ep.lam[a + v.cplx] = pt.lam[a];
    ep.lam[d - 2 + v.cplx] = pt.lam[d - 2] + s.y0[pt.p];  // this part's rows of axis d-2
    ep.shift = e.shift;
    ep.dt = e.dt;
    ep.cplx = v.cplx;
    ep.active = e.active ? e.active[i] : nullptr;
    run_pass(ctx, ctx.scratch[0], ctx.scratch[1], v, d - 1 + v.cplx, pt.fwd[d - 1], pt.lda[d - 1],
             s.n[d - 1], ep);
    EpiParams st;
    st.active = ep.active;
    run_pass(ctx, ctx.scratch[1], ctx.scratch[0], v, d - 1 + v.cplx, pt.bwd[d - 1], pt.lda[d - 1],
             s.n[d - 1], st);
    ysrc[i] = ctx.scratch[0];
    zdst[i] = pt.zx;
  }
  exchange_y_to_z(s, ysrc, zdst, c);
  // backward passes on axes 0..d-2, the last with the FullOperator AXPY epilogue
  for (size_t i = 0; i < s.parts.size(); ++i) {
    SlabPart& pt = s.parts[i];
    part_device(pt);
    kronop_ctx& ctx = *pt.ctx;
    int shp[KRONOP_MAX_DIM];
    for (int a = 0; a < d - 1; ++a) shp[a] = s.n[a];
    shp[d - 1] = s.zs[pt.p];
    View v = make_view(d, shp, cplx);
    const double* cur = pt.zx;
    for (int a = 0; a < d - 1; ++a) {
      const bool last = a == d - 2;
      double* dst = last ? out[i] : ctx.scratch[a % 2];
      EpiParams ep;
      ep.active = e.active ? e.active[i] : nullptr;
      const double* dg = e.diag.empty() ? nullptr : e.diag[i];
      if (last && (dg != nullptr || e.sigma != 0.0)) {
        ep.kind = EPI_AXPY_DIAG;
        ep.diag = dg;
        ep.u = in[i];
        ep.sigma = e.sigma;
        ep.cplx = v.cplx;
      }
      run_pass(ctx, cur, dst, v, a + v.cplx, pt.bwd[a], pt.lda[a], s.n[a], ep);
      cur = dst;
    }
  }
}

// ------------------------------------------------------------------------- scalars --
// Every local part computes `k` local partial sums into its ring slot (fill(part, slot_ptr)),
// then all parts receive sum_p partial_p[j] (part order) into dst[part] (device, k doubles).
template <class Fill>
static void slab_allgather_sum(kronop_slab& s, int k, Fill fill, const std::vector<double*>& dst) {
  const int slot = s.ring;
  s.ring = (s.ring + 1) % kSlabRing;
  for (size_t i = 0; i < s.parts.size(); ++i) {
    part_device(s.parts[i]);
    fill(i, s.parts[i].red + slot * kSlabSlots);
  }
  if (!s.nccl) {
    barrier_a(s);
    for (size_t i = 0; i < s.parts.size(); ++i) {
      SlabPart& pt = s.parts[i];
      part_device(pt);
      k_gather_sum<<<1, 32, 0, pt.ctx->stream>>>(pt.srcs_ring[slot], s.P, k, dst[i]);
      KCUDA(cudaGetLastError());
      pt.ctx->ws.launches += 1;
    }
    return;
  }
  SlabPart& me = s.parts[0];
  KNCCL(g_nccl.AllGather(me.red + slot * kSlabSlots, me.gathered + slot * s.P * kSlabSlots,
                         kSlabSlots, ncclDouble, s.comm, me.ctx->stream));
  k_gather_sum<<<1, 32, 0, me.ctx->stream>>>(me.srcs_ring[slot], s.P, k, dst[0]);
  KCUDA(cudaGetLastError());
  me.ctx->ws.launches += 1;
}

static IndexGeomHost slab_geom(const kronop_slab& s, const SlabPart& pt) {
  IndexGeomHost g;
  g.d = s.d;
  for (int a = 0; a < s.d; ++a) {
    g.n[a] = a == s.d - 1 ? s.zs[pt.p] : s.n[a];
    g.mass[a] = pt.mass[a];
  }
  g.mass[s.d - 1] = pt.mass[s.d - 1] ? pt.mass[s.d - 1] + s.z0[pt.p] : nullptr;
  return g;
}

// global (optionally mass-weighted) dots of pairs (a_j, b_j), j < k, into dst[part][j]
static void slab_dots(kronop_slab& s, int k, const std::vector<const double*>* a,
                      const std::vector<const double*>* b, bool weighted,
                      const std::vector<double*>& dst) {
  slab_allgather_sum(
      s, k,
      [&](size_t i, double* red) {
        SlabPart& pt = s.parts[i];
        const IndexGeomHost g = slab_geom(s, pt);
        for (int j = 0; j < k; ++j)
          launch_dot(pt.ctx->stream, pt.ctx->ws, a[j][i], b[j][i], zslab_elems(s, pt.p), 0,
                     weighted ? &g : nullptr, red + j);
      },
      dst);
}

static std::vector<double> read_part0(kronop_slab& s, const double* dev, int k) {
  std::vector<double> h(k);
  SlabPart& pt = s.parts[0];
  part_device(pt);
  KCUDA(cudaMemcpyAsync(h.data(), dev, k * sizeof(double), cudaMemcpyDeviceToHost,
                        pt.ctx->stream));
  KCUDA(cudaStreamSynchronize(pt.ctx->stream));
  return h;
}

static void slab_sync(kronop_slab& s) {
  for (auto& pt : s.parts) {
    part_device(pt);
    KCUDA(cudaStreamSynchronize(pt.ctx->stream));
  }
}

static void check_slab_shift(kronop_slab& s, double shift) {
  kronop_op tmp;  // lambda-only view for the gap check of operators.cpp:44-52
  tmp.d = s.d;
  tmp.N = s.N;
  for (int a = 0; a < s.d; ++a) {
    tmp.n[a] = s.n[a];
    tmp.lam[a] = s.parts[0].lam[a];
  }
  tmp.lmin = s.lmin;
  tmp.lmax = s.lmax;
  part_device(s.parts[0]);
  check_solve_shift(*s.parts[0].ctx, tmp, shift);
}

// ----------------------------------------------------------------------------- PCG --
struct SlabVecs {  // one device vector per local part, from that part's pool
  kronop_slab* s = nullptr;
  std::vector<double*> v;
  SlabVecs(kronop_slab& sl, int c = 1) : s(&sl) {
    for (auto& pt : sl.parts) {
      part_device(pt);
      v.push_back(pool_get(*pt.ctx, static_cast<size_t>(std::max(zslab_elems(sl, pt.p), 1LL)) * c));
    }
  }
  ~SlabVecs() {
    for (size_t i = 0; i < v.size(); ++i) {
      cudaSetDevice(s->parts[i].ctx->device);
      pool_put(*s->parts[i].ctx, v[i]);
    }
  }
  std::vector<const double*> c() const { return {v.begin(), v.end()}; }
  SlabVecs(const SlabVecs&) = delete;
  SlabVecs& operator=(const SlabVecs&) = delete;
};

static std::vector<double*> offset(const std::vector<double*>& base, int k) {
  std::vector<double*> o(base.size());
  for (size_t i = 0; i < base.size(); ++i) o[i] = base[i] + k;
  return o;
}

// pcg.cpp:8-81 with apply_a = FullOperator{slab(shift), diag}.apply - sigma, precond =
// slab.solve (shift p_shift). x in/out. History (optional) of max_iter + 1 doubles.
static void slab_pcg_run(kronop_slab& s, const std::vector<const double*>& diag, double sigma,
                         double p_shift, const std::vector<const double*>& b,
                         const std::vector<double*>& x, const kronop_pcg_config& cfg,
                         kronop_pcg_report& rep, double* history_host) {
  param_check(cfg.rel_tol > 0.0, "pcg: rel_tol must be positive");
  param_check(cfg.max_iter >= 1, "pcg: max_iter must be >= 1");
  const size_t L = s.parts.size();
  rep = kronop_pcg_report{};
  // per part: PcgScalars at scal + 0, slots at scal + 64.., history buffer
  std::vector<double*> scal(L), hist(L);
  std::vector<std::unique_ptr<DBuf>> hold;
  for (size_t i = 0; i < L; ++i) {
    part_device(s.parts[i]);
    hold.emplace_back(new DBuf(*s.parts[i].ctx, 128));
    scal[i] = hold.back()->p;
    hold.emplace_back(new DBuf(*s.parts[i].ctx, static_cast<size_t>(cfg.max_iter) + 2));
    hist[i] = hold.back()->p;
  }
  auto sc = [&](size_t i) { return reinterpret_cast<PcgScalars*>(scal[i]); };
  std::vector<double*> slot0 = offset(scal, 64);
  SlabVecs r(s), z(s), p(s), q(s), best(s);
  auto bvec = b;
  std::vector<const double*> xc(x.begin(), x.end());
  // ||b||, ||x0|| (pcg.cpp:15-26)
  {
    std::vector<const double*> aa[2] = {bvec, xc};
    slab_dots(s, 2, aa, aa, false, slot0);
  }
  const std::vector<double> nb = read_part0(s, slot0[0], 2);
  const double norm_b = std::sqrt(nb[0]);
  if (norm_b == 0.0) {
    for (size_t i = 0; i < L; ++i) {
      part_device(s.parts[i]);
      KCUDA(cudaMemsetAsync(x[i], 0, zslab_elems(s, s.parts[i].p) * sizeof(double),
                            s.parts[i].ctx->stream));
    }
    slab_sync(s);
    rep.converged = 1;
    return;
  }
  SlabEpi eA;
  eA.kind = EPI_SPEC_MUL;
  eA.shift = s.shift;
  eA.diag = diag;
  eA.sigma = sigma;
  SlabEpi eM;
  eM.kind = EPI_SPEC_DIV;
  eM.shift = p_shift;
  if (std::sqrt(nb[1]) != 0.0) {  // r = b - A x
    slab_transform(s, xc, q.v, 0, eA);
    for (size_t i = 0; i < L; ++i) {
      part_device(s.parts[i]);
      launch_sub(s.parts[i].ctx->stream, s.parts[i].ctx->ws, r.v[i], b[i], q.v[i],
                 zslab_elems(s, s.parts[i].p));
    }
  } else {
    for (size_t i = 0; i < L; ++i) {
      part_device(s.parts[i]);
      KCUDA(cudaMemcpyAsync(r.v[i], b[i], zslab_elems(s, s.parts[i].p) * sizeof(double),
                            cudaMemcpyDeviceToDevice, s.parts[i].ctx->stream));
    }
  }
  slab_transform(s, r.c(), z.v, 0, eM);  // z = M r
  for (size_t i = 0; i < L; ++i) {
    part_device(s.parts[i]);
    const long long ne = zslab_elems(s, s.parts[i].p);
    cudaStream_t st = s.parts[i].ctx->stream;
    KCUDA(cudaMemcpyAsync(p.v[i], z.v[i], ne * sizeof(double), cudaMemcpyDeviceToDevice, st));
    KCUDA(cudaMemcpyAsync(best.v[i], x[i], ne * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  {
    std::vector<const double*> aa[2] = {r.c(), r.c()}, bb[2] = {z.c(), r.c()};
    slab_dots(s, 2, aa, bb, false, offset(scal, 66));  // [r.z, r.r]
  }
  PcgScalars init{};
  init.rel_tol = cfg.rel_tol;
  init.max_iter = cfg.max_iter;
  init.stagnation_window = cfg.stagnation_window;
  init.preconditioned_norm = cfg.preconditioned_norm;
  init.record_history = history_host != nullptr || cfg.record_history;
  for (size_t i = 0; i < L; ++i) {
    part_device(s.parts[i]);
    cudaStream_t st = s.parts[i].ctx->stream;
    KCUDA(cudaMemcpyAsync(sc(i), &init, sizeof(init), cudaMemcpyHostToDevice, st));
    launch_pcg_init(st, s.parts[i].ctx->ws, sc(i), scal[i] + 66, scal[i] + 67, norm_b, hist[i]);
  }
  slab_sync(s);  // `init` is a host stack struct
  std::vector<const int*> act(L);
  for (size_t i = 0; i < L; ++i) act[i] = &sc(i)->active;
  eA.active = act.data();
  eM.active = act.data();
  // host-enqueued loop with a one-iteration lookahead on the device-side `active` flag
  int* hflag = nullptr;
  KCUDA(cudaHostAlloc(&hflag, 2 * sizeof(int), cudaHostAllocDefault));
  cudaEvent_t evf[2];
  part_device(s.parts[0]);
  for (auto& e : evf) KCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct Cleanup {
    int* h;
    cudaEvent_t* e;
    ~Cleanup() {
      cudaFreeHost(h);
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } cleanup{hflag, evf};
  PcgScalars first{};
  part_device(s.parts[0]);
  KCUDA(cudaMemcpy(&first, sc(0), sizeof(first), cudaMemcpyDeviceToHost));
  const unsigned long long launches0 = s.parts[0].ctx->ws.launches;
  int enqueued = 0;
  if (first.active) {
    for (int it = 0; it < cfg.max_iter; ++it) {
      slab_transform(s, p.c(), q.v, 0, eA);  // q = A p
      {
        std::vector<const double*> aa[1] = {p.c()}, bb[1] = {q.c()};
        slab_dots(s, 1, aa, bb, false, offset(scal, 72));  // p.q
      }
      for (size_t i = 0; i < L; ++i) {
        part_device(s.parts[i]);
        cudaStream_t st = s.parts[i].ctx->stream;
        Workspace& ws = s.parts[i].ctx->ws;
        k_pcg_take<<<1, 1, 0, st>>>(sc(i), scal[i] + 72, 0);
        ws.launches += 1;
        launch_pcg_alpha(st, ws, sc(i));
        // x += alpha p ; r -= alpha q ; local r.r (all-gathered with r.z below)
        launch_pcg_update_xr(st, ws, x[i], r.v[i], p.v[i], q.v[i], sc(i),
                             zslab_elems(s, s.parts[i].p), scal[i] + 74);
      }
      slab_transform(s, r.c(), z.v, 0, eM);  // z = M r
      slab_allgather_sum(
          s, 2,
          [&](size_t i, double* red) {
            SlabPart& pt = s.parts[i];
            k_copy_scalar<<<1, 1, 0, pt.ctx->stream>>>(red, scal[i] + 74);
            pt.ctx->ws.launches += 1;
            launch_dot(pt.ctx->stream, pt.ctx->ws, r.v[i], z.v[i], zslab_elems(s, pt.p), 0,
                       nullptr, red + 1);
          },
          offset(scal, 72));  // [r.r, r.z]
      for (size_t i = 0; i < L; ++i) {
        part_device(s.parts[i]);
        cudaStream_t st = s.parts[i].ctx->stream;
        Workspace& ws = s.parts[i].ctx->ws;
        const long long ne = zslab_elems(s, s.parts[i].p);
        k_pcg_take<<<1, 1, 0, st>>>(sc(i), scal[i] + 72, 1);
        ws.launches += 1;
        launch_pcg_beta(st, ws, sc(i));
        launch_pcg_update_p(st, ws, p.v[i], z.v[i], sc(i), ne);
        launch_pcg_finish(st, ws, sc(i), hist[i]);
        launch_copy_if(st, ws, best.v[i], x[i], ne, &sc(i)->improved);
      }
      ++enqueued;
      part_device(s.parts[0]);
      cudaStream_t st0 = s.parts[0].ctx->stream;
      KCUDA(cudaMemcpyAsync(hflag + (it & 1), &sc(0)->active, sizeof(int), cudaMemcpyDeviceToHost,
                            st0));
      KCUDA(cudaEventRecord(evf[it & 1], st0));
      if (it >= 1) {
        KCUDA(cudaEventSynchronize(evf[(it - 1) & 1]));
        if (!hflag[(it - 1) & 1]) break;  // iteration `it` was speculative (gated no-ops)
      }
    }
  }
  slab_sync(s);
  (void)launches0;
  (void)enqueued;
  PcgScalars fin{};
  part_device(s.parts[0]);
  KCUDA(cudaMemcpy(&fin, sc(0), sizeof(fin), cudaMemcpyDeviceToHost));
  if (fin.breakdown)
    fail(KRONOP_ENUMERICAL,
         "pcg: indefinite direction at iteration " + std::to_string(fin.iterations + 1));
  double rel = fin.rel;
  if (rel <= cfg.rel_tol) {  // pcg.cpp:73-79
    rep.converged = 1;
  } else if (fin.best_rel < rel) {
    for (size_t i = 0; i < L; ++i) {
      part_device(s.parts[i]);
      KCUDA(cudaMemcpyAsync(x[i], best.v[i], zslab_elems(s, s.parts[i].p) * sizeof(double),
                            cudaMemcpyDeviceToDevice, s.parts[i].ctx->stream));
    }
    rel = fin.best_rel;
  }
  rep.iterations = fin.iterations;
  rep.final_residual = rel;
  rep.history_len = fin.record_history ? fin.history_len : 0;
  if (history_host && rep.history_len > 0) {
    part_device(s.parts[0]);
    KCUDA(cudaMemcpy(history_host, hist[0], rep.history_len * sizeof(double),
                     cudaMemcpyDeviceToHost));
  }
  slab_sync(s);
}

// global (optionally mass-weighted) dots read back to the host
static std::vector<double> slab_dots_host(kronop_slab& s, int k, const std::vector<const double*>* a,
                                          const std::vector<const double*>* b, bool weighted,
                                          const std::vector<double*>& slots) {
  slab_dots(s, k, a, b, weighted, slots);
  return read_part0(s, slots[0], k);
}

// E(u) = 1/2 <u, H u>_M + beta/4 sum m u^4 (gpe.cpp:10-18); hu, sq scratch vectors
static double slab_gpe_energy(kronop_slab& s, const std::vector<const double*>& v2, double beta,
                              const std::vector<const double*>& u, SlabVecs& hu, SlabVecs& sq,
                              const std::vector<double*>& slots) {
  SlabEpi e;
  e.kind = EPI_SPEC_MUL;
  e.shift = s.shift;
  e.diag = v2;
  slab_transform(s, u, hu.v, 0, e);
  for (size_t i = 0; i < s.parts.size(); ++i) {
    part_device(s.parts[i]);
    launch_square2(s.parts[i].ctx->stream, s.parts[i].ctx->ws, sq.v[i], u[i],
                   zslab_elems(s, s.parts[i].p));
  }
  std::vector<const double*> aa[2] = {u, sq.c()}, bb[2] = {hu.c(), sq.c()};
  const std::vector<double> r = slab_dots_host(s, 2, aa, bb, true, slots);
  return 0.5 * r[0] + 0.25 * beta * r[1];
}

}  // namespace kronop_dev

// ============================================================================== C-ABI ==
extern "C" {

int kronop_slab_plan(int n, int parts, int* extents, int* offsets_out) {
  return guard_slab([&] {
    param_check(n >= 1 && parts >= 1 && parts <= n, "slab_plan: need 1 <= parts <= n");
    std::vector<int> e, o;
    split_extent(n, parts, e, o);
    std::copy(e.begin(), e.end(), extents);
    if (offsets_out) std::copy(o.begin(), o.end(), offsets_out);
  });
}

int kronop_nccl_load(const char* path) {
  return guard_slab([&] { nccl_load(path); });
}

int kronop_nccl_unique_id(unsigned char* id) {
  return guard_slab([&] {
    nccl_load(nullptr);
    ncclUniqueId u;
    KNCCL(g_nccl.GetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  });
}

static void slab_init_common(kronop_slab* s, int nparts, int d, const int* n,
                             const double* const* T, const double* const* Tinv,
                             const double* const* lambda, const double* const* mass, double shift) {
  param_check(n && T && Tinv && lambda, "slab: null argument");
  param_check(d >= 2 && d <= KRONOP_MAX_DIM, "slab: need 2 <= d <= 9 (slabs of the slowest axis)");
  s->d = d;
  s->P = nparts;
  s->N = 1;
  s->shift = shift;
  s->has_mass = mass != nullptr;
  double lmin = 0.0, lmax = 0.0;
  for (int a = 0; a < d; ++a) {
    param_check(n[a] >= 1 && T[a] && Tinv[a] && lambda[a], "slab: bad axis");
    s->n[a] = n[a];
    s->N *= n[a];
    lmin += *std::min_element(lambda[a], lambda[a] + n[a]);
    lmax += *std::max_element(lambda[a], lambda[a] + n[a]);
  }
  s->lmin = lmin;
  s->lmax = lmax;
  for (int a = 0; a < d - 2; ++a) s->R *= n[a];
  param_check(nparts >= 1 && nparts <= n[d - 1] && nparts <= n[d - 2],
              "slab: more parts than planes of the two slowest axes");
  split_extent(n[d - 1], nparts, s->zs, s->z0);
  split_extent(n[d - 2], nparts, s->ys, s->y0);
}

// matrices, eigenvalues, mass vectors and reduction buffers of one local part (on its device)
static void slab_init_part(kronop_slab* s, SlabPart& pt, const double* const* T,
                           const double* const* Tinv, const double* const* lambda,
                           const double* const* mass) {
  part_device(pt);
  for (int a = 0; a < s->d; ++a) {
    // reuse the transforms of an identical earlier axis (isotropic grids)
    int same = -1;
    const size_t nn = static_cast<size_t>(s->n[a]) * s->n[a];
    for (int b = 0; b < a && same < 0; ++b)
      if (s->n[b] == s->n[a] && !std::memcmp(T[a], T[b], nn * sizeof(double)) &&
          !std::memcmp(Tinv[a], Tinv[b], nn * sizeof(double)))
        same = b;
    if (same >= 0) {
      pt.fwd[a] = pt.fwd[same];
      pt.bwd[a] = pt.bwd[same];
      pt.lda[a] = pt.lda[same];
    } else {
      const int lda = pad_up(s->n[a], kMatPadM), kp = pad_up(s->n[a], kMatPadK);
      for (int dir = 0; dir < 2; ++dir) {
        const double* h = dir ? T[a] : Tinv[a];
        std::vector<double> hp(static_cast<size_t>(lda) * kp, 0.0);
        for (int j = 0; j < s->n[a]; ++j)
          std::memcpy(&hp[static_cast<size_t>(lda) * j], h + static_cast<size_t>(s->n[a]) * j,
                      sizeof(double) * s->n[a]);
        double*& dst = dir ? pt.bwd[a] : pt.fwd[a];
        KCUDA(cudaMalloc(&dst, hp.size() * sizeof(double)));
        KCUDA(cudaMemcpy(dst, hp.data(), hp.size() * sizeof(double), cudaMemcpyHostToDevice));
      }
      pt.lda[a] = lda;
    }
    KCUDA(cudaMalloc(&pt.lam[a], s->n[a] * sizeof(double)));
    KCUDA(cudaMemcpy(pt.lam[a], lambda[a], s->n[a] * sizeof(double), cudaMemcpyHostToDevice));
    if (mass) {
      param_check(mass[a] != nullptr, "slab: mass vector missing");
      KCUDA(cudaMalloc(&pt.mass[a], s->n[a] * sizeof(double)));
      KCUDA(cudaMemcpy(pt.mass[a], mass[a], s->n[a] * sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  KCUDA(cudaMalloc(&pt.red, kSlabRing * kSlabSlots * sizeof(double)));
  KCUDA(cudaMemset(pt.red, 0, kSlabRing * kSlabSlots * sizeof(double)));
  if (s->nccl) {
    KCUDA(cudaMalloc(&pt.gathered, static_cast<size_t>(kSlabRing) * s->P * kSlabSlots * sizeof(double)));
  }
  KCUDA(cudaEventCreateWithFlags(&pt.ev_a, cudaEventDisableTiming));
  KCUDA(cudaEventCreateWithFlags(&pt.ev_b, cudaEventDisableTiming));
}

// per ring slot, the device array of the P partial-sum sources this part adds up
static void slab_init_sources(kronop_slab* s) {
  for (auto& pt : s->parts) {
    part_device(pt);
    for (int slot = 0; slot < kSlabRing; ++slot) {
      std::vector<const double*> src(s->P);
      for (int q = 0; q < s->P; ++q)
        src[q] = s->nccl ? pt.gathered + (static_cast<size_t>(slot) * s->P + q) * kSlabSlots
                         : s->parts[q].red + slot * kSlabSlots;
      const double** dev = nullptr;
      KCUDA(cudaMalloc(&dev, s->P * sizeof(double*)));
      KCUDA(cudaMemcpy(dev, src.data(), s->P * sizeof(double*), cudaMemcpyHostToDevice));
      pt.srcs_ring.push_back(dev);
    }
  }
}

int kronop_slab_destroy(kronop_slab* s);

int kronop_slab_create(int nparts, const int* devices, int d, const int* n,
                       const double* const* T, const double* const* Tinv,
                       const double* const* lambda, const double* const* mass, double shift,
                       kronop_slab** out) {
  return guard_slab([&] {
    param_check(devices && out, "slab_create: null argument");
    auto* s = new kronop_slab();
    try {
      slab_init_common(s, nparts, d, n, T, Tinv, lambda, mass, shift);
      s->parts.resize(nparts);
      for (int p = 0; p < nparts; ++p) {
        SlabPart& pt = s->parts[p];
        pt.p = p;
        const int rc = kronop_ctx_create(devices[p], nullptr, &pt.ctx);
        if (rc != KRONOP_OK) fail(rc, kronop_last_error());
        pt.own_ctx = true;
      }
      // peer access between the distinct devices (NVLink / NVSwitch P2P)
      for (int p = 0; p < nparts; ++p)
        for (int q = 0; q < nparts; ++q) {
          const int dp = devices[p], dq = devices[q];
          if (dp == dq) continue;
          int ok = 0;
          KCUDA(cudaDeviceCanAccessPeer(&ok, dp, dq));
          if (!ok) fail(KRONOP_ECAPABILITY, "slab_create: no peer access between devices");
          KCUDA(cudaSetDevice(dp));
          const cudaError_t e = cudaDeviceEnablePeerAccess(dq, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) KCUDA(e);
          (void)cudaGetLastError();
          // the exchange reads / writes the parts' stream-ordered scratch (device dq's pool)
          cudaMemPool_t pool;
          KCUDA(cudaDeviceGetDefaultMemPool(&pool, dq));
          cudaMemAccessDesc acc{};
          acc.location.type = cudaMemLocationTypeDevice;
          acc.location.id = dp;
          acc.flags = cudaMemAccessFlagsProtReadWrite;
          KCUDA(cudaMemPoolSetAccess(pool, &acc, 1));
        }
      for (auto& pt : s->parts) slab_init_part(s, pt, T, Tinv, lambda, mass);
      slab_init_sources(s);
    } catch (...) {
      kronop_slab_destroy(s);
      throw;
    }
    *out = s;
  });
}

int kronop_slab_create_nccl(kronop_ctx* ctx, const unsigned char* unique_id, int nranks, int rank,
                            int d, const int* n, const double* const* T,
                            const double* const* Tinv, const double* const* lambda,
                            const double* const* mass, double shift, kronop_slab** out) {
  return guard_slab([&] {
    param_check(ctx && unique_id && out, "slab_create_nccl: null argument");
    param_check(rank >= 0 && rank < nranks, "slab_create_nccl: bad rank");
    nccl_load(nullptr);
    auto* s = new kronop_slab();
    try {
      s->nccl = true;
      slab_init_common(s, nranks, d, n, T, Tinv, lambda, mass, shift);
      s->parts.resize(1);
      s->parts[0].p = rank;
      s->parts[0].ctx = ctx;
      KCUDA(cudaSetDevice(ctx->device));
      ncclUniqueId id;
      std::memcpy(&id, unique_id, sizeof(id));
      KNCCL(g_nccl.CommInitRank(&s->comm, nranks, id, rank));
      slab_init_part(s, s->parts[0], T, Tinv, lambda, mass);
      slab_init_sources(s);
    } catch (...) {
      kronop_slab_destroy(s);
      throw;
    }
    *out = s;
  });
}

int kronop_slab_destroy(kronop_slab* s) {
  if (!s) return KRONOP_OK;
  for (auto& pt : s->parts) {
    if (!pt.ctx) continue;
    cudaSetDevice(pt.ctx->device);
    cudaStreamSynchronize(pt.ctx->stream);
    for (int a = 0; a < s->d; ++a) {
      bool shared = false;
      for (int b = 0; b < a; ++b) shared = shared || pt.fwd[b] == pt.fwd[a];
      if (!shared) {
        cudaFree(pt.fwd[a]);
        cudaFree(pt.bwd[a]);
      }
      cudaFree(pt.lam[a]);
      cudaFree(pt.mass[a]);
    }
    cudaFree(pt.zx);
    cudaFree(pt.yx);
    cudaFree(pt.red);
    cudaFree(pt.gathered);
    for (auto* p : pt.srcs_ring) cudaFree(p);
    if (pt.ev_a) cudaEventDestroy(pt.ev_a);
    if (pt.ev_b) cudaEventDestroy(pt.ev_b);
    if (pt.own_ctx) kronop_ctx_destroy(pt.ctx);
  }
  for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
  if (s->bar) cudaFree(s->bar);
  if (s->comm) g_nccl.CommDestroy(s->comm);
  delete s;
  return KRONOP_OK;
}

int kronop_slab_info(const kronop_slab* s, int* nparts, int* nlocal, int* first_part) {
  return guard_slab([&] {
    param_check(s, "slab_info: null slab");
    if (nparts) *nparts = s->P;
    if (nlocal) *nlocal = static_cast<int>(s->parts.size());
    if (first_part) *first_part = s->parts.empty() ? 0 : s->parts[0].p;
  });
}

int kronop_slab_stats(const kronop_slab* s, long long* fused_transforms) {
  return guard_slab([&] {
    param_check(s, "slab_stats: null slab");
    if (fused_transforms) *fused_transforms = s->fused_transforms;
  });
}

int kronop_slab_part(const kronop_slab* s, int local, int* device, void** stream,
                     long long* z0, long long* nz, long long* elems) {
  return guard_slab([&] {
    param_check(s && local >= 0 && local < static_cast<int>(s->parts.size()),
                "slab_part: bad local part index");
    const SlabPart& pt = s->parts[local];
    if (device) *device = pt.ctx->device;
    if (stream) *stream = pt.ctx->stream;
    if (z0) *z0 = s->z0[pt.p];
    if (nz) *nz = s->zs[pt.p];
    if (elems) *elems = zslab_elems(*s, pt.p);
  });
}

int kronop_slab_field_alloc(kronop_slab* s, int local, size_t doubles, double** out) {
  return guard_slab([&] {
    param_check(s && out && local >= 0 && local < static_cast<int>(s->parts.size()),
                "slab_field_alloc: bad argument");
    part_device(s->parts[local]);
    KCUDA(cudaMalloc(out, std::max<size_t>(doubles, 1) * sizeof(double)));
  });
}

int kronop_slab_field_free(kronop_slab* s, int local, double* p) {
  return guard_slab([&] {
    param_check(s && local >= 0 && local < static_cast<int>(s->parts.size()),
                "slab_field_free: bad argument");
    part_device(s->parts[local]);
    KCUDA(cudaFree(p));
  });
}

// host = the FULL field (all planes, axis 0 fastest); each local part gets / gives its planes
int kronop_slab_scatter(kronop_slab* s, const double* host, int is_complex, double* const* parts) {
  return guard_slab([&] {
    param_check(s && host && parts, "slab_scatter: null argument");
    const long long c = is_complex ? 2 : 1;
    for (size_t i = 0; i < s->parts.size(); ++i) {
      SlabPart& pt = s->parts[i];
      part_device(pt);
      const long long plane = zslab_elems(*s, pt.p) / std::max(1, s->zs[pt.p]);
      KCUDA(cudaMemcpyAsync(parts[i], host + c * plane * s->z0[pt.p],
                            c * zslab_elems(*s, pt.p) * sizeof(double), cudaMemcpyHostToDevice,
                            pt.ctx->stream));
    }
    slab_sync(*s);
  });
}

int kronop_slab_gather(kronop_slab* s, const double* const* parts, int is_complex, double* host) {
  return guard_slab([&] {
    param_check(s && host && parts, "slab_gather: null argument");
    const long long c = is_complex ? 2 : 1;
    for (size_t i = 0; i < s->parts.size(); ++i) {
      SlabPart& pt = s->parts[i];
      part_device(pt);
      const long long plane = zslab_elems(*s, pt.p) / std::max(1, s->zs[pt.p]);
      KCUDA(cudaMemcpyAsync(host + c * plane * s->z0[pt.p], parts[i],
                            c * zslab_elems(*s, pt.p) * sizeof(double), cudaMemcpyDeviceToHost,
                            pt.ctx->stream));
    }
    slab_sync(*s);
  });
}

int kronop_slab_set_shift(kronop_slab* s, double shift) {
  return guard_slab([&] {
    param_check(s, "slab_set_shift: null slab");
    s->shift = shift;
  });
}

int kronop_slab_synchronize(kronop_slab* s) {
  return guard_slab([&] { slab_sync(*s); });
}

static std::vector<const double*> cvec(const kronop_slab* s, const double* const* p) {
  return std::vector<const double*>(p, p + s->parts.size());
}
static std::vector<double*> mvec(const kronop_slab* s, double* const* p) {
  return std::vector<double*>(p, p + s->parts.size());
}

int kronop_slab_apply(kronop_slab* s, const double* const* u, int is_complex,
                      const double* const* diag, double sigma, double* const* out) {
  return guard_slab([&] {
    param_check(s && u && out, "slab_apply: null argument");
    SlabEpi e;
    e.kind = EPI_SPEC_MUL;
    e.shift = s->shift;
    if (diag) e.diag = cvec(s, diag);
    e.sigma = sigma;
    slab_transform(*s, cvec(s, u), mvec(s, out), is_complex, e);
  });
}

int kronop_slab_solve(kronop_slab* s, const double* const* b, int is_complex, double* const* out) {
  return guard_slab([&] {
    param_check(s && b && out, "slab_solve: null argument");
    check_slab_shift(*s, s->shift);
    SlabEpi e;
    e.kind = EPI_SPEC_DIV;
    e.shift = s->shift;
    slab_transform(*s, cvec(s, b), mvec(s, out), is_complex, e);
  });
}

int kronop_slab_propagate(kronop_slab* s, const double* const* psi, double dt,
                          double* const* out) {
  return guard_slab([&] {
    param_check(s && psi && out, "slab_propagate: null argument");
    if (dt == 0.0) {  // operators.cpp:64
      for (size_t i = 0; i < s->parts.size(); ++i) {
        part_device(s->parts[i]);
        KCUDA(cudaMemcpyAsync(out[i], psi[i], 2 * zslab_elems(*s, s->parts[i].p) * sizeof(double),
                              cudaMemcpyDeviceToDevice, s->parts[i].ctx->stream));
      }
      return;
    }
    SlabEpi e;
    e.kind = EPI_SPEC_PHASE;
    e.shift = s->shift;
    e.dt = dt;
    slab_transform(*s, cvec(s, psi), mvec(s, out), 1, e);
  });
}

int kronop_slab_dot(kronop_slab* s, const double* const* a, const double* const* b, int weighted,
                    double* result) {
  return guard_slab([&] {
    param_check(s && a && b && result, "slab_dot: null argument");
    param_check(!weighted || s->has_mass, "slab_dot: no mass weights attached");
    std::vector<const double*> aa[1] = {cvec(s, a)}, bb[1] = {cvec(s, b)};
    std::vector<double*> slots;
    std::vector<std::unique_ptr<DBuf>> hold;
    for (auto& pt : s->parts) {
      part_device(pt);
      hold.emplace_back(new DBuf(*pt.ctx, 8));
      slots.push_back(hold.back()->p);
    }
    *result = slab_dots_host(*s, 1, aa, bb, weighted != 0, slots)[0];
  });
}

int kronop_slab_pcg(kronop_slab* s, const double* const* diag, double sigma,
                    const double* const* b, double* const* x, const kronop_pcg_config* cfg,
                    kronop_pcg_report* report, double* history) {
  return guard_slab([&] {
    param_check(s && b && x && cfg && report, "slab_pcg: null argument");
    check_slab_shift(*s, s->shift);
    std::vector<const double*> dg;
    if (diag) dg = cvec(s, diag);
    slab_pcg_run(*s, dg, sigma, s->shift, cvec(s, b), mvec(s, x), *cfg, *report, history);
  });
}

// a_u gradient flow (gpe.cpp:55-165, AdaptiveMetric branch :118-134) on the slab-decomposed
// Hamiltonian H = slab (shift) + V2 (diag, per part or NULL). init CONSTANT or SUPPLIED.
int kronop_slab_gpe_au(kronop_slab* s, const double* const* diag, double beta,
                       const kronop_gpe_config* cfg, const double* const* initial,
                       double* const* state, kronop_gpe_result* result, double* history) {
  return guard_slab([&] {
    param_check(s && cfg && state && result, "slab_gpe_au: null argument");
    param_check(cfg->kind == KRONOP_GPE_AU, "slab_gpe_au: only the a_u (AdaptiveMetric) flow");
    param_check(beta >= 0.0, "gpe_gradient_flow: beta must be >= 0");
    param_check(cfg->step > 0.0, "gpe_gradient_flow: step must be positive");
    param_check(s->has_mass, "gpe_gradient_flow: problem needs mass weights");
    param_check(cfg->init == KRONOP_GPE_INIT_CONSTANT ||
                    (cfg->init == KRONOP_GPE_INIT_SUPPLIED && initial),
                "slab_gpe_au: init must be constant or supplied (with an initial state)");
    kronop_slab& sl = *s;
    const size_t L = sl.parts.size();
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<const double*> v2;
    if (diag) v2 = cvec(s, diag);
    SlabVecs u(sl), w(sl), grad(sl), hu(sl), sq(sl), dg(sl);
    std::vector<double*> slots;
    std::vector<std::unique_ptr<DBuf>> hold;
    for (auto& pt : sl.parts) {
      part_device(pt);
      hold.emplace_back(new DBuf(*pt.ctx, 8));
      slots.push_back(hold.back()->p);
    }
    for (size_t i = 0; i < L; ++i) {
      SlabPart& pt = sl.parts[i];
      part_device(pt);
      const long long ne = zslab_elems(sl, pt.p);
      if (cfg->init == KRONOP_GPE_INIT_SUPPLIED)
        KCUDA(cudaMemcpyAsync(u.v[i], initial[i], ne * sizeof(double), cudaMemcpyDeviceToDevice,
                              pt.ctx->stream));
      else
        launch_fill(pt.ctx->stream, pt.ctx->ws, u.v[i], 1.0, ne);
      KCUDA(cudaMemsetAsync(w.v[i], 0, ne * sizeof(double), pt.ctx->stream));
    }
    auto normalise = [&]() {  // u /= sqrt(<u,u>_M)
      std::vector<const double*> aa[1] = {u.c()};
      slab_dots(sl, 1, aa, aa, true, slots);
      for (size_t i = 0; i < L; ++i) {
        part_device(sl.parts[i]);
        launch_div_by(sl.parts[i].ctx->stream, sl.parts[i].ctx->ws, u.v[i], u.v[i],
                      zslab_elems(sl, sl.parts[i].p), slots[i], 1);
      }
    };
    normalise();
    *result = kronop_gpe_result{};
    double e_old = slab_gpe_energy(sl, v2, beta, u.c(), hu, sq, slots);
    int increases = 0;
    check_slab_shift(sl, sl.shift);
    for (int it = 0; it < cfg->max_iterations; ++it) {
      for (size_t i = 0; i < L; ++i) {  // diag = beta u^2 + V2 (gpe.cpp:120-122)
        part_device(sl.parts[i]);
        launch_beta_square(sl.parts[i].ctx->stream, sl.parts[i].ctx->ws, dg.v[i], u.v[i], beta,
                           v2.empty() ? nullptr : v2[i], zslab_elems(sl, sl.parts[i].p));
      }
      kronop_pcg_report rep;
      slab_pcg_run(sl, dg.c(), 0.0, sl.shift, u.c(), w.v, cfg->inner, rep, nullptr);
      result->linear_solves += rep.iterations;
      std::vector<const double*> aa[2] = {u.c(), w.c()}, bb[2] = {u.c(), u.c()};
      const std::vector<double> pr = slab_dots_host(sl, 2, aa, bb, true, slots);
      const double proj = pr[0] / pr[1];
      for (size_t i = 0; i < L; ++i) {
        SlabPart& pt = sl.parts[i];
        part_device(pt);
        const long long ne = zslab_elems(sl, pt.p);
        launch_sub_scaled(pt.ctx->stream, pt.ctx->ws, grad.v[i], u.v[i], w.v[i], proj, ne);
        launch_sub_scaled(pt.ctx->stream, pt.ctx->ws, u.v[i], u.v[i], grad.v[i], cfg->step, ne);
      }
      normalise();
      const double energy = slab_gpe_energy(sl, v2, beta, u.c(), hu, sq, slots);
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
    // eigenvalue = <u,Hu>_M + beta sum m u^4 (gpe.cpp:159-161); hu, sq hold H u and u^2 of the
    // final state (the last energy evaluation)
    std::vector<const double*> aa[2] = {u.c(), sq.c()}, bb[2] = {hu.c(), sq.c()};
    const std::vector<double> q = slab_dots_host(sl, 2, aa, bb, true, slots);
    result->eigenvalue = q[0] + beta * q[1];
    result->energy = e_old;
    for (size_t i = 0; i < L; ++i) {
      part_device(sl.parts[i]);
      KCUDA(cudaMemcpyAsync(state[i], u.v[i], zslab_elems(sl, sl.parts[i].p) * sizeof(double),
                            cudaMemcpyDeviceToDevice, sl.parts[i].ctx->stream));
    }
    slab_sync(sl);
  });
}

}  // extern "C"
