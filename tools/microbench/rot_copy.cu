// Microbenchmark: HBM bandwidth of the rotating-layout copy (contiguous tile reads of QT planes of
// F complex values, writes of F runs of QT complex values at stride Q) vs QT, i.e. what the output
// run length of a group kernel costs. nvcc -gencode arch=compute_100a,code=sm_100a -O3 rot_copy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int QT, int F, int STAGES>
__global__ void __launch_bounds__(512) rotcopy(const double2* __restrict__ x, double2* __restrict__ y, long long Q, long long ntiles) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ uint64_t bar[STAGES];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long long t, int s) {
    const uint32_t bytes = QT * F * 16;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + s * QT * F)),
                 "l"(x + t * QT * F), "r"(bytes), "r"(smem_u32(&bar[s])) : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) if (blockIdx.x + (long long)s * gridDim.x < ntiles) issue(blockIdx.x + (long long)s * gridDim.x, s);
  for (int it = 0;; ++it) {
    const long long t = blockIdx.x + (long long)it * gridDim.x;
    if (t >= ntiles) break;
    const int s = it % STAGES;
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(smem_u32(&bar[s])), "r"((it / STAGES) & 1) : "memory");
    const double2* tile = sm + s * QT * F;
    const long long q0 = t * QT;
    for (int u = tid; u < QT * F; u += blockDim.x) {
      const int qi = u % QT, g = u / QT;
      y[q0 + qi + Q * g] = tile[g + F * qi];
    }
    __syncthreads();
    if (tid == 0 && t + (long long)STAGES * gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t + (long long)STAGES * gridDim.x, s);
    }
  }
}

template <int QT, int STAGES, int CTAS>
void run(const double2* x, double2* y, long long N) {
  constexpr int F = 729;
  const long long Q = N / F, ntiles = Q / QT;
  const size_t smem = (size_t)STAGES * QT * F * 16;
  cudaFuncSetAttribute(rotcopy<QT, F, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148 * CTAS;
  rotcopy<QT, F, STAGES><<<grid, 512, smem>>>(x, y, Q, ntiles);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) rotcopy<QT, F, STAGES><<<grid, 512, smem>>>(x, y, Q, ntiles);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("QT=%2d stages=%d ctas=%d: %.3f ms  %.0f GB/s (err %s)\n", QT, STAGES, CTAS, ms, 2.0 * N * 16 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}


// Cluster variant: the K CTAs of a cluster hold K consecutive tiles (K*QT consecutive q); after a
// cluster barrier CTA r writes the g range r of all K*QT q from the K CTAs' shared memory (DSMEM),
// i.e. runs of K*QT complex values.
template <int QT, int F, int K, int STAGES>
__global__ void __launch_bounds__(512) rotcopy_cl(const double2* __restrict__ x, double2* __restrict__ y, long long Q, long long nsuper) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ uint64_t bar[STAGES];
  const int tid = threadIdx.x;
  uint32_t r; asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  const long long cid = blockIdx.x / K, ncl = gridDim.x / K;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long long T, int s) {
    const uint32_t bytes = QT * F * 16;
    const long long t = T * K + r;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + s * QT * F)),
                 "l"(x + t * QT * F), "r"(bytes), "r"(smem_u32(&bar[s])) : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) if (cid + (long long)s * ncl < nsuper) issue(cid + (long long)s * ncl, s);
  constexpr int GR = (F + K - 1) / K;  // g per CTA
  for (int it = 0;; ++it) {
    const long long T = cid + (long long)it * ncl;
    if (T >= nsuper) break;
    const int s = it % STAGES;
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(smem_u32(&bar[s])), "r"((it / STAGES) & 1) : "memory");
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t base = smem_u32(sm + s * QT * F);
    const long long q0 = T * K * QT;
    for (int u = tid; u < GR * K * QT; u += blockDim.x) {
      const int qq = u % (K * QT), gl = u / (K * QT);
      const int g = r * GR + gl;
      if (g >= F) continue;
      const int src = qq / QT, qi = qq % QT;
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + (g + F * qi) * 16), "r"(src));
      double2 v;
      asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra));
      y[q0 + qq + Q * g] = v;
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (tid == 0 && T + (long long)STAGES * ncl < nsuper) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(T + (long long)STAGES * ncl, s);
    }
  }
}

template <int QT, int K, int STAGES, int CTAS>
void run_cl(const double2* x, double2* y, long long N) {
  constexpr int F = 729;
  const long long Q = N / F, nsuper = Q / (QT * K);
  const size_t smem = (size_t)STAGES * QT * F * 16;
  auto kern = rotcopy_cl<QT, F, K, STAGES>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 * CTAS / K * K); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = K; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, x, y, Q, nsuper);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int rr = 0; rr < 5; ++rr) cudaLaunchKernelEx(&cfg, kern, x, y, Q, nsuper);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("cluster QT=%d K=%d stages=%d ctas=%d: %.3f ms  %.0f GB/s (err %s)\n", QT, K, STAGES, CTAS, ms, 2.0 * (nsuper * QT * K * F) * 16 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}


// ORDER 1: each CTA walks a contiguous range of tiles; ST 1: streaming stores (st.global.cs),
// ST 2: 2 q per thread (32-byte stores... as two 16-byte stores issued back to back)
template <int QT, int F, int STAGES, int ORDER, int ST>
__global__ void __launch_bounds__(512) rotcopy2(const double2* __restrict__ x, double2* __restrict__ y, long long Q, long long ntiles) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ uint64_t bar[STAGES];
  const int tid = threadIdx.x;
  const long long per = (ntiles + gridDim.x - 1) / gridDim.x;
  auto tile_of = [&](long long it) { return ORDER ? blockIdx.x * per + it : blockIdx.x + it * gridDim.x; };
  auto valid = [&](long long it) { return ORDER ? (it < per && tile_of(it) < ntiles) : tile_of(it) < ntiles; };
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long long t, int s) {
    const uint32_t bytes = QT * F * 16;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + s * QT * F)),
                 "l"(x + t * QT * F), "r"(bytes), "r"(smem_u32(&bar[s])) : "memory");
  };
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) if (valid(s)) issue(tile_of(s), s);
  for (int it = 0;; ++it) {
    if (!valid(it)) break;
    const long long t = tile_of(it);
    const int s = it % STAGES;
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(smem_u32(&bar[s])), "r"((it / STAGES) & 1) : "memory");
    const double2* tile = sm + s * QT * F;
    const long long q0 = t * QT;
    for (int u = tid; u < QT * F; u += blockDim.x) {
      const int qi = u % QT, g = u / QT;
      if (ST == 1) __stcs(&y[q0 + qi + Q * g], tile[g + F * qi]);
      else y[q0 + qi + Q * g] = tile[g + F * qi];
    }
    __syncthreads();
    if (tid == 0 && valid(it + STAGES)) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile_of(it + STAGES), s);
    }
  }
}
template <int QT, int STAGES, int CTAS, int ORDER, int ST>
void run2(const double2* x, double2* y, long long N) {
  constexpr int F = 729;
  const long long Q = N / F, ntiles = Q / QT;
  const size_t smem = (size_t)STAGES * QT * F * 16;
  cudaFuncSetAttribute(rotcopy2<QT, F, STAGES, ORDER, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148 * CTAS;
  rotcopy2<QT, F, STAGES, ORDER, ST><<<grid, 512, smem>>>(x, y, Q, ntiles);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) rotcopy2<QT, F, STAGES, ORDER, ST><<<grid, 512, smem>>>(x, y, Q, ntiles);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("QT=%2d stages=%d ctas=%d order=%d st=%d: %.3f ms  %.0f GB/s (err %s)\n", QT, STAGES, CTAS, ORDER, ST, ms, 2.0 * N * 16 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long long N = 387420489LL;  // 9^9
  double2 *x, *y;
  cudaMalloc(&x, N * 16); cudaMalloc(&y, N * 16);
  cudaMemset(x, 0, N * 16);
  run<2, 2, 4>(x, y, N);
  run<4, 2, 2>(x, y, N);
  run<4, 1, 4>(x, y, N);
  run<8, 2, 1>(x, y, N);
  run<8, 1, 2>(x, y, N);
  run<16, 1, 1>(x, y, N);
  run2<4, 2, 2, 0, 0>(x, y, N);
  run2<4, 2, 2, 1, 0>(x, y, N);
  run2<4, 2, 2, 0, 1>(x, y, N);
  run2<4, 2, 2, 1, 1>(x, y, N);
  run2<8, 2, 1, 1, 0>(x, y, N);
  run2<4, 4, 1, 1, 0>(x, y, N);
  run2<4, 4, 1, 0, 0>(x, y, N);
  // plain copy reference
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) cudaMemcpy(y, x, N * 16, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("cudaMemcpy D2D: %.3f ms %.0f GB/s\n", ms, 2.0 * N * 16 / ms / 1e6);
  return 0;
}
