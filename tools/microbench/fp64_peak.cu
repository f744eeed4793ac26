// FP64 issue-rate microbenchmark for B200 (sm_100a): DFMA vs the warp-level
// DMMA shapes (mma.sync m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16 .f64).
// Decides which instruction the mode-product kernel is built on.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;

__global__ void k_dfma(double* out, double s) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  double b = s, c = 1.0 - s;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], b, c);
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += acc[i];
  if (t == 12345.0) out[threadIdx.x] = t;
}

template <int K>
__device__ __forceinline__ void mma16(double (&d)[4], const double* a, const double* b);

template <>
__device__ __forceinline__ void mma16<4>(double (&d)[4], const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
template <>
__device__ __forceinline__ void mma16<8>(double (&d)[4], const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
template <>
__device__ __forceinline__ void mma16<16>(double (&d)[4], const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int K, int NACC>
__global__ void k_dmma16(double* out, double s) {
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = s * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = s * (threadIdx.x - i);
  double d[NACC][4];
#pragma unroll
  for (int j = 0; j < NACC; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[j][i] = 0.0;
  const int iters = ITERS * 4 / K;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) mma16<K>(d[j], a, b);
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) t += d[j][i];
  if (t == 12345.0) out[threadIdx.x] = t;
}

template <int NACC>
__global__ void k_dmma884(double* out, double s) {
  double a = s * threadIdx.x, b = s * (threadIdx.x + 1);
  double d[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; ++j) d[j][0] = d[j][1] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) t += d[j][0] + d[j][1];
  if (t == 12345.0) out[threadIdx.x] = t;
}

template <typename F>
int timeit(const char* name, F launch, double flops_per_launch) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) launch();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  printf("%-28s %8.3f ms  %7.2f TFLOP/s\n", name, best, flops_per_launch / (best * 1e-3) / 1e12);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s, %d SMs, clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out;
  CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int sms = p.multiProcessorCount;
  for (int bps : {2, 4, 8}) {
    const int blocks = sms * bps, threads = 256;
    char nm[64];
    snprintf(nm, sizeof nm, "DFMA  blocks/SM=%d", bps);
    timeit(nm, [&] { k_dfma<<<blocks, threads>>>(out, 0.999); },
           2.0 * 16 * ITERS * double(blocks) * threads);
  }
  for (int wps : {4, 8, 12, 16}) {
    // one block per SM with wps warps: DMMA throughput vs resident warps
    const int blocks = sms, threads = 32 * wps;
    const double warps = double(blocks) * wps;
    char nm[64];
    snprintf(nm, sizeof nm, "DMMA m8n8k4 x8 warps/SM=%d", wps);
    timeit(nm, [&] { k_dmma884<8><<<blocks, threads>>>(out, 0.5); }, warps * 8 * ITERS * 2.0 * 8 * 8 * 4);
    snprintf(nm, sizeof nm, "DMMA m8n8k4 x32 warps/SM=%d", wps);
    timeit(nm, [&] { k_dmma884<32><<<blocks, threads>>>(out, 0.5); }, warps * 32 * ITERS * 2.0 * 8 * 8 * 4);
  }
  for (int bps : {2, 4}) {
    const int blocks = sms * bps, threads = 256;
    const double warps = double(blocks) * threads / 32;
    char nm[64];
    snprintf(nm, sizeof nm, "DMMA m8n8k4 x8 bps=%d", bps);
    timeit(nm, [&] { k_dmma884<8><<<blocks, threads>>>(out, 0.5); }, warps * 8 * ITERS * 2.0 * 8 * 8 * 4);
    snprintf(nm, sizeof nm, "DMMA m16n8k4 x8 bps=%d", bps);
    timeit(nm, [&] { k_dmma16<4, 8><<<blocks, threads>>>(out, 0.5); },
           warps * 8 * (ITERS * 4 / 4) * 2.0 * 16 * 8 * 4);
    snprintf(nm, sizeof nm, "DMMA m16n8k8 x8 bps=%d", bps);
    timeit(nm, [&] { k_dmma16<8, 8><<<blocks, threads>>>(out, 0.5); },
           warps * 8 * (ITERS * 4 / 8) * 2.0 * 16 * 8 * 8);
    snprintf(nm, sizeof nm, "DMMA m16n8k16 x8 bps=%d", bps);
    timeit(nm, [&] { k_dmma16<16, 8><<<blocks, threads>>>(out, 0.5); },
           warps * 8 * (ITERS * 4 / 16) * 2.0 * 16 * 8 * 16);
    snprintf(nm, sizeof nm, "DMMA m16n8k16 x4 bps=%d", bps);
    timeit(nm, [&] { k_dmma16<16, 4><<<blocks, threads>>>(out, 0.5); },
           warps * 4 * (ITERS * 4 / 16) * 2.0 * 16 * 8 * 16);
  }
  return 0;
}
