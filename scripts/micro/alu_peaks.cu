// Microbenchmark of the peaks the rooflines in DESIGN.md use (SURVEY 8(d) "missing peaks"):
// FP32 FFMA and FP64 DFMA throughput per SM, and L2 read bandwidth (a 64 MB buffer, L2 126 MB,
// read repeatedly after a warm-up pass).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <class T>
__global__ void k_fma(T* out, int iters) {
  T a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (T)1 + (T)0.001 * (T)(threadIdx.x + i);
  const T m = (T)0.999999, c = (T)0.000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] * m + c;  // 8 independent FMA chains per thread
  }
  T acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += a[i];
  if (acc == (T)12345) out[0] = acc;
}

__global__ void k_l2(const float4* __restrict__ p, size_t n4, float* out, int reps) {
  float s = 0.f;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(p + i);  // cache in L2 only
      s += v.x + v.y + v.z + v.w;
    }
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* outf; double* outd;
  cudaMalloc(&outf, 4); cudaMalloc(&outd, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 8192, threads = 1024, blocks = sms * 2;
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_fma<float><<<blocks, threads>>>(outf, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  double n = (double)blocks * threads * iters * 8;
  printf("FFMA      %.3f ms  %.3e FMA/s  %.1f FMA/clk/SM  (%.1f TFLOP/s; at %d MHz nominal)\n", ms, n / (ms * 1e-3),
         n / (ms * 1e-3) / sms / (clk * 1e3), 2 * n / (ms * 1e-3) / 1e12, clk / 1000);
  const int diters = 1024;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_fma<double><<<blocks, threads>>>(outd, diters); cudaEventRecord(b); cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  n = (double)blocks * threads * diters * 8;
  printf("DFMA      %.3f ms  %.3e FMA/s  %.1f FMA/clk/SM  (%.1f TFLOP/s)\n", ms, n / (ms * 1e-3),
         n / (ms * 1e-3) / sms / (clk * 1e3), 2 * n / (ms * 1e-3) / 1e12);
  const size_t bytes = 64ull << 20, n4 = bytes / 16;
  float4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 0, bytes);
  const int reps = 20;
  k_l2<<<sms * 4, 1024>>>(buf, n4, outf, 1);
  cudaEventRecord(a); k_l2<<<sms * 4, 1024>>>(buf, n4, outf, reps); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("L2 read   %.3f ms  %.1f GB/s  (64 MB buffer x %d, __ldcg)\n", ms, (double)bytes * reps / (ms * 1e-3) / 1e9, reps);
  return 0;
}
