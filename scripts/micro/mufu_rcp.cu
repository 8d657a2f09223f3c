// Microbenchmark: MUFU.RCP (rcp.approx.ftz.f32) throughput per SM on this GPU, and the FMA-pipe
// Newton reciprocal, and a 3:1 mix.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float rcp_approx(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float rcp_nr(float x) {
  float y = __int_as_float(0x7EF311C3 - __float_as_int(x));
  float e = fmaf(-x, y, 1.0f); y = fmaf(y, e, y);
  e = fmaf(-x, y, 1.0f); y = fmaf(y, e, y);
  e = fmaf(-x, y, 1.0f); return fmaf(y, e, y);
}
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0f + 0.001f * (threadIdx.x + i);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float r;
      if (MODE == 0) r = rcp_approx(a[i]);
      else if (MODE == 1) r = rcp_nr(a[i]);
      else r = (i & 3) == 3 ? rcp_nr(a[i]) : rcp_approx(a[i]);
      a[i] = r + 1.0f;  // dependent chain per lane slot, 8 independent chains
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += a[i];
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, 4);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  const char* names[3] = {"MUFU.RCP", "Newton FMA", "3 MUFU : 1 Newton"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
      else if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
      else k<2><<<blocks, threads>>>(out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    double n = (double)blocks * threads * iters * 8;
    double per_s = n / (ms * 1e-3);
    printf("%-20s %.3f ms  %.3e rcp/s  %.2f rcp/clk/SM (at %d MHz nominal)\n", names[mode], ms, per_s,
           per_s / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
