// Microbenchmark: FP32 FFMA vs packed FFMA2 (fma.rn.f32x2) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_ffma(float* sink, int iters, float b, float c) {
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = threadIdx.x * 1e-7f + k;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = fmaf(v[k], b, c);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += v[k];
  if (s == 1234.5f) sink[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_ffma2(float* sink, int iters, float b, float c) {
  unsigned long long v[8];
  float2 bb = make_float2(b, b), cc = make_float2(c, c);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&bb);
  unsigned long long C = *reinterpret_cast<unsigned long long*>(&cc);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float2 t = make_float2(threadIdx.x * 1e-7f + k, k + 0.5f);
    v[k] = *reinterpret_cast<unsigned long long*>(&t);
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[k]) : "l"(B), "l"(C));
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) { float2 t = *reinterpret_cast<float2*>(&v[k]); s += t.x + t.y; }
  if (s == 1234.5f) sink[blockIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink; cudaMalloc(&sink, 1 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    k_ffma<<<blocks, threads>>>(sink, 16, 0.999f, 1e-6f);
    cudaEventRecord(a); k_ffma<<<blocks, threads>>>(sink, iters, 0.999f, 1e-6f); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * blocks * threads * (double)iters * 8 * 16;
    printf("FFMA : %.1f TFLOP/s\n", fl / ms / 1e9);
    k_ffma2<<<blocks, threads>>>(sink, 16, 0.999f, 1e-6f);
    cudaEventRecord(a); k_ffma2<<<blocks, threads>>>(sink, iters, 0.999f, 1e-6f); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    fl = 2.0 * blocks * threads * (double)iters * 8 * 8 * 2;
    printf("FFMA2: %.1f TFLOP/s\n", fl / ms / 1e9);
  }
  return 0;
}
