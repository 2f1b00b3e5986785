// ABI plumbing: version, thread-local error text, device query, FFMA probe.
#include <cstring>

#include "common.cuh"

namespace dpm {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

// FP32 FFMA throughput probe: 8 independent chains per thread so each
// SMSP always has an FFMA ready; the result is stored so nothing is elided.
constexpr int PROBE_CHAINS = 8;
constexpr int PROBE_UNROLL = 16;

__global__ void __launch_bounds__(256) ffma_probe_kernel(float* sink, int iters, float b, float c) {
  float v[PROBE_CHAINS];
#pragma unroll
  for (int k = 0; k < PROBE_CHAINS; ++k) v[k] = threadIdx.x * 1e-7f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < PROBE_UNROLL; ++u)
#pragma unroll
      for (int k = 0; k < PROBE_CHAINS; ++k) v[k] = fmaf(v[k], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < PROBE_CHAINS; ++k) s += v[k];
  if (s == 1234.5f) sink[blockIdx.x] = s;  // practically never true
}

}  // namespace dpm

using namespace dpm;

extern "C" int dpm_abi_version(void) { return DPM_ABI_VERSION; }

extern "C" const char* dpm_last_error(void) { return last_error(); }

extern "C" int dpm_device_query(int device, int* sm_count, int* cc_major, int* cc_minor) {
  DPM_REQUIRE(sm_count && cc_major && cc_minor, "dpm_device_query: null output");
  DPM_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  DPM_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  DPM_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return DPM_OK;
}

extern "C" int dpm_ffma_probe(float* sink, int iters, double* flops, void* stream) {
  DPM_REQUIRE(sink && flops && iters > 0, "dpm_ffma_probe: bad arguments");
  int dev = 0, sms = 148;
  DPM_CUDA(cudaGetDevice(&dev));
  DPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = sms * 8, threads = 256;
  ffma_probe_kernel<<<blocks, threads, 0, as_stream(stream)>>>(sink, iters, 0.999999f, 1e-6f);
  DPM_LAUNCHED("ffma_probe_kernel");
  *flops = 2.0 * blocks * threads * (double)iters * PROBE_UNROLL * PROBE_CHAINS;
  return DPM_OK;
}
