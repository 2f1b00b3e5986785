// Shared helpers of libdpm_b200.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdarg>
#include <cstdio>

#include "dpm_b200.h"

namespace dpm {

// Thread-local message of the last failing ABI call (dpm_last_error()).
void set_error(const char* fmt, ...);
const char* last_error();

#define DPM_REQUIRE(cond, ...)                  \
  do {                                          \
    if (!(cond)) {                              \
      ::dpm::set_error(__VA_ARGS__);            \
      return DPM_ERR_ARG;                       \
    }                                           \
  } while (0)

#define DPM_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      ::dpm::set_error("%s failed: %s", #call, cudaGetErrorString(e_));         \
      return DPM_ERR_CUDA;                                                      \
    }                                                                           \
  } while (0)

// Launch-error check after <<<>>>.
#define DPM_LAUNCHED(name)                                                      \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess) {                                                    \
      ::dpm::set_error("%s launch failed: %s", name, cudaGetErrorString(e_));   \
      return DPM_ERR_CUDA;                                                      \
    }                                                                           \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Bounds checks of the checked build (make checked -> libdpm_b200_checked.so,
// -DDPM_CHECKED): shared- and global-memory indices of the hot kernels are
// asserted; a violation prints the site and traps.  compute-sanitizer is
// closed on this GPU pool, so the parity suite run against the checked
// library stands in for memcheck (profiles/r2_checked_build.txt).  The
// product build compiles the checks away.
#ifdef DPM_CHECKED
#define DPM_CHECK(cond, what)                                                              \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("DPM_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                           \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define DPM_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

// Row pitch (floats) of a response map S of width w: rows are padded to 16
// bytes, so band / row copies can move whole 16-byte chunks and a map can be
// described to the TMA unit (strides must be multiples of 16 B).
__host__ __device__ constexpr int s_pitch(int w) { return (w + 3) & ~3; }

// Order-preserving float <-> uint32 key (max over keys == max over floats).
__device__ __forceinline__ uint32_t float_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// Find the job owning CTA `b` in a table sorted by block0 (binary search).
template <typename Job>
__device__ __forceinline__ int find_job(const Job* jobs, int njobs, int64_t b) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].block0 <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// The same as a 32-ary search by a whole warp (every lane calls it with the
// same b): each round one load per lane and a ballot narrow the range 32-fold,
// so a 15k-job table costs three dependent loads instead of fourteen.  `key`
// picks the start field (block0 by default); zero-size jobs share their
// successor's start and are skipped (the owner is the LAST job starting <= b).
template <typename Job, typename Key>
__device__ __forceinline__ int find_job_warp(const Job* jobs, int njobs, int64_t b, Key key) {
  const int lane = threadIdx.x & 31;
  int lo = 0, n = njobs;  // key(jobs[lo]) <= b; the owner lies in [lo, lo + n)
  while (n > 1) {
    const int step = (n + 31) >> 5;
    const int idx = lo + lane * step;
    const bool le = idx < lo + n && key(jobs[idx]) <= b;
    const unsigned m = __ballot_sync(0xffffffffu, le);  // lane 0 is always set
    const int k = 31 - __clz(m);
    lo += k * step;
    n = min(step, n - k * step);
  }
  return lo;
}
template <typename Job>
__device__ __forceinline__ int find_job_warp(const Job* jobs, int njobs, int64_t b) {
  return find_job_warp(jobs, njobs, b, [](const Job& j) { return j.block0; });
}

}  // namespace dpm
