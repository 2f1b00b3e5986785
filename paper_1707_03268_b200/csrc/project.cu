// K1: channel projection of HOG pyramid levels onto the rank-R basis.
//
//   P[r][y][x] = sum_l X[y][x][l] * C[l][r]
//
// Reference: the contraction `img.reshape(H*W, L) @ factors_c` of
// _term_stack (correlation.py:128).  HBM-bound: 4*(L+R) algorithmic bytes
// per cell.  Each CTA stages a contiguous run of K1_CELLS cells with
// coalesced 16-byte loads into shared memory (row pitch L+1 so the per-cell
// reads below are bank-conflict free), then one thread per cell contracts
// its channels against C (broadcast from shared memory) and writes R planar
// outputs; consecutive threads write consecutive x, so every plane store is
// coalesced.
#include "common.cuh"

namespace dpm {

constexpr int K1_CELLS = 256;
constexpr int K1_RC = 8;  // output channels per register chunk

__global__ void __launch_bounds__(K1_CELLS)
project_kernel(const float* __restrict__ X, float* __restrict__ P, const float* __restrict__ C,
               int L, int R, const dpm_proj_job* __restrict__ jobs, int njobs) {
  extern __shared__ __align__(16) float smem[];
  const int Rp = (R + K1_RC - 1) / K1_RC * K1_RC;
  float* sC = smem;                 // [L][Rp]
  float* sX = smem + L * Rp;        // [K1_CELLS][L+1]

  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_proj_job job = jobs[jid];
  const int64_t ncells_level = (int64_t)job.H * job.W;
  const int64_t cell0 = (int64_t)(blockIdx.x - job.block0) * K1_CELLS;
  const int ncell = (int)min((int64_t)K1_CELLS, ncells_level - cell0);
  const int t = threadIdx.x;
  DPM_CHECK(ncell > 0 && ncell <= K1_CELLS, "CTA cells inside its level");

  for (int i = t; i < L * Rp; i += blockDim.x) {
    const int l = i / Rp, r = i % Rp;
    sC[i] = r < R ? C[l * R + r] : 0.f;
  }
  const float* src = X + job.x_off + cell0 * L;
  const int nflt = ncell * L;
  if (L == 32 && ncell == K1_CELLS && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    // full tile of HOG cells: all 8 loads per thread in flight before the
    // shared-memory stores (one memory latency per CTA, not eight)
    const float4* src4 = reinterpret_cast<const float4*>(src);
    float4 q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = __ldcs(src4 + t + k * K1_CELLS);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int v = t + k * K1_CELLS;
      float* d = sX + (v >> 3) * 33 + ((v & 7) << 2);
      d[0] = q[k].x; d[1] = q[k].y; d[2] = q[k].z; d[3] = q[k].w;
    }
  } else if ((L & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    const float4* src4 = reinterpret_cast<const float4*>(src);
    for (int v = t; v < (nflt >> 2); v += blockDim.x) {
      const float4 q = __ldg(src4 + v);
      const int e = v << 2;
      const int c = e / L, l = e - c * L;
      float* d = sX + c * (L + 1) + l;
      d[0] = q.x; d[1] = q.y; d[2] = q.z; d[3] = q.w;
    }
  } else {
    for (int e = t; e < nflt; e += blockDim.x) {
      const int c = e / L, l = e - c * L;
      sX[c * (L + 1) + l] = __ldg(src + e);
    }
  }
  __syncthreads();
  if (t >= ncell) return;

  const int64_t cell = cell0 + t;
  const int y = (int)(cell / job.W), x = (int)(cell - (int64_t)y * job.W);
  const float* xr = sX + t * (L + 1);
  const int64_t plane = (int64_t)job.H * job.pitch;
  float* dst = P + job.p_off + (int64_t)y * job.pitch + x;
  // FFMA2: the channel value broadcast as {x, x}, C read as 64-bit pairs
  // straight into register pairs -- the same per-element fma as a scalar
  // loop, half the FMA issue slots.
  for (int r0 = 0; r0 < R; r0 += K1_RC) {
    unsigned long long acc[K1_RC / 2];
#pragma unroll
    for (int k = 0; k < K1_RC / 2; ++k) acc[k] = 0ull;
    for (int l = 0; l < L; ++l) {
      const float xv = xr[l];
      unsigned long long xx;
      asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(xv));
      const unsigned long long* cr = reinterpret_cast<const unsigned long long*>(sC + l * Rp + r0);
#pragma unroll
      for (int k = 0; k < K1_RC / 2; ++k)
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[k]) : "l"(xx), "l"(cr[k]));
    }
#pragma unroll
    for (int k = 0; k < K1_RC / 2; ++k) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[k]));
      if (r0 + 2 * k < R) dst[(int64_t)(r0 + 2 * k) * plane] = lo;
      if (r0 + 2 * k + 1 < R) dst[(int64_t)(r0 + 2 * k + 1) * plane] = hi;
    }
  }
}

}  // namespace dpm

using namespace dpm;

extern "C" int64_t dpm_project_prepare(dpm_proj_job* jobs, int njobs) {
  if (njobs < 0 || (njobs > 0 && jobs == nullptr)) {
    set_error("dpm_project_prepare: bad job table");
    return DPM_ERR_ARG;
  }
  int64_t b = 0;
  for (int i = 0; i < njobs; ++i) {
    const dpm_proj_job& j = jobs[i];
    if (j.H < 1 || j.W < 1 || j.pitch < j.W || (j.pitch & 3)) {
      set_error("dpm_project_prepare: job %d has H=%d W=%d pitch=%d", i, j.H, j.W, j.pitch);
      return DPM_ERR_ARG;
    }
    jobs[i].block0 = (int32_t)b;
    b += ((int64_t)j.H * j.W + K1_CELLS - 1) / K1_CELLS;
  }
  if (b > INT32_MAX) {
    set_error("dpm_project_prepare: too many CTAs (%lld)", (long long)b);
    return DPM_ERR_ARG;
  }
  return b;
}

extern "C" int dpm_project(const float* X, float* P, const float* C, int L, int R,
                           const dpm_proj_job* jobs, int njobs, int64_t nblocks, void* stream) {
  DPM_REQUIRE(X && P && C && jobs, "dpm_project: null pointer");
  DPM_REQUIRE(L >= 1 && L <= 256, "dpm_project: channels L=%d out of [1, 256]", L);
  DPM_REQUIRE(R >= 1 && R <= 1024, "dpm_project: rank R=%d out of [1, 1024]", R);
  DPM_REQUIRE(njobs >= 0 && nblocks >= 0 && nblocks <= INT32_MAX, "dpm_project: bad sizes");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  const int Rp = (R + K1_RC - 1) / K1_RC * K1_RC;
  const size_t smem = sizeof(float) * ((size_t)L * Rp + (size_t)K1_CELLS * (L + 1));
  DPM_REQUIRE(smem <= 227 * 1024, "dpm_project: L=%d R=%d needs %zu B shared memory", L, R, smem);
  if (smem > 48 * 1024)
    DPM_CUDA(cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  project_kernel<<<(unsigned)nblocks, K1_CELLS, smem, as_stream(stream)>>>(X, P, C, L, R, jobs, njobs);
  DPM_LAUNCHED("project_kernel");
  return DPM_OK;
}
