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
#include <cstdlib>

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

// K1 on mma.sync (the default for L = 32): the same projection with the
// contraction as m16n8k8 TF32 tensor-core tiles, operands split hi + lo
// (3xTF32: lo*hi + hi*lo + hi*hi, FP32 accumulate), so the shared-memory
// staging, its barrier and the per-channel LDS of project_kernel disappear
// and the kernel is eight 16-byte loads, 24 MMAs and eight stores per warp
// and 32 cells.  A warp owns 32 consecutive cells as two 16-row A tiles
// (and K1_TPW such tiles one after the other, all loads issued up front).
// The MMA's k index is a free permutation of the channels: lane (g, t)
// loads chunks t and t + 4 (channels 4t.., 16 + 4t..) of cells g and g + 8,
// and k-step e takes element e of both chunks, so column t of step e is
// channel 4t + e and column t + 4 is channel 16 + 4t + e; B rows follow the
// same map.  Each output column r is its own dot product (prefixes of C
// give bit-identical planes).  Lanes (g, t) hold P[2t, 2t+1][cells g, g+8]:
// every store instruction writes 32-byte runs of four planes.
// hi = v rounded to TF32 (10 mantissa bits, half away from zero, integer
// arithmetic on the bits); lo = v - hi, exact.  lo goes to the MMA as raw
// FP32 bits: the tensor core reads the upper 19 bits only, and because hi is
// round-to-nearest lo has either sign, so that truncation is unbiased
// (|error| <= 2^-21 |v|).  Finite inputs (check_feature_map's contract).
__device__ __forceinline__ void split_tf32(float v, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(v) + 0x1000u) & 0xffffe000u;
  lo = __float_as_uint(v - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Tiles (32 cells) per warp: a CTA still owns K1_CELLS cells, with
// K1_CELLS / (32 K1_TPW) warps.  Two tiles per warp share the job lookup and
// the B operands and keep 8 KB of loads per warp in flight.
#ifndef DPM_K1_TPW
#define DPM_K1_TPW 2
#endif
constexpr int K1_TPW = DPM_K1_TPW;
constexpr int K1_MMA_THREADS = K1_CELLS / K1_TPW;

#ifndef DPM_K1_CTAS
#define DPM_K1_CTAS (K1_TPW == 1 ? 3 : 5)
#endif
__global__ void __launch_bounds__(K1_MMA_THREADS, DPM_K1_CTAS)
project_mma_kernel(const float* __restrict__ X, float* __restrict__ P, const float* __restrict__ C,
                   int R, const dpm_proj_job* __restrict__ jobs, int njobs) {
  constexpr int L = 32;
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_proj_job job = jobs[jid];
  const int ncl = job.H * job.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int cw = (blockIdx.x - job.block0) * K1_CELLS + warp * (32 * K1_TPW);
  DPM_CHECK(cw >= 0, "CTA cells inside its level");
  if (cw >= ncl) return;  // no CTA barrier below: a warp past the level's end just leaves

  // ---- loads: all eight 16-byte chunks of each of the warp's tiles in flight.
  // q[i][k][v]: chunk t + 4v of cell cw + 32i + 8k + g (k = 2h + u: A tile h, row half u)
  const float* src = X + job.x_off + (int64_t)(cw + g) * L + 4 * t;
  const bool al16 = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  float4 q[K1_TPW][4][2];
#pragma unroll
  for (int i = 0; i < K1_TPW; ++i) {
    const int c0 = cw + 32 * i;
    const float* s = src + 32 * i * L;
    if (c0 + 32 <= ncl && al16) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int v = 0; v < 2; ++v)
          // plain cached loads: the two 64-byte halves of a cell's line are fetched by two
          // instructions, and evict-first (__ldcs) loads cost 0.07 ms here (0.85 -> 0.78 ms)
          q[i][k][v] = __ldg(reinterpret_cast<const float4*>(s + 8 * k * L + 16 * v));
    } else {  // a level's last cells, or a feature block off 16-byte alignment
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const float* a = s + 8 * k * L + 16 * v;
          q[i][k][v] = c0 + 8 * k + g < ncl
                           ? make_float4(__ldg(a), __ldg(a + 1), __ldg(a + 2), __ldg(a + 3))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
  }

  const int64_t plane = (int64_t)job.H * job.pitch;

  // ---- B operands (R <= 8: one 8-column tile): rows t / t + 4 of k-step e, column g
  uint32_t bhi[4][2], blo[4][2];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int v = 0; v < 2; ++v)
      split_tf32(g < R ? __ldg(C + (16 * v + 4 * t + e) * R + g) : 0.f, bhi[e][v], blo[e][v]);
  const int ra = 2 * t;
  float* const Pr = P + job.p_off + (int64_t)ra * plane;
  int y = (cw + g) / job.W, x = (cw + g) - y * job.W;  // the other cells follow by +8 with row wraps
#pragma unroll
  for (int i = 0; i < K1_TPW; ++i) {
    if (cw + 32 * i >= ncl) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // A operands of k-step e: element e of the four chunks, a[u + 2v]
        uint32_t ahi[4], alo[4];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const float4 f = q[i][2 * h + u][v];
            split_tf32(e == 0 ? f.x : e == 1 ? f.y : e == 2 ? f.z : f.w, ahi[u + 2 * v], alo[u + 2 * v]);
          }
        mma_tf32(d, alo, bhi[e][0], bhi[e][1]);  // small terms first
        mma_tf32(d, ahi, blo[e][0], blo[e][1]);
        mma_tf32(d, ahi, bhi[e][0], bhi[e][1]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (cw + 32 * i + 16 * h + 8 * u + g < ncl) {
          const int o = y * job.pitch + x;
          DPM_CHECK(y >= 0 && y < job.H && x >= 0 && x < job.W, "output cell inside its level");
          if (ra < R) Pr[o] = d[2 * u];
          if (ra + 1 < R) Pr[plane + o] = d[2 * u + 1];
        }
        x += 8;
        while (x >= job.W) { x -= job.W; ++y; }
      }
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
    if ((int64_t)j.H * j.pitch > INT32_MAX) {  // the kernels index a level's plane with 32 bits
      set_error("dpm_project_prepare: job %d level %dx%d (pitch %d) too large", i, j.H, j.W, j.pitch);
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

// DPM_K1MMA=0 keeps 32-channel levels on project_kernel (A/B)
static bool mma_enabled() {
  static const bool on = [] {
    const char* e = getenv("DPM_K1MMA");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

extern "C" int dpm_project(const float* X, float* P, const float* C, int L, int R,
                           const dpm_proj_job* jobs, int njobs, int64_t nblocks, void* stream) {
  DPM_REQUIRE(X && P && C && jobs, "dpm_project: null pointer");
  DPM_REQUIRE(L >= 1 && L <= 256, "dpm_project: channels L=%d out of [1, 256]", L);
  DPM_REQUIRE(R >= 1 && R <= 1024, "dpm_project: rank R=%d out of [1, 1024]", R);
  DPM_REQUIRE(njobs >= 0 && nblocks >= 0 && nblocks <= INT32_MAX, "dpm_project: bad sizes");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  if (L == 32 && R <= 8 && mma_enabled()) {
    project_mma_kernel<<<(unsigned)nblocks, K1_MMA_THREADS, 0, as_stream(stream)>>>(X, P, C, R, jobs, njobs);
    DPM_LAUNCHED("project_mma_kernel");
    return DPM_OK;
  }
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
