// K2 in rank-prefix mode: every cumulative rank prefix of a CP filter from
// one pass over the filter's ranks (convolution shortening, paper
// Algorithm 1 / PAPER.md:135-178).
//
// Reference: cp_partial_stack = cumsum of _term_stack (correlation.py:115-180)
// -- per rank r the term T_r[y][x] = sum_{i,j} w_r a_ir b_jr (X c_r)[y+i][x+j],
// then prefix_k = T_0 + ... + T_{k-1}.  Here, in the same structure:
//
//   T_r      = sum_{j < w} sum_{i < h} G[i][j][r] * P[chan_off + r][y+i][x+j]
//   prefix_k = prefix_{k-1} + T_{k-1}       (FP32, rank order)
//
// so one launch writes all K prefix maps at the cost of ONE full correlation
// (h*w FMAs per rank and position) plus K stores, instead of K independent
// correlations with ranks >= k zeroed.  correlate3_cp(upto = k) and
// cp_partial_stack both read these maps, so the reference's prefix
// bit-identity (test_correlation.py:158-178) holds by construction.
//
// Tiling: CTA = 4 warps = a 32 x 32 tile of output positions of one job;
// lane = column, warp = 8 rows.  Rank planes of the projected level (tile +
// (h-1, w-1) halo) are staged in shared memory one rank at a time,
// double-buffered with cp.async; the core values of a rank are broadcast
// from shared memory.  Each thread keeps an (8 + FH - 1)-tall register
// column per tap column j (FH compile-time).
#include "common.cuh"

namespace dpm {

constexpr int PX_THREADS = 128;
constexpr int PX_MP = 8;                  // output rows per thread
constexpr int PX_TH = 4 * PX_MP;          // tile rows
constexpr int PX_HMAX = 16, PX_WMAX = 16;  // filter extent limits
constexpr int PX_TPITCH = 32 + PX_WMAX - 1;
constexpr int PX_PLANE = (PX_TH + PX_HMAX - 1) * PX_TPITCH;

struct PrefixArgs {
  const float* P;
  const float* G;
  float* S;
  const dpm_corr_job* jobs;
  const dpm_corr_tile* tiles;
  int ntiles;
  uint32_t* ranges;
};

__device__ __forceinline__ void px_stage(float* dst, const PrefixArgs& a, const dpm_corr_job& job,
                                         int r, int y0, int x0) {
  const int rows = PX_TH + job.h - 1, cols = 32 + job.w - 1;
  const int64_t plane = (int64_t)job.H * job.pitch;
  const float* src = a.P + job.p_off + (int64_t)(job.chan_off + r) * plane;
  for (int e = threadIdx.x; e < rows * cols; e += PX_THREADS) {
    const int row = e / cols, col = e - row * cols;
    const int gy = y0 + row, gx = x0 + col;
    const bool ok = gy < job.H && gx < job.W;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + row * PX_TPITCH + col);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa),
                 "l"(ok ? src + (int64_t)gy * job.pitch + gx : a.P), "r"(ok ? 4 : 0));
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

template <int FH>
__global__ void __launch_bounds__(PX_THREADS) prefix_kernel(const PrefixArgs a) {
  __shared__ __align__(16) float sP[2][PX_PLANE];
  __shared__ float sG[2][PX_HMAX * PX_WMAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int COL = PX_MP + FH - 1;
  for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const dpm_corr_tile tile = a.tiles[t];
    const dpm_corr_job job = a.jobs[tile.job];
    const int y0 = tile.ty * PX_TH, x0 = tile.tx * 32;
    const int ho = job.H - FH + 1, wo = job.W - job.w + 1, wp = s_pitch(wo);
    const int x = x0 + lane, yb = y0 + warp * PX_MP;
    const int K = job.nf;  // prefixes to write (ranks 0 .. K-1)
    __syncthreads();       // the previous tile's buffers are free
    px_stage(sP[0], a, job, 0, y0, x0);
    float pre[PX_MP];
#pragma unroll
    for (int p = 0; p < PX_MP; ++p) pre[p] = 0.f;
    for (int r = 0; r < K; ++r) {
      const int b = r & 1;
      // core values of rank r (column 0 of the [h][w][R][nf_pad] block)
      for (int e = threadIdx.x; e < FH * job.w; e += PX_THREADS)
        sG[b][e] = __ldg(a.G + job.g_off + ((int64_t)e * job.R + r) * job.nf_pad);
      if (r + 1 < K) {
        px_stage(sP[b ^ 1], a, job, r + 1, y0, x0);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      __syncthreads();  // plane r and its core values resident
      float term[PX_MP];
#pragma unroll
      for (int p = 0; p < PX_MP; ++p) term[p] = 0.f;
      const float* pw = sP[b] + (warp * PX_MP) * PX_TPITCH + lane;
      for (int j = 0; j < job.w; ++j) {
        float col[COL];
#pragma unroll
        for (int q = 0; q < COL; ++q) col[q] = pw[q * PX_TPITCH + j];
#pragma unroll
        for (int i = 0; i < FH; ++i) {
          const float g = sG[b][i * job.w + j];
#pragma unroll
          for (int p = 0; p < PX_MP; ++p) term[p] = fmaf(g, col[p + i], term[p]);
        }
      }
      float vmax = -INFINITY, vmin = INFINITY;
      float* dst = a.S + job.s_off + (int64_t)r * ho * wp;
#pragma unroll
      for (int p = 0; p < PX_MP; ++p) {
        pre[p] = __fadd_rn(pre[p], term[p]);
        const int y = yb + p;
        if (x < wo && y < ho) {
          dst[(int64_t)y * wp + x] = pre[p];
          vmax = fmaxf(vmax, pre[p]);
          vmin = fminf(vmin, pre[p]);
        }
      }
      if (a.ranges != nullptr && job.range_idx >= 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
          vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        }
        if (lane == 0 && vmax >= vmin) {
          atomicMax(a.ranges + 2 * (job.range_idx + r), float_key(vmax));
          atomicMin(a.ranges + 2 * (job.range_idx + r) + 1, float_key(vmin));
        }
      }
      __syncthreads();  // every warp done with plane r before it is refilled
    }
  }
}

}  // namespace dpm

using namespace dpm;

extern "C" int dpm_correlate_prefix_tile(int* tile_w, int* tile_h) {
  DPM_REQUIRE(tile_w && tile_h, "dpm_correlate_prefix_tile: null output");
  *tile_w = 32;
  *tile_h = PX_TH;
  return DPM_OK;
}

extern "C" int dpm_correlate_prefix(const float* P, const float* G, float* S,
                                    const dpm_corr_job* jobs, const dpm_corr_tile* tiles,
                                    int ntiles, int h, uint32_t* ranges, void* stream) {
  DPM_REQUIRE(P && G && S && jobs && tiles, "dpm_correlate_prefix: null pointer");
  DPM_REQUIRE(ntiles >= 0, "dpm_correlate_prefix: ntiles=%d", ntiles);
  DPM_REQUIRE(h >= 1 && h <= PX_HMAX, "dpm_correlate_prefix: filter height %d outside [1, %d]", h,
              PX_HMAX);
  if (ntiles == 0) return DPM_OK;
  PrefixArgs a{P, G, S, jobs, tiles, ntiles, ranges};
  void (*fn)(const PrefixArgs) = nullptr;
  switch (h) {
#define DPM_PX(H) case H: fn = prefix_kernel<H>; break;
    DPM_PX(1) DPM_PX(2) DPM_PX(3) DPM_PX(4) DPM_PX(5) DPM_PX(6) DPM_PX(7) DPM_PX(8)
    DPM_PX(9) DPM_PX(10) DPM_PX(11) DPM_PX(12) DPM_PX(13) DPM_PX(14) DPM_PX(15) DPM_PX(16)
#undef DPM_PX
  }
  int dev = 0, sms = 148;
  DPM_CUDA(cudaGetDevice(&dev));
  DPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = ntiles < 8 * sms ? ntiles : 8 * sms;
  fn<<<grid, PX_THREADS, 0, as_stream(stream)>>>(a);
  DPM_LAUNCHED("prefix_kernel");
  return DPM_OK;
}

// Host-side validation of a prefix job table (mode 1): called by the planner.
extern "C" int dpm_correlate_prefix_check(const dpm_corr_job* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_correlate_prefix_check: bad table");
  for (int i = 0; i < njobs; ++i) {
    const dpm_corr_job& j = jobs[i];
    DPM_REQUIRE(j.mode == 1, "dpm_correlate_prefix_check: job %d is not a prefix job", i);
    DPM_REQUIRE(j.nf >= 1 && j.nf <= j.R && j.h >= 1 && j.h <= PX_HMAX && j.w >= 1 &&
                    j.w <= PX_WMAX && j.H >= j.h && j.W >= j.w,
                "dpm_correlate_prefix_check: job %d has nf=%d R=%d filter %dx%d level %dx%d", i,
                j.nf, j.R, j.h, j.w, j.H, j.W);
  }
  return DPM_OK;
}
