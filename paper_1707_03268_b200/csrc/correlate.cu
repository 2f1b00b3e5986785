// K2: shortened multi-filter cross-correlation (implicit GEMM, FP32 FFMA).
//
//   S_f[y][x] = sum_{i<h, j<w, r<R} G[i][j][r][f] * P[chan_off + r][y+i][x+j]
//
// GEMM view: M = output positions, N = filters, K = h*w*R.  Reference:
// _term_stack + cumsum (correlation.py:115-180) for per-filter CP models and
// correlate3_full (correlation.py:92-112) for dense filters (C = identity).
//
// Tiling.  A CTA owns a 32-wide x (nwy*MP)-tall tile of output positions of
// one (image, level) and all filters of one group.  Warp w takes filter
// subset w % nwf (NF filters) and row band w / nwf (MP rows); lane = x.
// The projected tile (+ (h-1, w-1) halo) and the group's core are staged in
// shared memory channel-chunk by channel-chunk (8 ranks at a time), planar,
// so a warp's 32 column reads of one (r, row) hit 32 consecutive words.
// Each thread keeps an (MP + FH - 1)-tall register column of P for a fixed
// (j, r) and slides it over the FH filter rows: per (j, r) it issues
// MP + FH - 1 conflict-free LDS.32 plus FH broadcast vector loads of G for
// FH*MP*NF FFMAs (6*8*8 = 384 FFMAs per 25 loads for 6x6 parts).
//
// Persistent CTAs walk the tile list with a grid stride; a group's core is
// re-staged only when the group changes (all part tiles of a DPM model
// share one group, so it is staged once per CTA when R <= 8).
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace dpm {

constexpr int K2_MP = 8;       // output rows per thread
constexpr int K2_RCH = 8;      // ranks staged per chunk
constexpr int K2_MAX_WARPS = 12;

template <int NF>
__device__ __forceinline__ void load_g(float (&g)[NF], const float* p) {
  if constexpr (NF % 4 == 0) {
#pragma unroll
    for (int q = 0; q < NF / 4; ++q) {
      const float4 v = reinterpret_cast<const float4*>(p)[q];
      g[4 * q] = v.x; g[4 * q + 1] = v.y; g[4 * q + 2] = v.z; g[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < NF / 2; ++q) {
      const float2 v = reinterpret_cast<const float2*>(p)[q];
      g[2 * q] = v.x; g[2 * q + 1] = v.y;
    }
  }
}

// Packed FP32 pair (one 64-bit register pair) for FFMA2: sm_100a issues
// fma.rn.f32x2 as a single instruction at the scalar FFMA's FLOP rate, which
// halves the FMA issue slots of the outer-product loop.  A scalar first
// operand packed as {c, c} folds into FFMA2's broadcast operand (no MOV).
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void ffma2(unsigned long long& acc, float a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pack2(a, a)), "l"(b));
}

struct CorrArgs {
  const float* P;
  const float* G;
  float* S;
  const dpm_corr_job* jobs;
  const dpm_corr_tile* tiles;
  int ntiles;
  int nwf, nwy;
  int w_max;
  int R_max;
  int nf_max;
  uint32_t* ranges;
};

__device__ __forceinline__ void fold_range(uint32_t* ranges, int slot, float vmax, float vmin) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
  }
  if ((threadIdx.x & 31) == 0 && vmax >= vmin) {
    atomicMax(ranges + 2 * slot, float_key(vmax));
    atomicMin(ranges + 2 * slot + 1, float_key(vmin));
  }
}

// Stage the P chunk of one tile (nr planes x TROWS x (32 + w - 1)) with
// cp.async; zero-fill outside the level.
__device__ __forceinline__ void stage_p(float* dst, const CorrArgs& a, const dpm_corr_job& job,
                                        int rc, int nr, int y0, int x0, int TROWS, int TPITCH) {
  const int tcols = 32 + job.w - 1;
  const int per_plane = TROWS * tcols;
  const int64_t plane = (int64_t)job.H * job.pitch;
  const float* pbase = a.P + job.p_off + (int64_t)(job.chan_off + rc) * plane;
  (void)per_plane;
  const int nwarps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int rr = threadIdx.x >> 5; rr < nr * TROWS; rr += nwarps) {
    const int r = rr / TROWS, row = rr - r * TROWS;
    const int gy = y0 + row;
    const float* srow = pbase + r * plane + (int64_t)gy * job.pitch;
    float* drow = dst + (r * TROWS + row) * TPITCH;
    DPM_CHECK(tcols <= TPITCH && r < K2_RCH, "P tile row fits its buffer");
    for (int col = lane; col < tcols; col += 32) {
      const int gx = x0 + col;
      const bool ok = gy < job.H && gx < job.W;
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(drow + col);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa),
                   "l"(ok ? srow + gx : a.P), "r"(ok ? 4 : 0));
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

__device__ __forceinline__ void stage_g(float* sG, const CorrArgs& a, const dpm_corr_job& job,
                                        int FH, int rc, int nr) {
  const int nfp = job.nf_pad;
  const int per_ij = nr * nfp;
  const int total = FH * job.w * per_ij;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int ij = e / per_ij, rem = e - ij * per_ij;
    sG[ij * per_ij + rem] = __ldg(a.G + job.g_off + ((int64_t)ij * job.R + rc) * nfp + rem);
  }
}

// One rank chunk of a tile: every warp accumulates its MP output rows x NF
// filters over the staged P chunk (nr ranks) and core chunk.
template <int FH, int NF>
__device__ __forceinline__ void chunk_fma(unsigned long long (&acc)[K2_MP][NF / 2],
                                          const float* sP, const float* sG, int wy, int wf,
                                          int lane, int nr, int w, int nfp, int TROWS,
                                          int TPITCH) {
  constexpr int MP = K2_MP;
  constexpr int COL = MP + FH - 1;
  constexpr int NP = NF / 2;
  const float* pw = sP + (wy * MP) * TPITCH + lane;
  const float* gw = sG + wf * NF;
  const int gstride_i = w * nr * nfp;
  for (int j = 0; j < w; ++j) {
    for (int r = 0; r < nr; ++r) {
      const float* pc = pw + r * TROWS * TPITCH + j;
      DPM_CHECK(wy * MP + COL <= TROWS && lane + j < TPITCH, "compute reads inside the P tile");
      float col[COL];
#pragma unroll
      for (int q = 0; q < COL; ++q) col[q] = pc[q * TPITCH];
      const float* gp = gw + (j * nr + r) * nfp;
#pragma unroll
      for (int i = 0; i < FH; ++i) {
        float g[NF];
        load_g<NF>(g, gp + i * gstride_i);
        unsigned long long g2[NP];
#pragma unroll
        for (int f = 0; f < NP; ++f) g2[f] = pack2(g[2 * f], g[2 * f + 1]);
#pragma unroll
        for (int p = 0; p < MP; ++p)
#pragma unroll
          for (int f = 0; f < NP; ++f) ffma2(acc[p][f], col[p + i], g2[f]);
      }
    }
  }
}

// chunk_fma with compile-time strides (filter width FW, a full K2_RCH-rank
// chunk, core stride NFP, two row warps): every LDS of a (j, r) step is the
// step's base register plus an immediate.  With runtime strides the loop
// spends ~31 IMADs per 192 FFMA2 on addresses, and IMAD issues to the same
// FMA-heavy pipe as FFMA2 (ncu: fmaheavy 78% busy, math-pipe throttle the top
// stall at config 5, R = 32).  Same fma order as chunk_fma.
template <int FH, int NF, int FW, int NFP>
__device__ __forceinline__ void chunk_fma_fixed(unsigned long long (&acc)[K2_MP][NF / 2],
                                                const float* sP, const float* sG, int wy, int wf,
                                                int lane) {
  constexpr int MP = K2_MP;
  constexpr int COL = MP + FH - 1;
  constexpr int NP = NF / 2;
  constexpr int NR = K2_RCH;
  constexpr int TROWS = 2 * MP + FH - 1;
  constexpr int TPITCH = 32 + FW - 1;
  constexpr int GI = FW * NR * NFP;  // core stride of a filter row
  const float* pw = sP + (wy * MP) * TPITCH + lane;
  const float* gw = sG + wf * NF;
#pragma unroll 1
  for (int j = 0; j < FW; ++j) {
    const float* pj = pw + j;
    const float* gj = gw + j * (NR * NFP);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float col[COL];
#pragma unroll
      for (int q = 0; q < COL; ++q) col[q] = pj[r * TROWS * TPITCH + q * TPITCH];
#pragma unroll
      for (int i = 0; i < FH; ++i) {
        float g[NF];
        load_g<NF>(g, gj + r * NFP + i * GI);
        unsigned long long g2[NP];
#pragma unroll
        for (int f = 0; f < NP; ++f) g2[f] = pack2(g[2 * f], g[2 * f + 1]);
#ifdef DPM_K2_POUTER
#pragma unroll
        for (int p = 0; p < MP; ++p)
#pragma unroll
          for (int f = 0; f < NP; ++f) ffma2(acc[p][f], col[p + i], g2[f]);
#else
        // filter pair outer: consecutive FFMA2 reuse the 64-bit core pair (operand
        // reuse cache) and read only the scalar P value and the accumulator
#pragma unroll
        for (int f = 0; f < NP; ++f)
#pragma unroll
          for (int p = 0; p < MP; ++p) ffma2(acc[p][f], col[p + i], g2[f]);
#endif
      }
    }
  }
}

// epilogue: coalesced stores (lane = x), optional per-map range fold
template <int FH, int NF>
__device__ __forceinline__ void tile_epilogue(unsigned long long (&acc)[K2_MP][NF / 2],
                                              const CorrArgs& a, const dpm_corr_job& job, int x0,
                                              int y0, int wy, int wf, int lane) {
  constexpr int MP = K2_MP;
  constexpr int NP = NF / 2;
  const int ho = job.H - FH + 1, wo = job.W - job.w + 1;
  const int x = x0 + lane;
  const int yb = y0 + wy * MP;
  float out[MP][NF];
#pragma unroll
  for (int p = 0; p < MP; ++p)
#pragma unroll
    for (int f = 0; f < NP; ++f) unpack2(acc[p][f], out[p][2 * f], out[p][2 * f + 1]);
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int fg = wf * NF + f;
    float vmax = -INFINITY, vmin = INFINITY;
    if (fg < job.nf) {
      const int wp = s_pitch(wo);
      float* dst = a.S + job.s_off + (int64_t)fg * ho * wp;
#pragma unroll
      for (int p = 0; p < MP; ++p) {
        const int y = yb + p;
        if (x < wo && y < ho) {
          dst[(int64_t)y * wp + x] = out[p][f];
          vmax = fmaxf(vmax, out[p][f]);
          vmin = fminf(vmin, out[p][f]);
        }
      }
    }
    if (a.ranges != nullptr && job.range_idx >= 0 && wf * NF + f < job.nf)
      fold_range(a.ranges, job.range_idx + fg, vmax, vmin);
  }
}

// Core chunk (ranks rc .. rc+nr of every tap) with 16-byte cp.async (cores
// are 16-byte aligned, nf_pad % 8 == 0).
__device__ __forceinline__ void stage_g_async(float* sG, const CorrArgs& a,
                                              const dpm_corr_job& job, int FH, int rc, int nr) {
  const int nfp = job.nf_pad;
  const int per_ij4 = (nr * nfp) >> 2;
  const int total4 = FH * job.w * per_ij4;
  for (int e = threadIdx.x; e < total4; e += blockDim.x) {
    const int ij = e / per_ij4, rem = e - ij * per_ij4;
    const float* src = a.G + job.g_off + ((int64_t)ij * job.R + rc) * nfp + 4 * rem;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sG + ij * (nr * nfp) + 4 * rem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
  }
}

// Rank-chunk pipeline for R > K2_RCH: a step is (tile, rank chunk); the P and
// core chunks of step s+1 are copied (cp.async) while step s computes, into
// the other half of double buffers; accumulators live across a tile's chunks.
template <int FH, int NF, int FW = 0, int NFP = 0>
__device__ __forceinline__ void corr_chunked(const CorrArgs& a, float* smem, int PBUF, int GBUF,
                                             int TY, int TROWS, int TPITCH) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wf = warp % a.nwf, wy = warp / a.nwf;
  float* sG0 = smem + 2 * PBUF;
  auto issue = [&](int t, int rc, int buf) {
    const dpm_corr_tile tl = a.tiles[t];
    const dpm_corr_job jb = a.jobs[tl.job];
    const int nr = min(K2_RCH, jb.R - rc);
    stage_g_async(sG0 + buf * GBUF, a, jb, FH, rc, nr);  // joins stage_p's commit group
    stage_p(smem + buf * PBUF, a, jb, rc, nr, tl.ty * TY, tl.tx * 32, TROWS, TPITCH);
  };
  int t = blockIdx.x, rc = 0, buf = 0;
  if (t < a.ntiles) issue(t, 0, 0);
  unsigned long long acc[K2_MP][NF / 2];
  while (t < a.ntiles) {
    const dpm_corr_tile tile = a.tiles[t];
    const dpm_corr_job job = a.jobs[tile.job];
    if (rc == 0) {
#pragma unroll
      for (int p = 0; p < K2_MP; ++p)
#pragma unroll
        for (int f = 0; f < NF / 2; ++f) acc[p][f] = 0ull;
    }
    int nt = t, nrc = rc + K2_RCH;
    if (nrc >= job.R) {
      nt = t + gridDim.x;
      nrc = 0;
    }
    __syncthreads();  // every warp is done with buffer buf ^ 1 (step s-1)
    if (nt < a.ntiles) {
      issue(nt, nrc, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();  // step s resident for every warp
    const int nr = min(K2_RCH, job.R - rc);
    if constexpr (FW > 0) {
      if (nr == K2_RCH && job.w == FW && job.nf_pad == NFP) {
        DPM_CHECK(TPITCH == 32 + FW - 1 && TROWS == 2 * K2_MP + FH - 1, "fixed strides");
        chunk_fma_fixed<FH, NF, FW, NFP>(acc, smem + buf * PBUF, sG0 + buf * GBUF, wy, wf, lane);
      } else {
        chunk_fma<FH, NF>(acc, smem + buf * PBUF, sG0 + buf * GBUF, wy, wf, lane, nr, job.w,
                          job.nf_pad, TROWS, TPITCH);
      }
    } else {
      chunk_fma<FH, NF>(acc, smem + buf * PBUF, sG0 + buf * GBUF, wy, wf, lane, nr, job.w,
                        job.nf_pad, TROWS, TPITCH);
    }
    if (nrc == 0 || nt != t)  // last chunk of this tile
      tile_epilogue<FH, NF>(acc, a, job, tile.tx * 32, tile.ty * TY, wy, wf, lane);
    t = nt;
    rc = nrc;
    buf ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

template <int FH, int NF, int FW = 0, int NFP = 0>
__global__ void __launch_bounds__(32 * K2_MAX_WARPS)
corr_kernel(const CorrArgs a) {
  constexpr int MP = K2_MP;
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wf = warp % a.nwf, wy = warp / a.nwf;
  const int TY = a.nwy * MP;
  const int TROWS = TY + FH - 1;
  const int TPITCH = 32 + a.w_max - 1;
  const int PBUF = (K2_RCH * TROWS * TPITCH + 3) & ~3;
  if (a.R_max > K2_RCH) {  // several rank chunks per tile: chunk pipeline
    const int GBUF = (FH * a.w_max * K2_RCH * ((a.nf_max + 7) & ~7) + 3) & ~3;
    corr_chunked<FH, NF, FW, NFP>(a, smem, PBUF, GBUF, TY, TROWS, TPITCH);
    return;
  }
  // P double buffer [2][RCH][TROWS][TPITCH] at smem, core [FH][w][RCH][nf_pad] after it
  float* sG = smem + 2 * PBUF;
  // one rank chunk per tile: prefetch the next tile's P during this one
  const bool pipelined = a.R_max <= K2_RCH;

  int64_t staged_g = -1;
  int staged_chunk = -1;
  int it = 0;
  if (pipelined && blockIdx.x < a.ntiles) {
    const dpm_corr_tile t0 = a.tiles[blockIdx.x];
    const dpm_corr_job j0 = a.jobs[t0.job];
    stage_p(smem, a, j0, 0, j0.R, t0.ty * TY, t0.tx * 32, TROWS, TPITCH);
  }
  for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
    const dpm_corr_tile tile = a.tiles[t];
    const dpm_corr_job job = a.jobs[tile.job];
    const int y0 = tile.ty * TY, x0 = tile.tx * 32;
    const int w = job.w, nfp = job.nf_pad;

    constexpr int NP = NF / 2;  // filter pairs (FFMA2 lanes)
    unsigned long long acc[MP][NP];
#pragma unroll
    for (int p = 0; p < MP; ++p)
#pragma unroll
      for (int f = 0; f < NP; ++f) acc[p][f] = 0ull;

    for (int rc = 0; rc < job.R; rc += K2_RCH) {
      const int nr = min(K2_RCH, job.R - rc);
      float* sP = smem + ((pipelined && (it & 1)) ? PBUF : 0);
      __syncthreads();  // every warp is done with the buffers about to be refilled
      if (pipelined) {
        const int tn = t + gridDim.x;
        if (tn < a.ntiles) {
          const dpm_corr_tile nt = a.tiles[tn];
          const dpm_corr_job nj = a.jobs[nt.job];
          stage_p(smem + (((it + 1) & 1) ? PBUF : 0), a, nj, 0, nj.R, nt.ty * TY, nt.tx * 32, TROWS,
                  TPITCH);
          asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::);
        }
      } else {
        stage_p(sP, a, job, rc, nr, y0, x0, TROWS, TPITCH);
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      if (staged_g != job.g_off || staged_chunk != rc) {
        stage_g(sG, a, job, FH, rc, nr);
        staged_g = job.g_off;
        staged_chunk = rc;
      }
      __syncthreads();

      chunk_fma<FH, NF>(acc, sP, sG, wy, wf, lane, nr, w, nfp, TROWS, TPITCH);
    }

    tile_epilogue<FH, NF>(acc, a, job, x0, y0, wy, wf, lane);
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// Generic fallback: any h, any nf; one thread per (position, filter loop).
__global__ void __launch_bounds__(256)
corr_generic_kernel(const CorrArgs a) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const dpm_corr_tile tile = a.tiles[t];
    const dpm_corr_job job = a.jobs[tile.job];
    const int ho = job.H - job.h + 1, wo = job.W - job.w + 1;
    const int x = tile.tx * 32 + tx, y = tile.ty * 8 + ty;
    if (x >= wo || y >= ho) continue;
    const int64_t plane = (int64_t)job.H * job.pitch;
    const float* pb = a.P + job.p_off + (int64_t)job.chan_off * plane + (int64_t)y * job.pitch + x;
    for (int f = 0; f < job.nf; ++f) {
      float acc = 0.f;
      for (int j = 0; j < job.w; ++j)
        for (int r = 0; r < job.R; ++r)
          for (int i = 0; i < job.h; ++i)
            acc = fmaf(__ldg(pb + r * plane + (int64_t)i * job.pitch + j),
                       __ldg(a.G + job.g_off + (((int64_t)i * job.w + j) * job.R + r) * job.nf_pad + f),
                       acc);
      a.S[job.s_off + ((int64_t)f * ho + y) * s_pitch(wo) + x] = acc;
      if (a.ranges != nullptr && job.range_idx >= 0) {
        atomicMax(a.ranges + 2 * (job.range_idx + f), float_key(acc));
        atomicMin(a.ranges + 2 * (job.range_idx + f) + 1, float_key(acc));
      }
    }
  }
}

__global__ void ranges_init_kernel(uint32_t* ranges, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    ranges[2 * i] = 0u;             // key(-inf) > 0, any value beats it
    ranges[2 * i + 1] = 0xffffffffu;
  }
}

// ------------------------------------------------------------ dispatch
struct Shape {
  int nf_kernel, nwf, nwy;
};

static bool pick(int h, int nf, Shape* s) {
  if (nf < 1) return false;
  if (nf <= 8) {
    s->nf_kernel = nf <= 2 ? 2 : nf <= 4 ? 4 : nf <= 6 ? 6 : 8;
    s->nwf = 1;
    s->nwy = 2;
  } else {
    s->nf_kernel = 8;
    s->nwf = (nf + 7) / 8;
    if (s->nwf > 6) return false;
    s->nwy = 2;  // <= K2_MAX_WARPS (12) warps per CTA
  }
  switch (h) {
    case 2: case 3: case 4: case 5: case 6: case 7: case 8: case 11: case 15: return true;
    default: return false;
  }
}

typedef void (*corr_fn)(const CorrArgs);

int launch_corr_few(const float* P, const float* G, float* S, const dpm_corr_job* jobs,
                    const dpm_corr_tile* tiles, int ntiles, int h, int nf, int w_max,
                    uint32_t* ranges, cudaStream_t st);
// DPM_K2FEW=0 keeps few-filter groups on corr_kernel (A/B)
static bool few_enabled() {
  static const bool on = [] {
    const char* e = getenv("DPM_K2FEW");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// DPM_K2FIXED=0 keeps the runtime-stride inner loop for R > 8 (A/B)
static bool fixed_enabled() {
  static const bool on = [] {
    const char* e = getenv("DPM_K2FIXED");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

template <int FH>
static corr_fn by_nf(int nfk) {
  switch (nfk) {
    case 2: return corr_kernel<FH, 2>;
    case 4: return corr_kernel<FH, 4>;
    case 6: return corr_kernel<FH, 6>;
    default: return corr_kernel<FH, 8>;
  }
}

static corr_fn kernel_for(int h, int nfk) {
  switch (h) {
    case 2: return by_nf<2>(nfk);
    case 3: return by_nf<3>(nfk);
    case 4: return by_nf<4>(nfk);
    case 5: return by_nf<5>(nfk);
    case 6: return by_nf<6>(nfk);
    case 7: return by_nf<7>(nfk);
    case 8: return by_nf<8>(nfk);
    case 11: return by_nf<11>(nfk);
    default: return by_nf<15>(nfk);
  }
}

}  // namespace dpm

using namespace dpm;

extern "C" int dpm_correlate_tile_shape(int h, int nf, int* tile_w, int* tile_h) {
  DPM_REQUIRE(tile_w && tile_h, "dpm_correlate_tile_shape: null output");
  Shape s;
  *tile_w = 32;
  if (pick(h, nf, &s)) {
    *tile_h = s.nwy * K2_MP;
    return s.nwf * s.nwy;
  }
  *tile_h = 8;
  return DPM_ERR_UNSUPPORTED;
}

extern "C" int dpm_ranges_init(uint32_t* ranges, int n, void* stream) {
  DPM_REQUIRE(ranges && n >= 0, "dpm_ranges_init: bad arguments");
  if (n == 0) return DPM_OK;
  ranges_init_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(ranges, n);
  DPM_LAUNCHED("ranges_init_kernel");
  return DPM_OK;
}

extern "C" int dpm_correlate(const float* P, const float* G, float* S, const dpm_corr_job* jobs,
                             const dpm_corr_tile* tiles, int ntiles, int h, int nf, int R,
                             int w_max, uint32_t* ranges, void* stream) {
  DPM_REQUIRE(P && G && S && jobs && tiles, "dpm_correlate: null pointer");
  DPM_REQUIRE(ntiles >= 0, "dpm_correlate: ntiles=%d", ntiles);
  DPM_REQUIRE(h >= 1 && w_max >= 1 && w_max <= 64, "dpm_correlate: h=%d w_max=%d", h, w_max);
  DPM_REQUIRE(R >= 1 && nf >= 1, "dpm_correlate: R=%d nf=%d", R, nf);
  if (ntiles == 0) return DPM_OK;
  int dev = 0, sms = 148;
  DPM_CUDA(cudaGetDevice(&dev));
  DPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (nf <= 8 && few_enabled()) {  // few-filter groups: correlate_few.cu
    const int rc = launch_corr_few(P, G, S, jobs, tiles, ntiles, h, nf, w_max, ranges,
                                   as_stream(stream));
    if (rc != DPM_ERR_UNSUPPORTED) return rc;
  }
  CorrArgs a{P, G, S, jobs, tiles, ntiles, 1, 1, w_max, R, nf, ranges};
  Shape s;
  if (!pick(h, nf, &s)) {
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * 8);
    corr_generic_kernel<<<grid, 256, 0, as_stream(stream)>>>(a);
    DPM_LAUNCHED("corr_generic_kernel");
    return DPM_OK;
  }
  a.nwf = s.nwf;
  a.nwy = s.nwy;
  const int TROWS = s.nwy * K2_MP + h - 1;
  const int TPITCH = 32 + w_max - 1;
  const int nfp = (nf + 7) & ~7;  // core filter stride (dpm_corr_job.nf_pad)
  // P double buffer + one core chunk; R > K2_RCH double-buffers the core chunk too
  const size_t gbuf = (((size_t)h * w_max * K2_RCH * nfp) + 3) & ~(size_t)3;
  const size_t smem = sizeof(float) * (2 * ((((size_t)K2_RCH * TROWS * TPITCH) + 3) & ~(size_t)3) +
                                       (R > K2_RCH ? 2 : 1) * gbuf);
  DPM_REQUIRE(smem <= 227 * 1024, "dpm_correlate: h=%d w=%d nf=%d needs %zu B shared memory",
              h, w_max, nf, smem);
  corr_fn fn = kernel_for(h, s.nf_kernel);
  // R > 8 with 6x6 filters in groups of 16 / 48: compile-time strides (chunk_fma_fixed)
  if (R > K2_RCH && h == 6 && w_max == 6 && s.nf_kernel == 8 && s.nwy == 2 && fixed_enabled()) {
    if (nfp == 48) fn = corr_kernel<6, 8, 6, 48>;
    else if (nfp == 16) fn = corr_kernel<6, 8, 6, 16>;
  }
  DPM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  const int threads = 32 * s.nwf * s.nwy;
  DPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm < 1) per_sm = 1;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
  fn<<<grid, threads, smem, as_stream(stream)>>>(a);
  DPM_LAUNCHED("corr_kernel");
  return DPM_OK;
}
