// K2 for few-filter groups (nf <= 8): roots and other small filter groups.
//
//   S_f[y][x] = sum_{i<h, j<w, r<R} G[i][j][r][f] * P[chan_off + r][y+i][x+j]
//
// Reference: _term_stack + cumsum (correlation.py:115-180) and
// correlate3_full (correlation.py:92-112), as corr_kernel (correlate.cu).
//
// Why a second FFMA kernel.  corr_kernel gives a few-filter group one warp
// per 8 output rows and stages the core at the 8-filter stride and the P tile
// double-buffered at 8 ranks: a 15x15 root pair then needs ~200 KB of shared
// memory, runs ONE 2-warp CTA per SM and reached 5-7% of the FFMA peak
// (config 5), and the many 2-8 filter root groups of config 3 10-20%.  Here
//   - the reduction is split across warps by filter rows: S_K warps share an
//     8-row x 32-column output block, warp k sums filter rows
//     [k KS, (k+1) KS), and the partial sums are added in a fixed order
//     (deterministic) through shared memory at the end of the tile, so a
//     tile carries 2 S_K warps instead of 2;
//   - ranks are staged FEW_RCH at a time (double-buffered cp.async), and the
//     core at the kernel's own filter stride NF, which keeps the footprint
//     at 3 CTAs per SM for 15x15 filters;
//   - the tile geometry (32 x 16) and the tile lists are corr_kernel's.
// Inner loop as in corr_kernel: a register column of P slides over the
// warp's filter rows, FFMA2 (fma.rn.f32x2) over filter pairs.
#include <algorithm>

#include "common.cuh"

namespace dpm {

constexpr int FEW_MP = 8;    // output rows per thread
constexpr int FEW_TY = 16;   // output rows per tile (2 row warps)
constexpr int FEW_RCH = 4;   // ranks per staged chunk

// K-split of the filter rows: S_K warps per 8-row block
__host__ __device__ constexpr int few_split(int fh, int nf) {
  return nf >= 6 ? (fh >= 6 ? 2 : 1) : (fh >= 8 ? 4 : fh >= 6 ? 3 : fh >= 4 ? 2 : 1);
}
__host__ __device__ constexpr int few_ks(int fh, int nf) {
  return (fh + few_split(fh, nf) - 1) / few_split(fh, nf);
}

struct FewArgs {
  const float* P;
  const float* G;
  float* S;
  const dpm_corr_job* jobs;
  const dpm_corr_tile* tiles;
  int ntiles;
  int w_max;
  uint32_t* ranges;
  int prow, pbuf, gbuf;  // P rows per plane, P / core chunk buffer floats
};

__device__ __forceinline__ unsigned long long f_pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f_ffma2(unsigned long long& acc, float a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(f_pack2(a, a)), "l"(b));
}

// One staged chunk of a warp's filter-row slice (NKS rows starting at the
// warp's i0): every shared-memory address is a per-j base plus an immediate
// (compile-time tile pitch TP, plane stride PROW * TP, core layout
// [j][r][i][NF]); full chunks unroll the ranks.  Same fma order as before
// (j, r, i), so the sums are unchanged bit for bit.
template <int NKS, int MP, int NF, int FH, int TP, int PROW>
__device__ __forceinline__ void few_chunk(unsigned long long (&acc)[MP][NF / 2], const float* sp,
                                          const float* sg, int w, int nr) {
  constexpr int NP = NF / 2, COL = MP + NKS - 1, PLANE = PROW * TP;
  const bool full = nr == FEW_RCH;
#pragma unroll 1
  for (int j = 0; j < w; ++j) {
    const float* pj = sp + j;
    const float* gj = sg + j * nr * FH * NF;
#pragma unroll
    for (int r = 0; r < FEW_RCH; ++r) {
      if (!full && r >= nr) break;
      float col[COL];
#pragma unroll
      for (int q = 0; q < COL; ++q) col[q] = pj[r * PLANE + q * TP];
#pragma unroll
      for (int i = 0; i < NKS; ++i) {
        unsigned long long g2[NP];
        const float* gp = gj + (r * FH + i) * NF;
        if constexpr (NF % 4 == 0) {
#pragma unroll
          for (int f = 0; f < NP; f += 2) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(gp + 2 * f);
            g2[f] = v.x;
            g2[f + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int f = 0; f < NP; ++f) g2[f] = *reinterpret_cast<const unsigned long long*>(gp + 2 * f);
        }
#pragma unroll
        for (int p = 0; p < MP; ++p)
#pragma unroll
          for (int f = 0; f < NP; ++f) f_ffma2(acc[p][f], col[p + i], g2[f]);
      }
    }
  }
}

template <int FH, int NF, int TP>
__global__ void __launch_bounds__(64 * few_split(FH, NF))
corr_few_kernel(const FewArgs a) {
  constexpr int SK = few_split(FH, NF), KS = few_ks(FH, NF);
  constexpr int KS_LAST = FH - (SK - 1) * KS;  // rows of the last slice
  static_assert(KS_LAST >= 1 && KS_LAST <= KS, "every filter-row slice is non-empty");
  constexpr int MP = FEW_MP, NP = NF / 2;
  constexpr int NT = 64 * SK;
  constexpr int PROW = FEW_TY + SK * KS - 1;   // P rows per plane (= a.prow)
  constexpr int TPITCH = TP;                   // P tile pitch (>= 32 + w - 1)
  extern __shared__ __align__(16) float smem[];
  float* const sP0 = smem;                      // [2][RCH][PROW][TP]
  float* const sG0 = smem + 2 * a.pbuf;         // [2][w][RCH][FH][NF]
  float* const sX = sG0 + 2 * a.gbuf;           // [SK-1][2][MP][NF][32] partial sums
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wy = warp & 1, wk = warp >> 1;     // row block, filter-row slice
  const int i0 = wk * KS;                       // first filter row of this warp
  DPM_CHECK(a.prow == PROW && 32 + a.w_max - 1 <= TP, "compile-time tile geometry");

  // stage the P and core chunk (ranks rc .. rc + nr) of tile t into buffer b
  auto issue = [&](int t, int rc, int b) {
    const dpm_corr_tile tl = a.tiles[t];
    const dpm_corr_job& jb = a.jobs[tl.job];
    const int nr = min(FEW_RCH, jb.R - rc);
    // core: (i, j, r) rows of NF floats (the job's nf_pad stride is 32-byte aligned)
    float* sg = sG0 + b * a.gbuf;
    const int rows = FH * jb.w * nr;
    for (int e = threadIdx.x; e < rows; e += NT) {
      const int ij = e / nr, r = e - ij * nr;
      const int i = ij / jb.w, j = ij - i * jb.w;
      const float* src = a.G + jb.g_off + ((int64_t)ij * jb.R + rc + r) * jb.nf_pad;
      const int d = (j * nr + r) * FH + i;  // smem layout [j][r][i][NF]
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sg + d * NF);
      DPM_CHECK((d + 1) * NF <= a.gbuf, "core chunk fits its buffer");
      if constexpr (NF % 4 == 0) {
#pragma unroll
        for (int q = 0; q < NF / 4; ++q)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa + 16 * q),
                       "l"(src + 4 * q));
      } else {
#pragma unroll
        for (int q = 0; q < NF / 2; ++q)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa + 8 * q),
                       "l"(src + 2 * q));
      }
    }
    // P rows of the tile (zero-filled outside the level)
    const int y0 = tl.ty * FEW_TY, x0 = tl.tx * 32;
    const int tcols = 32 + jb.w - 1, trows = FEW_TY + FH - 1;
    const int64_t plane = (int64_t)jb.H * jb.pitch;
    const float* pbase = a.P + jb.p_off + (int64_t)(jb.chan_off + rc) * plane;
    float* sp = sP0 + b * a.pbuf;
    for (int rr = warp; rr < nr * trows; rr += NT / 32) {
      const int r = rr / trows, row = rr - r * trows;
      const int gy = y0 + row;
      const float* srow = pbase + r * plane + (int64_t)gy * jb.pitch;
      float* drow = sp + (r * a.prow + row) * TPITCH;
      DPM_CHECK(row < a.prow && (r * a.prow + row + 1) * TPITCH <= a.pbuf && tcols <= TPITCH,
                "P chunk fits its buffer");
      for (int col = lane; col < tcols; col += 32) {
        const int gx = x0 + col;
        const bool ok = gy < jb.H && gx < jb.W;
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(drow + col);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa),
                     "l"(ok ? srow + gx : a.P), "r"(ok ? 4 : 0));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  int t = blockIdx.x, rc = 0, buf = 0;
  if (t < a.ntiles) issue(t, 0, 0);
  unsigned long long acc[MP][NP];
  while (t < a.ntiles) {
    const dpm_corr_tile tile = a.tiles[t];
    const dpm_corr_job& job = a.jobs[tile.job];
    const int R = job.R, w = job.w;
    if (rc == 0) {
#pragma unroll
      for (int p = 0; p < MP; ++p)
#pragma unroll
        for (int f = 0; f < NP; ++f) acc[p][f] = 0ull;
    }
    int nt = t, nrc = rc + FEW_RCH;
    if (nrc >= R) {
      nt = t + gridDim.x;
      nrc = 0;
    }
    __syncthreads();  // buffer buf ^ 1 (step s-1) and the partial sums are free
    if (nt < a.ntiles) {
      issue(nt, nrc, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();  // step s resident
    const int nr = min(FEW_RCH, R - rc);
    const float* sp = sP0 + buf * a.pbuf + (wy * MP + i0) * TPITCH + lane;
    const float* sg = sG0 + buf * a.gbuf + i0 * NF;
    DPM_CHECK(((nr - 1) * PROW + wy * MP + i0 + MP + KS - 1) * TPITCH <= a.pbuf && w <= a.w_max &&
                  (w * nr * FH) * NF <= a.gbuf,
              "compute reads stay inside the staged chunk");
    if (wk == SK - 1)
      few_chunk<KS_LAST, MP, NF, FH, TPITCH, PROW>(acc, sp, sg, w, nr);
    else
      few_chunk<KS, MP, NF, FH, TPITCH, PROW>(acc, sp, sg, w, nr);
    if (nt != t) {  // last chunk of the tile: sum the filter-row slices, store
      if constexpr (SK > 1) {
        if (wk > 0) {
          unsigned long long* x = reinterpret_cast<unsigned long long*>(sX) +
                                  (((wk - 1) * 2 + wy) * MP * NP) * 32 + lane;
#pragma unroll
          for (int p = 0; p < MP; ++p)
#pragma unroll
            for (int f = 0; f < NP; ++f) x[(p * NP + f) * 32] = acc[p][f];
        }
        __syncthreads();
        if (wk == 0) {
#pragma unroll 1
          for (int k = 1; k < SK; ++k) {  // fixed order: deterministic sums
            const unsigned long long* x = reinterpret_cast<const unsigned long long*>(sX) +
                                          (((k - 1) * 2 + wy) * MP * NP) * 32 + lane;
#pragma unroll
            for (int p = 0; p < MP; ++p)
#pragma unroll
              for (int f = 0; f < NP; ++f) {
                unsigned long long v = x[(p * NP + f) * 32], s;
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(acc[p][f]), "l"(v));
                acc[p][f] = s;
              }
          }
        }
      }
      if (wk == 0) {
        const int ho = job.H - FH + 1, wo = job.W - w + 1;
        const int x = tile.tx * 32 + lane, yb = tile.ty * FEW_TY + wy * MP;
        const int wp = s_pitch(wo);
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          float vmax = -INFINITY, vmin = INFINITY;
          if (f < job.nf) {
            float* dst = a.S + job.s_off + (int64_t)f * ho * wp;
#pragma unroll
            for (int p = 0; p < MP; ++p) {
              float lo, hi;
              asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[p][f / 2]));
              const float v = (f & 1) ? hi : lo;
              const int y = yb + p;
              if (x < wo && y < ho) {
                dst[(int64_t)y * wp + x] = v;
                vmax = fmaxf(vmax, v);
                vmin = fminf(vmin, v);
              }
            }
          }
          if (a.ranges != nullptr && job.range_idx >= 0 && f < job.nf) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
              vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
            }
            if (lane == 0 && vmax >= vmin) {
              atomicMax(a.ranges + 2 * (job.range_idx + f), float_key(vmax));
              atomicMin(a.ranges + 2 * (job.range_idx + f) + 1, float_key(vmin));
            }
          }
        }
      }
    }
    t = nt;
    rc = nrc;
    buf ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

typedef void (*few_fn)(const FewArgs);

// compile-time tile pitch: 40 floats for filters up to 9 wide, 48 up to 17
template <int FH, int TP>
static few_fn few_by_nf(int nf) {
  if (nf <= 2) return corr_few_kernel<FH, 2, TP>;
  if (nf <= 4) return corr_few_kernel<FH, 4, TP>;
  if (nf <= 6) return corr_few_kernel<FH, 6, TP>;
  return corr_few_kernel<FH, 8, TP>;
}

template <int FH>
static few_fn few_by_w(int nf, int tp) {
  return tp == 40 ? few_by_nf<FH, 40>(nf) : few_by_nf<FH, 48>(nf);
}

static int few_pitch(int w_max) { return w_max <= 9 ? 40 : w_max <= 17 ? 48 : 0; }

static few_fn few_kernel_for(int h, int nf, int tp) {
  switch (h) {
    case 2: return few_by_w<2>(nf, tp);
    case 3: return few_by_w<3>(nf, tp);
    case 4: return few_by_w<4>(nf, tp);
    case 5: return few_by_w<5>(nf, tp);
    case 6: return few_by_w<6>(nf, tp);
    case 7: return few_by_w<7>(nf, tp);
    case 8: return few_by_w<8>(nf, tp);
    case 11: return few_by_w<11>(nf, tp);
    case 15: return few_by_w<15>(nf, tp);
    default: return nullptr;
  }
}

static int nf_kernel(int nf) { return nf <= 2 ? 2 : nf <= 4 ? 4 : nf <= 6 ? 6 : 8; }

// Launch for a few-filter class (called by dpm_correlate); returns
// DPM_ERR_UNSUPPORTED when the class has no few-filter kernel.
int launch_corr_few(const float* P, const float* G, float* S, const dpm_corr_job* jobs,
                    const dpm_corr_tile* tiles, int ntiles, int h, int nf, int w_max,
                    uint32_t* ranges, cudaStream_t st) {
  const int tpitch = few_pitch(w_max);
  few_fn fn = nf >= 1 && nf <= 8 && tpitch > 0 ? few_kernel_for(h, nf, tpitch) : nullptr;
  if (fn == nullptr) return DPM_ERR_UNSUPPORTED;
  const int nfk = nf_kernel(nf);
  const int sk = few_split(h, nfk), ks = few_ks(h, nfk);
  FewArgs a{P, G, S, jobs, tiles, ntiles, w_max, ranges, 0, 0, 0};
  a.prow = FEW_TY + sk * ks - 1;  // rows the last filter-row slice may touch
  a.pbuf = (FEW_RCH * a.prow * tpitch + 3) & ~3;
  a.gbuf = (h * w_max * FEW_RCH * nfk + 3) & ~3;
  const size_t xbuf = (size_t)(sk - 1) * 2 * FEW_MP * nfk * 32;
  const size_t smem = sizeof(float) * (2 * (size_t)a.pbuf + 2 * (size_t)a.gbuf + xbuf);
  DPM_REQUIRE(smem <= 227 * 1024, "dpm_correlate: h=%d w=%d nf=%d needs %zu B shared memory", h,
              w_max, nf, smem);
  DPM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148, per_sm = 0;
  DPM_CUDA(cudaGetDevice(&dev));
  DPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int threads = 64 * sk;
  DPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm < 1) per_sm = 1;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
  fn<<<grid, threads, smem, st>>>(a);
  DPM_LAUNCHED("corr_few_kernel");
  return DPM_OK;
}

}  // namespace dpm
