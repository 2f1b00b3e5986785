// 32-channel HOG feature pyramid on the device:
// images in, the X arena ([H][W][32] float32 per level, the layout K1
// reads) out.  Generalises the reference's 9-bin demo extractor
// (cpdetect/features.py:16-68) to the DPM v5 feature layout on the
// pyramid geometry of geometry.build_pyramid; oracle/hog_oracle.py states
// the algorithm and is the parity checker.
//
//   dpm_resample : level k = box-filter resampled to floor(H 2^-k/10) x
//                  floor(W 2^-k/10) pixels -- levels 0..9 from the image
//                  (uint8 or float32), level k >= 10 from level k-10's
//                  resampled image (one launch per octave wave);
//   dpm_hog      : per-pixel gradient (max-magnitude colour channel,
//                  clamped central differences) and 18-way orientation,
//                  bilinear soft binning into 4x4-pixel cells, the 4
//                  block normalisations, 18 + 9 + 4 + 1 features.
//
// The discrete steps are computed with round-to-nearest FP32 operations in a
// fixed order (no FMA contraction), the oracle emulates them bit for bit, so
// orientation bins agree exactly; histograms and features are FP32 sums
// compared at 1e-5.
#include <type_traits>

#include "common.cuh"

namespace dpm {

constexpr int HOG_SBIN = 4;
constexpr int HOG_TC = 16;                       // cells per tile side
constexpr int HOG_TP = HOG_TC * HOG_SBIN + 4;    // staged pixels per side (2 each side)
constexpr int HOG_THREADS = HOG_TC * HOG_TC;     // one thread per cell
constexpr int HOG_HPITCH = 19;                   // shared histogram row pitch (18 bins)
constexpr int RS_THREADS = 256;

__constant__ float kHogU[9] = {0x1p+0f,         0x1.e11f64p-1f,  0x1.8836fap-1f,
                               0x1p-1f,         0x1.63a1a8p-3f,  -0x1.63a1a8p-3f,
                               -0x1p-1f,        -0x1.8836fap-1f, -0x1.e11f64p-1f};
__constant__ float kHogV[9] = {0.0f,           0x1.5e3a88p-2f, 0x1.491b76p-1f,
                               0x1.bb67aep-1f, 0x1.f838b8p-1f, 0x1.f838b8p-1f,
                               0x1.bb67aep-1f, 0x1.491b76p-1f, 0x1.5e3a88p-2f};

template <typename T>
__device__ __forceinline__ float pix(const T* p) { return (float)*p; }

// Box-filter resampling, one thread per output pixel (all channels).  CC > 0
// fixes the channel count at compile time (unrolled, 32-bit pixel indices);
// the float operations and their order are the same for every CC.
template <typename T, int CC>
__device__ __forceinline__ void resample_body(const T* __restrict__ img, float* __restrict__ out,
                                              const dpm_resample_job& j, int blk) {
  const int C = CC ? CC : j.C;
  constexpr int CM = CC ? CC : 4;
  const int e = blk * RS_THREADS + (int)threadIdx.x;  // Hs * Ws * C fits 31 bits (prepare)
  if (e >= j.Hs * j.Ws) return;
  const int oy = e / j.Ws, ox = e - oy * j.Ws;
  const float sy = __fdiv_rn((float)j.H, (float)j.Hs), sx = __fdiv_rn((float)j.W, (float)j.Ws);
  const float ay = __fmul_rn((float)oy, sy), by = __fmul_rn((float)(oy + 1), sy);
  const float ax = __fmul_rn((float)ox, sx), bx = __fmul_rn((float)(ox + 1), sx);
  const int iy0 = (int)floorf(ay), iy1 = min((int)ceilf(by), j.H);
  const int ix0 = (int)floorf(ax), ix1 = min((int)ceilf(bx), j.W);
  const T* base = img + j.img_off;
  const int nx = ix1 - ix0;
  DPM_CHECK(iy0 >= 0 && ix0 >= 0 && iy1 <= j.H && ix1 <= j.W && nx >= 1, "box support inside the source");
  float acc[CM];
#pragma unroll
  for (int c = 0; c < CM; ++c) acc[c] = 0.f;
  if (nx <= 4) {  // every pyramid step (scale < 3): column weights once, not once per row
    float wxs[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      wxs[k] = __fsub_rn(fminf((float)(ix0 + k + 1), bx), fmaxf((float)(ix0 + k), ax));
    for (int iy = iy0; iy < iy1; ++iy) {
      const float wy = __fsub_rn(fminf((float)(iy + 1), by), fmaxf((float)iy, ay));
      float row[CM];
#pragma unroll
      for (int c = 0; c < CM; ++c) row[c] = 0.f;
      const T* p = base + (iy * j.W + ix0) * C;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nx) {
#pragma unroll
          for (int c = 0; c < CM; ++c)
            if (c < C) row[c] = __fadd_rn(row[c], __fmul_rn(wxs[k], pix(p + k * C + c)));
        }
#pragma unroll
      for (int c = 0; c < CM; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(wy, row[c]));
    }
  } else {
    for (int iy = iy0; iy < iy1; ++iy) {
      const float wy = __fsub_rn(fminf((float)(iy + 1), by), fmaxf((float)iy, ay));
      float row[CM];
#pragma unroll
      for (int c = 0; c < CM; ++c) row[c] = 0.f;
      for (int ix = ix0; ix < ix1; ++ix) {
        const float wx = __fsub_rn(fminf((float)(ix + 1), bx), fmaxf((float)ix, ax));
        const T* p = base + (iy * j.W + ix) * C;
#pragma unroll
        for (int c = 0; c < CM; ++c)
          if (c < C) row[c] = __fadd_rn(row[c], __fmul_rn(wx, pix(p + c)));
      }
#pragma unroll
      for (int c = 0; c < CM; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(wy, row[c]));
    }
  }
  const float d = __fmul_rn(sy, sx);
  float* o = out + j.out_off + e * C;
#pragma unroll
  for (int c = 0; c < CM; ++c)
    if (c < C) o[c] = __fdiv_rn(acc[c], d);
}

template <typename T>
__global__ void __launch_bounds__(RS_THREADS)
resample_kernel(const T* __restrict__ img, float* __restrict__ out,
                const dpm_resample_job* __restrict__ jobs, int njobs) {
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_resample_job j = jobs[jid];
  const int blk = blockIdx.x - j.block0;
  if (j.C == 3) resample_body<T, 3>(img, out, j, blk);
  else if (j.C == 1) resample_body<T, 1>(img, out, j, blk);
  else resample_body<T, 0>(img, out, j, blk);
}

// Gradient magnitude and orientation bin (0..17) of resampled pixel (y, x).
template <int CC>
__device__ __forceinline__ void grad_bin(const float* __restrict__ R, int Hs, int Ws, int Cj, int y,
                                         int x, float& v, int& bin) {
  const int C = CC ? CC : Cj;  // CC > 0: compile-time channel count (unrolled)
  const int xr = min(x + 1, Ws - 1), xl = max(x - 1, 0);
  const int yd = min(y + 1, Hs - 1), yu = max(y - 1, 0);
  const float* pr = R + (y * Ws + xr) * C;  // Hs * Ws * C fits 31 bits (prepare)
  const float* pl = R + (y * Ws + xl) * C;
  const float* pd = R + (yd * Ws + x) * C;
  const float* pu = R + (yu * Ws + x) * C;
  float best = -1.f, bdx = 0.f, bdy = 0.f;
#pragma unroll
  for (int c = 0; c < (CC ? CC : 4); ++c) {
    if (c >= C) break;
    const float dx = __fsub_rn(pr[c], pl[c]);
    const float dy = __fsub_rn(pd[c], pu[c]);
    const float m = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
    if (c == 0 || m > best) {
      best = m;
      bdx = dx;
      bdy = dy;
    }
  }
  v = __fsqrt_rn(best);
  float bd = 0.f;
  int bo = 0;
#pragma unroll
  for (int o = 0; o < 9; ++o) {
    const float dot = __fadd_rn(__fmul_rn(kHogU[o], bdx), __fmul_rn(kHogV[o], bdy));
    if (dot > bd) {
      bd = dot;
      bo = o;
    } else if (-dot > bd) {
      bd = -dot;
      bo = o + 9;
    }
  }
  bin = bo;
}

// Cell histograms of one 16 x 16-cell tile: (v, bin) of the tile's pixels
// plus a 2-pixel apron staged in shared memory, then each thread gathers
// its cell's 8 x 8-pixel bilinear support in a fixed order.  Writes the 18
// bins and the energy E of every cell.
__global__ void __launch_bounds__(HOG_THREADS)
hog_cells_kernel(const float* __restrict__ R, float* __restrict__ hist,
                 const dpm_hog_job* __restrict__ jobs, int njobs) {
  __shared__ float sv[HOG_TP * HOG_TP];
  __shared__ uint8_t sb[HOG_TP * HOG_TP];
  __shared__ float sh[HOG_THREADS * HOG_HPITCH];
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_hog_job j = jobs[jid];
  const int Hc = j.Hs / HOG_SBIN, Wc = j.Ws / HOG_SBIN;
  const int ntx = (Wc + HOG_TC - 1) / HOG_TC;
  const int tile = blockIdx.x - j.block0;
  const int cy0 = (tile / ntx) * HOG_TC, cx0 = (tile % ntx) * HOG_TC;
  const int py0 = cy0 * HOG_SBIN - 2, px0 = cx0 * HOG_SBIN - 2;
  const float* Rl = R + j.r_off;
  auto stage = [&](auto cc) {
    for (int e = threadIdx.x; e < HOG_TP * HOG_TP; e += HOG_THREADS) {
      const int ry = e / HOG_TP, rx = e - ry * HOG_TP;
      const int y = py0 + ry, x = px0 + rx;
      float v = 0.f;
      int b = 0;
      // only pixels of whole cells contribute
      if (y >= 0 && x >= 0 && y < Hc * HOG_SBIN && x < Wc * HOG_SBIN)
        grad_bin<decltype(cc)::value>(Rl, j.Hs, j.Ws, j.C, y, x, v, b);
      sv[e] = v;
      sb[e] = (uint8_t)b;
    }
  };
  if (j.C == 3) stage(std::integral_constant<int, 3>{});
  else if (j.C == 1) stage(std::integral_constant<int, 1>{});
  else stage(std::integral_constant<int, 0>{});
  float* h = sh + threadIdx.x * HOG_HPITCH;
#pragma unroll
  for (int o = 0; o < 18; ++o) h[o] = 0.f;
  __syncthreads();
  const int cy = cy0 + (int)threadIdx.x / HOG_TC, cx = cx0 + (int)threadIdx.x % HOG_TC;
  if (cy >= Hc || cx >= Wc) return;
  // support: pixels 4c-2 .. 4c+5 on each axis (bilinear weights over cell centres)
  const int ly = (cy - cy0) * HOG_SBIN, lx = (cx - cx0) * HOG_SBIN;  // staged index of pixel 4c-2
  // Bilinear weight of support pixel a (pixel 4c - 2 + a) towards cell c:
  // ((p + 0.5) / 4 - 0.5 has fraction (2a + 1) / 8 below the cell centre and
  // 1 - that above it; every step is exact in FP32, so these constants are
  // the values the rounded intrinsics produce (oracle/hog_oracle.py).
  constexpr float kW[2 * HOG_SBIN] = {0.125f, 0.375f, 0.625f, 0.875f, 0.875f, 0.625f, 0.375f, 0.125f};
  const float* pv = sv + ly * HOG_TP + lx;
  const uint8_t* pb = sb + ly * HOG_TP + lx;
#pragma unroll
  for (int a = 0; a < 2 * HOG_SBIN; ++a) {
#pragma unroll
    for (int b = 0; b < 2 * HOG_SBIN; ++b) {
      const int si = a * HOG_TP + b;
      float* hb = h + pb[si];
      *hb = __fadd_rn(*hb, __fmul_rn(__fmul_rn(kW[a], kW[b]), pv[si]));
    }
  }
  float* g = hist + j.h_off + ((int64_t)cy * Wc + cx) * 20;  // 18 bins, E, pad
  float E = 0.f;
#pragma unroll
  for (int o = 0; o < 9; ++o) {
    const float s = __fadd_rn(h[o], h[o + 9]);
    E = __fadd_rn(E, __fmul_rn(s, s));
  }
#pragma unroll
  for (int o = 0; o < 18; ++o) g[o] = h[o];
  g[18] = E;
}

// Normalisations and the 32 features of every cell, written to the level's
// X block [Hc][Wc][32].
__global__ void __launch_bounds__(256)
hog_feat_kernel(const float* __restrict__ hist, float* __restrict__ X,
                const dpm_hog_job* __restrict__ jobs, int njobs, int64_t nblocks_total) {
  (void)nblocks_total;
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_hog_job j = jobs[jid];
  const int Hc = j.Hs / HOG_SBIN, Wc = j.Ws / HOG_SBIN;
  const int ntx = (Wc + HOG_TC - 1) / HOG_TC;
  const int tile = blockIdx.x - j.block0;
  const int cy = (tile / ntx) * HOG_TC + (int)threadIdx.x / HOG_TC;
  const int cx = (tile % ntx) * HOG_TC + (int)threadIdx.x % HOG_TC;
  if (cy >= Hc || cx >= Wc) return;
  const float* H = hist + j.h_off;
  auto E = [&](int y, int x) {
    y = min(max(y, 0), Hc - 1);
    x = min(max(x, 0), Wc - 1);
    return H[((int64_t)y * Wc + x) * 20 + 18];
  };
  auto nrm = [&](int dy, int dx) {  // 2x2 block with top-left (cy+dy, cx+dx)
    const float s = __fadd_rn(__fadd_rn(__fadd_rn(E(cy + dy, cx + dx), E(cy + dy, cx + dx + 1)),
                                        E(cy + dy + 1, cx + dx)),
                              E(cy + dy + 1, cx + dx + 1));
    return __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(s, 1e-4f)));
  };
  const float n[4] = {nrm(0, 0), nrm(-1, 0), nrm(0, -1), nrm(-1, -1)};
  const float* h = H + ((int64_t)cy * Wc + cx) * 20;
  float f[32];
  float tex[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int o = 0; o < 18; ++o) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float t = fminf(__fmul_rn(h[o], n[k]), 0.2f);
      acc = __fadd_rn(acc, t);
      tex[k] = __fadd_rn(tex[k], t);
    }
    f[o] = __fmul_rn(0.5f, acc);
  }
#pragma unroll
  for (int o = 0; o < 9; ++o) {
    const float s = __fadd_rn(h[o], h[o + 9]);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc = __fadd_rn(acc, fminf(__fmul_rn(s, n[k]), 0.2f));
    f[18 + o] = __fmul_rn(0.5f, acc);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) f[27 + k] = __fmul_rn(0.2357f, tex[k]);
  f[31] = 0.f;
  float4* dst = reinterpret_cast<float4*>(X + j.x_off + ((int64_t)cy * Wc + cx) * 32);
#pragma unroll
  for (int q = 0; q < 8; ++q) dst[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
}

}  // namespace dpm

using namespace dpm;

extern "C" int64_t dpm_resample_prepare(dpm_resample_job* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_resample_prepare: bad table");
  int64_t b = 0;
  for (int i = 0; i < njobs; ++i) {
    dpm_resample_job& j = jobs[i];
    DPM_REQUIRE(j.H >= 1 && j.W >= 1 && j.Hs >= 1 && j.Ws >= 1 && j.Hs <= j.H && j.Ws <= j.W &&
                    j.C >= 1 && j.C <= 4 && j.img_off >= 0 && j.out_off >= 0,
                "dpm_resample_prepare: job %d resamples %dx%dx%d to %dx%d", i, j.H, j.W, j.C, j.Hs,
                j.Ws);
    DPM_REQUIRE((int64_t)j.H * j.W * j.C < INT32_MAX, "dpm_resample_prepare: job %d too large", i);
    j.block0 = (int32_t)b;
    b += ((int64_t)j.Hs * j.Ws + RS_THREADS - 1) / RS_THREADS;
  }
  DPM_REQUIRE(b <= INT32_MAX, "dpm_resample_prepare: too many blocks");
  return b;
}

extern "C" int dpm_resample(const void* img, int u8, float* out, const dpm_resample_job* jobs,
                            int njobs, int64_t nblocks, void* stream) {
  DPM_REQUIRE(img && out && jobs, "dpm_resample: null pointer");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  if (u8)
    resample_kernel<uint8_t><<<(unsigned)nblocks, RS_THREADS, 0, as_stream(stream)>>>(
        static_cast<const uint8_t*>(img), out, jobs, njobs);
  else
    resample_kernel<float><<<(unsigned)nblocks, RS_THREADS, 0, as_stream(stream)>>>(
        static_cast<const float*>(img), out, jobs, njobs);
  DPM_LAUNCHED("resample_kernel");
  return DPM_OK;
}

extern "C" int64_t dpm_hog_prepare(dpm_hog_job* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_hog_prepare: bad table");
  int64_t b = 0;
  for (int i = 0; i < njobs; ++i) {
    dpm_hog_job& j = jobs[i];
    DPM_REQUIRE(j.Hs >= HOG_SBIN && j.Ws >= HOG_SBIN && j.C >= 1 && j.C <= 4 && j.r_off >= 0 &&
                    j.x_off >= 0 && j.h_off >= 0 && j.x_off % 4 == 0,
                "dpm_hog_prepare: job %d (%dx%dx%d)", i, j.Hs, j.Ws, j.C);
    DPM_REQUIRE((int64_t)j.Hs * j.Ws * j.C < INT32_MAX, "dpm_hog_prepare: job %d too large", i);
    j.block0 = (int32_t)b;
    const int Hc = j.Hs / HOG_SBIN, Wc = j.Ws / HOG_SBIN;
    b += (int64_t)((Hc + HOG_TC - 1) / HOG_TC) * ((Wc + HOG_TC - 1) / HOG_TC);
  }
  DPM_REQUIRE(b <= INT32_MAX, "dpm_hog_prepare: too many blocks");
  return b;
}

extern "C" int dpm_hog(const float* R, float* hist, float* X, const dpm_hog_job* jobs, int njobs,
                       int64_t nblocks, void* stream) {
  DPM_REQUIRE(R && hist && X && jobs, "dpm_hog: null pointer");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  hog_cells_kernel<<<(unsigned)nblocks, HOG_THREADS, 0, as_stream(stream)>>>(R, hist, jobs, njobs);
  DPM_LAUNCHED("hog_cells_kernel");
  hog_feat_kernel<<<(unsigned)nblocks, 256, 0, as_stream(stream)>>>(hist, X, jobs, njobs, nblocks);
  DPM_LAUNCHED("hog_feat_kernel");
  return DPM_OK;
}
