// K3 (part placement) and K4 (root + parts assembly).
//
// Reference: _placement_grid (detection.py:320-373), best_part_placement
// (detection.py:180-207) and the assembly of detect / dense_detect
// (detection.py:449, 509-538; 590-613).
//
// Exact semantics (bit-identical values and argmaxes for a given FP32 map):
//   x pass: for every map row y and centre cx = scale*rx + ax,
//           best over dx = -r..r (ascending, strict '>') of
//           S[y][cx+dx] - (c_dx*dx + (c_dxx*dx)*dx), -inf outside the map;
//   y pass: best over dy = -r..r (ascending, strict '>') of
//           xbest[cy+dy] - (c_dy*dy + (c_dyy*dy)*dy), cy = scale*ry + ay;
//   total = root + sum_parts best + bias, summed in part order.
// Penalties use round-to-nearest intrinsics (no FMA contraction), matching
// the reference's unfused float64 evaluation.
//
// One kernel: each CTA owns a 32 x 64 tile of roots of one (image,
// component, root level).  Per part it stages the S band its windows touch
// in shared memory, runs the x pass for every band row at the 32 centre
// columns (64-row tiles keep the band overlap between vertically adjacent
// tiles at 2r / 128 rows), then the y pass for its roots; exact FP64 values
// are recomputed from the staged band.  Root + parts + bias are summed in
// registers and written with the part positions; detections >= tau are
// compacted with one atomic per warp.
// Candidates are screened in FP32, branch free: the scan keeps the running
// maximum m1 (first index on ties, strict '>') and the best value m2 of all
// other candidates.  With E2 = 2^-19 * (max|S| + max pen_x + max pen_y) at
// least twice the FP32 error of any candidate value, m2 < m1 - E2 proves the
// FP32 winner is the unique exact winner; otherwise (ties, near ties) the
// candidates within E2 of m1 are rescanned in FP64 in the reference's order.
//
// radius < 0 selects the unbounded generalised distance transform, realised
// as the window of radius r* computed from the map's
// range, beyond which no maximiser lies.  Radii above RCAP use unstaged loops
// with the same arithmetic.
#include <math.h>

#include "common.cuh"

namespace dpm {

constexpr int RCAP = 16;                                  // staged-path radius cap
constexpr int PT_W = 32;                                  // root columns per tile (lanes)
constexpr int PT_H = 64;                                  // root rows per tile
constexpr int PT_THREADS = 512;
constexpr int PT_WARPS = PT_THREADS / 32;
constexpr int BAND_MAX = 2 * (PT_H - 1) + 1 + 2 * RCAP;   // 159 (scale <= 2)
constexpr int COLS_PITCH = 2 * (PT_W - 1) + 1 + 2 * RCAP + 2;  // 97

__device__ __forceinline__ double pen(double c1, double c2, int d) {
  const double dd = (double)d;
  return __dadd_rn(__dmul_rn(c1, dd), __dmul_rn(__dmul_rn(c2, dd), dd));
}

__device__ __forceinline__ double pen_absmax(double c1, double c2, int r) {
  double m = fmax(fabs(pen(c1, c2, -r)), fabs(pen(c1, c2, r)));
  if (c2 > 0.0) m = fmax(m, c1 * c1 / (4.0 * c2));
  return m;
}

// r* of App. A.2 for one axis from the map range; +1 guards the floor.
__device__ __forceinline__ int radius_of(const dpm_place_job& j, float vmax, float vmin, bool x_axis) {
  if (j.radius >= 0) return j.radius;
  const double a = x_axis ? j.cdxx : j.cdyy, b = x_axis ? j.cdx : j.cdy;
  const double ao = x_axis ? j.cdyy : j.cdxx, bo = x_axis ? j.cdy : j.cdx;
  const double dprime = ((double)vmax - (double)vmin) + bo * bo / (4.0 * ao);
  return (int)floor((fabs(b) + sqrt(b * b + 4.0 * a * dprime)) / (2.0 * a)) + 1;
}

struct JobRange {
  float vmax, vmin;
  int rx, ry;
  float E2;
};

__device__ __forceinline__ JobRange job_range(const dpm_place_job& pj, const uint32_t* ranges) {
  JobRange jr;
  jr.vmax = key_float(ranges[2 * pj.range_idx]);
  jr.vmin = key_float(ranges[2 * pj.range_idx + 1]);
  jr.rx = radius_of(pj, jr.vmax, jr.vmin, true);
  jr.ry = radius_of(pj, jr.vmax, jr.vmin, false);
  const double mabs = fmax(fabs((double)jr.vmax), fabs((double)jr.vmin));
  jr.E2 = (float)ldexp(mabs + pen_absmax(pj.cdx, pj.cdxx, jr.rx) + pen_absmax(pj.cdy, pj.cdyy, jr.ry),
                       -19);
  return jr;
}

__device__ __forceinline__ uint32_t pack_pos(int y, int x) {
  return ((uint32_t)(uint16_t)(int16_t)y << 16) | (uint32_t)(uint16_t)(int16_t)x;
}

// Branch-free FP32 screen of one window (see file comment).
struct Screen {
  float m1, m2;
  int i1;
};

__device__ __forceinline__ void screen_init(Screen& sc, int r) {
  sc.m1 = -INFINITY;
  sc.m2 = -INFINITY;
  sc.i1 = -r;
}

__device__ __forceinline__ void screen_add(Screen& sc, float v, int d) {
  const bool gt = v > sc.m1;
  sc.m2 = fmaxf(sc.m2, fminf(sc.m1, v));
  sc.i1 = gt ? d : sc.i1;
  sc.m1 = fmaxf(sc.m1, v);
}

// Placement of one part for one root via direct global loads (any radius).
__device__ void place_unstaged(const float* __restrict__ sm, const dpm_place_job& pj, int cy,
                               int cx, int rx_, int ry_, double& best, int& bdy, int& bdx) {
  best = -INFINITY;
  bdy = -ry_;
  bdx = -rx_;
  for (int dy = -ry_; dy <= ry_; ++dy) {
    const int y = cy + dy;
    if (y < 0 || y >= pj.Hp) continue;
    double xb = -INFINITY;
    int xd = -rx_;
    const int lo = max(-rx_, -cx), hi = min(rx_, pj.Wp - 1 - cx);
    for (int dx = lo; dx <= hi; ++dx) {
      const double c = __dadd_rn((double)__ldg(sm + (int64_t)y * pj.Wp + cx + dx),
                                 -pen(pj.cdx, pj.cdxx, dx));
      if (c > xb) { xb = c; xd = dx; }
    }
    const double cand = __dadd_rn(xb, -pen(pj.cdy, pj.cdyy, dy));
    if (cand > best) { best = cand; bdy = dy; bdx = xd; }
  }
}

struct __align__(16) PlaceSmem {
  float s[BAND_MAX * COLS_PITCH];  // staged S band (-inf outside the map)
  float x32[BAND_MAX * PT_W];      // x-pass winners' FP32 screen values
  int8_t xdx[BAND_MAX * PT_W];     // x-pass winning dx
  float npx[2 * RCAP + 1];         // -pen_x(dx) in FP32 (screening only)
  float npy[2 * RCAP + 1];
  JobRange jr;                     // r*, E2 of the current part (computed once per CTA)
};

__global__ void __launch_bounds__(PT_THREADS, 2)
place_assemble_kernel(const float* __restrict__ S, const dpm_place_job* __restrict__ pjobs,
                      const dpm_asm_job* __restrict__ ajobs, int najobs,
                      const uint32_t* __restrict__ ranges, double* __restrict__ total,
                      uint32_t* __restrict__ pos, double* __restrict__ placed, double tau,
                      dpm_detection* __restrict__ dets, int max_dets, int* __restrict__ det_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PlaceSmem& sh = *reinterpret_cast<PlaceSmem*>(smem_raw);
  const int jid = find_job(ajobs, najobs, blockIdx.x);
  const dpm_asm_job aj = ajobs[jid];
  const int hr = aj.ry1 - aj.ry0 + 1, wr = aj.rx1 - aj.rx0 + 1;
  const int ntx = (wr + PT_W - 1) / PT_W;
  const int tile = blockIdx.x - aj.block0;
  const int ty0 = (tile / ntx) * PT_H, tx0 = (tile % ntx) * PT_W;  // offsets inside the rect
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int RPT = PT_H / PT_WARPS;  // roots per thread (4)
  const int ix = tx0 + lane;
  const bool col_ok = ix < wr;
  const int rx = aj.rx0 + ix;
  const int ry_lo = aj.ry0 + ty0;
  const int ry_hi = aj.ry0 + min(ty0 + PT_H, hr) - 1;
  const int rx_lo = aj.rx0 + tx0;

  double tot[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int iy = ty0 + warp + PT_WARPS * k;
    tot[k] = 0.0;
    if (aj.root_off >= 0 && col_ok && iy < hr)
      tot[k] = (double)__ldg(S + aj.root_off + (int64_t)(aj.ry0 + iy) * aj.root_pitch + rx);
  }

  for (int p = 0; p < aj.nparts; ++p) {
    const dpm_place_job pj = pjobs[aj.part_job0 + p];
    __syncthreads();  // previous part done with the shared band and parameters
    if (threadIdx.x == 0) sh.jr = job_range(pj, ranges);
    if (threadIdx.x >= 32 && threadIdx.x <= 32 + 2 * RCAP) {
      const int d = threadIdx.x - 32 - RCAP;
      sh.npx[d + RCAP] = (float)(-pen(pj.cdx, pj.cdxx, d));
      sh.npy[d + RCAP] = (float)(-pen(pj.cdy, pj.cdyy, d));
    }
    __syncthreads();
    const JobRange jr = sh.jr;
    const float* sm = S + pj.s_off;
    const int cx = pj.scale * rx + pj.ax;
    if (!(jr.rx <= RCAP && jr.ry <= RCAP && pj.scale <= 2)) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int iy = ty0 + warp + PT_WARPS * k;
        if (!col_ok || iy >= hr) continue;
        const int cy = pj.scale * (aj.ry0 + iy) + pj.ay;
        double best;
        int bdy, bdx;
        place_unstaged(sm, pj, cy, cx, jr.rx, jr.ry, best, bdy, bdx);
        tot[k] = __dadd_rn(tot[k], best);
        const int64_t o = ((int64_t)p * hr + iy) * wr + ix;
        if (aj.pos_off >= 0) pos[aj.pos_off + o] = pack_pos(cy + bdy, cx + bdx);
        if (aj.placed_off >= 0) placed[aj.placed_off + o] = best;
      }
      continue;
    }
    // band: map rows / cols the windows of this tile reach
    const int yb0 = pj.scale * ry_lo + pj.ay - jr.ry;
    const int nrows = pj.scale * (ry_hi - ry_lo) + 1 + 2 * jr.ry;
    const int xb0 = pj.scale * rx_lo + pj.ax - jr.rx;
    const int ncols = pj.scale * (PT_W - 1) + 1 + 2 * jr.rx;

    // stage the band: warp per row, up to 3 loads in flight per lane, -inf outside
    for (int r = warp; r < nrows; r += PT_WARPS) {
      const int y = yb0 + r;
      const bool yok = y >= 0 && y < pj.Hp;
      const float* srow = sm + (int64_t)(yok ? y : 0) * pj.Wp;
      float v[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int c = lane + 32 * q, x = xb0 + c;
        v[q] = (yok && c < ncols && x >= 0 && x < pj.Wp) ? __ldg(srow + x) : -INFINITY;
      }
      float* drow = sh.s + r * COLS_PITCH;
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (lane + 32 * q < ncols) drow[lane + 32 * q] = v[q];
    }
    __syncthreads();

    // x pass: band row r (warp-strided), centre column = lane
    const float* npx = sh.npx + RCAP;
    for (int r = warp; r < nrows; r += PT_WARPS) {
      const float* srow = sh.s + r * COLS_PITCH + pj.scale * lane + jr.rx;  // dx = 0
      Screen sc;
      screen_init(sc, jr.rx);
      for (int dx = -jr.rx; dx <= jr.rx; ++dx) screen_add(sc, srow[dx] + npx[dx], dx);
      // the y-pass screen only needs the winner's value to FP32 accuracy
      // (the FP32 screen max is within 2^-22 M of it); exact values are
      // recomputed from the band for y winners and ties
      int xi = sc.i1;
      if (sc.m1 == -INFINITY) {  // no candidate inside the map: reference gives (-inf, -r)
        xi = -jr.rx;
      } else if (sc.m2 >= sc.m1 - jr.E2) {  // tie or near tie: exact rescan, reference order
        const float lo = sc.m1 - jr.E2;
        double xv = -INFINITY;
        xi = -jr.rx;
        for (int dx = -jr.rx; dx <= jr.rx; ++dx) {
          if (srow[dx] + npx[dx] >= lo) {
            const double e = __dadd_rn((double)srow[dx], -pen(pj.cdx, pj.cdxx, dx));
            if (e > xv) { xv = e; xi = dx; }
          }
        }
      }
      sh.x32[r * PT_W + lane] = sc.m1;
      sh.xdx[r * PT_W + lane] = (int8_t)xi;
    }
    __syncthreads();

    // y pass for this thread's roots; exact values from the staged band
    const float* npy = sh.npy + RCAP;
    const float* scol = sh.s + pj.scale * lane + jr.rx;  // band column of the centre
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int iy = ty0 + warp + PT_WARPS * k;
      if (!col_ok || iy >= hr) continue;
      const int ry = aj.ry0 + iy;
      const int cy = pj.scale * ry + pj.ay;
      const int r0 = cy - yb0;  // band row of dy = 0
      const float* xcol = sh.x32 + r0 * PT_W + lane;
      Screen sc;
      screen_init(sc, jr.ry);
      for (int dy = -jr.ry; dy <= jr.ry; ++dy) screen_add(sc, xcol[dy * PT_W] + npy[dy], dy);
      auto exact = [&](int dy) -> double {
        const int row = r0 + dy;
        const int dx = sh.xdx[row * PT_W + lane];
        const double xv = __dadd_rn((double)scol[row * COLS_PITCH + dx], -pen(pj.cdx, pj.cdxx, dx));
        return __dadd_rn(xv, -pen(pj.cdy, pj.cdyy, dy));
      };
      double best;
      int bi = sc.i1;
      if (sc.m1 == -INFINITY) {
        best = -INFINITY;
        bi = -jr.ry;
      } else if (sc.m2 >= sc.m1 - jr.E2) {
        const float lo = sc.m1 - jr.E2;
        best = -INFINITY;
        bi = -jr.ry;
        for (int dy = -jr.ry; dy <= jr.ry; ++dy) {
          if (xcol[dy * PT_W] + npy[dy] >= lo) {
            const double e = exact(dy);
            if (e > best) { best = e; bi = dy; }
          }
        }
      } else {
        best = exact(bi);
      }
      const int bdx = sh.xdx[(r0 + bi) * PT_W + lane];
      tot[k] = __dadd_rn(tot[k], best);
      const int64_t o = ((int64_t)p * hr + iy) * wr + ix;
      if (aj.pos_off >= 0) pos[aj.pos_off + o] = pack_pos(cy + bi, cx + bdx);
      if (aj.placed_off >= 0) placed[aj.placed_off + o] = best;
    }
  }

  // bias, totals, tau compaction (part positions read back from `pos`)
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int iy = ty0 + warp + PT_WARPS * k;
    const bool live = col_ok && iy < hr;
    if (live) {
      tot[k] = __dadd_rn(tot[k], aj.bias);
      if (aj.total_off >= 0) total[aj.total_off + (int64_t)iy * wr + ix] = tot[k];
    }
    if (dets == nullptr) continue;
    const bool hit = live && tot[k] >= tau;
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask == 0u) continue;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(det_count, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!hit) continue;
    const int slot = base + __popc(mask & ((1u << lane) - 1u));
    if (slot >= max_dets) continue;
    dpm_detection dd;
    dd.image = aj.image;
    dd.level = aj.level;
    dd.component = aj.component;
    dd.ry = aj.ry0 + iy;
    dd.rx = rx;
    dd.nparts = aj.nparts;
    dd.score = tot[k];
    for (int q = 0; q < DPM_MAX_PARTS; ++q)
      dd.parts[q] = (q < aj.nparts && aj.pos_off >= 0)
                        ? pos[aj.pos_off + ((int64_t)q * hr + iy) * wr + ix]
                        : 0u;
    dets[slot] = dd;
  }
}

}  // namespace dpm

using namespace dpm;

extern "C" int64_t dpm_place_prepare(dpm_place_job* jobs, int njobs) {
  if (njobs < 0 || (njobs > 0 && !jobs)) {
    set_error("dpm_place_prepare: bad job table");
    return DPM_ERR_ARG;
  }
  int64_t b = 0;
  for (int i = 0; i < njobs; ++i) {
    const dpm_place_job& j = jobs[i];
    if (j.Hp < 1 || j.Wp < 1 || j.wr < 1 || j.scale < 1 || j.radius > 32000 || j.range_idx < 0) {
      set_error("dpm_place_prepare: placement job %d has Hp=%d Wp=%d wr=%d scale=%d radius=%d "
                "range_idx=%d", i, j.Hp, j.Wp, j.wr, j.scale, j.radius, j.range_idx);
      return DPM_ERR_ARG;
    }
    if (j.radius < 0 && !(j.cdxx > 0.0 && j.cdyy > 0.0)) {
      set_error("dpm_place_prepare: placement job %d: the unbounded transform needs "
                "c_dxx, c_dyy > 0", i);
      return DPM_ERR_ARG;
    }
    jobs[i].block0 = 0;
  }
  return b;
}

extern "C" int64_t dpm_assemble_prepare(dpm_asm_job* jobs, int njobs, const dpm_place_job* pjobs,
                                        int npjobs) {
  if (njobs < 0 || (njobs > 0 && !jobs) || npjobs < 0 || (npjobs > 0 && !pjobs)) {
    set_error("dpm_assemble_prepare: bad job tables");
    return DPM_ERR_ARG;
  }
  int64_t b = 0;
  for (int i = 0; i < njobs; ++i) {
    const dpm_asm_job& j = jobs[i];
    if (j.ry1 < j.ry0 || j.rx1 < j.rx0 || j.nparts < 0 || j.nparts > DPM_MAX_PARTS ||
        j.part_job0 < 0 || j.part_job0 + j.nparts > npjobs) {
      set_error("dpm_assemble_prepare: job %d has rect (%d,%d,%d,%d) parts [%d, +%d)", i, j.ry0,
                j.ry1, j.rx0, j.rx1, j.part_job0, j.nparts);
      return DPM_ERR_ARG;
    }
    for (int p = 0; p < j.nparts; ++p) {
      const dpm_place_job& pj = pjobs[j.part_job0 + p];
      if (pj.rx0 != j.rx0 || pj.wr != j.rx1 - j.rx0 + 1) {
        set_error("dpm_assemble_prepare: job %d part %d: x-pass columns [%d, +%d) differ from the "
                  "root columns", i, p, pj.rx0, pj.wr);
        return DPM_ERR_ARG;
      }
    }
    jobs[i].block0 = (int32_t)b;
    const int64_t hr = j.ry1 - j.ry0 + 1, wr = j.rx1 - j.rx0 + 1;
    b += ((hr + PT_H - 1) / PT_H) * ((wr + PT_W - 1) / PT_W);
  }
  if (b > INT32_MAX) {
    set_error("dpm_assemble_prepare: too many CTAs");
    return DPM_ERR_ARG;
  }
  return b;
}

extern "C" int dpm_assemble(const float* S, const dpm_place_job* pjobs, const dpm_asm_job* ajobs,
                            int najobs, int64_t nblocks, const uint32_t* ranges, double* total,
                            uint32_t* pos, double* placed, double tau, dpm_detection* dets,
                            int max_dets, int* det_count, void* stream) {
  DPM_REQUIRE(S && pjobs && ajobs && ranges, "dpm_assemble: null pointer");
  DPM_REQUIRE(!dets || (det_count && pos), "dpm_assemble: detections need a counter and positions");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_assemble: nblocks");
  if (najobs == 0 || nblocks == 0) return DPM_OK;
  const size_t smem = sizeof(PlaceSmem);
  DPM_CUDA(cudaFuncSetAttribute(place_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  place_assemble_kernel<<<(unsigned)nblocks, PT_THREADS, smem, as_stream(stream)>>>(
      S, pjobs, ajobs, najobs, ranges, total, pos, placed, tau, dets, max_dets, det_count);
  DPM_LAUNCHED("place_assemble_kernel");
  return DPM_OK;
}
