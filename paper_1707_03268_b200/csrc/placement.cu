// K3 (part placement) and K4 (root + parts assembly), FP64 arithmetic on
// FP32 response maps.
//
// Reference: _placement_grid (detection.py:320-373), best_part_placement
// (detection.py:180-207) and the assembly lines of detect / dense_detect
// (detection.py:449, 509-538; 590-613).
//
// Semantics reproduced exactly (bit-identical values and argmaxes for the
// same input map, checked against the oracle):
//   x pass: for every map row y and centre column cx = scale*rx + ax,
//           best over dx = -r..r (ascending, strict '>') of
//           S[y][cx+dx] - (c_dx*dx + (c_dxx*dx)*dx), -inf outside the map;
//   y pass: best over dy = -r..r (ascending, strict '>') of
//           xbest[cy+dy] - (c_dy*dy + (c_dyy*dy)*dy), cy = scale*ry + ay.
// All penalty products/sums use round-to-nearest intrinsics so the compiler
// cannot contract them into FMAs (the reference evaluates them unfused).
// The x pass stores only the winning dx (int16); the y pass recomputes the
// winning x-pass value from S, which is the same double again.
//
// radius < 0 selects the unbounded generalised distance transform: the
// window radius becomes r* from the map's range, past
// which no maximiser can lie, so the window result equals the unbounded one.
#include <math.h>

#include "common.cuh"

namespace dpm {

constexpr int K3_THREADS = 256;

__device__ __forceinline__ double pen(double c1, double c2, int d) {
  const double dd = (double)d;
  return __dadd_rn(__dmul_rn(c1, dd), __dmul_rn(__dmul_rn(c2, dd), dd));
}

// r* of App. A.2 for one axis (a = quadratic, b = linear coefficient of that
// axis, (a_o, b_o) of the other), from the map's [min, max]; +1 guards the
// floor against rounding (any radius >= r* gives the identical result).
__device__ __forceinline__ int radius_of(const dpm_place_job& j, const uint32_t* ranges, bool x_axis) {
  if (j.radius >= 0) return j.radius;
  const float vmax = key_float(ranges[2 * j.range_idx]);
  const float vmin = key_float(ranges[2 * j.range_idx + 1]);
  const double a = x_axis ? j.cdxx : j.cdyy, b = x_axis ? j.cdx : j.cdy;
  const double ao = x_axis ? j.cdyy : j.cdxx, bo = x_axis ? j.cdy : j.cdx;
  const double dprime = ((double)vmax - (double)vmin) + bo * bo / (4.0 * ao);
  const double r = (fabs(b) + sqrt(b * b + 4.0 * a * dprime)) / (2.0 * a);
  return (int)floor(r) + 1;
}

__global__ void __launch_bounds__(K3_THREADS)
xpass_kernel(const float* __restrict__ S, int16_t* __restrict__ DX,
             const dpm_place_job* __restrict__ jobs, int njobs, const uint32_t* __restrict__ ranges) {
  const int jid = find_job(jobs, njobs, blockIdx.x);
  const dpm_place_job j = jobs[jid];
  const int64_t e = (int64_t)(blockIdx.x - j.block0) * K3_THREADS + threadIdx.x;
  if (e >= (int64_t)j.Hp * j.wr) return;
  const int y = (int)(e / j.wr), c = (int)(e - (int64_t)y * j.wr);
  const int cx = j.scale * (j.rx0 + c) + j.ax;
  const int r = radius_of(j, ranges, true);
  const float* row = S + j.s_off + (int64_t)y * j.Wp;
  const int lo = max(-r, -cx), hi = min(r, j.Wp - 1 - cx);
  double best = -INFINITY;
  int bdx = -r;
  for (int dx = lo; dx <= hi; ++dx) {
    const double cand = __dadd_rn((double)__ldg(row + cx + dx), -pen(j.cdx, j.cdxx, dx));
    if (cand > best) {
      best = cand;
      bdx = dx;
    }
  }
  DX[j.dx_off + e] = (int16_t)bdx;
}

__device__ __forceinline__ uint32_t pack_pos(int y, int x) {
  return ((uint32_t)(uint16_t)(int16_t)y << 16) | (uint32_t)(uint16_t)(int16_t)x;
}

__global__ void __launch_bounds__(K3_THREADS)
assemble_kernel(const float* __restrict__ S, const int16_t* __restrict__ DX,
                const dpm_place_job* __restrict__ pjobs, const dpm_asm_job* __restrict__ ajobs,
                int najobs, const uint32_t* __restrict__ ranges, double* __restrict__ total,
                uint32_t* __restrict__ pos, double* __restrict__ placed, double tau,
                dpm_detection* __restrict__ dets, int max_dets, int* __restrict__ det_count) {
  const int jid = find_job(ajobs, najobs, blockIdx.x);
  const dpm_asm_job aj = ajobs[jid];
  const int hr = aj.ry1 - aj.ry0 + 1, wr = aj.rx1 - aj.rx0 + 1;
  const int64_t e = (int64_t)(blockIdx.x - aj.block0) * K3_THREADS + threadIdx.x;
  const bool live = e < (int64_t)hr * wr;
  const int iy = live ? (int)(e / wr) : 0, ix = live ? (int)(e - (int64_t)iy * wr) : 0;
  const int ry = aj.ry0 + iy, rx = aj.rx0 + ix;

  double tot = 0.0;
  uint32_t parts[DPM_MAX_PARTS];
  if (live) {
    if (aj.root_off >= 0) tot = (double)__ldg(S + aj.root_off + (int64_t)ry * aj.root_pitch + rx);
    for (int p = 0; p < aj.nparts; ++p) {
      const dpm_place_job pj = pjobs[aj.part_job0 + p];
      const int c = rx - pj.rx0;
      const int cx = pj.scale * rx + pj.ax, cy = pj.scale * ry + pj.ay;
      const int r = radius_of(pj, ranges, false);
      const int lo = max(-r, -cy), hi = min(r, pj.Hp - 1 - cy);
      const float* sm = S + pj.s_off;
      const int16_t* dxt = DX + pj.dx_off + c;
      double best = -INFINITY;
      int bdy = -r, bdx = -r;
      for (int dy = lo; dy <= hi; ++dy) {
        const int y = cy + dy;
        const int dx = dxt[(int64_t)y * pj.wr];
        const int x = cx + dx;
        double vx = -INFINITY;
        if (x >= 0 && x < pj.Wp)
          vx = __dadd_rn((double)__ldg(sm + (int64_t)y * pj.Wp + x), -pen(pj.cdx, pj.cdxx, dx));
        const double cand = __dadd_rn(vx, -pen(pj.cdy, pj.cdyy, dy));
        if (cand > best) {
          best = cand;
          bdy = dy;
          bdx = dx;
        }
      }
      tot = __dadd_rn(tot, best);
      const uint32_t pk = pack_pos(cy + bdy, cx + bdx);
      if (p < DPM_MAX_PARTS) parts[p] = pk;
      const int64_t o = ((int64_t)p * hr + iy) * wr + ix;
      if (aj.pos_off >= 0) pos[aj.pos_off + o] = pk;
      if (aj.placed_off >= 0) placed[aj.placed_off + o] = best;
    }
    tot = __dadd_rn(tot, aj.bias);
    if (aj.total_off >= 0) total[aj.total_off + (int64_t)iy * wr + ix] = tot;
  }
  if (dets == nullptr) return;
  const bool hit = live && tot >= tau;
  const unsigned mask = __ballot_sync(0xffffffffu, hit);
  if (mask == 0u) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(det_count, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
  if (!hit) return;
  const int slot = base + __popc(mask & ((1u << lane) - 1u));
  if (slot >= max_dets) return;
  dpm_detection d;
  d.image = aj.image;
  d.level = aj.level;
  d.component = aj.component;
  d.ry = ry;
  d.rx = rx;
  d.nparts = aj.nparts;
  d.score = tot;
  for (int p = 0; p < DPM_MAX_PARTS; ++p) d.parts[p] = p < aj.nparts ? parts[p] : 0u;
  dets[slot] = d;
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
    if (j.Hp < 1 || j.Wp < 1 || j.wr < 1 || j.scale < 1) {
      set_error("dpm_place_prepare: job %d has Hp=%d Wp=%d wr=%d scale=%d", i, j.Hp, j.Wp, j.wr,
                j.scale);
      return DPM_ERR_ARG;
    }
    if (j.radius > 32000) {
      set_error("dpm_place_prepare: job %d radius %d too large", i, j.radius);
      return DPM_ERR_ARG;
    }
    if (j.radius < 0 && !(j.cdxx > 0.0 && j.cdyy > 0.0)) {
      set_error("dpm_place_prepare: job %d: the unbounded transform needs c_dxx, c_dyy > 0", i);
      return DPM_ERR_ARG;
    }
    if (j.radius < 0 && j.range_idx < 0) {
      set_error("dpm_place_prepare: job %d: GDT mode needs a range slot", i);
      return DPM_ERR_ARG;
    }
    jobs[i].block0 = (int32_t)b;
    b += ((int64_t)j.Hp * j.wr + K3_THREADS - 1) / K3_THREADS;
  }
  return b;
}

extern "C" int64_t dpm_assemble_prepare(dpm_asm_job* jobs, int njobs) {
  if (njobs < 0 || (njobs > 0 && !jobs)) {
    set_error("dpm_assemble_prepare: bad job table");
    return DPM_ERR_ARG;
  }
  int64_t b = 0;
  for (int i = 0; i < njobs; ++i) {
    const dpm_asm_job& j = jobs[i];
    if (j.ry1 < j.ry0 || j.rx1 < j.rx0 || j.nparts < 0 || j.nparts > DPM_MAX_PARTS) {
      set_error("dpm_assemble_prepare: job %d has rect (%d,%d,%d,%d) nparts=%d", i, j.ry0, j.ry1,
                j.rx0, j.rx1, j.nparts);
      return DPM_ERR_ARG;
    }
    jobs[i].block0 = (int32_t)b;
    b += ((int64_t)(j.ry1 - j.ry0 + 1) * (j.rx1 - j.rx0 + 1) + K3_THREADS - 1) / K3_THREADS;
  }
  return b;
}

extern "C" int dpm_place_xpass(const float* S, int16_t* dx, const dpm_place_job* jobs, int njobs,
                               int64_t nblocks, const uint32_t* ranges, void* stream) {
  DPM_REQUIRE(S && dx && jobs, "dpm_place_xpass: null pointer");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_place_xpass: nblocks");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  xpass_kernel<<<(unsigned)nblocks, K3_THREADS, 0, as_stream(stream)>>>(S, dx, jobs, njobs, ranges);
  DPM_LAUNCHED("xpass_kernel");
  return DPM_OK;
}

extern "C" int dpm_assemble(const float* S, const int16_t* dx, const dpm_place_job* pjobs,
                            const dpm_asm_job* ajobs, int najobs, int64_t nblocks,
                            const uint32_t* ranges, double* total, uint32_t* pos, double* placed,
                            double tau, dpm_detection* dets, int max_dets, int* det_count,
                            void* stream) {
  DPM_REQUIRE(S && pjobs && ajobs, "dpm_assemble: null pointer");
  DPM_REQUIRE(!dets || det_count, "dpm_assemble: detections need a counter");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_assemble: nblocks");
  if (najobs == 0 || nblocks == 0) return DPM_OK;
  assemble_kernel<<<(unsigned)nblocks, K3_THREADS, 0, as_stream(stream)>>>(
      S, dx, pjobs, ajobs, najobs, ranges, total, pos, placed, tau, dets, max_dets, det_count);
  DPM_LAUNCHED("assemble_kernel");
  return DPM_OK;
}
