// Pruned detection (paper Algorithm 1, reference detect(pruning=True),
// detection.py:433-503): first failing rank per root hypothesis.
//
// Inputs are the rank-prefix maps K2 produces (prefix k = the filter's core
// with ranks >= k zeroed, bit-identical to cp_partial_stack[k-1],
// correlation.py:170-180).  For every root (ry, rx) of a job's rectangle:
//   root job : first r with prefix_r[ry][rx] < thr[r]            (detection.py:452-460)
//   part job : first r with max over the (2*radius+1)^2 window around the
//              centre scale*root + anchor of prefix_r < thr[r], -inf outside
//              the map                                           (detection.py:471-503)
// written as r + 1 (0 = never fails) into out[out_off + iy * wr + ix].
// The comparison is the reference's: (double) map value < double threshold.
// Which hypotheses are alive when a part is checked (kill / lenient modes)
// and the work accounting are composed on the host from these ranks.
#include <math.h>

#include "common.cuh"

namespace dpm {

__global__ void __launch_bounds__(256)
prune_ranks_kernel(const float* __restrict__ S, const int64_t* __restrict__ map_offs,
                   const double* __restrict__ thr, const dpm_prune_job* __restrict__ jobs,
                   int njobs, uint8_t* __restrict__ out) {
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_prune_job j = jobs[jid];
  const int hr = j.ry1 - j.ry0 + 1, wr = j.rx1 - j.rx0 + 1;
  const int64_t e = (int64_t)(blockIdx.x - j.block0) * 256 + threadIdx.x;
  if (e >= (int64_t)hr * wr) return;
  const int iy = (int)(e / wr), ix = (int)(e - (int64_t)iy * wr);
  const int ry = j.ry0 + iy, rx = j.rx0 + ix;
  int fail = 0;
  if (j.radius < 0) {  // root: the prefix value at the root itself
    for (int r = 0; r < j.R && !fail; ++r) {
      const float v = __ldg(S + map_offs[j.offs0 + r] + (int64_t)ry * s_pitch(j.Wp) + rx);
      if ((double)v < thr[j.thr0 + r]) fail = r + 1;
    }
  } else {
    const int cy = j.scale * ry + j.ay, cx = j.scale * rx + j.ax;
    const int y0 = max(cy - j.radius, 0), y1 = min(cy + j.radius, j.Hp - 1);
    const int x0 = max(cx - j.radius, 0), x1 = min(cx + j.radius, j.Wp - 1);
    for (int r = 0; r < j.R && !fail; ++r) {
      const float* m = S + map_offs[j.offs0 + r];
      float wmax = -INFINITY;
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) wmax = fmaxf(wmax, __ldg(m + (int64_t)y * s_pitch(j.Wp) + x));
      if ((double)wmax < thr[j.thr0 + r]) fail = r + 1;
    }
  }
  out[j.out_off + e] = (uint8_t)fail;
}

}  // namespace dpm

using namespace dpm;

extern "C" int64_t dpm_prune_prepare(dpm_prune_job* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_prune_prepare: bad table");
  int64_t blocks = 0;
  for (int i = 0; i < njobs; ++i) {
    dpm_prune_job& j = jobs[i];
    DPM_REQUIRE(j.ry1 >= j.ry0 && j.rx1 >= j.rx0 && j.R >= 1 && j.R <= 255 && j.Hp >= 1 &&
                    j.Wp >= 1 && j.offs0 >= 0 && j.thr0 >= 0 && j.out_off >= 0,
                "dpm_prune_prepare: job %d has a bad rectangle / rank / offset", i);
    if (j.radius < 0)
      DPM_REQUIRE(j.ry0 >= 0 && j.rx0 >= 0 && j.ry1 < j.Hp && j.rx1 < j.Wp,
                  "dpm_prune_prepare: root job %d rectangle outside its map", i);
    else
      DPM_REQUIRE(j.scale >= 1, "dpm_prune_prepare: part job %d scale", i);
    j.block0 = (int32_t)blocks;
    blocks += ((int64_t)(j.ry1 - j.ry0 + 1) * (j.rx1 - j.rx0 + 1) + 255) / 256;
  }
  return blocks;
}

extern "C" int dpm_prune_ranks(const float* S, const int64_t* map_offs, const double* thr,
                               const dpm_prune_job* jobs, int njobs, int64_t nblocks,
                               uint8_t* out, void* stream) {
  DPM_REQUIRE(S && map_offs && thr && jobs && out, "dpm_prune_ranks: null pointer");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_prune_ranks: nblocks");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  prune_ranks_kernel<<<(unsigned)nblocks, 256, 0, as_stream(stream)>>>(S, map_offs, thr, jobs,
                                                                       njobs, out);
  DPM_LAUNCHED("prune_ranks_kernel");
  return DPM_OK;
}

// ------------------------------------------------ pruned-detection composition
// detect(pruning=True) after the per-rank checks (detection.py:433-542), per
// root in the reference's part order; see dpm_b200.h (dpm_prune_compose).
namespace dpm {
__device__ __forceinline__ uint32_t pack_yx(int y, int x) {
  return ((uint32_t)(uint16_t)(int16_t)y << 16) | (uint32_t)(uint16_t)(int16_t)x;
}

__global__ void __launch_bounds__(256)
prune_compose_kernel(const uint8_t* __restrict__ ranks, const float* __restrict__ S,
                     const double* __restrict__ total, const uint32_t* __restrict__ pos,
                     const double* __restrict__ placed, const dpm_prune_asm* __restrict__ jobs,
                     int njobs, int kill_mode, double tau, uint8_t* __restrict__ lim,
                     uint32_t* __restrict__ hist, dpm_detection* __restrict__ dets, int max_dets,
                     int* __restrict__ det_count) {
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_prune_asm& j = jobs[jid];
  const int hr = j.ry1 - j.ry0 + 1, wr = j.rx1 - j.rx0 + 1;
  const int64_t n = (int64_t)hr * wr;
  const int64_t e = (int64_t)(blockIdx.x - j.block0) * 256 + threadIdx.x;
  const bool live = e < n;
  const int iy = live ? (int)(e / wr) : 0, ix = live ? (int)(e - (int64_t)iy * wr) : 0;
  const int ry = j.ry0 + iy, rx = j.rx0 + ix;
  bool alive = false, hit = false;
  uint32_t part_alive = 0u;  // bit i: part i's term counts (lenient)
  double score = 0.0;
  if (live) {
    const int rr = ranks[j.rank_off + e];
    atomicAdd(hist + j.hist_off + rr, 1u);  // root (detection.py:452-460)
    alive = rr == 0;
    for (int i = 0; i < j.nparts; ++i) {  // parts in order (detection.py:462-503)
      const int pr = ranks[j.rank_off + (int64_t)(1 + i) * n + e];
      const bool pa0 = alive;  // alive when part i is checked
      lim[j.lim_off + i * n + e] = (uint8_t)(pa0 ? (pr == 0 ? j.part_R[i] : pr) : 0);
      lim[j.lim_off + (j.nparts + i) * n + e] = (uint8_t)(pa0 && pr >= 1 ? pr : 0);
      if (pa0) atomicAdd(hist + j.hist_off + (1 + i) * 256, 1u);  // bin 0: alive at part i
      if (pa0 && pr >= 1) {
        atomicAdd(hist + j.hist_off + (1 + i) * 256 + pr, 1u);
        if (kill_mode) alive = false;  // positions_killed_by_parts
      }
      if (pa0 && pr == 0) part_alive |= 1u << i;
    }
    if (kill_mode) {
      score = total[j.total_off + e];
    } else {  // root + sum_i (alive_i ? placed_i : 0) + bias, in the reference's order
      score = (double)S[j.root_off + (int64_t)ry * j.root_pitch + rx];
      for (int i = 0; i < j.nparts; ++i)
        score = __dadd_rn(score, (part_alive >> i) & 1u ? placed[j.placed_off + i * n + e] : 0.0);
      score = __dadd_rn(score, j.bias);
    }
    hit = alive && score >= tau;
  }
  if (dets == nullptr) return;
  const unsigned bal = __ballot_sync(0xffffffffu, hit);
  if (bal == 0u) return;
  const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(det_count, __popc(bal));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!hit) return;
  const int slot = base + __popc(bal & ((1u << lane) - 1u));
  if (slot >= max_dets) return;
  dpm_detection d;
  d.image = j.image;
  d.level = j.level;
  d.component = 0;
  d.ry = ry;
  d.rx = rx;
  d.nparts = j.nparts;
  d.score = score;
  for (int q = 0; q < DPM_MAX_PARTS; ++q) {
    uint32_t v = 0u;
    if (q < j.nparts)
      v = (!kill_mode && !((part_alive >> q) & 1u)) ? pack_yx(ry + j.ay[q], rx + j.ax[q])
                                                    : pos[j.pos_off + q * n + e];
    d.parts[q] = v;
  }
  dets[slot] = d;
}

__global__ void __launch_bounds__(256)
prune_cover_kernel(const uint8_t* __restrict__ lim, const dpm_cover_job* __restrict__ jobs,
                   int njobs, uint32_t* __restrict__ hist) {
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_cover_job& j = jobs[jid];
  const int bw = j.x1 - j.x0 + 1;
  const int64_t e = (int64_t)(blockIdx.x - j.block0) * 256 + threadIdx.x;
  if (e >= (int64_t)(j.y1 - j.y0 + 1) * bw) return;
  const int y = j.y0 + (int)(e / bw), x = j.x0 + (int)(e % bw);
  const int cy = y - j.oy, cx = x - j.ox;  // root index whose window centre is the cell
  const int iy0 = max(cy - j.radius, 0), iy1 = min(cy + j.radius, j.hr - 1);
  const int ix0 = max(cx - j.radius, 0), ix1 = min(cx + j.radius, j.wr - 1);
  int m = 0;
  for (int iy = iy0; iy <= iy1; ++iy)
    for (int ix = ix0; ix <= ix1; ++ix) m = max(m, (int)lim[j.lim_off + (int64_t)iy * j.wr + ix]);
  DPM_CHECK(m < 256, "cover histogram bin");
  if (m > 0) atomicAdd(hist + j.hist_off + m, 1u);
}
}  // namespace dpm

extern "C" int64_t dpm_prune_compose_prepare(dpm_prune_asm* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_prune_compose_prepare: bad table");
  int64_t blocks = 0;
  for (int i = 0; i < njobs; ++i) {
    dpm_prune_asm& j = jobs[i];
    DPM_REQUIRE(j.ry1 >= j.ry0 && j.rx1 >= j.rx0 && j.nparts >= 0 && j.nparts <= DPM_MAX_PARTS &&
                    j.rank_off >= 0 && j.lim_off >= 0 && j.hist_off >= 0 && j.total_off >= 0 &&
                    (j.nparts == 0 || (j.pos_off >= 0 && j.placed_off >= 0)) && j.root_off >= 0,
                "dpm_prune_compose_prepare: job %d has a bad rectangle / part count / offset", i);
    for (int q = 0; q < j.nparts; ++q)
      DPM_REQUIRE(j.part_R[q] >= 1 && j.part_R[q] <= 255,
                  "dpm_prune_compose_prepare: job %d part %d rank %d", i, q, j.part_R[q]);
    j.block0 = (int32_t)blocks;
    blocks += ((int64_t)(j.ry1 - j.ry0 + 1) * (j.rx1 - j.rx0 + 1) + 255) / 256;
  }
  DPM_REQUIRE(blocks <= INT32_MAX, "dpm_prune_compose_prepare: too many CTAs");
  return blocks;
}

extern "C" int dpm_prune_compose(const uint8_t* ranks, const float* S, const double* total,
                                 const uint32_t* pos, const double* placed,
                                 const dpm_prune_asm* jobs, int njobs, int64_t nblocks,
                                 int kill_mode, double tau, uint8_t* lim, uint32_t* hist,
                                 dpm_detection* dets, int max_dets, int* det_count, void* stream) {
  DPM_REQUIRE(ranks && S && total && jobs && lim && hist, "dpm_prune_compose: null pointer");
  DPM_REQUIRE(!dets || det_count, "dpm_prune_compose: detections need a counter");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_prune_compose: nblocks");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  prune_compose_kernel<<<(unsigned)nblocks, 256, 0, as_stream(stream)>>>(
      ranks, S, total, pos, placed, jobs, njobs, kill_mode, tau, lim, hist, dets, max_dets,
      det_count);
  DPM_LAUNCHED("prune_compose_kernel");
  return DPM_OK;
}

extern "C" int64_t dpm_prune_cover_prepare(dpm_cover_job* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_prune_cover_prepare: bad table");
  int64_t blocks = 0;
  for (int i = 0; i < njobs; ++i) {
    dpm_cover_job& j = jobs[i];
    DPM_REQUIRE(j.hr >= 1 && j.wr >= 1 && j.radius >= 0 && j.lim_off >= 0 && j.hist_off >= 0,
                "dpm_prune_cover_prepare: job %d has a bad extent / radius / offset", i);
    j.block0 = (int32_t)blocks;
    if (j.y1 >= j.y0 && j.x1 >= j.x0)
      blocks += ((int64_t)(j.y1 - j.y0 + 1) * (j.x1 - j.x0 + 1) + 255) / 256;
  }
  DPM_REQUIRE(blocks <= INT32_MAX, "dpm_prune_cover_prepare: too many CTAs");
  return blocks;
}

extern "C" int dpm_prune_cover(const uint8_t* lim, const dpm_cover_job* jobs, int njobs,
                               int64_t nblocks, uint32_t* hist, void* stream) {
  DPM_REQUIRE(lim && jobs && hist, "dpm_prune_cover: null pointer");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_prune_cover: nblocks");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  prune_cover_kernel<<<(unsigned)nblocks, 256, 0, as_stream(stream)>>>(lim, jobs, njobs, hist);
  DPM_LAUNCHED("prune_cover_kernel");
  return DPM_OK;
}

// ------------------------------------------------------------ mixture max
// Per (image, root level): for every root position of the union rectangle
// of the level's component assemblies, the max over components of their
// totals at that position (components whose rectangle holds it), ties to the
// lowest component index (the reference defines no
// combination, SPEC.md:358 asks for a max).
namespace dpm {
__global__ void __launch_bounds__(256)
mixture_max_kernel(const double* __restrict__ total, const dpm_asm_job* __restrict__ ajobs,
                   const int32_t* __restrict__ members, const dpm_mix_job* __restrict__ jobs,
                   int njobs, double* __restrict__ best, int32_t* __restrict__ comp) {
  const int jid = find_job_warp(jobs, njobs, blockIdx.x);
  const dpm_mix_job j = jobs[jid];
  const int hu = j.ry1 - j.ry0 + 1, wu = j.rx1 - j.rx0 + 1;
  const int64_t e = (int64_t)(blockIdx.x - j.block0) * 256 + threadIdx.x;
  if (e >= (int64_t)hu * wu) return;
  const int ry = j.ry0 + (int)(e / wu), rx = j.rx0 + (int)(e % wu);
  double b = -INFINITY;
  int bc = -1;
  for (int m = 0; m < j.nmembers; ++m) {
    const dpm_asm_job a = ajobs[members[j.member0 + m]];
    if (ry < a.ry0 || ry > a.ry1 || rx < a.rx0 || rx > a.rx1) continue;
    const double v = total[a.total_off + (int64_t)(ry - a.ry0) * (a.rx1 - a.rx0 + 1) + (rx - a.rx0)];
    if (bc < 0 || v > b || (v == b && a.component < bc)) {
      b = v;
      bc = a.component;
    }
  }
  best[j.out_off + e] = b;
  comp[j.out_off + e] = bc;
}
}  // namespace dpm

extern "C" int64_t dpm_mixture_prepare(dpm_mix_job* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_mixture_prepare: bad table");
  int64_t blocks = 0;
  for (int i = 0; i < njobs; ++i) {
    dpm_mix_job& j = jobs[i];
    DPM_REQUIRE(j.ry1 >= j.ry0 && j.rx1 >= j.rx0 && j.nmembers >= 0 && j.member0 >= 0 &&
                    j.out_off >= 0,
                "dpm_mixture_prepare: job %d has a bad rectangle / member range", i);
    j.block0 = (int32_t)blocks;
    blocks += ((int64_t)(j.ry1 - j.ry0 + 1) * (j.rx1 - j.rx0 + 1) + 255) / 256;
  }
  return blocks;
}

extern "C" int dpm_mixture_max(const double* total, const dpm_asm_job* ajobs,
                               const int32_t* members, const dpm_mix_job* jobs, int njobs,
                               int64_t nblocks, double* best, int32_t* comp, void* stream) {
  DPM_REQUIRE(total && ajobs && members && jobs && best && comp, "dpm_mixture_max: null pointer");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_mixture_max: nblocks");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  mixture_max_kernel<<<(unsigned)nblocks, 256, 0, as_stream(stream)>>>(total, ajobs, members, jobs,
                                                                       njobs, best, comp);
  DPM_LAUNCHED("mixture_max_kernel");
  return DPM_OK;
}
