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
