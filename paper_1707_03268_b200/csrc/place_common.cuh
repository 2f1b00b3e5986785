// Device helpers shared by the K3/K4 placement kernels (placement.cu: the
// round-1 kernel, place2.cu: the two-phase kernel).  Reference semantics:
// _placement_grid (detection.py:320-373) and best_part_placement
// (detection.py:180-207).
#pragma once

#include <math.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace dpm {

constexpr int RCAP = 16;                                  // staged-path radius cap
constexpr int PT_W = 32;                                  // root columns per tile (lanes)
constexpr int PT_H = 64;                                  // root rows per tile
constexpr int PT_THREADS = 512;
constexpr int PT_WARPS = PT_THREADS / 32;
constexpr int BAND_ROWS = 2 * (PT_H - 1) + 1 + 2 * RCAP;  // 159 band rows (scale <= 2)
constexpr int TMA_BH = DPM_SMAP_BOX_H;                      // band rows per TMA box
constexpr int BAND_MAX = (BAND_ROWS + TMA_BH - 1) / TMA_BH * TMA_BH;  // 160: whole boxes
// even, so band rows start 8-byte aligned (packed pairs in the x pass)
// band row pitch in shared memory = the TMA box width (the box lands dense)
constexpr int COLS_PITCH = DPM_SMAP_BOX_W;  // 100 >= 2 * (PT_W - 1) + 1 + 2 * RCAP = 95
static_assert(COLS_PITCH >= 2 * (PT_W - 1) + 1 + 2 * RCAP && COLS_PITCH % 4 == 0, "band width");
constexpr uint32_t TMA_BOX_BYTES = DPM_SMAP_BOX_W * DPM_SMAP_BOX_H * 4;

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

using JobRange = dpm_place_range;

__device__ __forceinline__ JobRange job_range(const dpm_place_job& pj, const uint32_t* ranges) {
  JobRange jr;
  const float vmax = key_float(ranges[2 * pj.range_idx]);
  const float vmin = key_float(ranges[2 * pj.range_idx + 1]);
  jr.rx = radius_of(pj, vmax, vmin, true);
  jr.ry = radius_of(pj, vmax, vmin, false);
  const double mabs = fmax(fabs((double)vmax), fabs((double)vmin));
  // floor: the index code of values near 0 lives in denormals (< 64 * 2^-149)
  jr.E2 = (float)fmax(ldexp(mabs + pen_absmax(pj.cdx, pj.cdxx, jr.rx) +
                                pen_absmax(pj.cdy, pj.cdyy, jr.ry), -15),
                      0x1p-120);
  jr.E2in = (float)fmax(ldexp(mabs + pen_absmax(pj.cdx, pj.cdxx, min(jr.rx, 6)) +
                                  pen_absmax(pj.cdy, pj.cdyy, min(jr.ry, 6)), -15),
                        0x1p-120);
  return jr;
}

__device__ __forceinline__ uint32_t pack_pos(int y, int x) {
  return ((uint32_t)(uint16_t)(int16_t)y << 16) | (uint32_t)(uint16_t)(int16_t)x;
}

constexpr float OUT_SENTINEL = -1.0e37f;  // x-pass result of a band row without candidates
constexpr float NONE_BELOW = -1.0e36f;    // m1 below this: no candidate inside the map

// (bits(v) & mask) | code in ONE lop3 (LUT 0xEA = (a & b) | c): the mask
// lives in a register so the code can be the instruction's immediate
template <int CODE>
__device__ __forceinline__ float enc_idx(float v, uint32_t mask) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(__float_as_uint(v)), "r"(mask), "n"(CODE));
  return __uint_as_float(r);
}

// min that propagates NaN (FMNMX.NAN): cells outside the map arrive as NaN
// (TMA out-of-bounds fill); in the top-2 merge below a NaN candidate must
// drop out of both m1 and m2 -- with the NaN-ignoring fminf it would make m2
// equal to the winner and force a needless exact rescan.
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Placement of one part for one root via direct global loads (any radius).
static __device__ void place_unstaged(const float* __restrict__ sm, const dpm_place_job& pj, int cy,
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
      const double c = __dadd_rn((double)__ldg(sm + (int64_t)y * s_pitch(pj.Wp) + cx + dx),
                                 -pen(pj.cdx, pj.cdxx, dx));
      if (c > xb) { xb = c; xd = dx; }
    }
    const double cand = __dadd_rn(xb, -pen(pj.cdy, pj.cdyy, dy));
    if (cand > best) { best = cand; bdy = dy; bdx = xd; }
  }
}

__device__ __forceinline__ uint32_t pl_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// Band copy: one TMA tensor load of a DPM_SMAP_BOX_W x DPM_SMAP_BOX_H box of
// map z starting at (x, y) (signed; cells outside the map arrive as NaN).
__device__ __forceinline__ void tma_band_box(uint32_t dst, const void* map, int x, int y, int z,
                                             uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void pl_mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (int spin = 0; spin < 2000 && !done; ++spin)  // each try suspends up to 10 ms
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(10000000u)
        : "memory");
  if (!done) asm volatile("trap;");  // a band that never lands is a bug, not a hang
}


// Tiles of the specialised K3 kernel (place2.cu): the leading tile columns
// at least FAST_MINW roots wide of a job whose parts are all at scale 2 with
// radius < 0 (r* from the device's map ranges; a part whose r* falls outside
// (6, RCAP] takes the kernel's exact per-root path) or 7 <= radius <= RCAP.
// Host (dpm_assemble_prepare) and device (tile numbering) evaluate the same
// rule.  Returns the number of such tile columns.
constexpr int FAST_MINW = 17;
constexpr int FAST_R1 = 6;  // inner screen radius of the two-phase kernel
__host__ __device__ inline bool k3_fast_part(const dpm_place_job& pj) {
  return pj.scale == 2 && (pj.radius < 0 || (pj.radius > FAST_R1 && pj.radius <= RCAP));
}
bool k3_fast_enabled();  // DPM_K3F=0 turns the specialised kernel off (place2.cu)
__host__ inline int k3_fast_cols(const dpm_asm_job& j, const dpm_place_job* pjobs, int wr) {
  if (j.nparts <= 0 || !k3_fast_enabled()) return 0;
  for (int q = 0; q < j.nparts; ++q)
    if (!k3_fast_part(pjobs[j.part_job0 + q])) return 0;
  const int ntx = (wr + PT_W - 1) / PT_W;
  return wr - PT_W * (ntx - 1) >= FAST_MINW ? ntx : ntx - 1;
}
// the same on the device, by a whole warp (lane q tests part q)
__device__ __forceinline__ int k3_fast_cols_warp(const dpm_asm_job& j, const dpm_place_job* pjobs,
                                                 int wr, int lane) {
  if (j.nparts <= 0) return 0;
  const bool ok = lane >= j.nparts || k3_fast_part(pjobs[j.part_job0 + lane]);
  if (!__all_sync(0xffffffffu, ok)) return 0;
  const int ntx = (wr + PT_W - 1) / PT_W;
  return wr - PT_W * (ntx - 1) >= FAST_MINW ? ntx : ntx - 1;
}

// the two-phase K3/K4 kernels (place2.cu) and their tile height in root rows
int k3v2_tile_rows();
int launch_place2(const float* S, const void* smaps, const dpm_place_job* pjobs,
                  const dpm_asm_job* ajobs, int najobs, int64_t nfast, int64_t ngeneric,
                  const dpm_place_range* prep, double* total, uint32_t* pos, double* placed,
                  double tau, dpm_detection* dets, int max_dets, int* det_count, cudaStream_t st);

}  // namespace dpm
