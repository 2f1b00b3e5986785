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
// in shared memory (TMA tensor boxes, one thread, mbarrier completion; the
// next part's band lands during this part's y pass), runs the x pass for
// every band row at the 32 centre
// columns (64-row tiles keep the band overlap between vertically adjacent
// tiles at 2r / 128 rows), then the y pass for its roots; exact FP64 values
// are recomputed from the staged band.  Root + parts + bias are summed in
// registers and written with the part positions; detections >= tau are
// compacted with one atomic per warp.
// Candidates are screened in FP32, branch free, by a loop fully unrolled for
// the part's radius (switch over 0..RCAP): each candidate value carries its
// window index in the low 6 mantissa bits, candidates are merged in pairs
// (max/min), and the scan keeps the top value m1 (whose low bits name the
// winner) and the best value m2 of all other candidates.  Encoding moves a
// value by < 64 ulps; with E2 = 2^-15 * (max|S| + max pen_x + max pen_y) at
// least twice the FP32 error plus the encoding error of any candidate,
// m2 < m1 - E2 proves the decoded winner is the unique exact winner;
// otherwise (ties, near ties) the candidates within E2 of m1 are rescanned
// in FP64 in the reference's order.  Cells outside the map arrive as NaN
// (TMA out-of-bounds fill): fmaxf ignores them and the NaN-propagating min of
// the merge keeps them out of m2, so a window without any in-map cell ends
// with m1 = -inf, the reference's "no candidate".
//
// radius < 0 selects the unbounded generalised distance transform, realised
// as the window of radius r* computed from the map's
// range, beyond which no maximiser lies.  Radii above RCAP use unstaged loops
// with the same arithmetic.
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "place_common.cuh"

namespace dpm {

// K3 prologue: r* and the screening bound of every placement job, once per
// run (after K2 has filled the map ranges)
__global__ void __launch_bounds__(256)
place_ranges_kernel(const dpm_place_job* __restrict__ pjobs, int njobs,
                    const uint32_t* __restrict__ ranges, dpm_place_range* __restrict__ prep) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i < njobs) prep[i] = job_range(pjobs[i], ranges);
}

// Window of 2R+1 candidates src[d*STRIDE] + np[d], d = -R..R (pointers at
// d = 0); m1 = top encoded value (code d + R in its low bits), m2 = best of
// the others.
template <int R, int STRIDE, int D>
__device__ __forceinline__ void screen_pairs(const float* __restrict__ src,
                                             const float* __restrict__ np, uint32_t mask,
                                             float& m1, float& m2) {
  if constexpr (D < R) {
    const float a = enc_idx<D + R>(src[D * STRIDE] + np[D], mask);
    const float b = enc_idx<D + 1 + R>(src[(D + 1) * STRIDE] + np[D + 1], mask);
    const float hi = fmaxf(a, b), lo = fmin_nan(a, b);
    m2 = fmaxf(m2, fmaxf(lo, fmin_nan(m1, hi)));
    m1 = fmaxf(m1, hi);
    screen_pairs<R, STRIDE, D + 2>(src, np, mask, m1, m2);
  }
}

// Contiguous candidates (x pass at scale 2): src + D and np + D are 8-byte
// aligned for every pair start D = -R, -R+2, ..., so each pair is one
// 64-bit load per operand and one packed add.f32x2.
template <int R, int D>
__device__ __forceinline__ void screen_pairs_packed(const float* __restrict__ src,
                                                    const float* __restrict__ np, uint32_t mask,
                                                    float& m1, float& m2) {
  if constexpr (D < R) {
    const unsigned long long s2 = *reinterpret_cast<const unsigned long long*>(src + D);
    const unsigned long long p2 = *reinterpret_cast<const unsigned long long*>(np + D);
    unsigned long long v2;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(v2) : "l"(s2), "l"(p2));
    float va, vb;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(va), "=f"(vb) : "l"(v2));
    const float a = enc_idx<D + R>(va, mask);
    const float b = enc_idx<D + 1 + R>(vb, mask);
    const float hi = fmaxf(a, b), lo = fmin_nan(a, b);
    m2 = fmaxf(m2, fmaxf(lo, fmin_nan(m1, hi)));
    m1 = fmaxf(m1, hi);
    screen_pairs_packed<R, D + 2>(src, np, mask, m1, m2);
  }
}

// Packed x pass (scale 2): candidates d = -R..R at src[d] (pointer at d = 0).
// The band may be staged with an odd float shift (`odd`), which decides the
// 8-byte pair alignment: pairs start at d = odd - R and carry codes
// 0..2R-1 (d = code - R + odd); the remaining single candidate (d = R, or
// d = -R when odd) carries code 2R.  One code path for both parities keeps
// the hot code small (a per-parity instantiation doubled it and the kernel
// stalled on instruction fetch).  np_odd: the penalty table shifted by one
// element, for the pair alignment of the table side.
template <int R, int STRIDE, bool PACKED>
__device__ __forceinline__ void screen_window(const float* __restrict__ src,
                                              const float* __restrict__ np,
                                              const float* __restrict__ np_odd, uint32_t mask,
                                              int odd, float& m1, float& m2) {
  m1 = -INFINITY;
  m2 = -INFINITY;
  if constexpr (PACKED) {
    const float* npp = (((R + odd) & 1) ? np_odd : np) + (odd - R);
    screen_pairs_packed<R, -R>(src + (odd - R) + R, npp + R, mask, m1, m2);
    const int sd = odd ? -R : R;
    const float c = enc_idx<2 * R>(src[sd] + np[sd], mask);
    m2 = fmaxf(m2, fmin_nan(m1, c));
    m1 = fmaxf(m1, c);
  } else {
    screen_pairs<R, STRIDE, -R>(src, np, mask, m1, m2);
    const float c = enc_idx<2 * R>(src[R * STRIDE] + np[R], mask);
    m2 = fmaxf(m2, fmin_nan(m1, c));
    m1 = fmaxf(m1, c);
  }
}

// runtime radius -> unrolled instantiation (radius <= RCAP on the staged path)
template <int STRIDE, bool PACKED>
__device__ __forceinline__ void screen_dispatch(int r, const float* __restrict__ src,
                                                const float* __restrict__ np,
                                                const float* __restrict__ np_odd, uint32_t mask,
                                                int odd, float& m1, float& m2) {
  switch (r) {
#define DPM_SCREEN_CASE(R) \
  case R: screen_window<R, STRIDE, PACKED>(src, np, np_odd, mask, odd, m1, m2); break;
    DPM_SCREEN_CASE(0) DPM_SCREEN_CASE(1) DPM_SCREEN_CASE(2) DPM_SCREEN_CASE(3)
    DPM_SCREEN_CASE(4) DPM_SCREEN_CASE(5) DPM_SCREEN_CASE(6) DPM_SCREEN_CASE(7)
    DPM_SCREEN_CASE(8) DPM_SCREEN_CASE(9) DPM_SCREEN_CASE(10) DPM_SCREEN_CASE(11)
    DPM_SCREEN_CASE(12) DPM_SCREEN_CASE(13) DPM_SCREEN_CASE(14) DPM_SCREEN_CASE(15)
    DPM_SCREEN_CASE(16)
#undef DPM_SCREEN_CASE
    default: m1 = m2 = -INFINITY;
  }
}
static_assert(2 * RCAP + 1 <= 63, "window index must fit the 6-bit code");

// Exact rescans of a near-tie window in the reference's order (ascending
// offset, strict '>'), over the candidates whose FP32 screen value reaches
// lo.  Rare; kept out of line so the screening loops do not reserve their
// FP64 registers.
__device__ __noinline__ int x_rescan(const float* srow, const float* npx, float lo, int rx,
                                     const dpm_place_job* pj) {
  const double cdx = pj->cdx, cdxx = pj->cdxx;
  double xv = -INFINITY;
  int xi = -rx;
  for (int dx = -rx; dx <= rx; ++dx) {
    if (srow[dx] + npx[dx] >= lo) {
      const double e = __dadd_rn((double)srow[dx], -pen(cdx, cdxx, dx));
      if (e > xv) { xv = e; xi = dx; }
    }
  }
  return xi;
}

// y: xcol / xsv / xdx point at the dy = 0 row of the root's column (stride PT_W)
__device__ __noinline__ int y_rescan(const float* xcol, const float* xsv, const int8_t* xdx,
                                     const float* npy, float lo, int ry, const dpm_place_job* pj,
                                     double& best) {
  const double cdx = pj->cdx, cdxx = pj->cdxx, cdy = pj->cdy, cdyy = pj->cdyy;
  best = -INFINITY;
  int bi = -ry;
  for (int dy = -ry; dy <= ry; ++dy) {
    if (xcol[dy * PT_W] + npy[dy] >= lo) {
      const double xv = __dadd_rn((double)xsv[dy * PT_W], -pen(cdx, cdxx, xdx[dy * PT_W]));
      const double e = __dadd_rn(xv, -pen(cdy, cdyy, dy));
      if (e > best) { best = e; bi = dy; }
    }
  }
  return bi;
}

struct __align__(128) PlaceSmem {
  float s[BAND_MAX * COLS_PITCH];  // S band, TMA-staged (NaN outside the map)
  float x32[BAND_MAX * PT_W];      // x-pass winners' FP32 screen values
  float xsv[BAND_MAX * PT_W];      // x-pass winners' S values (exact y values)
  int8_t xdx[BAND_MAX * PT_W];     // x-pass winning dx
  float npx[2][2 * RCAP + 4];      // -pen_x(dx) in FP32 (screening only), by part parity
  float npx_odd[2][2 * RCAP + 4];  // the same, shifted by one element (packed pairs, odd r)
  float npy[2][2 * RCAP + 4];
  alignas(16) JobRange jr[2];      // r*, E2 of the current / next part (16-B cp.async)
  alignas(16) dpm_place_job pj[2]; // placement job of the current / next part
  dpm_asm_job aj;                  // this CTA's assembly job
  alignas(8) uint64_t band_bar;    // TMA completion of the current band (one phase per band)
};
static_assert(TMA_BOX_BYTES % 128 == 0, "TMA boxes land 128-byte aligned");

// x pass over one warp's band rows rb0, rb0 + step, ... (< r_hi) for a
// compile-time radius: the radius switch sits outside the row loop, so the
// loop carries no per-row dispatch and the winner decode folds R.
template <int R, bool PACKED>
__device__ __forceinline__ void x_rows(PlaceSmem& sh, int buf, const float* srow0, int rb0,
                                       int r_hi, int step, int xsub, int xc, uint32_t mask,
                                       int xodd, float E2) {
  const float* npx = sh.npx[buf] + RCAP;
  const float* npx_odd = sh.npx_odd[buf] + RCAP + 1;
  for (int rb = rb0; rb < r_hi; rb += step) {
    const int r = rb + xsub;
    if (r >= r_hi) continue;
    const float* srow = srow0 + r * COLS_PITCH;
    float m1, m2;
    screen_window<R, 1, PACKED>(srow, npx, npx_odd, mask, xodd, m1, m2);
    // the y-pass screen only needs the winner's value to the screening
    // accuracy; exact values are recomputed from xsv for y winners and ties
    const int code = __float_as_int(m1) & 63;
    int xi = code == 2 * R ? (xodd ? -R : R) : code - R + xodd;
    if (m1 < NONE_BELOW) {  // no candidate inside the map: reference gives (-inf, -r)
      xi = -R;
      m1 = OUT_SENTINEL;
    } else if (m2 >= m1 - E2) {  // tie or near tie: exact rescan, reference order
      xi = x_rescan(srow, npx, m1 - E2, R, &sh.pj[buf]);
    }
    sh.x32[r * PT_W + xc] = m1;
    sh.xsv[r * PT_W + xc] = srow[xi];
    sh.xdx[r * PT_W + xc] = (int8_t)xi;
  }
}

__global__ void __launch_bounds__(PT_THREADS, 2)
place_assemble_kernel(const float* __restrict__ S, const unsigned char* __restrict__ smaps,
                      const dpm_place_job* __restrict__ pjobs,
                      const dpm_asm_job* __restrict__ ajobs, int najobs,
                      const dpm_place_range* __restrict__ prep, double* __restrict__ total,
                      uint32_t* __restrict__ pos, double* __restrict__ placed, double tau,
                      dpm_detection* __restrict__ dets, int max_dets, int* __restrict__ det_count) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PlaceSmem& sh = *reinterpret_cast<PlaceSmem*>(smem_raw);
  const int jid = find_job_warp(ajobs, najobs, blockIdx.x);
  if (threadIdx.x == 0) sh.aj = ajobs[jid];
  __syncthreads();
  const dpm_asm_job& aj = sh.aj;
  const int hr = aj.ry1 - aj.ry0 + 1, wr = aj.rx1 - aj.rx0 + 1;
  const int ntx = (wr + PT_W - 1) / PT_W;
  const int tile = blockIdx.x - aj.block0;
  const int ty0 = (tile / ntx) * PT_H, tx0 = (tile % ntx) * PT_W;  // offsets inside the rect
  // thread index read once through a volatile asm: the compiler may not
  // re-derive it (S2R + shifts) at every use, which it did under the
  // 64-register cap (7% of the kernel's instructions, with S2R latency)
  int tid_, lane_, warp_;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid_));
  asm volatile("and.b32 %0, %1, 31;" : "=r"(lane_) : "r"(tid_));
  asm volatile("shr.u32 %0, %1, 5;" : "=r"(warp_) : "r"(tid_));
  const int tid = tid_, lane = lane_, warp = warp_;
  constexpr int RPT = PT_H / PT_WARPS;  // roots per thread (4)
  // Narrow tiles pack: lpr = lanes per band row / per root row (power of two
  // >= the tile's valid columns), so a warp screens 32 / lpr rows at once and
  // the roots map compactly onto threads.
  const int wt = min(PT_W, wr - tx0), h_tile = min(PT_H, hr - ty0);
  const int lpr_log = wt > 16 ? 5 : wt > 8 ? 4 : wt > 4 ? 3 : wt > 2 ? 2 : wt > 1 ? 1 : 0;
  const int lpr = 1 << lpr_log;
  auto root_of = [&](int k, int& iyr, int& ixr) -> bool {  // k-th root of this thread
    const int e = tid + PT_THREADS * k;
    iyr = e >> lpr_log;
    ixr = e & (lpr - 1);
    return iyr < h_tile && ixr < wt;
  };
  const int ry_lo = aj.ry0 + ty0;
  const int ry_hi = aj.ry0 + min(ty0 + PT_H, hr) - 1;
  const int rx_lo = aj.rx0 + tx0;
  // ~63 from a value the compiler cannot fold (najobs > 0), so the index
  // code, not the mask, is each encoding lop3's immediate
  const uint32_t code_mask = ~63u | ((uint32_t)najobs >> 31);

  double tot[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    int iyr, ixr;
    tot[k] = 0.0;
    if (aj.root_off >= 0 && root_of(k, iyr, ixr))
      tot[k] = (double)__ldg(S + aj.root_off + (int64_t)(ry_lo + iyr) * aj.root_pitch + rx_lo + ixr);
  }

  // Per part: [band p resident] x pass -> sync -> async copy of band p+1 into
  // the same buffer (the y pass only reads x32/xdx/xsv) overlapped with the
  // y pass of part p.  Penalty tables are double buffered by part parity.
  auto staged_ok = [&](const dpm_place_job& pj, const JobRange& jr) {
    return jr.rx <= RCAP && jr.ry <= RCAP && pj.scale <= 2;
  };
  // Band of a part: one thread issues the TMA boxes covering band rows
  // 0..nrows-1 and columns xb0..xb0+COLS_PITCH-1 (outside the map: NaN, which
  // the screens treat as no candidate); the band barrier completes when all
  // bytes landed.  The buffer's previous band was last read before the
  // __syncthreads preceding this call.
  const uint32_t band_bar = pl_smem(&sh.band_bar);
  auto stage_issue = [&](const dpm_place_job& pj, const JobRange& jr, int buf) {
    const int yb0 = pj.scale * ry_lo + pj.ay - jr.ry;
    const int nrows = pj.scale * (ry_hi - ry_lo) + 1 + 2 * jr.ry;
    const int xb0 = pj.scale * rx_lo + pj.ax - jr.rx;
    if (tid == 0) {
      const int nbox = (nrows + TMA_BH - 1) / TMA_BH;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(band_bar),
                   "r"((uint32_t)nbox * TMA_BOX_BYTES)
                   : "memory");
      const void* map = smaps + (int64_t)pj.smap * DPM_SMAP_BYTES;
      const uint32_t dst = pl_smem(sh.s);
      // the box's first column must be 16-byte aligned in the map: start at
      // xb0 & ~3; band column c then lands at shared column c + (xb0 & 3)
      for (int k = 0; k < nbox; ++k)
        tma_band_box(dst + (uint32_t)k * TMA_BOX_BYTES, map, xb0 & ~3, yb0 + k * TMA_BH, pj.smap_z,
                     band_bar);
    }
    if (tid >= PT_THREADS - 2 * (2 * RCAP + 1)) {  // last warps: penalty tables
      const int t = tid - (PT_THREADS - 2 * (2 * RCAP + 1));
      const int d = (t % (2 * RCAP + 1)) - RCAP;
      if (t < 2 * RCAP + 1) {
        const float v = (float)(-pen(pj.cdx, pj.cdxx, d));
        sh.npx[buf][d + RCAP] = v;
        sh.npx_odd[buf][d + RCAP + 1] = v;
      }
      else sh.npy[buf][d + RCAP] = (float)(-pen(pj.cdy, pj.cdyy, d));
    }
  };

  // r*/E2 of every part come from the prologue (dpm_place_ranges)
  // The placement job and r*/E2 record of part q are cp.async-copied into
  // shared slot q & 1 one part ahead (warp 0), so no thread waits on their
  // global loads at a part boundary.
  auto fetch_job = [&](int q, int buf) {
    if (warp != 0) return;
    if (lane < (int)(sizeof(dpm_place_job) / 8)) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(
          reinterpret_cast<unsigned char*>(&sh.pj[buf]) + 8 * lane);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa),
                   "l"(reinterpret_cast<const unsigned char*>(pjobs + aj.part_job0 + q) + 8 * lane));
    } else if (lane == 31) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&sh.jr[buf]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                   "l"(prep + aj.part_job0 + q));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  auto issue_part = [&](int buf) {  // band + tables of the part whose job is in slot buf
    const dpm_place_job pn = sh.pj[buf];
    const JobRange jn = sh.jr[buf];
    if (staged_ok(pn, jn)) stage_issue(pn, jn, buf);
  };
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(band_bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t bands = 0;  // bands staged so far: band k completes barrier phase k
  if (aj.nparts > 0) {
    fetch_job(0, 0);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    issue_part(0);
  }
  // this job's position / placed outputs (nullptr: not requested)
  uint32_t* const posb = aj.pos_off >= 0 ? pos + aj.pos_off : nullptr;
  double* const placedb = aj.placed_off >= 0 ? placed + aj.placed_off : nullptr;
  for (int p = 0; p < aj.nparts; ++p) {
    const int buf = p & 1;
    // the job record of part p landed before the previous barrier
    const dpm_place_job& pj = sh.pj[buf];
    const JobRange& jr = sh.jr[buf];
    asm volatile("cp.async.wait_group 0;\n" ::);
    const bool staged = staged_ok(pj, jr);
    if (staged) pl_mbar_wait(band_bar, bands++ & 1);  // band p landed
    __syncthreads();  // penalty tables of part p visible; part p-1 finished
    const float* sm = S + pj.s_off;
    const bool have_next = p + 1 < aj.nparts;
    if (have_next) fetch_job(p + 1, buf ^ 1);
    if (!staged) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        int iyr, ixr;
        if (!root_of(k, iyr, ixr)) continue;
        const int iy = ty0 + iyr, ix = tx0 + ixr;
        const int cy = pj.scale * (aj.ry0 + iy) + pj.ay;
        const int cx = pj.scale * (aj.rx0 + ix) + pj.ax;
        double best;
        int bdy, bdx;
        place_unstaged(sm, pj, cy, cx, jr.rx, jr.ry, best, bdy, bdx);
        tot[k] = __dadd_rn(tot[k], best);
        const int o = (p * hr + iy) * wr + ix;  // < nparts * hr * wr: 32-bit
        if (posb) posb[o] = pack_pos(cy + bdy, cx + bdx);
        if (placedb) placedb[o] = best;
      }
      if (have_next) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();  // job p+1 visible
        issue_part(buf ^ 1);
      }
      continue;
    }
    const int yb0 = pj.scale * ry_lo + pj.ay - jr.ry;
    const int nrows = pj.scale * (ry_hi - ry_lo) + 1 + 2 * jr.ry;
    const int xsh = (pj.scale * rx_lo + pj.ax - jr.rx) & 3;  // band column 0's shared column
    const int xodd = pj.scale == 2 ? (xsh & 1) : 0;           // packed-pair parity (screen_window)

    // x pass: band row r (warp-strided), centre column = lane
    // band rows outside the map have no candidate (reference: (-inf, -r))
    // clamped so that a band entirely above or below the map (anchors far
    // outside it) gives r_lo = r_hi and every row takes the no-candidate fill
    const int r_lo = min(max(0, -yb0), nrows);
    const int r_hi = max(min(nrows, pj.Hp - yb0), r_lo);
    const int n_out = r_lo + (nrows - r_hi);
    for (int i = tid; i < n_out * PT_W; i += PT_THREADS) {
      const int k = i / PT_W, l = i - k * PT_W;
      const int r = k < r_lo ? k : r_hi + (k - r_lo);
      sh.x32[r * PT_W + l] = OUT_SENTINEL;
      sh.xsv[r * PT_W + l] = OUT_SENTINEL;
      sh.xdx[r * PT_W + l] = (int8_t)(-jr.rx);
    }
    const int xsub = lane >> lpr_log, xc = lane & (lpr - 1);
    const int rpw = PT_W >> lpr_log;  // band rows per warp step
    const float* srow0 = sh.s + xsh + pj.scale * xc + jr.rx;  // band row 0, dx = 0
    {  // in-map rows only, warp-strided
      const int rb0 = r_lo + warp * rpw, step = PT_WARPS * rpw;
      const float E2 = jr.E2;
      if (pj.scale == 2) {  // even row base + 2*lane: pair alignment follows the shift parity
        switch (jr.rx) {
#define DPM_X_CASE(R) \
  case R: x_rows<R, true>(sh, buf, srow0, rb0, r_hi, step, xsub, xc, code_mask, xodd, E2); break;
          DPM_X_CASE(0) DPM_X_CASE(1) DPM_X_CASE(2) DPM_X_CASE(3) DPM_X_CASE(4) DPM_X_CASE(5)
          DPM_X_CASE(6) DPM_X_CASE(7) DPM_X_CASE(8) DPM_X_CASE(9) DPM_X_CASE(10) DPM_X_CASE(11)
          DPM_X_CASE(12) DPM_X_CASE(13) DPM_X_CASE(14) DPM_X_CASE(15) DPM_X_CASE(16)
#undef DPM_X_CASE
        }
      } else {
        switch (jr.rx) {
#define DPM_X_CASE(R) \
  case R: x_rows<R, false>(sh, buf, srow0, rb0, r_hi, step, xsub, xc, code_mask, 0, E2); break;
          DPM_X_CASE(0) DPM_X_CASE(1) DPM_X_CASE(2) DPM_X_CASE(3) DPM_X_CASE(4) DPM_X_CASE(5)
          DPM_X_CASE(6) DPM_X_CASE(7) DPM_X_CASE(8) DPM_X_CASE(9) DPM_X_CASE(10) DPM_X_CASE(11)
          DPM_X_CASE(12) DPM_X_CASE(13) DPM_X_CASE(14) DPM_X_CASE(15) DPM_X_CASE(16)
#undef DPM_X_CASE
        }
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);  // job p+1 (warp 0's copies)
    __syncthreads();  // x pass done: the band buffer is free for part p+1
    if (have_next) issue_part(buf ^ 1);

    // y pass for this thread's roots; exact values from the x winners
    const float* npy = sh.npy[buf] + RCAP;
    // the radius switch sits outside the per-root loop (R compile-time inside)
    auto y_roots = [&](auto rc) {
      constexpr int R = decltype(rc)::value;
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        int iyr, ixr;
        if (!root_of(k, iyr, ixr)) continue;
        const int iy = ty0 + iyr, ix = tx0 + ixr;
        const int ry = aj.ry0 + iy;
        const int cy = pj.scale * ry + pj.ay;
        const int cx = pj.scale * (aj.rx0 + ix) + pj.ax;
        const int r0 = cy - yb0;  // band row of dy = 0
        const float* xcol = sh.x32 + r0 * PT_W + ixr;
        float m1, m2;
        screen_window<R, PT_W, false>(xcol, npy, npy, code_mask, 0, m1, m2);
        auto exact = [&](int dy) -> double {
          const int row = (r0 + dy) * PT_W + ixr;
          const int dx = sh.xdx[row];
          const double xv = __dadd_rn((double)sh.xsv[row], -pen(pj.cdx, pj.cdxx, dx));
          return __dadd_rn(xv, -pen(pj.cdy, pj.cdyy, dy));
        };
        double best;
        int bi = (__float_as_int(m1) & 63) - R;
        if (m1 < NONE_BELOW) {
          best = -INFINITY;
          bi = -R;
        } else if (m2 >= m1 - jr.E2) {
          bi = y_rescan(xcol, sh.xsv + r0 * PT_W + ixr, sh.xdx + r0 * PT_W + ixr, npy, m1 - jr.E2,
                        R, &sh.pj[buf], best);
        } else {
          best = exact(bi);
        }
        const int bdx = sh.xdx[(r0 + bi) * PT_W + ixr];
        tot[k] = __dadd_rn(tot[k], best);
        const int o = (p * hr + iy) * wr + ix;
        if (posb) posb[o] = pack_pos(cy + bi, cx + bdx);
        if (placedb) placedb[o] = best;
      }
    };
    switch (jr.ry) {
#define DPM_Y_CASE(R) \
  case R: y_roots(std::integral_constant<int, R>{}); break;
      DPM_Y_CASE(0) DPM_Y_CASE(1) DPM_Y_CASE(2) DPM_Y_CASE(3) DPM_Y_CASE(4) DPM_Y_CASE(5)
      DPM_Y_CASE(6) DPM_Y_CASE(7) DPM_Y_CASE(8) DPM_Y_CASE(9) DPM_Y_CASE(10) DPM_Y_CASE(11)
      DPM_Y_CASE(12) DPM_Y_CASE(13) DPM_Y_CASE(14) DPM_Y_CASE(15) DPM_Y_CASE(16)
#undef DPM_Y_CASE
    }
  }

  // bias, totals, tau compaction (part positions read back from `pos`)
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    int iyr, ixr;
    const bool live = root_of(k, iyr, ixr);
    const int iy = ty0 + iyr, ix = tx0 + ixr;
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
    dd.rx = aj.rx0 + ix;
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

// DPM_K3=v1 selects the round-1 kernel (A/B); its tiles are PT_H root rows
// tall, the two-phase kernel's k3v2 tile rows (place2.cu)
static bool k3_use_v1() {
  static const bool v1 = [] {
    const char* e = getenv("DPM_K3");
    return e != nullptr && e[0] == 'v' && e[1] == '1';
  }();
  return v1;
}

extern "C" int64_t dpm_assemble_prepare(dpm_asm_job* jobs, int njobs, const dpm_place_job* pjobs,
                                        int npjobs, int64_t* nfast) {
  if (njobs < 0 || (njobs > 0 && !jobs) || npjobs < 0 || (npjobs > 0 && !pjobs)) {
    set_error("dpm_assemble_prepare: bad job tables");
    return DPM_ERR_ARG;
  }
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
    const int64_t hr = j.ry1 - j.ry0 + 1, wr = j.rx1 - j.rx0 + 1;
    if ((int64_t)(j.nparts > 0 ? j.nparts : 1) * hr * wr > INT32_MAX) {  // 32-bit output offsets
      set_error("dpm_assemble_prepare: job %d: %d parts x %lld x %lld roots exceed 2^31 outputs", i,
                j.nparts, (long long)hr, (long long)wr);
      return DPM_ERR_ARG;
    }
  }
  // tiles: the specialised kernel's (leading tile columns of eligible jobs)
  // numbered by block0 over [0, nf), the generic kernel's by block1 over
  // [0, ng); the round-1 kernel (DPM_K3=v1) numbers every tile by block0
  const bool v1 = k3_use_v1();
  const int th = v1 ? PT_H : k3v2_tile_rows();
  int64_t nf = 0, ng = 0;
  for (int i = 0; i < njobs; ++i) {
    const dpm_asm_job& j = jobs[i];
    const int hr = j.ry1 - j.ry0 + 1, wr = j.rx1 - j.rx0 + 1;
    const int64_t nty = (hr + th - 1) / th, ntx = (wr + PT_W - 1) / PT_W;
    const int fc = v1 ? 0 : k3_fast_cols(j, pjobs, wr);
    jobs[i].block0 = (int32_t)(v1 ? ng : nf);
    jobs[i].block1 = (int32_t)ng;
    if (v1) {
      ng += nty * ntx;
    } else {
      nf += nty * fc;
      ng += nty * (ntx - fc);
    }
  }
  if (nf + ng > INT32_MAX) {
    set_error("dpm_assemble_prepare: too many CTAs");
    return DPM_ERR_ARG;
  }
  if (nfast) *nfast = nf;
  return nf + ng;
}

extern "C" int dpm_place_ranges(const dpm_place_job* pjobs, int njobs, const uint32_t* ranges,
                                dpm_place_range* prep, void* stream) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || (pjobs && ranges && prep)),
              "dpm_place_ranges: null pointer");
  if (njobs == 0) return DPM_OK;
  place_ranges_kernel<<<(unsigned)((njobs + 255) / 256), 256, 0, as_stream(stream)>>>(pjobs, njobs,
                                                                                    ranges, prep);
  DPM_LAUNCHED("place_ranges_kernel");
  return DPM_OK;
}

extern "C" int dpm_assemble(const float* S, const void* smaps, const dpm_place_job* pjobs,
                            const dpm_asm_job* ajobs, int najobs, int64_t nfast, int64_t nblocks,
                            const dpm_place_range* prep, double* total, uint32_t* pos,
                            double* placed, double tau, dpm_detection* dets, int max_dets,
                            int* det_count, void* stream) {
  DPM_REQUIRE(S && smaps && pjobs && ajobs && prep, "dpm_assemble: null pointer");
  DPM_REQUIRE((reinterpret_cast<uintptr_t>(smaps) & 63) == 0,
              "dpm_assemble: tensor maps must be 64-byte aligned");
  DPM_REQUIRE(!dets || (det_count && pos), "dpm_assemble: detections need a counter and positions");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX && nfast >= 0 && nfast <= nblocks,
              "dpm_assemble: nfast / nblocks");
  if (najobs == 0 || nblocks == 0) return DPM_OK;
  if (!k3_use_v1())
    return launch_place2(S, smaps, pjobs, ajobs, najobs, nfast, nblocks - nfast, prep, total, pos,
                         placed, tau, dets, max_dets, det_count, as_stream(stream));
  DPM_REQUIRE(nfast == 0, "dpm_assemble: the round-1 kernel has no specialised tiles");
  const size_t smem = sizeof(PlaceSmem);
  DPM_CUDA(cudaFuncSetAttribute(place_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  place_assemble_kernel<<<(unsigned)nblocks, PT_THREADS, smem, as_stream(stream)>>>(
      S, static_cast<const unsigned char*>(smaps), pjobs, ajobs, najobs, prep, total, pos, placed,
      tau, dets, max_dets, det_count);
  DPM_LAUNCHED("place_assemble_kernel");
  return DPM_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link); host only, no context work.
extern "C" int dpm_smap_encode(const float* S, const dpm_smap_desc* descs, int n, void* maps_host) {
  DPM_REQUIRE(S && (n == 0 || (descs && maps_host)), "dpm_smap_encode: null pointer");
  if (n == 0) return DPM_OK;
  DPM_REQUIRE((reinterpret_cast<uintptr_t>(S) & 15) == 0, "dpm_smap_encode: S must be 16-byte aligned");
  DPM_REQUIRE((reinterpret_cast<uintptr_t>(maps_host) & 63) == 0,
              "dpm_smap_encode: maps_host must be 64-byte aligned");
  static_assert(sizeof(CUtensorMap) == DPM_SMAP_BYTES, "CUtensorMap size");
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (encode == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    DPM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    DPM_REQUIRE(q == cudaDriverEntryPointSuccess && fn != nullptr,
                "dpm_smap_encode: cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  for (int i = 0; i < n; ++i) {
    const dpm_smap_desc& d = descs[i];
    DPM_REQUIRE(d.Ho >= 1 && d.Wo >= 1 && d.nf >= 1 && d.s_off >= 0 && d.s_off % 4 == 0,
                "dpm_smap_encode: descriptor %d has Ho=%d Wo=%d nf=%d s_off=%lld", i, d.Ho, d.Wo,
                d.nf, (long long)d.s_off);
    const int pitch = s_pitch(d.Wo);
    const cuuint64_t dims[3] = {(cuuint64_t)d.Wo, (cuuint64_t)d.Ho, (cuuint64_t)d.nf};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)pitch * 4 * d.Ho};
    const cuuint32_t box[3] = {DPM_SMAP_BOX_W, DPM_SMAP_BOX_H, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(reinterpret_cast<CUtensorMap*>(maps_host) + i,
                              CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                              const_cast<float*>(S + d.s_off), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA);
    DPM_REQUIRE(r == CUDA_SUCCESS, "dpm_smap_encode: descriptor %d rejected (CUresult %d)", i,
                (int)r);
  }
  return DPM_OK;
}
