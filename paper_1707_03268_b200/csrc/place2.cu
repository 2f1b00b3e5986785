// K3 (part placement) + K4 (assembly), two-phase window screen.
//
// Reference: _placement_grid (detection.py:320-373), best_part_placement
// (detection.py:180-207), the assembly of detect / dense_detect
// (detection.py:449, 509-538; 590-613).  Same results as placement.cu (the
// round-1 kernel, kept for A/B as DPM_K3=v1): bit-identical values and
// argmaxes for a given FP32 map -- x pass then y pass, ties to the smallest
// offset, the penalty subtracted in two stages with round-to-nearest FP64
// operations.
//
// Inner screen + outer bound.  The unbounded transform is a window of
// radius r* (App. A.2; r* ~ 10 at the benchmark's maps) but the winner
// almost always lies a few cells from the centre.  Each window is screened
// in FP32 over its inner part |d| <= R1 = min(r, 6) only.  The outer
// candidates are bounded from above by
//   x pass: max of the band row + max over outer d of the screen penalty,
//   y pass: max of the column's x results + the same for y,
// (FP32 rounding is monotone, so the bound dominates every outer screen
// value).  The decoded inner winner is the exact winner of the whole window
// when both the inner runner-up and the outer bound stay below m1 - E2;
// otherwise the lane scans exactly in FP64, in the reference's order: the
// inner window for a near tie, the whole window when the bound fails (rare:
// ~0.1% of x rows at the benchmark's maps).
//
// Screen values carry the candidate's code in their 4 low mantissa bits
// (16 ulps).  E2x = 2^-17 M and E2y = 2^-16 M (M = max|S| + the largest
// penalties of the inner windows, E2in = 2^-15 M from the prologue) cover
// twice the FP32 error plus the encodings, so m2 < m1 - E2 proves the winner
// exact; the outer-bound comparisons add the full-window margin.  The x result
// of a row is one 32-bit word: the winner's screen value with the x code in
// its low 4 bits (13 = no candidate, 14 = a row resolved by an exact scan,
// whose dx the y pass recovers by the same exact scan from global memory),
// so the x loop stores its screen maximum as is.
//
// Structure.  CTA = 8 warps, 32 x 32 root tile of one (image, component,
// root level), three CTAs per SM (24 warps, 85 registers; 64 KB of shared
// memory each).  Per part:
//   wait for the part's S band (TMA boxes, NaN outside the map, mbarrier),
//   x pass over the band rows (lane = centre column), column maxima (shared
//   atomic max),
//   one CTA barrier (x words complete, band buffer free, the next part's job
//   record and tables visible) -> thread 0 issues the next part's band,
//   y pass for the thread's 4 roots: screen the x words of the column; the
//   winner's exact FP64 value from its S value in global memory (L2
//   resident: the TMA just streamed it), so the y pass never reads the band
//   and the next band lands underneath it,
//   a second barrier before the next part's x pass overwrites the x words.
// Job records / tables are triple-buffered; warp 0 copies the next part's
// job record (cp.async) and builds its penalty tables (FP32 screen values,
// exact FP64 penalties) during the x pass.
// Geometry, measured at config 4 (7.77 -> 7.47 ms came from screening work;
// these are the same kernel at other shapes): 12 warps x 48 rows, two CTAs
// per SM, x words double-buffered (one barrier per part): 7.47 ms; the same
// with one x buffer: 7.76; 8 warps x 32 rows at two CTAs per SM (128
// registers): 8.14; 8 warps x 32 rows, one x buffer, THREE CTAs per SM:
// 7.28 ms (the default).  More independent CTAs per SM hide the per-part
// barrier better than the second barrier costs: with the column maxima kept
// as one shared atomic-max row per part (instead of per-warp rows), two x
// buffers also fit three CTAs per SM (75.5 KB) and measured the same 7.28 ms.
// DPM_K3_THREADS / _TH / _XBUF / _MINB rebuild the others.
//
// Two kernels over disjoint tile lists (dpm_assemble_prepare numbers them):
// place2f_kernel, one compile-time instantiation of the above for the bulk
// tiles (at least 17 roots wide, every part at scale 2 with r* in (6, 16]:
// 95% of config 4's roots; per-part geometry computed once by warp 0, rare
// roots resolved out of line), and place2_kernel, the generic form (any
// width, scale, radius) for the rest.  With both at three CTAs per SM the
// pair took K3 from 7.27 to 6.99 ms at config 4; at two 12-warp CTAs per SM
// the specialised kernel had lost (57% against 66% issue).
#include <math.h>
#include <stdlib.h>

#include "place_common.cuh"

namespace dpm {
namespace k3v2 {

#ifndef DPM_K3_THREADS
#define DPM_K3_THREADS 256
#endif
#ifndef DPM_K3_TH
#define DPM_K3_TH 32
#endif
#ifndef DPM_K3_XBUF
#define DPM_K3_XBUF 1
#endif
#ifndef DPM_K3_MINB
#define DPM_K3_MINB 3
#endif
constexpr int THREADS = DPM_K3_THREADS;  // tile geometry: see "Shape" above (A/B macros)
constexpr int XBUF = DPM_K3_XBUF;         // x-word buffers (2: one barrier per part)
constexpr int RMASK = 16;                 // x-pass row iterations per warp and part (<= 12 here)
constexpr int WARPS = THREADS / 32;
constexpr int TH = DPM_K3_TH;               // root rows per tile (32 columns)
constexpr int RPT = TH * PT_W / THREADS;    // roots per thread
static_assert(RPT * THREADS == TH * PT_W, "whole roots per thread");
constexpr int BAND2 = (2 * (TH - 1) + 1 + 2 * RCAP + TMA_BH - 1) / TMA_BH * TMA_BH;  // 128 band rows
constexpr int R1MAX = 6;                    // inner screen radius
constexpr int CODE_NONE = 13;               // x word: no candidate in the window
constexpr int CODE_RARE = 14;               // x word: winner from an exact scan
constexpr int TD = 36;                      // table stride: index d + 16, d in [-16, 16]
static_assert(2 * R1MAX + 1 <= CODE_NONE, "inner codes fit below the special codes");
static_assert(R1MAX == 6, "the prologue's E2in (place_common.cuh) is computed for |d| <= 6");

struct PartTab {
  float npx[TD];    // FP32 screen penalty -pen_x(d) at [d + 16]
  float npx1[TD];   // the same shifted by one element (8-byte aligned odd pairs)
  float npy[TD];
  double px[33];    // exact FP64 pen_x(d) at [d + 16] (reference expression)
  double py[33];
  float out_x, out_y;  // max screen penalty over the outer offsets
  float E2x, E2y, E2o;
};

struct __align__(128) Smem {
  float s[BAND2 * COLS_PITCH];     // S band (TMA, NaN outside the map)
  float x32[XBUF][BAND2 * PT_W];   // x words by part parity
  double tot[RPT][THREADS];        // running totals of the roots, summed in part order
  uint32_t cmk[3][PT_W];           // column maxima of the x words (float_key), part q at q % 3
  uint32_t rmask[WARPS][RMASK];    // x pass: lane masks of the rows to rescan exactly
  PartTab tab[3];                  // tables of part q at slot q % 3
  alignas(16) JobRange jr[3];
  alignas(16) dpm_place_job pj[3];
  dpm_asm_job aj;
  alignas(8) uint64_t band_bar;
};

template <int CODE>
__device__ __forceinline__ float enc4(float v, uint32_t mask) { return enc_idx<CODE>(v, mask); }
__device__ __forceinline__ float enc_code(float v, int code) {
  return __uint_as_float((__float_as_uint(v) & ~15u) | (uint32_t)code);
}
__device__ __forceinline__ int code_of(float w) { return (int)(__float_as_uint(w) & 15u); }
// (bits(v) & mask) | code in one lop3; code is a constant after unrolling
__device__ __forceinline__ float enc_idx_rt(float v, uint32_t mask, int code) {
  return __uint_as_float((__float_as_uint(v) & mask) | (uint32_t)code);
}

// Top-2 reduction tree.  A node is (h, l): its best candidate and the best
// of the others; NaN candidates (outside the map) drop out of both.  A
// balanced tree keeps the dependency chain short (the screens run at 4 warps
// per scheduler, so chain latency is not hidden).
__device__ __forceinline__ void leaf2(float a, float b, float& h, float& l) {
  h = fmaxf(a, b);
  l = fmin_nan(a, b);
}
__device__ __forceinline__ void join2(float& h, float& l, float h2, float l2) {
  l = fmaxf(fmaxf(l, l2), fmin_nan(h, h2));
  h = fmaxf(h, h2);
}
template <int N>
__device__ __forceinline__ void tree_reduce(float (&h)[N > 0 ? N : 1], float (&l)[N > 0 ? N : 1]) {
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int k = 0; k + w < N; k += 2 * w) join2(h[k], l[k], h[k + w], l[k + w]);
}

// Leaves of the packed screen: pair k = candidates (d0 + 2k, d0 + 2k + 1)
// at p0 + 2k (8-byte aligned), codes 2k and 2k + 1 (compile-time: the
// encoding lop3 takes the code as its immediate).
template <int R1, int K>
__device__ __forceinline__ void leaves_packed(const float* __restrict__ p0,
                                              const unsigned long long (&pp)[R1 > 0 ? R1 : 1],
                                              uint32_t mask, float (&h)[R1 > 0 ? R1 : 1],
                                              float (&l)[R1 > 0 ? R1 : 1]) {
  if constexpr (K < R1) {
    const unsigned long long s2 = *reinterpret_cast<const unsigned long long*>(p0 + 2 * K);
    unsigned long long v2;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(v2) : "l"(s2), "l"(pp[K]));
    float va, vb;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(va), "=f"(vb) : "l"(v2));
    leaf2(enc4<2 * K>(va, mask), enc4<2 * K + 1>(vb, mask), h[K], l[K]);
    leaves_packed<R1, K + 1>(p0, pp, mask, h, l);
  }
}
// Leaves of the strided screen: pair k = offsets (-R1 + 2k, -R1 + 2k + 1),
// codes d + R1.
template <int R1, int STRIDE, int K>
__device__ __forceinline__ void leaves_strided(const float* __restrict__ src,
                                               const float (&pr)[2 * R1 + 1], uint32_t mask,
                                               float (&h)[R1 > 0 ? R1 : 1],
                                               float (&l)[R1 > 0 ? R1 : 1]) {
  if constexpr (K < R1) {
    constexpr int D = -R1 + 2 * K;
    leaf2(enc4<D + R1>(src[D * STRIDE] + pr[D + R1], mask),
          enc4<D + 1 + R1>(src[(D + 1) * STRIDE] + pr[D + 1 + R1], mask), h[K], l[K]);
    leaves_strided<R1, STRIDE, K + 1>(src, pr, mask, h, l);
  }
}

// Packed inner screen (x pass at scale 2): the pairs, then the single
// candidate (code 2 R1).  m1 = top encoded value, m2 = best of the others.
template <int R1>
__device__ __forceinline__ void scr_packed(const float* __restrict__ p0,
                                           const unsigned long long (&pp)[R1 > 0 ? R1 : 1],
                                           float single, uint32_t mask, float& m1, float& m2) {
  const float c = enc4<2 * R1>(single, mask);
  if constexpr (R1 == 0) {
    m1 = fmaxf(c, -INFINITY);
    m2 = -INFINITY;
  } else {
    float h[R1], l[R1];
    leaves_packed<R1, 0>(p0, pp, mask, h, l);
    tree_reduce<R1>(h, l);
    m2 = fmaxf(l[0], fmin_nan(h[0], c));
    m1 = fmaxf(fmaxf(h[0], c), -INFINITY);  // all candidates outside the map: -inf, not NaN
  }
}

// Strided inner screen (x pass at scale 1, y pass): candidates src[d*STRIDE]
// + pr[d + R1], d = -R1..R1, code d + R1.
template <int R1, int STRIDE>
__device__ __forceinline__ void scr_strided(const float* __restrict__ src,
                                            const float (&pr)[2 * R1 + 1], uint32_t mask,
                                            float& m1, float& m2) {
  const float c = enc4<2 * R1>(src[R1 * STRIDE] + pr[2 * R1], mask);
  if constexpr (R1 == 0) {
    m1 = fmaxf(c, -INFINITY);
    m2 = -INFINITY;
  } else {
    float h[R1], l[R1];
    leaves_strided<R1, STRIDE, 0>(src, pr, mask, h, l);
    tree_reduce<R1>(h, l);
    m2 = fmaxf(l[0], fmin_nan(h[0], c));
    m1 = fmaxf(fmaxf(h[0], c), -INFINITY);
  }
}

// Exact x window scan in the reference's order (ascending dx, strict '>')
// over dx in [lo, hi], band cells (s0 = dx = 0; NaN = outside the map).
// Returns the winner, lo when there is no candidate.  Rare: out of line.
__device__ __noinline__ int x_exact_band(const float* s0, int lo, int hi, const double* px) {
  double best = -INFINITY;
  int bi = lo;
  for (int d = lo; d <= hi; ++d) {
    const float v = s0[d];
    if (v != v) continue;
    const double e = __dadd_rn((double)v, -px[d + 16]);
    if (e > best) { best = e; bi = d; }
  }
  return bi;
}

// The same scan over the map in global memory (row pointer at column cx):
// recovers the dx of an x word with CODE_RARE (the x pass found it with this
// very scan over the band, so both agree).
__device__ __noinline__ int x_exact_global(const float* __restrict__ srow, int cx, int Wp, int r,
                                           const double* px) {
  double best = -INFINITY;
  int bi = -r;
  const int lo = max(-r, -cx), hi = min(r, Wp - 1 - cx);
  for (int d = lo; d <= hi; ++d) {
    const double e = __dadd_rn((double)__ldg(srow + d), -px[d + 16]);
    if (e > best) { best = e; bi = d; }
  }
  return bi;
}

struct XDec {  // decoding of the x codes of one part in one tile
  int d0, ds, c2r1;
};

// Exact y scan over dy in [lo, hi] for one root in the reference's order:
// x words of the root's column (xcol at dy = 0), exact x values from the S
// values in global memory.  With thr > -inf (a near tie of the inner
// screen) only the rows whose screen value -- recomputed bit for bit: same
// add, same code -- reaches thr are candidates; the others are below the
// winner by more than the screening error.  Returns (dy + 64) | (dx + 64)
// << 8, or -1 when no row has a candidate.
__device__ __noinline__ int y_exact(const float* xcol, const float* __restrict__ smap, int pitch,
                                    int cy, int cx, int lo, int hi, int Wp, const PartTab* tb,
                                    XDec xd, int rx, float thr, uint32_t mask, int r1, int ta,
                                    int tb2) {
  // Two-row near tie (the common case): when exactly rows ta and tb2 (the
  // screen's top two) reach thr and both carry inner x codes, their two S
  // loads are issued together -- one L2 round trip, not one per row.
  if (ta <= hi && tb2 <= hi) {
    int n = 0;
    for (int dy = lo; dy <= hi; ++dy) {
      const float w = xcol[dy * PT_W];
      if (code_of(w) != CODE_NONE && enc_idx_rt(w + tb->npy[dy + 16], mask, dy + r1) >= thr) ++n;
    }
    const float wa = xcol[ta * PT_W], wb = xcol[tb2 * PT_W];
    const int ca = code_of(wa), cb = code_of(wb);
    if (n == 2 && ca <= 12 && cb <= 12 && ta != tb2) {
      const int da = ca == xd.c2r1 ? xd.ds : xd.d0 + ca;
      const int db = cb == xd.c2r1 ? xd.ds : xd.d0 + cb;
      const float sa = __ldg(smap + (int64_t)(cy + ta) * pitch + cx + da);
      const float sb = __ldg(smap + (int64_t)(cy + tb2) * pitch + cx + db);
      const double ea = __dadd_rn(__dadd_rn((double)sa, -tb->px[da + 16]), -tb->py[ta + 16]);
      const double eb = __dadd_rn(__dadd_rn((double)sb, -tb->px[db + 16]), -tb->py[tb2 + 16]);
      // the reference's order: ascending dy, strict '>'
      const bool a_first = ta < tb2;
      const double e1 = a_first ? ea : eb, e2 = a_first ? eb : ea;
      const int d1 = a_first ? ta : tb2, d2 = a_first ? tb2 : ta;
      const int x1 = a_first ? da : db, x2 = a_first ? db : da;
      if (e2 > e1) return (d2 + 64) | ((x2 + 64) << 8);
      if (e1 > -INFINITY) return (d1 + 64) | ((x1 + 64) << 8);
    }
  }
  double best = -INFINITY;
  int out = -1;
  for (int dy = lo; dy <= hi; ++dy) {
    const float w = xcol[dy * PT_W];
    const int c = code_of(w);
    if (c == CODE_NONE) continue;
    if (enc_idx_rt(w + tb->npy[dy + 16], mask, dy + r1) < thr) continue;
    const float* srow = smap + (int64_t)(cy + dy) * pitch;
    const int dx = c == CODE_RARE ? x_exact_global(srow + cx, cx, Wp, rx, tb->px)
                                  : (c == xd.c2r1 ? xd.ds : xd.d0 + c);
    const double xv = __dadd_rn((double)__ldg(srow + cx + dx), -tb->px[dx + 16]);
    const double e = __dadd_rn(xv, -tb->py[dy + 16]);
    if (e > best) {
      best = e;
      out = (dy + 64) | ((dx + 64) << 8);
    }
  }
  return out;
}

// x pass of one part over band rows rb0, rb0 + step, ... (< r_hi) at lane
// centre xc (FULLW: one row per warp iteration, lane = column; else lpr
// lanes per row, 32 / lpr rows per iteration).  Stores the x words and folds
// the column maxima into cmaxv.  Rows whose screen is not conclusive (near
// tie, failed outer bound, no inner candidate) are only flagged in the main
// loop -- one ballot per iteration, its mask parked in shared memory when
// non-zero -- and rescanned exactly afterwards, so the hot loop is straight
// line code.
template <int R1, bool PACKED, bool OUTER, bool FULLW>
__device__ __forceinline__ void x_pass(float* __restrict__ x32, const float* __restrict__ band,
                                       const PartTab& tb, uint32_t* __restrict__ rmask, int lane,
                                       int rb0, int r_hi, int step, int xsub, int xc, int lpr,
                                       int wt, int reach, int c0, int scale, XDec xd, int rx,
                                       uint32_t mask, float& cmaxv, int rin_lo, int rin_hi) {
  const float E2 = tb.E2x;
  float pr[2 * R1 + 1];
  unsigned long long pp[R1 > 0 ? R1 : 1];
  if constexpr (PACKED) {
    // pair k starts at d0 + 2k: table index d0 + 2k + 16, shifted table if odd
    const float* tp = ((xd.d0 + 16) & 1) ? tb.npx1 + xd.d0 + 17 : tb.npx + xd.d0 + 16;
#pragma unroll
    for (int k = 0; k < R1; ++k) pp[k] = *reinterpret_cast<const unsigned long long*>(tp + 2 * k);
    pr[0] = tb.npx[xd.ds + 16];
  } else {
#pragma unroll
    for (int d = -R1; d <= R1; ++d) pr[d + R1] = tb.npx[d + 16];
  }
  const float out = tb.out_x;
  const int xsh = c0 - rx;  // shared column of band column 0
  const int cstep = PACKED ? 2 : scale;
  uint32_t iters = 0;  // bit i: iteration i flagged a rare row
  int it = 0;
  // maximum of band row r over the columns this row's windows reach
  auto rowmax = [&](int r) {
    const float* row = band + r * COLS_PITCH;
    float mr;
    if constexpr (FULLW) {
      const float a = row[xsh + xc];
      const float b = xc + 32 < reach ? row[xsh + xc + 32] : -INFINITY;
      const float c = xc + 64 < reach ? row[xsh + xc + 64] : -INFINITY;
      const float l = fmaxf(a, fmaxf(b, c));
      asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(l));
    } else {
      mr = -INFINITY;
      for (int c = xc; c < reach; c += lpr) mr = fmaxf(mr, row[xsh + c]);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1)
        if (o < lpr) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    }
    return mr;
  };
  // screen of band row r (m1, m2, outer bound failed)
  auto screen = [&](int r, float& m1, float& m2, bool& full) {
    const float* row = band + r * COLS_PITCH;
    const float* s0 = row + c0 + cstep * xc;  // dx = 0
    DPM_CHECK(r >= 0 && r < BAND2, "x pass: band row");
    DPM_CHECK(c0 + cstep * xc - R1 >= 0 && c0 + cstep * xc + R1 < COLS_PITCH &&
                  (!PACKED || (c0 + cstep * xc + xd.d0 >= 0 &&
                               c0 + cstep * xc + xd.d0 + 2 * R1 < COLS_PITCH)),
              "x pass: band column");
    if constexpr (PACKED) scr_packed<R1>(s0 + xd.d0, pp, s0[xd.ds] + pr[0], mask, m1, m2);
    else scr_strided<R1, 1>(s0, pr, mask, m1, m2);
    full = false;
    if constexpr (OUTER) full = rowmax(r) + out + tb.E2o >= m1 - E2;
  };
  // flag / store the screen result of row r (loop iteration it)
  auto finish = [&](int r, bool live, int it, float m1, float m2, bool full) {
    const bool rare = live && (full || m1 < NONE_BELOW || m2 >= m1 - E2);
    const uint32_t bal = __ballot_sync(0xffffffffu, rare);
    if (bal != 0u) {
      DPM_CHECK(it < RMASK, "x pass: at most RMASK row iterations per warp");
      iters |= 1u << it;
      if (lane == 0) rmask[it] = bal;  // it < RMASK (checked above)
    }
    if (live) {  // certified: the screen maximum, its code names the winner
      DPM_CHECK(r >= 0 && r < BAND2 && xc >= 0 && xc < PT_W, "x pass: x word");
      x32[r * PT_W + xc] = m1;
      cmaxv = fmaxf(cmaxv, m1);
    }
  };
  int rb = rb0;
  for (; rb < r_hi; rb += step, ++it) {
    const int r = FULLW ? rb : min(rb + xsub, r_hi - 1);  // clamped: spare lanes still shuffle
    const bool live = (FULLW || rb + xsub < r_hi) && xc < wt;
    float m1, m2;
    bool full;
    screen(r, m1, m2, full);
    finish(r, live, it, m1, m2, full);
  }
  if (iters == 0u) return;
  __syncwarp();
  // exact rescans of the flagged rows over the whole window (the reference's
  // order); the winner's screen value with CODE_RARE, or no candidate
  while (iters != 0u) {
    const int i = __ffs(iters) - 1;
    iters &= iters - 1;
    if (!((rmask[i] >> lane) & 1u)) continue;
    const int r = rb0 + i * step + xsub;
    const float* s0 = band + r * COLS_PITCH + c0 + cstep * xc;
    const int xi = x_exact_band(s0, -rx, rx, tb.px);
    const float v = s0[xi];
    const float word = v == v ? enc_code(v + tb.npx[xi + 16], CODE_RARE)
                              : enc_code(OUT_SENTINEL, CODE_NONE);
    x32[r * PT_W + xc] = word;
    cmaxv = fmaxf(cmaxv, word);
  }
}

// y pass of one part for the thread's roots (R1 = inner y radius).  Adds
// the placed values to tot[] in part order, writes positions / placed.
template <int R1, bool OUTER, int K0, int G, typename RootOf>
__device__ __forceinline__ void y_group(const float* __restrict__ x32, const float* __restrict__ smap,
                                       int pitch, const dpm_place_job* pjs, const PartTab& tb,
                                       XDec xd, int rx, int ry, int yb0, int ty0, int tx0,
                                       uint32_t mask, RootOf root_of, const dpm_asm_job& aj, int p,
                                       int hr, int wr, double* __restrict__ tot, uint32_t* posb,
                                       double* placedb, float cmax) {
  const float E2 = tb.E2y;
  float pr[2 * R1 + 1];
#pragma unroll
  for (int d = -R1; d <= R1; ++d) pr[d + R1] = tb.npy[d + 16];
  const float bound = OUTER ? cmax + tb.out_y + tb.E2o : -INFINITY;  // outer rows of this column
  const int scale = pjs->scale, ay = pjs->ay, ax = pjs->ax;
  // phase 1: screen every root, start the S loads of the certified winners.
  // st = state (0 dead, 1 certified, 2 exact inner scan, 3 exact full scan,
  // 4 no candidate, 5 certified dy whose x row was scanned exactly)
  //      | (dy + 64) << 3 | (dx + 64) << 10
  int st[G];
  float sv[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int k = K0 + g;
    int iyr, ixr;
    int& stk = st[g];
    stk = 0;
    sv[g] = 0.f;
    if (!root_of(k, iyr, ixr)) continue;
    const int cy = scale * (aj.ry0 + ty0 + iyr) + ay;
    const float* xcol = x32 + (cy - yb0) * PT_W + ixr;
    DPM_CHECK(cy - yb0 - R1 >= 0 && cy - yb0 + R1 < BAND2 && ixr >= 0 && ixr < PT_W,
              "y pass: x words of the inner window");
    float m1 = -INFINITY, m2 = -INFINITY;
    scr_strided<R1, PT_W>(xcol, pr, mask, m1, m2);
    const float lo = m1 - E2;
    if (bound >= lo) {
      stk = 3;
    } else if (m1 < NONE_BELOW) {
      stk = 4;
    } else if (m2 >= lo) {
      // rescan only the rows whose screen value reaches lo; the two top rows
      // (codes of m1, m2) ride along for the common two-row near tie
      stk = 2 | ((code_of(m1) - R1 + 64) << 3) | ((code_of(m2) - R1 + 64) << 10);
      sv[g] = lo;
    } else {
      const int dy = code_of(m1) - R1;
      const int c = code_of(xcol[dy * PT_W]);
      if (c == CODE_RARE) {
        stk = 5 | ((dy + 64) << 3);
      } else {
        const int dx = c == xd.c2r1 ? xd.ds : xd.d0 + c;
        const int cx = scale * (aj.rx0 + tx0 + ixr) + ax;
        stk = 1 | ((dy + 64) << 3) | ((dx + 64) << 10);
        DPM_CHECK(cy + dy >= 0 && cy + dy < pjs->Hp && cx + dx >= 0 && cx + dx < pjs->Wp,
                  "y pass: winner inside the map");
        sv[g] = __ldg(smap + (int64_t)(cy + dy) * pitch + cx + dx);
      }
    }
  }
  // phase 2: exact FP64 values, totals and outputs
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int k = K0 + g;
    int state = st[g] & 7;
    if (state == 0) continue;
    int iyr, ixr;
    root_of(k, iyr, ixr);
    const int iy = ty0 + iyr, ix = tx0 + ixr;
    const int cy = scale * (aj.ry0 + iy) + ay;
    const int cx = scale * (aj.rx0 + ix) + ax;
    int dy = ((st[g] >> 3) & 127) - 64, dx = ((st[g] >> 10) & 127) - 64;
    float s = sv[g];
    if (state != 1) {
      if (state == 5) {
        dx = x_exact_global(smap + (int64_t)(cy + dy) * pitch + cx, cx, pjs->Wp, rx, tb.px);
      } else if (state != 4) {
        const float* xcol = x32 + (cy - yb0) * PT_W + ixr;
        const int q = y_exact(xcol, smap, pitch, cy, cx, state == 2 ? -R1 : -ry,
                              state == 2 ? R1 : ry, pjs->Wp, &tb, xd, rx,
                              state == 2 ? sv[g] : -INFINITY, mask, R1,
                              state == 2 ? dy : 1000, state == 2 ? dx : 1000);
        if (q < 0) {
          state = 4;
        } else {
          dy = (q & 255) - 64;
          dx = (q >> 8) - 64;
        }
      }
      if (state == 4) {  // no candidate: the reference's (-inf, first dy, first row's dx)
        dy = -ry;
        dx = -rx;
      } else {
        s = __ldg(smap + (int64_t)(cy + dy) * pitch + cx + dx);
      }
    }
    double best = -INFINITY;
    if (state != 4) best = __dadd_rn(__dadd_rn((double)s, -tb.px[dx + 16]), -tb.py[dy + 16]);
    tot[k * THREADS] = __dadd_rn(tot[k * THREADS], best);
    const int o = (p * hr + iy) * wr + ix;
    if (posb) posb[o] = pack_pos(cy + dy, cx + dx);
    if (placedb) placedb[o] = best;
  }
}

// y pass of one part for the thread's RPT roots in one group (the loads of
// a group are in flight together; two groups of 2 spill nothing but measured
// 7.77 ms against 7.47 ms for one group of 4 with ~400 B of rare-path spills)
template <int R1, bool OUTER, typename RootOf>
__device__ __forceinline__ void y_pass(const float* __restrict__ x32, const float* __restrict__ smap,
                                       int pitch, const dpm_place_job* pjs, const PartTab& tb,
                                       XDec xd, int rx, int ry, int yb0, int ty0, int tx0,
                                       uint32_t mask, RootOf root_of, const dpm_asm_job& aj, int p,
                                       int hr, int wr, double* __restrict__ tot, uint32_t* posb,
                                       double* placedb, float cmax) {
  constexpr int G0 = RPT;
  y_group<R1, OUTER, 0, G0>(x32, smap, pitch, pjs, tb, xd, rx, ry, yb0, ty0, tx0, mask, root_of, aj,
                            p, hr, wr, tot, posb, placedb, cmax);
  if constexpr (RPT > G0)
    y_group<R1, OUTER, G0, RPT - G0>(x32, smap, pitch, pjs, tb, xd, rx, ry, yb0, ty0, tx0, mask,
                                     root_of, aj, p, hr, wr, tot, posb, placedb, cmax);
}

// Penalty tables of a part (warp 0): FP32 screen values, exact FP64
// penalties in the reference's expression, the outer maxima and the
// screening bounds.
__device__ __forceinline__ void build_tab(PartTab& tb, const dpm_place_job& pj, const JobRange& jr,
                                          int lane) {
  for (int i = lane; i < 33; i += 32) {
    const int d = i - 16;
    const double qx = pen(pj.cdx, pj.cdxx, d), qy = pen(pj.cdy, pj.cdyy, d);
    tb.px[i] = qx;
    tb.py[i] = qy;
    tb.npx[i] = (float)(-qx);
    tb.npx1[i + 1] = (float)(-qx);
    tb.npy[i] = (float)(-qy);
  }
  __syncwarp();
  const int d = lane - 16;  // lanes cover d = -16..15; d = 16 is lane 0's too
  const bool ox = abs(d) > R1MAX && abs(d) <= jr.rx, oy = abs(d) > R1MAX && abs(d) <= jr.ry;
  float mx = ox ? tb.npx[lane] : -INFINITY, my = oy ? tb.npy[lane] : -INFINITY;
  if (16 <= jr.rx && lane == 0) mx = fmaxf(mx, tb.npx[32]);
  if (16 <= jr.ry && lane == 0) my = fmaxf(my, tb.npy[32]);
  float rmx, rmy;
  asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(rmx) : "f"(mx));
  asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(rmy) : "f"(my));
  if (lane == 0) {
    tb.out_x = rmx;
    tb.out_y = rmy;
    // screened values are bounded by M = max|S| + the inner windows' largest
    // penalties (E2in = 2^-15 M from the prologue; the full-window E2 covers
    // the outer-bound comparisons): E2x = 2^-17 M (4-bit codes), E2y =
    // 2^-16 M (the x words' codes too)
    tb.E2x = jr.E2in * 0.25f;
    tb.E2y = jr.E2in * 0.5f;
    tb.E2o = jr.E2 * 0.25f;
  }
}

// Bias, totals and tau compaction of a tile's roots (part positions read back
// from `pos`); root k of the thread at (iyr, ixr) when live.
__device__ __forceinline__ void emit_root(const dpm_asm_job& aj, bool live, int iy, int ix, int wr,
                                          double t0, double* __restrict__ total,
                                          const uint32_t* __restrict__ pos, double tau,
                                          dpm_detection* __restrict__ dets, int max_dets,
                                          int* __restrict__ det_count, int lane, int hr) {
  const double t = __dadd_rn(t0, aj.bias);
  if (live && aj.total_off >= 0) total[aj.total_off + (int64_t)iy * wr + ix] = t;
  if (dets == nullptr) return;
  const bool hit = live && t >= tau;
  const unsigned bal = __ballot_sync(0xffffffffu, hit);
  if (bal == 0u) return;
  const int leader = __ffs(bal) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(det_count, __popc(bal));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!hit) return;
  const int slot = base + __popc(bal & ((1u << lane) - 1u));
  if (slot >= max_dets) return;
  dpm_detection d;
  d.image = aj.image;
  d.level = aj.level;
  d.component = aj.component;
  d.ry = aj.ry0 + iy;
  d.rx = aj.rx0 + ix;
  d.nparts = aj.nparts;
  d.score = t;
  for (int q = 0; q < DPM_MAX_PARTS; ++q)
    d.parts[q] = (q < aj.nparts && aj.pos_off >= 0)
                     ? pos[aj.pos_off + ((int64_t)q * hr + iy) * wr + ix]
                     : 0u;
  dets[slot] = d;
}

__global__ void __launch_bounds__(THREADS, DPM_K3_MINB)
place2_kernel(const float* __restrict__ S, const unsigned char* __restrict__ smaps,
              const dpm_place_job* __restrict__ pjobs, const dpm_asm_job* __restrict__ ajobs,
              int najobs, const dpm_place_range* __restrict__ prep, double* __restrict__ total,
              uint32_t* __restrict__ pos, double* __restrict__ placed, double tau,
              dpm_detection* __restrict__ dets, int max_dets, int* __restrict__ det_count,
              int fast_on) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& sh = *reinterpret_cast<Smem*>(smem_raw);
  const int jid = find_job_warp(ajobs, najobs, blockIdx.x,
                                [](const dpm_asm_job& j) { return j.block1; });
  int tid_, lane_, warp_;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid_));
  asm volatile("and.b32 %0, %1, 31;" : "=r"(lane_) : "r"(tid_));
  asm volatile("shr.u32 %0, %1, 5;" : "=r"(warp_) : "r"(tid_));
  const int tid = tid_, lane = lane_, warp = __shfl_sync(0xffffffffu, warp_, 0);
  const uint32_t band_bar = pl_smem(&sh.band_bar);
  if (warp == 0) {  // this CTA's tile among the job's generic ones (block1 numbering)
    const dpm_asm_job& g = ajobs[jid];
    const int w = g.rx1 - g.rx0 + 1, nt = (w + PT_W - 1) / PT_W;
    const int fc = fast_on ? k3_fast_cols_warp(g, pjobs, w, lane) : 0;
    const int t = (int)blockIdx.x - g.block1;
    if (lane == 0) sh.rmask[0][0] = fc > 0 ? (t << 16) | (nt - 1) : ((t / nt) << 16) | (t % nt);
  }
  if (tid == 0) {
    sh.aj = ajobs[jid];
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(band_bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 3 * PT_W) (&sh.cmk[0][0])[tid] = 0u;  // float_key(-inf) > 0: every value beats it
  __syncthreads();
  const dpm_asm_job& aj = sh.aj;
  const int hr = aj.ry1 - aj.ry0 + 1, wr = aj.rx1 - aj.rx0 + 1;
  const int ty0 = (int)(sh.rmask[0][0] >> 16) * TH, tx0 = (int)(sh.rmask[0][0] & 0xffffu) * PT_W;
  const int wt = min(PT_W, wr - tx0), h_tile = min(TH, hr - ty0);
  const int lpr_log = wt > 16 ? 5 : wt > 8 ? 4 : wt > 4 ? 3 : wt > 2 ? 2 : wt > 1 ? 1 : 0;
  const int lpr = 1 << lpr_log;
  auto root_of = [=](int k, int& iyr, int& ixr) -> bool {
    const int e = tid + THREADS * k;
    iyr = e >> lpr_log;
    ixr = e & (lpr - 1);
    return iyr < h_tile && ixr < wt;
  };
  const int ry_lo = aj.ry0 + ty0;
  const int ry_hi = aj.ry0 + ty0 + h_tile - 1;
  const int rx_lo = aj.rx0 + tx0;
  // ~15 from a value the compiler cannot fold (najobs > 0): the code, not the
  // mask, is each encoding lop3's immediate
  const uint32_t mask = ~15u | ((uint32_t)najobs >> 31);

  double* const tot = &sh.tot[0][tid];  // tot[k * THREADS]: root k of this thread
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    int iyr, ixr;
    double t = 0.0;
    if (aj.root_off >= 0 && root_of(k, iyr, ixr))
      t = (double)__ldg(S + aj.root_off + (int64_t)(ry_lo + iyr) * aj.root_pitch + rx_lo + ixr);
    tot[k * THREADS] = t;
  }

  auto staged_ok = [&](const dpm_place_job& pj, const JobRange& jr) {
    return jr.rx <= RCAP && jr.ry <= RCAP && pj.scale <= 2;
  };
  // job record + r*/E2 of part q into slot q % 3 (warp 0, cp.async)
  auto fetch_job = [&](int q) {
    const int slot = q % 3;
    if (lane < (int)(sizeof(dpm_place_job) / 8)) {
      const uint32_t sa = pl_smem(reinterpret_cast<unsigned char*>(&sh.pj[slot]) + 8 * lane);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa),
                   "l"(reinterpret_cast<const unsigned char*>(pjobs + aj.part_job0 + q) + 8 * lane));
    } else if (lane == 31) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(pl_smem(&sh.jr[slot])),
                   "l"(prep + aj.part_job0 + q));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  auto finish_job = [&](int q) {  // warp 0: wait for the copy, build the tables
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();
    build_tab(sh.tab[q % 3], sh.pj[q % 3], sh.jr[q % 3], lane);
  };
  // band of part q (thread 0): TMA boxes covering the band rows; the buffer's
  // previous band was last read before the barrier preceding this call
  auto issue_band = [&](int q) {
    const dpm_place_job& pj = sh.pj[q % 3];
    const JobRange& jr = sh.jr[q % 3];
    if (tid != 0 || !staged_ok(pj, jr)) return;
    const int yb0 = pj.scale * ry_lo + pj.ay - jr.ry;
    const int nrows = pj.scale * (ry_hi - ry_lo) + 1 + 2 * jr.ry;
    const int xb0 = pj.scale * rx_lo + pj.ax - jr.rx;
    const int nbox = (nrows + TMA_BH - 1) / TMA_BH;
    DPM_CHECK(nbox * TMA_BH <= BAND2 && xb0 - (xb0 & ~3) + pj.scale * (PT_W - 1) + 1 + 2 * jr.rx <= COLS_PITCH,
              "band boxes fit the band buffer");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(band_bar),
                 "r"((uint32_t)nbox * TMA_BOX_BYTES)
                 : "memory");
    const void* map = smaps + (int64_t)pj.smap * DPM_SMAP_BYTES;
    const uint32_t dst = pl_smem(sh.s);
    for (int k = 0; k < nbox; ++k)
      tma_band_box(dst + (uint32_t)k * TMA_BOX_BYTES, map, xb0 & ~3, yb0 + k * TMA_BH, pj.smap_z,
                   band_bar);
  };

  uint32_t bands = 0;  // bands staged so far: band k completes barrier phase k
  if (aj.nparts > 0) {
    if (warp == 0) {
      fetch_job(0);
      finish_job(0);
    }
    __syncthreads();
    issue_band(0);
  }
  uint32_t* const posb = aj.pos_off >= 0 ? pos + aj.pos_off : nullptr;
  double* const placedb = aj.placed_off >= 0 ? placed + aj.placed_off : nullptr;
  const int xsub = lane >> lpr_log, xc = lane & (lpr - 1);
  for (int p = 0; p < aj.nparts; ++p) {
    const int slot = p % 3, buf = XBUF == 2 ? p & 1 : 0;
    if (XBUF == 1 && p > 0) __syncthreads();  // y(p-1) done with the single x-word buffer
    // column maxima of part p+1 go to slot (p+1) % 3, last read by y(p-2), which
    // every warp finished before the barrier after x(p-1)
    if (warp == 0) sh.cmk[(p + 1) % 3][lane] = 0u;
    const dpm_place_job& pj = sh.pj[slot];
    const JobRange& jr = sh.jr[slot];
    const PartTab& tb = sh.tab[slot];
    // job p+1 into slot (p+1) % 3 = (p-2) % 3, whose last readers (part p-2's
    // y pass) finished before the previous barrier
    const bool have_next = p + 1 < aj.nparts;
    if (warp == 0 && have_next) fetch_job(p + 1);
    const bool staged = staged_ok(pj, jr);
    const int rx = jr.rx, ry = jr.ry;
    const int yb0 = pj.scale * ry_lo + pj.ay - ry;
    const int xsh = (pj.scale * rx_lo + pj.ax - rx) & 3;  // band column 0's shared column
    const int c0 = xsh + rx;                               // shared column of lane 0's dx = 0
    const int r1x = min(rx, R1MAX), r1y = min(ry, R1MAX);
    XDec xd;
    if (pj.scale == 2) {  // packed pairs start on an even shared column
      const int s = ((c0 & 1) + r1x) & 1;
      xd.d0 = -r1x + s;
      xd.ds = s ? -r1x : r1x;
    } else {
      xd.d0 = -r1x;
      xd.ds = r1x;
    }
    xd.c2r1 = 2 * r1x;
    float* x32 = sh.x32[buf];
    if (staged) {
      pl_mbar_wait(band_bar, bands++ & 1);
      const int nrows = pj.scale * (ry_hi - ry_lo) + 1 + 2 * ry;
      // rows outside the map: no candidate (reference: (-inf, -r))
      const int r_lo = min(max(0, -yb0), nrows);
      const int r_hi = max(min(nrows, pj.Hp - yb0), r_lo);
      const int n_out = r_lo + (nrows - r_hi);
      const float sent = enc_code(OUT_SENTINEL, CODE_NONE);
      for (int i = tid; i < n_out * PT_W; i += THREADS) {
        const int k = i / PT_W, l = i - k * PT_W;
        DPM_CHECK((k < r_lo ? k : r_hi + (k - r_lo)) < BAND2, "rows outside the map");
        x32[(k < r_lo ? k : r_hi + (k - r_lo)) * PT_W + l] = sent;
      }
      const int rpw = PT_W >> lpr_log;
      const int rb0 = r_lo + warp * rpw, step = WARPS * rpw;
      const int reach = pj.scale * (wt - 1) + 1 + 2 * rx;  // band columns the windows reach
      float cmaxv = n_out > 0 ? sent : -INFINITY;
      const bool outer = rx > R1MAX;
      // band rows some root's inner y window (|dy| <= min(ry, R1MAX)) reaches
      const int rin_lo = ry - r1y, rin_hi = nrows - 1 - (ry - r1y);
#define DPM_XARGS x32, sh.s, tb, sh.rmask[warp], lane, rb0, r_hi, step, xsub, xc, lpr, wt, reach, c0, pj.scale, xd, rx, mask, cmaxv, rin_lo, rin_hi
      if (pj.scale == 2) {
        if (outer) {
          if (lpr == 32) x_pass<R1MAX, true, true, true>(DPM_XARGS);
          else x_pass<R1MAX, true, true, false>(DPM_XARGS);
        } else {
          switch (r1x) {
#define DPM_XC(R) case R: x_pass<R, true, false, false>(DPM_XARGS); break;
            DPM_XC(0) DPM_XC(1) DPM_XC(2) DPM_XC(3) DPM_XC(4) DPM_XC(5) DPM_XC(6)
#undef DPM_XC
          }
        }
      } else {
        if (outer) {
          x_pass<R1MAX, false, true, false>(DPM_XARGS);
        } else {
          switch (r1x) {
#define DPM_XC(R) case R: x_pass<R, false, false, false>(DPM_XARGS); break;
            DPM_XC(0) DPM_XC(1) DPM_XC(2) DPM_XC(3) DPM_XC(4) DPM_XC(5) DPM_XC(6)
#undef DPM_XC
          }
        }
      }
#undef DPM_XARGS
      // column maxima: fold the row groups of a packed warp, group 0 writes
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1)
        if (o >= lpr) cmaxv = fmaxf(cmaxv, __shfl_xor_sync(0xffffffffu, cmaxv, o));
      if (xsub == 0) atomicMax(&sh.cmk[slot][xc], float_key(cmaxv));
    }
    if (warp == 0 && have_next) finish_job(p + 1);
    __syncthreads();  // x(p) done: x words visible, band buffer free, tables of p+1 built
    if (have_next) issue_band(p + 1);
    const float* sm = S + pj.s_off;
    const int pitch = s_pitch(pj.Wp);
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
        place_unstaged(sm, pj, cy, cx, rx, ry, best, bdy, bdx);
        tot[k * THREADS] = __dadd_rn(tot[k * THREADS], best);
        const int o = (p * hr + iy) * wr + ix;
        if (posb) posb[o] = pack_pos(cy + bdy, cx + bdx);
        if (placedb) placedb[o] = best;
      }
      continue;
    }
    // the column maximum of this thread's roots (every root of a thread has
    // the column tid & (lpr - 1))
    float cmax = -INFINITY;
    if (ry > R1MAX) cmax = key_float(sh.cmk[slot][tid & (lpr - 1)]);
#define DPM_YARGS x32, sm, pitch, &pj, tb, xd, rx, ry, yb0, ty0, tx0, mask, root_of, aj, p, hr, wr, tot, posb, placedb, cmax
    if (ry > R1MAX) {
      y_pass<R1MAX, true>(DPM_YARGS);
    } else {
      switch (r1y) {
#define DPM_YC(R) case R: y_pass<R, false>(DPM_YARGS); break;
        DPM_YC(0) DPM_YC(1) DPM_YC(2) DPM_YC(3) DPM_YC(4) DPM_YC(5) DPM_YC(6)
#undef DPM_YC
      }
    }
#undef DPM_YARGS
  }

  // bias, totals, tau compaction (part positions read back from `pos`)
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    int iyr, ixr;
    const bool live = root_of(k, iyr, ixr);
    const int iy = ty0 + iyr, ix = tx0 + ixr;
    const double t = __dadd_rn(tot[k * THREADS], aj.bias);
    if (live && aj.total_off >= 0) total[aj.total_off + (int64_t)iy * wr + ix] = t;
    if (dets == nullptr) continue;
    const bool hit = live && t >= tau;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (bal == 0u) continue;
    const int leader = __ffs(bal) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(det_count, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!hit) continue;
    const int slot = base + __popc(bal & ((1u << lane) - 1u));
    if (slot >= max_dets) continue;
    dpm_detection d;
    d.image = aj.image;
    d.level = aj.level;
    d.component = aj.component;
    d.ry = aj.ry0 + iy;
    d.rx = aj.rx0 + ix;
    d.nparts = aj.nparts;
    d.score = t;
    for (int q = 0; q < DPM_MAX_PARTS; ++q)
      d.parts[q] = (q < aj.nparts && aj.pos_off >= 0)
                       ? pos[aj.pos_off + ((int64_t)q * hr + iy) * wr + ix]
                       : 0u;
    dets[slot] = d;
  }
}

// Specialised kernel for the bulk tiles (fast_tile): scale 2, both radii in
// (R1MAX, RCAP], full-width tiles (lane = root column, one band row per warp
// iteration).  Same algorithm, bounds and results as place2_kernel -- the
// generic kernel's instantiation <R1MAX, PACKED, OUTER, FULLW> of the x pass
// and <R1MAX, OUTER> of the y pass -- with the per-part geometry computed
// once per CTA by warp 0 (PartHdr) instead of by every warp, per-thread root
// offsets advanced by compile-time strides, and no radius / scale / lane
// packing dispatch, so the part loop carries far fewer live values.
struct PartHdr {
  const float* sm;    // S + s_off of the part's map
  int r_lo, r_hi;     // band rows inside the map: [r_lo, r_hi)
  int n_out;          // band rows outside the map
  int c0;             // shared column of lane 0's dx = 0
  int d0, ds;         // packed screen: first pair's dx, the single candidate's dx
  int reach;          // band columns the tile's windows reach
  int rx, ry;
  int pitch, Wp;
  int cyb, cxb;       // window centre of root (ty0, tx0) in map rows / columns
  int soff0;          // its S offset, cyb * pitch + cxb
  int xb0, yb0, nbox; // TMA band boxes: first column (16-byte aligned), row, count
  int map, map_z;     // TMA descriptor index, map index in its group
  int ok;             // both radii in (R1MAX, RCAP]: staged two-phase path
};

// A part of a fast tile whose r* falls outside (R1MAX, RCAP]: every root of
// the thread by direct global loads (exact, the reference's order).  Out of
// line so the hot loop's register allocation does not carry it.
__device__ __noinline__ void fast_unstaged(const dpm_place_job& pj, const PartHdr& h,
                                           double* tot, int warp, int lane, int h_tile, int o0,
                                           int wr, uint32_t* posb, double* placedb) {
  for (int k = 0; k < RPT; ++k) {
    const int iyr = warp + WARPS * k;
    if (iyr >= h_tile) continue;
    const int cy = h.cyb + 2 * iyr, cx = h.cxb + 2 * lane;
    double best;
    int bdy, bdx;
    place_unstaged(h.sm, pj, cy, cx, h.rx, h.ry, best, bdy, bdx);
    tot[k * THREADS] = __dadd_rn(tot[k * THREADS], best);
    const int o = o0 + WARPS * k * wr;
    if (posb) posb[o] = pack_pos(cy + bdy, cx + bdx);
    if (placedb) placedb[o] = best;
  }
}

// y-pass roots of a fast tile that need an exact scan (near tie, failed
// outer bound, or an x row resolved exactly), resolved after the hot loop and
// out of line, in the reference's order, exactly as the generic kernel's
// y_group phase 2 does (state and screening threshold of each root passed in).
static_assert(RPT == 4, "fast_rare_roots takes four roots");
__device__ __noinline__ void fast_rare_roots(uint32_t rare, int st0, int st1, int st2, int st3,
                                             float sv0, float sv1, float sv2, float sv3,
                                             const float* x32, const PartHdr& h,
                                             const PartTab& tb, double* tot, int warp, int lane,
                                             int o0, int wr, uint32_t* posb, double* placedb,
                                             uint32_t mask) {
  const int ry = h.ry, rx = h.rx, pitch = h.pitch;
  XDec xd;
  xd.d0 = h.d0;
  xd.ds = h.ds;
  xd.c2r1 = 2 * R1MAX;
  while (rare) {
    const int k = __ffs(rare) - 1;
    rare &= rare - 1;
    const int st = k == 0 ? st0 : k == 1 ? st1 : k == 2 ? st2 : st3;
    const float thr = k == 0 ? sv0 : k == 1 ? sv1 : k == 2 ? sv2 : sv3;
    int state = st & 7;
    int dy = ((st >> 3) & 127) - 64, dx = ((st >> 10) & 127) - 64;
    const int iyr = warp + WARPS * k;
    const int cy = h.cyb + 2 * iyr, cx = h.cxb + 2 * lane;
    const int so = cy * pitch + cx;
    if (state == 5) {
      dx = x_exact_global(h.sm + so + dy * pitch, cx, h.Wp, rx, tb.px);
    } else {
      const float* xcol = x32 + (2 * iyr + ry) * PT_W + lane;
      const int q = y_exact(xcol, h.sm, pitch, cy, cx, state == 2 ? -R1MAX : -ry,
                            state == 2 ? R1MAX : ry, h.Wp, &tb, xd, rx,
                            state == 2 ? thr : -INFINITY, mask, R1MAX,
                            state == 2 ? dy : 1000, state == 2 ? dx : 1000);
      if (q < 0) {
        state = 4;
      } else {
        dy = (q & 255) - 64;
        dx = (q >> 8) - 64;
      }
    }
    double best = -INFINITY;
    if (state == 4) {
      dy = -ry;
      dx = -rx;
    } else {
      const float s = __ldg(h.sm + so + dy * pitch + dx);
      best = __dadd_rn(__dadd_rn((double)s, -tb.px[dx + 16]), -tb.py[dy + 16]);
    }
    tot[k * THREADS] = __dadd_rn(tot[k * THREADS], best);
    const int o = o0 + WARPS * k * wr;
    if (posb) posb[o] = pack_pos(cy + dy, cx + dx);
    if (placedb) placedb[o] = best;
  }
}

struct __align__(128) SmemF {
  float s[BAND2 * COLS_PITCH];
  float x32[XBUF][BAND2 * PT_W];
  double tot[RPT][THREADS];
  uint32_t cmk[3][PT_W];           // column maxima (float_key), part q at q % 3
  uint32_t rmask[WARPS][RMASK];
  PartTab tab[3];
  PartHdr hdr[3];
  alignas(16) JobRange jr[3];
  alignas(16) dpm_place_job pj[3];
  dpm_asm_job aj;
  alignas(8) uint64_t band_bar;
  int tile;  // (tile row << 16) | tile column
};

__device__ __forceinline__ void fast_tile_run(
    const float* __restrict__ S, const unsigned char* __restrict__ smaps,
    const dpm_place_job* __restrict__ pjobs, const dpm_asm_job* __restrict__ ajobs, int najobs,
    const dpm_place_range* __restrict__ prep, double* __restrict__ total,
    uint32_t* __restrict__ pos, double* __restrict__ placed, double tau,
    dpm_detection* __restrict__ dets, int max_dets, int* __restrict__ det_count, int jid) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  SmemF& sh = *reinterpret_cast<SmemF*>(smem_raw);
  int tid_, lane_, warp_;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid_));
  asm volatile("and.b32 %0, %1, 31;" : "=r"(lane_) : "r"(tid_));
  asm volatile("shr.u32 %0, %1, 5;" : "=r"(warp_) : "r"(tid_));
  const int tid = tid_, lane = lane_, warp = __shfl_sync(0xffffffffu, warp_, 0);
  const uint32_t band_bar = pl_smem(&sh.band_bar);
  if (warp == 0) {  // this CTA's tile among the job's fast ones (block0 numbering)
    const dpm_asm_job& g = ajobs[jid];
    const int fc = k3_fast_cols_warp(g, pjobs, g.rx1 - g.rx0 + 1, lane);
    const int t = (int)blockIdx.x - g.block0;
    if (lane == 0) sh.tile = ((t / fc) << 16) | (t % fc);
  }
  if (tid == 0) {
    sh.aj = ajobs[jid];
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(band_bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 3 * PT_W) (&sh.cmk[0][0])[tid] = 0u;
  __syncthreads();
  const dpm_asm_job& aj = sh.aj;
  const int hr = aj.ry1 - aj.ry0 + 1, wr = aj.rx1 - aj.rx0 + 1;
  const int ty0 = (sh.tile >> 16) * TH, tx0 = (sh.tile & 0xffff) * PT_W;
  const int wt = min(PT_W, wr - tx0), h_tile = min(TH, hr - ty0);
  const int ry_lo = aj.ry0 + ty0, ry_hi = ry_lo + h_tile - 1, rx_lo = aj.rx0 + tx0;
  const bool lane_live = lane < wt;
  const uint32_t mask = ~15u | ((uint32_t)najobs >> 31);  // see place2_kernel

  // root k of this thread: row warp + WARPS k, column lane
  double* const tot = &sh.tot[0][tid];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int iyr = warp + WARPS * k;
    double t = 0.0;
    if (aj.root_off >= 0 && lane_live && iyr < h_tile)
      t = (double)__ldg(S + aj.root_off + (int64_t)(ry_lo + iyr) * aj.root_pitch + rx_lo + lane);
    tot[k * THREADS] = t;
  }

  auto fetch_job = [&](int q) {  // warp 0
    const int slot = q % 3;
    if (lane < (int)(sizeof(dpm_place_job) / 8)) {
      const uint32_t sa = pl_smem(reinterpret_cast<unsigned char*>(&sh.pj[slot]) + 8 * lane);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa),
                   "l"(reinterpret_cast<const unsigned char*>(pjobs + aj.part_job0 + q) + 8 * lane));
    } else if (lane == 31) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(pl_smem(&sh.jr[slot])),
                   "l"(prep + aj.part_job0 + q));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  auto finish_job = [&](int q) {  // warp 0: tables and the part's geometry
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();
    const int slot = q % 3;
    const dpm_place_job& pj = sh.pj[slot];
    const JobRange& jr = sh.jr[slot];
    build_tab(sh.tab[slot], pj, jr, lane);
    if (lane == 0) {
      PartHdr& h = sh.hdr[slot];
      const int yb0 = 2 * ry_lo + pj.ay - jr.ry;
      const int nrows = 2 * (ry_hi - ry_lo) + 1 + 2 * jr.ry;
      const int xb0 = 2 * rx_lo + pj.ax - jr.rx;
      h.sm = S + pj.s_off;
      h.r_lo = min(max(0, -yb0), nrows);
      h.r_hi = max(min(nrows, pj.Hp - yb0), h.r_lo);
      h.n_out = h.r_lo + (nrows - h.r_hi);
      h.c0 = (xb0 & 3) + jr.rx;
      const int s = h.c0 & 1;  // packed pairs start on an even shared column
      h.d0 = -R1MAX + s;
      h.ds = s ? -R1MAX : R1MAX;
      h.reach = 2 * (wt - 1) + 1 + 2 * jr.rx;
      h.rx = jr.rx;
      h.ry = jr.ry;
      h.pitch = s_pitch(pj.Wp);
      h.Wp = pj.Wp;
      h.cyb = 2 * ry_lo + pj.ay;
      h.cxb = 2 * rx_lo + pj.ax;
      h.soff0 = h.cyb * h.pitch + h.cxb;
      h.xb0 = xb0 & ~3;
      h.yb0 = yb0;
      h.nbox = (nrows + TMA_BH - 1) / TMA_BH;
      h.map = pj.smap;
      h.map_z = pj.smap_z;
      h.ok = jr.rx > R1MAX && jr.rx <= RCAP && jr.ry > R1MAX && jr.ry <= RCAP;
    }
  };
  auto issue_band = [&](int q) {  // thread 0; the buffer's last readers passed a barrier
    const PartHdr& h = sh.hdr[q % 3];
    if (tid != 0 || !h.ok) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(band_bar),
                 "r"((uint32_t)h.nbox * TMA_BOX_BYTES)
                 : "memory");
    const void* map = smaps + (int64_t)h.map * DPM_SMAP_BYTES;
    const uint32_t dst = pl_smem(sh.s);
    for (int k = 0; k < h.nbox; ++k)
      tma_band_box(dst + (uint32_t)k * TMA_BOX_BYTES, map, h.xb0, h.yb0 + k * TMA_BH, h.map_z,
                   band_bar);
  };

  uint32_t bands = 0;
  if (warp == 0) {
    fetch_job(0);
    finish_job(0);
  }
  __syncthreads();
  issue_band(0);
  uint32_t* const posb = aj.pos_off >= 0 ? pos + aj.pos_off : nullptr;
  double* const placedb = aj.placed_off >= 0 ? placed + aj.placed_off : nullptr;
  const int obase = (ty0 + warp) * wr + tx0 + lane;  // output offset of root 0 in part 0
  const float sent = enc_code(OUT_SENTINEL, CODE_NONE);
  for (int p = 0; p < aj.nparts; ++p) {
    const int slot = p % 3, buf = XBUF == 2 ? p & 1 : 0;
    if (XBUF == 1 && p > 0) __syncthreads();  // y(p-1) done with the single x-word buffer
    if (warp == 0) sh.cmk[(p + 1) % 3][lane] = 0u;  // slot of part p+1 (see place2_kernel)
    const PartTab& tb = sh.tab[slot];
    const PartHdr& h = sh.hdr[slot];
    const bool have_next = p + 1 < aj.nparts;
    if (warp == 0 && have_next) fetch_job(p + 1);
    float* x32 = sh.x32[buf];
    const bool staged = h.ok;
    float cmaxv = -INFINITY;
    if (staged) pl_mbar_wait(band_bar, bands++ & 1);
    if (staged && h.n_out > 0) {  // rows outside the map: no candidate (reference: (-inf, -r))
      const int r_lo = h.r_lo, r_hi = h.r_hi, n_out = h.n_out;
      for (int i = tid; i < n_out * PT_W; i += THREADS) {
        const int k = i >> 5, l = i & 31;
        x32[(k < r_lo ? k : r_hi + (k - r_lo)) * PT_W + l] = sent;
      }
      cmaxv = sent;
    }
    // ---- x pass: band rows r_lo + warp, + WARPS, ...; lane = centre column
    if (staged) {
      const float E2 = tb.E2x, outx = tb.out_x, e2o = tb.E2o;
      unsigned long long pp[R1MAX];
      const float* tp = ((h.d0 + 16) & 1) ? tb.npx1 + h.d0 + 17 : tb.npx + h.d0 + 16;
#pragma unroll
      for (int k = 0; k < R1MAX; ++k) pp[k] = *reinterpret_cast<const unsigned long long*>(tp + 2 * k);
      const float pr0 = tb.npx[h.ds + 16];
      const int r_hi = h.r_hi, d0 = h.d0, ds = h.ds;
      const float* s0row = sh.s + h.c0 + 2 * lane;         // dx = 0 of lane's centre, row 0
      const float* mrow = sh.s + (h.c0 - h.rx) + lane;     // band column 0 + lane
      const bool b1 = lane + 32 < h.reach, b2 = lane + 64 < h.reach;
      uint32_t iters = 0;
      int it = 0;
      const int rb0 = h.r_lo + warp;
      for (int r = rb0; r < r_hi; r += WARPS, ++it) {
        const float* s0 = s0row + r * COLS_PITCH;
        float m1, m2;
        scr_packed<R1MAX>(s0 + d0, pp, s0[ds] + pr0, mask, m1, m2);
        const float* mr_ = mrow + r * COLS_PITCH;
        const float l = fmaxf(mr_[0], fmaxf(b1 ? mr_[32] : -INFINITY, b2 ? mr_[64] : -INFINITY));
        float mr;
        asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mr) : "f"(l));
        const bool rare =
            lane_live && (mr + outx + e2o >= m1 - E2 || m1 < NONE_BELOW || m2 >= m1 - E2);
        const uint32_t bal = __ballot_sync(0xffffffffu, rare);
        if (bal != 0u) {
          iters |= 1u << it;
          if (lane == 0) sh.rmask[warp][it] = bal;  // it < RMASK
        }
        if (lane_live) {
          x32[r * PT_W + lane] = m1;
          cmaxv = fmaxf(cmaxv, m1);
        }
      }
      if (iters != 0u) {
        __syncwarp();
        while (iters != 0u) {
          const int i = __ffs(iters) - 1;
          iters &= iters - 1;
          if (!((sh.rmask[warp][i] >> lane) & 1u)) continue;
          const int r = rb0 + i * WARPS;
          const float* s0 = s0row + r * COLS_PITCH;
          const int xi = x_exact_band(s0, -h.rx, h.rx, tb.px);
          const float v = s0[xi];
          const float word = v == v ? enc_code(v + tb.npx[xi + 16], CODE_RARE)
                                    : enc_code(OUT_SENTINEL, CODE_NONE);
          x32[r * PT_W + lane] = word;
          cmaxv = fmaxf(cmaxv, word);
        }
      }
    }
    if (staged) atomicMax(&sh.cmk[slot][lane], float_key(cmaxv));
    if (warp == 0 && have_next) finish_job(p + 1);
    __syncthreads();  // x(p) done: x words visible, band buffer free, part p+1 ready
    if (have_next) issue_band(p + 1);
    if (!staged) {  // r* outside (R1MAX, RCAP]: the exact per-root path (rare)
      if (lane_live)
        fast_unstaged(sh.pj[slot], h, tot, warp, lane, h_tile, p * hr * wr + obase, wr, posb,
                      placedb);
      continue;
    }
    // ---- y pass: roots (warp + WARPS k, lane)
    {
      const float cmax = key_float(sh.cmk[slot][lane]);
      const float E2 = tb.E2y, bound = cmax + tb.out_y + tb.E2o;
      float pr[2 * R1MAX + 1];
#pragma unroll
      for (int d = -R1MAX; d <= R1MAX; ++d) pr[d + R1MAX] = tb.npy[d + 16];
      const int ry = h.ry, rx = h.rx, pitch = h.pitch, d0 = h.d0, ds = h.ds;
      const float* smap = h.sm;
      const float* xcol0 = x32 + (2 * warp + ry) * PT_W + lane;
      const int soff0 = h.soff0 + 2 * warp * pitch + 2 * lane;
      int st[RPT];
      float sv[RPT];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        st[k] = 0;
        sv[k] = 0.f;
        if (!lane_live || warp + WARPS * k >= h_tile) continue;
        const float* xcol = xcol0 + 2 * WARPS * k * PT_W;
        float m1, m2;
        scr_strided<R1MAX, PT_W>(xcol, pr, mask, m1, m2);
        const float lo = m1 - E2;
        if (bound >= lo) {
          st[k] = 3;
        } else if (m1 < NONE_BELOW) {
          st[k] = 4;
        } else if (m2 >= lo) {
          st[k] = 2 | ((code_of(m1) - R1MAX + 64) << 3) | ((code_of(m2) - R1MAX + 64) << 10);
          sv[k] = lo;
        } else {
          const int dy = code_of(m1) - R1MAX;
          const int c = code_of(xcol[dy * PT_W]);
          if (c == CODE_RARE) {
            st[k] = 5 | ((dy + 64) << 3);
          } else {
            const int dx = c == 2 * R1MAX ? ds : d0 + c;
            st[k] = 1 | ((dy + 64) << 3) | ((dx + 64) << 10);
            sv[k] = __ldg(smap + soff0 + 2 * WARPS * k * pitch + dy * pitch + dx);
          }
        }
      }
      const int o0 = p * hr * wr + obase;
      uint32_t rare = 0;  // roots whose winner needs an exact scan (~1%), after the loop
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int state = st[k] & 7;
        if (state == 0) continue;
        if (state != 1 && state != 4) {
          rare |= 1u << k;
          continue;
        }
        int dy = ((st[k] >> 3) & 127) - 64, dx = ((st[k] >> 10) & 127) - 64;
        double best = -INFINITY;
        if (state == 4) {  // no candidate: the reference's (-inf, first dy, first row's dx)
          dy = -ry;
          dx = -rx;
        } else {
          best = __dadd_rn(__dadd_rn((double)sv[k], -tb.px[dx + 16]), -tb.py[dy + 16]);
        }
        tot[k * THREADS] = __dadd_rn(tot[k * THREADS], best);
        const int o = o0 + WARPS * k * wr;
        if (posb) posb[o] = pack_pos(h.cyb + 2 * (warp + WARPS * k) + dy, h.cxb + 2 * lane + dx);
        if (placedb) placedb[o] = best;
      }
      if (rare)
        fast_rare_roots(rare, st[0], st[1], st[2], st[3], sv[0], sv[1], sv[2], sv[3], x32, h, tb,
                        tot, warp, lane, o0, wr, posb, placedb, mask);
    }
  }

#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int iyr = warp + WARPS * k;
    emit_root(aj, lane_live && iyr < h_tile, ty0 + iyr, tx0 + lane, wr, tot[k * THREADS], total,
              pos, tau, dets, max_dets, det_count, lane, hr);
  }
}


// The specialised path and the generic one as two kernels over disjoint tile
// lists (block0 / block1 numbering of dpm_assemble_prepare); one kernel
// calling both paths allocates registers for their union and spills ~2 KB.
__global__ void __launch_bounds__(THREADS, DPM_K3_MINB)
place2f_kernel(const float* __restrict__ S, const unsigned char* __restrict__ smaps,
               const dpm_place_job* __restrict__ pjobs, const dpm_asm_job* __restrict__ ajobs,
               int najobs, const dpm_place_range* __restrict__ prep, double* __restrict__ total,
               uint32_t* __restrict__ pos, double* __restrict__ placed, double tau,
               dpm_detection* __restrict__ dets, int max_dets, int* __restrict__ det_count) {
  const int jid = find_job_warp(ajobs, najobs, blockIdx.x);
  fast_tile_run(S, smaps, pjobs, ajobs, najobs, prep, total, pos, placed, tau, dets, max_dets,
                det_count, jid);
}

}  // namespace k3v2

int k3v2_tile_rows() { return k3v2::TH; }

// launched by dpm_assemble (placement.cu)
// DPM_K3F=0 keeps every tile on the generic kernel (A/B of the specialised
// one); read by dpm_assemble_prepare's tile numbering and by the launch
bool k3_fast_enabled() {
  static const bool on = [] {
    const char* e = getenv("DPM_K3F");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// launched by dpm_assemble (placement.cu): the specialised kernel over its
// nfast tiles, the generic kernel over the other ngeneric
int launch_place2(const float* S, const void* smaps, const dpm_place_job* pjobs,
                  const dpm_asm_job* ajobs, int najobs, int64_t nfast, int64_t ngeneric,
                  const dpm_place_range* prep, double* total, uint32_t* pos, double* placed,
                  double tau, dpm_detection* dets, int max_dets, int* det_count, cudaStream_t st) {
  const unsigned char* sm = static_cast<const unsigned char*>(smaps);
  if (nfast > 0) {
    const size_t smf = sizeof(k3v2::SmemF);
    DPM_CUDA(cudaFuncSetAttribute(k3v2::place2f_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf));
    k3v2::place2f_kernel<<<(unsigned)nfast, k3v2::THREADS, smf, st>>>(
        S, sm, pjobs, ajobs, najobs, prep, total, pos, placed, tau, dets, max_dets, det_count);
    DPM_LAUNCHED("place2f_kernel");
  }
  if (ngeneric > 0) {
    const size_t smem = sizeof(k3v2::Smem);
    DPM_CUDA(cudaFuncSetAttribute(k3v2::place2_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k3v2::place2_kernel<<<(unsigned)ngeneric, k3v2::THREADS, smem, st>>>(
        S, sm, pjobs, ajobs, najobs, prep, total, pos, placed, tau, dets, max_dets, det_count,
        k3_fast_enabled() ? 1 : 0);
    DPM_LAUNCHED("place2_kernel");
  }
  return DPM_OK;
}

}  // namespace dpm
