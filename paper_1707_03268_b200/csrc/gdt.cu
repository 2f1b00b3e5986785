// K3 as a Felzenszwalb generalised distance transform (lower envelope per
// row, then per column) fused with K4 (root + parts + bias, tau compaction),
// for the unbounded placement mode (radius < 0) on the GDT root domain.
//
// Reference semantics: _placement_grid (detection.py:320-373) with a window
// large enough to be unbounded.  The value of the chosen
// displacement is recomputed with the reference's expression and order
// ((S - (c_dx*dx + (c_dxx*dx)*dx)) - (c_dy*dy + (c_dyy*dy)*dy), unfused FP64,
// detection.py:346-347,361), so values are bit-identical to the windowed
// reference whenever the argmax is; argmaxes are bit-identical except at exact
// ties (displacements whose penalised values agree to a few ulps), where the
// envelope's tie-break may differ.
//
// 1-D max-plus transform, source q, query p, pen(d) = b*d + a*d*d, d = q - p:
//   V(q, p) = h(q) + 2a*q*p + (b*p - a*p*p),   h(q) = f(q) - (b*q + a*q*q),
// so the maximiser at p is the upper envelope of the lines h(q) + 2a*q*p.
// The envelope lives in a per-lane deque in shared memory (slots x 32 lanes,
// conflict free); intersection tests are cross-multiplied in FP64.  Sources
// stream in ascending order and query p is answered once every q <= p + r*
// has been pushed: by the App. A.2 lemma (centres inside the map) no
// maximiser lies farther than r*, so the deque never holds more than
// 2 r* + 2 lines (capacity GD_CAP; larger r* takes a plain full-row scan).
//
//   gdt_x_kernel : warp = 32 map rows (lane = row), S streamed through shared
//                  memory in 32 x 32 blocks (coalesced loads, transposed
//                  reads, next block prefetched in registers).  Queries are
//                  the centre columns s*rx + ax of the assembly's roots.
//                  Writes, row-major [Hp][wr], the S value and dx of every
//                  (row, centre) winner (again through a 32 x 32 transpose).
//   gdt_y_kernel : warp = 32 root columns of one assembly (lane = column).
//                  Per part, rows stream in; the source value of row y is the
//                  exact x-pass value sv - pen_x(dx); queries are the centre
//                  rows s*ry + ay.  Part values are summed into the totals in
//                  part order (root first); then bias, tau compaction.
#include <math.h>

#include "common.cuh"

namespace dpm {

constexpr int GD_CAP = 32;  // deque capacity per lane (power of two)
constexpr int GD_MASK = GD_CAP - 1;
constexpr int GX_WARPS = 4;
constexpr int GY_WARPS = 4;

// c1*d + (c2*d)*d, round-to-nearest, no contraction (reference penalty order)
__device__ __forceinline__ double gpen(double c1, double c2, int d) {
  const double dd = (double)d;
  return __dadd_rn(__dmul_rn(c1, dd), __dmul_rn(__dmul_rn(c2, dd), dd));
}

// r* of App. A.2 for one axis (+1 guards the floor)
__device__ __forceinline__ int gdt_rstar(double a, double b, double ao, double bo, float vmax,
                                         float vmin) {
  const double dprime = ((double)vmax - (double)vmin) + bo * bo / (4.0 * ao);
  return (int)floor((fabs(b) + sqrt(b * b + 4.0 * a * dprime)) / (2.0 * a)) + 1;
}

__device__ __forceinline__ uint32_t gpack(int y, int x) {
  return ((uint32_t)(uint16_t)(int16_t)y << 16) | (uint32_t)(uint16_t)(int16_t)x;
}

// back line B (after A) is useless once the new line N overtakes A no later
// than B does: x(A,N) <= x(A,B), qA < qB < qN.
__device__ __forceinline__ bool back_useless(int qa, double ha, int qb, double hb, int qn,
                                             double hn) {
  return __dmul_rn(ha - hn, (double)(qb - qa)) <= __dmul_rn(ha - hb, (double)(qn - qa));
}

// the second line is strictly better than the front at p: x(0,1) < p
__device__ __forceinline__ bool front_beaten(int q0, double h0, int q1, double h1, double twoa,
                                             int p) {
  return (h0 - h1) < __dmul_rn(twoa * (double)(q1 - q0), (double)p);
}

// ------------------------------------------------------------------ deque
// Per-lane envelope deque: line i has source index q_i and intercept h_i;
// slots [GD_CAP][32] in shared memory (lane fastest: conflict free for any
// per-lane slot).  The two front lines (positions 0, 1) and the two back
// lines (positions size-2, size-1) are cached in registers, so shared memory
// is read only when a pop exposes a new line.  `pay` is a per-line 32-bit
// payload (the x pass stores q, the y pass (y << 16) | dx) and `val` the
// line's float source value.
struct Env {
  int front, size;
  int qa, qb, q0, q1;
  double ha, hb, h0, h1;
};

__device__ __forceinline__ void env_init(Env& e) {
  e.front = e.size = 0;
  e.qa = e.qb = e.q0 = e.q1 = 0;
  e.ha = e.hb = e.h0 = e.h1 = 0.0;
}

__device__ __forceinline__ void env_push(Env& e, int q, double h, int pay, float val,
                                         int (*dq_pay)[32], double (*dq_h)[32],
                                         float (*dq_val)[32], int lane, int shift) {
  while (e.size >= 2 && back_useless(e.qa, e.ha, e.qb, e.hb, q, h)) {
    --e.size;
    e.qb = e.qa;
    e.hb = e.ha;
    if (e.size >= 2) {
      const int s2 = (e.front + e.size - 2) & GD_MASK;
      e.qa = dq_pay[s2][lane] >> shift;
      e.ha = dq_h[s2][lane];
    }
  }
  if (e.size == GD_CAP) {  // only reachable through rounding: drop the stale front
    e.front = (e.front + 1) & GD_MASK;
    --e.size;
    e.q0 = e.q1;
    e.h0 = e.h1;
    const int s1 = (e.front + 1) & GD_MASK;
    e.q1 = dq_pay[s1][lane] >> shift;
    e.h1 = dq_h[s1][lane];
  }
  const int sn = (e.front + e.size) & GD_MASK;
  dq_pay[sn][lane] = pay;
  dq_h[sn][lane] = h;
  dq_val[sn][lane] = val;
  ++e.size;
  e.qa = e.qb;
  e.ha = e.hb;
  e.qb = q;
  e.hb = h;
  if (e.size == 1) {
    e.q0 = q;
    e.h0 = h;
  } else if (e.size == 2) {
    e.q1 = q;
    e.h1 = h;
  }
}

// pops the front while the next line is strictly better at p; returns the
// front slot (the maximiser at p)
__device__ __forceinline__ int env_query(Env& e, double twoa, int p, int (*dq_pay)[32],
                                         double (*dq_h)[32], int lane, int shift) {
  while (e.size >= 2 && front_beaten(e.q0, e.h0, e.q1, e.h1, twoa, p)) {
    e.front = (e.front + 1) & GD_MASK;
    --e.size;
    e.q0 = e.q1;
    e.h0 = e.h1;
    if (e.size >= 2) {
      const int s1 = (e.front + 1) & GD_MASK;
      e.q1 = dq_pay[s1][lane] >> shift;
      e.h1 = dq_h[s1][lane];
    }
  }
  return e.front;
}

// ------------------------------------------------------------------ x pass

struct GxWarp {
  float blk[32][33];      // S block [col][row]
  float osv[32][33];      // winners' S value [query][row]
  int16_t odx[32][34];    // winners' dx      [query][row]
  int dq_pay[GD_CAP][32];
  double dq_h[GD_CAP][32];
  float dq_val[GD_CAP][32];
};

__global__ void __launch_bounds__(GX_WARPS * 32)
gdt_x_kernel(const float* __restrict__ S, float* __restrict__ SV, int16_t* __restrict__ DX,
             const dpm_place_job* __restrict__ jobs, int njobs, const uint32_t* __restrict__ ranges) {
  extern __shared__ __align__(16) unsigned char gx_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  GxWarp& sh = reinterpret_cast<GxWarp*>(gx_raw)[warp];
  const int64_t wb = (int64_t)blockIdx.x * GX_WARPS + warp;
  const int jid = find_job(jobs, njobs, wb);
  const dpm_place_job pj = jobs[jid];
  const int y0 = (int)(wb - pj.block0) * 32;
  if (y0 >= pj.Hp) return;
  const int Hp = pj.Hp, Wp = pj.Wp, wr = pj.wr, sc = pj.scale, sp = s_pitch(pj.Wp);
  const float vmax = key_float(ranges[2 * pj.range_idx]);
  const float vmin = key_float(ranges[2 * pj.range_idx + 1]);
  const int rs = gdt_rstar(pj.cdxx, pj.cdx, pj.cdyy, pj.cdy, vmax, vmin);
  const double a = pj.cdxx, b = pj.cdx, twoa = 2.0 * a;
  const float* sm = S + pj.s_off;
  float* svo = SV + pj.x_off;
  int16_t* dxo = DX + pj.x_off;
  const int cx0 = sc * pj.rx0 + pj.ax;

  auto flush = [&](int cq) {  // write queries (cq & ~31) .. cq of the 32 rows
    __syncwarp();
    const int base = cq & ~31, n = cq - base + 1;
    if (lane < n) {
      for (int r = 0; r < 32 && y0 + r < Hp; ++r) {
        const int64_t o = (int64_t)(y0 + r) * wr + base + lane;
        svo[o] = sh.osv[lane][r];
        dxo[o] = sh.odx[lane][r];
      }
    }
    __syncwarp();
  };

  if (2 * rs + 2 > GD_CAP) {  // r* beyond the deque: full-row scan (same winner rule)
    const int y = min(y0 + lane, Hp - 1);
    for (int cq = 0; cq < wr; ++cq) {
      const int p = cx0 + sc * cq;
      double best = -INFINITY;
      int bq = 0;
      for (int q = 0; q < Wp; ++q) {
        const double v = __dadd_rn((double)__ldg(sm + (int64_t)y * sp + q), -gpen(b, a, q - p));
        if (v > best) { best = v; bq = q; }
      }
      sh.osv[cq & 31][lane] = __ldg(sm + (int64_t)y * sp + bq);
      sh.odx[cq & 31][lane] = (int16_t)(bq - p);
      if ((cq & 31) == 31 || cq == wr - 1) flush(cq);
    }
    return;
  }

  Env e;
  env_init(e);
  int c = 0;  // next query
  auto answer = [&](int cq) {
    const int p = cx0 + sc * cq;
    const int s0 = env_query(e, twoa, p, sh.dq_pay, sh.dq_h, lane, 0);
    sh.osv[cq & 31][lane] = sh.dq_val[s0][lane];
    sh.odx[cq & 31][lane] = (int16_t)(e.q0 - p);
    if ((cq & 31) == 31 || cq == wr - 1) flush(cq);
  };

  const int nblk = (Wp + 31) / 32;
  float nxt[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const int yy = y0 + r, xx = lane;
    nxt[r] = (yy < Hp && xx < Wp) ? __ldg(sm + (int64_t)yy * sp + xx) : 0.f;
  }
  for (int kb = 0; kb < nblk; ++kb) {
    const int xb = kb * 32;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) sh.blk[lane][r] = nxt[r];
    __syncwarp();
    if (kb + 1 < nblk) {  // prefetch the next block while this one is consumed
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int yy = y0 + r, xx = xb + 32 + lane;
        nxt[r] = (yy < Hp && xx < Wp) ? __ldg(sm + (int64_t)yy * sp + xx) : 0.f;
      }
    }
    const int ncol = min(32, Wp - xb);
    double qd = (double)xb;
    for (int k = 0; k < ncol; ++k, qd += 1.0) {
      const int q = xb + k;
      const float f = sh.blk[k][lane];
      // h only feeds envelope decisions (stored, so every test sees one value)
      const double h = (double)f - __fma_rn(a, qd, b) * qd;
      env_push(e, q, h, q, f, sh.dq_pay, sh.dq_h, sh.dq_val, lane, 0);
      // answer every query whose window end p + r* has been reached
      while (c < wr && cx0 + sc * c + rs <= q) answer(c++);
    }
  }
  while (c < wr) answer(c++);  // centres within r* of the right edge
}

// ------------------------------------------------------- y pass + assembly

struct GyWarp {
  int dq_pay[GD_CAP][32];  // (y << 16) | (uint16)dx
  double dq_h[GD_CAP][32];
  float dq_val[GD_CAP][32];  // sv
};

__global__ void __launch_bounds__(GY_WARPS * 32)
gdt_y_kernel(const float* __restrict__ S, const float* __restrict__ SV,
             const int16_t* __restrict__ DX, const dpm_place_job* __restrict__ pjobs,
             const dpm_asm_job* __restrict__ ajobs, int najobs, const uint32_t* __restrict__ ranges,
             double* __restrict__ total, uint32_t* __restrict__ pos, double* __restrict__ placed,
             double tau, dpm_detection* __restrict__ dets, int max_dets, int* __restrict__ det_count) {
  extern __shared__ __align__(16) unsigned char gy_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  GyWarp& sh = reinterpret_cast<GyWarp*>(gy_raw)[warp];
  const int64_t wb = (int64_t)blockIdx.x * GY_WARPS + warp;
  const int jid = find_job(ajobs, najobs, wb);
  const dpm_asm_job aj = ajobs[jid];
  const int hr = aj.ry1 - aj.ry0 + 1, wr = aj.rx1 - aj.rx0 + 1;
  const int cb = (int)(wb - aj.block0);
  if (cb * 32 >= wr) return;
  const int c = cb * 32 + lane;
  const bool col_ok = c < wr;
  const int cc = col_ok ? c : wr - 1;  // idle lanes shadow a valid column
  double* tot = total + aj.total_off;

  for (int p = 0; p < aj.nparts; ++p) {
    const dpm_place_job pj = pjobs[aj.part_job0 + p];
    const int Hp = pj.Hp, sc = pj.scale;
    const float vmax = key_float(ranges[2 * pj.range_idx]);
    const float vmin = key_float(ranges[2 * pj.range_idx + 1]);
    const int rs = gdt_rstar(pj.cdyy, pj.cdy, pj.cdxx, pj.cdx, vmax, vmin);
    const double a = pj.cdyy, b = pj.cdy, twoa = 2.0 * a;
    const double cdx = pj.cdx, cdxx = pj.cdxx;
    const float* svc = SV + pj.x_off + cc;
    const int16_t* dxc = DX + pj.x_off + cc;
    const int cx = sc * (pj.rx0 + cc) + pj.ax;
    const int cy0 = sc * aj.ry0 + pj.ay;

    // exact reference value of the winner (ys, dxs) for root row iy
    auto emit = [&](int iy, int ys, int dxs, float svs) {
      const double v = __dadd_rn(__dadd_rn((double)svs, -gpen(cdx, cdxx, dxs)),
                                 -gpen(b, a, ys - (cy0 + sc * iy)));
      if (!col_ok) return;
      const int64_t o = (int64_t)iy * wr + c;
      double t;
      if (p == 0)
        t = aj.root_off >= 0
                ? (double)__ldg(S + aj.root_off + (int64_t)(aj.ry0 + iy) * aj.root_pitch + aj.rx0 + c)
                : 0.0;
      else
        t = tot[o];
      tot[o] = __dadd_rn(t, v);
      const int64_t po = ((int64_t)p * hr + iy) * wr + c;
      if (aj.pos_off >= 0) pos[aj.pos_off + po] = gpack(ys, cx + dxs);
      if (aj.placed_off >= 0) placed[aj.placed_off + po] = v;
    };

    if (2 * rs + 2 > GD_CAP) {  // plain scan over every map row
      for (int iy = 0; iy < hr; ++iy) {
        const int cy = cy0 + sc * iy;
        double best = -INFINITY;
        int by = 0;
        for (int yy = 0; yy < Hp; ++yy) {
          const int d = dxc[(int64_t)yy * wr];
          const double v = __dadd_rn(__dadd_rn((double)svc[(int64_t)yy * wr], -gpen(cdx, cdxx, d)),
                                     -gpen(b, a, yy - cy));
          if (v > best) { best = v; by = yy; }
        }
        emit(iy, by, dxc[(int64_t)by * wr], svc[(int64_t)by * wr]);
      }
      continue;
    }

    Env e;
    env_init(e);
    int iy = 0;
    auto answer = [&](int ry) {
      const int s0 = env_query(e, twoa, cy0 + sc * ry, sh.dq_pay, sh.dq_h, lane, 16);
      const int pay = sh.dq_pay[s0][lane];
      emit(ry, pay >> 16, (int16_t)pay, sh.dq_val[s0][lane]);
    };
    constexpr int U = 4;
    float nsv[U];
    int16_t ndx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      nsv[u] = u < Hp ? svc[(int64_t)u * wr] : 0.f;
      ndx[u] = u < Hp ? dxc[(int64_t)u * wr] : (int16_t)0;
    }
    for (int g = 0; g < Hp; g += U) {
      float csv[U];
      int16_t cdv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        csv[u] = nsv[u];
        cdv[u] = ndx[u];
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {  // prefetch the next group of rows
        const int yy = g + U + u;
        nsv[u] = yy < Hp ? svc[(int64_t)yy * wr] : 0.f;
        ndx[u] = yy < Hp ? dxc[(int64_t)yy * wr] : (int16_t)0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int yy = g + u;
        if (yy >= Hp) break;
        const double dd = (double)cdv[u], yd = (double)yy;
        // decision value only: x-pass value minus the y polynomial
        const double h = ((double)csv[u] - __fma_rn(cdxx, dd, cdx) * dd) - __fma_rn(a, yd, b) * yd;
        env_push(e, yy, h, (yy << 16) | (uint16_t)cdv[u], csv[u], sh.dq_pay, sh.dq_h, sh.dq_val,
                 lane, 16);
        while (iy < hr && cy0 + sc * iy + rs <= yy) answer(iy++);
      }
    }
    while (iy < hr) answer(iy++);
  }

  // bias, totals, tau compaction (one ballot per root row)
  for (int iy = 0; iy < hr; ++iy) {
    const int64_t o = (int64_t)iy * wr + c;
    double t = 0.0;
    if (col_ok) {
      if (aj.nparts == 0)
        t = aj.root_off >= 0
                ? (double)__ldg(S + aj.root_off + (int64_t)(aj.ry0 + iy) * aj.root_pitch + aj.rx0 + c)
                : 0.0;
      else
        t = tot[o];
      t = __dadd_rn(t, aj.bias);
      tot[o] = t;
    }
    if (dets == nullptr) continue;
    const bool hit = col_ok && t >= tau;
    const unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (mask == 0u) continue;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(det_count, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!hit) continue;
    const int slot = base + __popc(mask & ((1u << lane) - 1u));
    if (slot >= max_dets) continue;
    dpm_detection d;
    d.image = aj.image;
    d.level = aj.level;
    d.component = aj.component;
    d.ry = aj.ry0 + iy;
    d.rx = aj.rx0 + c;
    d.nparts = aj.nparts;
    d.score = t;
    for (int q = 0; q < DPM_MAX_PARTS; ++q)
      d.parts[q] = (q < aj.nparts && aj.pos_off >= 0) ? pos[aj.pos_off + ((int64_t)q * hr + iy) * wr + c] : 0u;
    dets[slot] = d;
  }
}

}  // namespace dpm

using namespace dpm;

static bool centres_inside(const dpm_place_job& j, int ry0, int ry1) {
  const int64_t x0 = (int64_t)j.scale * j.rx0 + j.ax, x1 = (int64_t)j.scale * (j.rx0 + j.wr - 1) + j.ax;
  const int64_t y0 = (int64_t)j.scale * ry0 + j.ay, y1 = (int64_t)j.scale * ry1 + j.ay;
  return x0 >= 0 && x1 < j.Wp && y0 >= 0 && y1 < j.Hp;
}

extern "C" int64_t dpm_gdt_x_prepare(dpm_place_job* jobs, int njobs) {
  DPM_REQUIRE(njobs >= 0 && (njobs == 0 || jobs), "dpm_gdt_x_prepare: bad table");
  int64_t warps = 0;
  for (int i = 0; i < njobs; ++i) {
    dpm_place_job& j = jobs[i];
    DPM_REQUIRE(j.radius < 0 && j.cdxx > 0.0 && j.cdyy > 0.0,
                "dpm_gdt_x_prepare: job %d is not an unbounded transform with c_dxx, c_dyy > 0", i);
    DPM_REQUIRE(j.Hp >= 1 && j.Wp >= 1 && j.Hp <= 32767 && j.Wp <= 32767 && j.wr >= 1 &&
                    j.x_off >= 0 && j.range_idx >= 0 && j.scale >= 1,
                "dpm_gdt_x_prepare: job %d has a bad shape/offset", i);
    const int64_t x0 = (int64_t)j.scale * j.rx0 + j.ax, x1 = (int64_t)j.scale * (j.rx0 + j.wr - 1) + j.ax;
    DPM_REQUIRE(x0 >= 0 && x1 < j.Wp, "dpm_gdt_x_prepare: job %d has centre columns outside the map", i);
    j.block0 = (int32_t)warps;
    warps += (j.Hp + 31) / 32;
  }
  return (warps + GX_WARPS - 1) / GX_WARPS;
}

extern "C" int64_t dpm_gdt_y_prepare(dpm_asm_job* ajobs, int najobs, const dpm_place_job* pjobs,
                                     int npjobs) {
  DPM_REQUIRE(najobs >= 0 && (najobs == 0 || (ajobs && pjobs)), "dpm_gdt_y_prepare: bad table");
  int64_t warps = 0;
  for (int i = 0; i < najobs; ++i) {
    dpm_asm_job& a = ajobs[i];
    DPM_REQUIRE(a.ry1 >= a.ry0 && a.rx1 >= a.rx0 && a.total_off >= 0,
                "dpm_gdt_y_prepare: assembly %d needs a non-empty rect and totals", i);
    DPM_REQUIRE(a.nparts >= 0 && a.nparts <= DPM_MAX_PARTS && a.part_job0 >= 0 &&
                    a.part_job0 + a.nparts <= npjobs,
                "dpm_gdt_y_prepare: assembly %d has bad part jobs", i);
    for (int p = 0; p < a.nparts; ++p) {
      const dpm_place_job& j = pjobs[a.part_job0 + p];
      DPM_REQUIRE(j.radius < 0 && j.cdxx > 0.0 && j.cdyy > 0.0 && j.x_off >= 0,
                  "dpm_gdt_y_prepare: assembly %d part %d is not a GDT placement", i, p);
      DPM_REQUIRE(j.rx0 == a.rx0 && j.wr == a.rx1 - a.rx0 + 1,
                  "dpm_gdt_y_prepare: assembly %d part %d columns differ from the assembly", i, p);
      DPM_REQUIRE(centres_inside(j, a.ry0, a.ry1),
                  "dpm_gdt_y_prepare: assembly %d part %d has centres outside its map", i, p);
    }
    a.block0 = (int32_t)warps;
    warps += (a.rx1 - a.rx0 + 1 + 31) / 32;
  }
  return (warps + GY_WARPS - 1) / GY_WARPS;
}

extern "C" int dpm_gdt_x(const float* S, float* sv, int16_t* dx, const dpm_place_job* jobs,
                         int njobs, int64_t nblocks, const uint32_t* ranges, void* stream) {
  DPM_REQUIRE(S && sv && dx && jobs && ranges, "dpm_gdt_x: null pointer");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_gdt_x: nblocks");
  if (njobs == 0 || nblocks == 0) return DPM_OK;
  const size_t smem = sizeof(GxWarp) * GX_WARPS;
  DPM_CUDA(cudaFuncSetAttribute(gdt_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gdt_x_kernel<<<(unsigned)nblocks, GX_WARPS * 32, smem, as_stream(stream)>>>(S, sv, dx, jobs, njobs,
                                                                           ranges);
  DPM_LAUNCHED("gdt_x_kernel");
  return DPM_OK;
}

extern "C" int dpm_gdt_y(const float* S, const float* sv, const int16_t* dx,
                         const dpm_place_job* pjobs, const dpm_asm_job* ajobs, int najobs,
                         int64_t nblocks, const uint32_t* ranges, double* total, uint32_t* pos,
                         double* placed, double tau, dpm_detection* dets, int max_dets,
                         int* det_count, void* stream) {
  DPM_REQUIRE(S && sv && dx && pjobs && ajobs && ranges && total, "dpm_gdt_y: null pointer");
  DPM_REQUIRE(!dets || (det_count && pos), "dpm_gdt_y: detections need a counter and positions");
  DPM_REQUIRE(nblocks >= 0 && nblocks <= INT32_MAX, "dpm_gdt_y: nblocks");
  if (najobs == 0 || nblocks == 0) return DPM_OK;
  const size_t smem = sizeof(GyWarp) * GY_WARPS;
  DPM_CUDA(cudaFuncSetAttribute(gdt_y_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gdt_y_kernel<<<(unsigned)nblocks, GY_WARPS * 32, smem, as_stream(stream)>>>(
      S, sv, dx, pjobs, ajobs, najobs, ranges, total, pos, placed, tau, dets, max_dets, det_count);
  DPM_LAUNCHED("gdt_y_kernel");
  return DPM_OK;
}
