// K2 on the 5th-generation tensor cores: shortened correlation as an
// implicit GEMM on tcgen05 (kind::tf32, 3xTF32 split for FP32 accuracy).
//
//   S_f[y][x] = sum_{i<h, j<w, r<R} G[i][j][r][f] * P[r][y+i][x+j]
//
// GEMM shape per MMA: M = 128 consecutive output positions of one output
// row, N = filters, K = 8 ranks of one tap (i, j).  The A operand of tap
// (i, j) is a plain shifted window of the staged input row y+i: in the
// K-major no-swizzle canonical layout each position is one 16-byte row per
// 4-rank quad, so shifting by j positions is just +16*j bytes on the smem
// descriptor's start address -- no im2col copy.
//
// 3xTF32: A = A_hi + A_lo, B = B_hi + B_lo with hi = fp32 truncated to tf32
// (low 13 mantissa bits cleared) and lo = the exact remainder; per tap
//   MMA1: D[:, 0:2N] += A_hi x [B_hi | B_lo]      (N2 = 2N)
//   MMA2: D[:, 0:N]  += A_lo x  B_hi
// and the epilogue adds D[:, f] + D[:, N+f]; the dropped A_lo*B_lo term is
// ~2^-22 relative, far inside the 1e-5 parity bar.
// The compile-time DPM shapes (R == 8) run the correction MMA2 in bf16
// (kind::f16) over two taps at once: A_lo is staged as bf16, 16 bytes per
// position, so a K-major descriptor with LBO = 16 B reads position m + j for
// K = 0..7 and position m + j + 1 for K = 8..15, i.e. taps j and j + 1,
// against a host-built bf16 [B_hi(j); B_hi(j+1)] block.  That halves MMA2's
// instructions and its shared-memory operand bytes (the tensor pipe here is
// bound by operand bandwidth); the added error (bf16 rounding of the ~2^-11
// correction) is ~2^-19 relative per product.
//
// Warp roles (256 threads, one persistent CTA per SM):
//   warp 0      : TMEM allocation; one elected lane issues tcgen05.mma
//   warps 1..3  : producers -- stream input rows of P (planar fp32) into an
//                 smem ring as quad-interleaved hi/lo tf32 (mbarrier full/empty)
//   warps 4..7  : epilogue -- tcgen05.ld the accumulator of an output row,
//                 add the split halves, store S (coalesced per filter) and
//                 fold per-map extrema for the placement kernel
// Each CTA walks 128-wide column strips of levels top to bottom; every input
// row is staged once per strip.  The group's core B (hi | lo) stays resident
// in shared memory for the whole launch.
#include "tc_common.cuh"

namespace dpm {



#ifdef DPM_TC_PROBE
// MMA-warp wait cycles (debug builds only, tools/tc_probe.py): accumulator
// free, input rows staged, output rows, total loop cycles
__device__ unsigned long long dpm_tc_probe[4];
#endif

// NMAX: max filters held by the epilogue registers.  FH, FW > 0: filter
// extent fixed at compile time (R == 8), fully unrolled MMA issue.
// EPI: epilogue warps (4, or 8 = two per TMEM lane quarter, each draining
// alternate 16-filter column chunks).
// KS > 1 (R == 8, FH/FW fixed, at most 8 filters): output rows stacked KS at
// a time into one accumulator group [hi(y) lo(y) hi(y+1) lo(y+1) ...] (16
// columns per row); see tc_stack() for the core layout.
template <int NMAX, int FH, int FW, int EPI = 4, int KS = 1>
__global__ void __launch_bounds__(32 * (1 + TC_PRODUCERS + EPI), 1) corr_tc_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  // warp index broadcast from lane 0: provably warp-uniform, so the role
  // branches below do not make the MMA warp's bookkeeping divergent
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int nq = a.R >> 2;                       // rank quads
  const int taps = a.h * a.w;
  const int tcols = TC_M + a.w - 1;
  constexpr bool BF = FH > 0;  // bf16 correction MMA (compile-time shapes, R == 8)
  constexpr int NB = FH + 2 * (KS - 1);  // stacked core: tap-row blocks per tap column
  const uint32_t npairs = (uint32_t)(a.w + 1) / 2;
  const uint32_t b_bytes = KS > 1 ? (uint32_t)FW * NB * 512u : (uint32_t)taps * nq * (2 * a.N) * 16u;
  const uint32_t b2_bytes = KS > 1 ? npairs * NB * 512u
                          : BF     ? (uint32_t)a.h * npairs * 2u * a.N * 16u : 0u;
  const uint32_t hi_bytes = (uint32_t)nq * tcols * 16u;
  const uint32_t slot_bytes = BF ? ((hi_bytes + (tcols + 1u) * 16u + 127u) & ~127u)
                                 : 2u * hi_bytes;  // hi then lo
  unsigned char* sB = smem;
  unsigned char* sB2 = smem + ((b_bytes + 1023u) & ~1023u);
  unsigned char* sA = sB2 + ((b2_bytes + 1023u) & ~1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + ((a.ring * slot_bytes + 15u) & ~15u));
  uint64_t* full = bars;
  uint64_t* empty = bars + TC_MAX_RING;
  uint64_t* tfull = bars + 2 * TC_MAX_RING;
  uint64_t* tempty = tfull + TC_MAX_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + TC_MAX_ACC);
  uint64_t* bdone = tempty + TC_MAX_ACC + 1;  // multi-group: issued MMAs complete
  uint64_t* bload = bdone + 1;                // multi-group: core B landed

  // ---- setup: core B -> smem (all threads), barriers, TMEM
  if (a.tc_off == nullptr) {
    const float4* src = reinterpret_cast<const float4*>(a.Gtc);
    float4* dst = reinterpret_cast<float4*>(sB);
    for (uint32_t e = threadIdx.x; e < b_bytes / 16u; e += blockDim.x) dst[e] = __ldg(src + e);
    if constexpr (BF) {  // bf16 tap-pair block follows the tf32 block in Gtc
      const float4* src2 = src + b_bytes / 16u;
      float4* dst2 = reinterpret_cast<float4*>(sB2);
      for (uint32_t e = threadIdx.x; e < b2_bytes / 16u; e += blockDim.x) dst2[e] = __ldg(src2 + e);
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.ring; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < a.nacc; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, EPI);
    }
    mbar_init(bdone, 1);
    mbar_init(bload, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // =================== MMA issuer ===================
    // The whole warp walks the loop (warp-uniform descriptors live in uniform
    // registers); one elected lane issues.  A descriptor differs from the
    // base only in its 14-bit start-address field, so per tap it is the base
    // plus (byte offset >> 4).
    const uint32_t idesc1 = idesc_tf32(2 * a.N), idesc2 = idesc_tf32(a.N);
    const uint32_t lboA = (uint32_t)tcols * 16u, lboB = (uint32_t)(2 * a.N) * 16u;
    const uint64_t dA0 = umma_desc(smem_u32(sA), lboA, 128);
    const uint64_t dB0 = umma_desc(smem_u32(sB), lboB, 128);
    const uint32_t lo_step = (uint32_t)nq * lboA >> 4;   // hi -> lo plane block
    const uint32_t slot_step = slot_bytes >> 4;
    const uint32_t tap_step = (uint32_t)nq * lboB >> 4;
    const uint32_t kcA = 2u * lboA >> 4, kcB = 2u * lboB >> 4;
    // bf16 correction operands: A_lo [position][8 ranks] after the hi planes
    // (LBO 16 B: K-chunk 1 = next position), B2 [h][pair][2][N][8] (LBO = N*16 B)
    const uint64_t dAlo0 = umma_desc(smem_u32(sA) + hi_bytes, 16u, 128u);
    const uint64_t dB2 = umma_desc(smem_u32(sB2), (uint32_t)a.N * 16u, 128u);
    const uint32_t b2_pair = (2u * a.N * 16u) >> 4;
    const uint32_t idescbf = idesc_bf16(a.N);
    uint32_t q_glob = 0, row_glob = 0;
    if constexpr (KS > 1) {
      // Stacked rows: input row y+t meets output row y+k through tap row
      // i = t-k, so ONE MMA per (input row, tap column) updates all KS rows of
      // the group with the core window [B(t), B(t-1), ..., B(t-KS+1)] (zero
      // blocks outside 0..FH-1).  Each staged row is read (KS+FH-1)/KS times
      // per output row instead of FH times.  With few filters each MMA's cost
      // is dominated by reading its 128-row A operand from shared memory, so
      // fewer, wider MMAs (N = 16*KS) are the saving.
      constexpr int NP = (FW + 1) / 2;
      const uint32_t idesc_s = idesc_tf32(16 * KS), idesc_sb = idesc_bf16(16 * KS);
      const uint64_t dBs = umma_desc(smem_u32(sB), NB * 256u, 128u);
      const uint64_t dB2s = umma_desc(smem_u32(sB2), NB * 256u, 128u);
      // ring slot / phase of each group's first input row advance
      // incrementally (no division on the issue path; see the FH > 0 branch)
      const uint32_t ring = (uint32_t)a.ring;
      uint32_t gs = 0, gph = 0;
      for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
        const dpm_corr_job job = a.jobs[a.strips[st].job];
        const int ho = job.H - FH + 1;
        DPM_CHECK(a.strips[st].pad == 0, "stacked-row strips are never segmented");
        int qready = 0;  // rows of this strip known to be staged
        int y = 0;
        for (; y < ho; y += KS, ++row_glob) {
          const int b = row_glob & (TC_MAX_ACC - 1);
          mbar_wait(tempty + b, ((row_glob / TC_MAX_ACC) & 1) ^ 1);
          const uint32_t d = tmem_base + (uint32_t)(b * a.acc_cols);
          const int tmax = min(KS + FH - 1, job.H - y);
          for (int t = 0; t < tmax; ++t) {
            uint32_t sl = gs + (uint32_t)t, ph = gph;
            if (sl >= ring) { sl -= ring; ph ^= 1; }
            if (y + t >= qready) {
              mbar_wait(full + sl, ph);
              qready = y + t + 1;
            }
            tc_fence_after();
            const uint64_t da = dA0 + sl * slot_step;
            const uint64_t dal = dAlo0 + sl * slot_step;
            const uint32_t s0 = (uint32_t)(FH - 1 + KS - 1 - t) * 16u;  // window start (>> 4)
            if (elect_one()) {
#pragma unroll
              for (int j = 0; j < FW; ++j)
                mma_tf32(d, da + (uint32_t)j, dBs + (uint32_t)(j * NB * 32) + s0, idesc_s,
                         (t | j) != 0);
#pragma unroll
              for (int jp = 0; jp < NP; ++jp)
                mma_bf16(d, dal + (uint32_t)(2 * jp), dB2s + (uint32_t)(jp * NB * 32) + s0, idesc_sb);
            }
            __syncwarp();
          }
          // one commit per group (each commit costs the tensor pipe a bubble);
          // the epilogue frees the group's dead input rows once it sees tfull
          if (elect_one()) tc_commit(tfull + b);
          __syncwarp();
          gs += KS;  // next group's first row (KS < ring)
          if (gs >= ring) { gs -= ring; gph ^= 1; }
        }
        // rows y .. H-1 of the strip were never first rows of a group
        for (int rr = y; rr < job.H; ++rr)
          if (++gs == ring) { gs = 0; gph ^= 1; }
        if (y > job.H) {  // the last group stepped past the strip end
          for (int rr = job.H; rr < y; ++rr) {
            if (gs == 0) { gs = ring; gph ^= 1; }
            --gs;
          }
        }
        q_glob += job.H;
      }
    } else if constexpr (FH > 0) {
      // Compile-time taps.  All bookkeeping stays on the uniform datapath: ring
      // slots / phases and accumulator indices advance incrementally (no
      // division), and every B descriptor is the base plus an immediate (the
      // padded filter count N equals NMAX here).  Descriptors that had to be
      // moved from vector registers (R2UR) per MMA throttled the issue.
      constexpr uint32_t LB4 = (2u * NMAX * 16u) >> 4;  // B tap stride (>> 4)
      constexpr uint32_t B2P = (2u * NMAX * 16u) >> 4;  // bf16 tap-pair block stride (>> 4)
      const uint32_t ring = (uint32_t)a.ring;
#ifdef DPM_TC_PROBE
      long long pr_empty = 0, pr_full = 0, pr_rows = 0;
      const long long pr_t0 = clock64();
#endif
      uint32_t qs = 0, qph = 0;    // ring slot / phase of the strip's input row 0
      uint32_t acc = 0, aph = 0;   // accumulator index / phase of the current output row
      for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
        const dpm_corr_tile strip = a.strips[st];
        const dpm_corr_job job = a.jobs[strip.job];
        const int ho = seg_out_rows(strip, job.H - FH + 1);  // this segment's output rows
        const int hs = seg_in_rows(strip, job.H, FH);        // and staged input rows
        for (int y = 0; y < ho; ++y) {
          uint32_t sl[FH], ph[FH];  // slots / phases of input rows y .. y+FH-1
          sl[0] = qs;
          ph[0] = qph;
#pragma unroll
          for (int i = 1; i < FH; ++i) {
            sl[i] = sl[i - 1] + 1;
            ph[i] = ph[i - 1];
            if (sl[i] == ring) { sl[i] = 0; ph[i] ^= 1; }
          }
#ifdef DPM_TC_PROBE
          const long long t0 = clock64();
#endif
          mbar_wait(tempty + acc, aph ^ 1);
#ifdef DPM_TC_PROBE
          const long long t1 = clock64();
          pr_empty += t1 - t0;
#endif
#pragma unroll
          for (int i = 0; i < FH; ++i)
            if (y == 0 || i == FH - 1) mbar_wait(full + sl[i], ph[i]);
#ifdef DPM_TC_PROBE
          pr_full += clock64() - t1;
          pr_rows += 1;
#endif
          tc_fence_after();
          const uint32_t d = tmem_base + acc * (uint32_t)a.acc_cols;
          // opaque per row: keeps the compiler from hoisting all FH*FW B
          // descriptors into vector registers (each then needing R2UR per MMA);
          // base + immediate is formed at the use, on the uniform datapath
          uint64_t bB = dB0, bB2 = dB2;
          asm volatile("" : "+l"(bB), "+l"(bB2));
          if (elect_one()) {
#pragma unroll
            for (int i = 0; i < FH; ++i) {
              const uint64_t da = dA0 + sl[i] * slot_step;
#pragma unroll
              for (int j = 0; j < FW; ++j)
                mma_tf32(d, da + (uint32_t)j, bB + (uint32_t)((i * FW + j) * 2) * LB4, idesc1,
                         (i | j) != 0);
            }
#pragma unroll
            for (int i = 0; i < FH; ++i) {
              const uint64_t dl = dAlo0 + sl[i] * slot_step;
#pragma unroll
              for (int jp = 0; jp < (FW + 1) / 2; ++jp)
                mma_bf16(d, dl + (uint32_t)(2 * jp), bB2 + (uint32_t)((i * ((FW + 1) / 2) + jp)) * B2P,
                         idescbf);
            }
            // one commit per row (each costs the tensor pipe a bubble): the
            // epilogue frees input row y's slot once it sees this row's tfull
            tc_commit(tfull + acc);
          }
          __syncwarp();
          qs = sl[1 % FH];
          qph = ph[1 % FH];
          if (FH == 1) { if (++qs == ring) { qs = 0; qph ^= 1; } }
          if (++acc == TC_MAX_ACC) { acc = 0; aph ^= 1; }
        }
        for (int rr = ho; rr < hs; ++rr)  // rows never first of an output row
          if (++qs == ring) { qs = 0; qph ^= 1; }
      }
#ifdef DPM_TC_PROBE
      if (lane == 0) {
        atomicAdd(&dpm_tc_probe[0], (unsigned long long)pr_empty);
        atomicAdd(&dpm_tc_probe[1], (unsigned long long)pr_full);
        atomicAdd(&dpm_tc_probe[2], (unsigned long long)pr_rows);
        atomicAdd(&dpm_tc_probe[3], (unsigned long long)(clock64() - pr_t0));
      }
#endif
    } else {
    int64_t b_res = -1;              // Gtc offset of the resident core (multi-group)
    uint32_t bdone_ph = 0, bload_ph = 0;
    bool issued = false;
    for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
      const dpm_corr_job job = a.jobs[a.strips[st].job];
      const int ho = job.H - a.h + 1;
      DPM_CHECK(a.strips[st].pad == 0, "generic-shape strips are never segmented");
      if (a.tc_off != nullptr) {
        const int64_t off = a.tc_off[a.strips[st].job];
        if (off != b_res) {
          // every MMA that read the old core has completed, then one bulk
          // copy brings the strip's core (the ring and TMEM are untouched)
          if (issued) {
            if (elect_one()) tc_commit(bdone);
            __syncwarp();
            mbar_wait(bdone, bdone_ph);
            bdone_ph ^= 1;
          }
          if (elect_one()) {
            mbar_expect_tx(bload, b_bytes);
            const unsigned char* src = reinterpret_cast<const unsigned char*>(a.Gtc + off);
            for (uint32_t o = 0; o < b_bytes; o += 32768u)
              bulk_g2s(sB + o, src + o, min(32768u, b_bytes - o), bload);
          }
          __syncwarp();
          mbar_wait(bload, bload_ph);
          bload_ph ^= 1;
          b_res = off;
        }
        issued = true;
      }
      for (int y = 0; y < ho; ++y, ++row_glob) {
        const int b = row_glob & (TC_MAX_ACC - 1);
        mbar_wait(tempty + b, ((row_glob / TC_MAX_ACC) & 1) ^ 1);
        for (int rr = (y == 0 ? 0 : a.h - 1); rr < a.h; ++rr) {
          const uint32_t q = q_glob + y + rr;
          mbar_wait(full + q % a.ring, (q / a.ring) & 1);
        }
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(b * a.acc_cols);
        {
          uint64_t db = dB0;
          for (int i = 0; i < a.h; ++i) {
            const uint64_t da_row = dA0 + ((q_glob + y + i) % a.ring) * slot_step;
            for (int j = 0; j < a.w; ++j, db += tap_step) {
              const uint64_t da = da_row + (uint32_t)j;
              for (int kc = 0; kc < nq; kc += 2) {
                const uint64_t ahi = da + (uint32_t)(kc >> 1) * kcA;
                const uint64_t bb = db + (uint32_t)(kc >> 1) * kcB;
                if (elect_one()) {
                  mma_tf32(d, ahi, bb, idesc1, (i | j | kc) != 0);
                  mma_tf32(d, ahi + lo_step, bb, idesc2, 1);
                }
                __syncwarp();
              }
            }
          }
        }
        if (elect_one()) {
          tc_commit(tfull + b);                      // accumulator ready
          tc_commit(empty + (q_glob + y) % a.ring);  // input row y no longer needed
        }
        __syncwarp();
      }
      if (elect_one())
        for (int rr = ho; rr < job.H; ++rr) tc_commit(empty + (q_glob + rr) % a.ring);
      __syncwarp();
      q_glob += job.H;
    }
    }
  } else if (warp <= TC_PRODUCERS) {
    // =================== producers ===================
    // Producer warp p stages input rows q = p, p+3, ... of every strip: each
    // lane issues all of its (up to PQ) quad-column loads before converting,
    // so one row costs one memory latency, and three rows are in flight.
    constexpr int PQ = 10;  // quad-columns per lane per batch (R = 8: one batch per row)
    const int pw = warp - 1;
    uint32_t q_glob = 0;
    for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
      const dpm_corr_tile strip = a.strips[st];
      const dpm_corr_job job = a.jobs[strip.job];
      const int x0 = strip.tx * TC_M;
      const int64_t plane = (int64_t)job.H * job.pitch;
      const float* pbase = a.P + job.p_off + (int64_t)job.chan_off * plane;
      const int nelem = nq * tcols;
      const int hs = seg_in_rows(strip, job.H, FH > 0 ? FH : a.h);  // rows staged for the strip
      for (int q = pw; q < hs; q += TC_PRODUCERS) {
        const uint32_t qg = q_glob + q;
        const uint32_t slot = qg % a.ring;
        mbar_wait(empty + slot, ((qg / a.ring) & 1) ^ 1);
        float4* hi = reinterpret_cast<float4*>(sA + slot * slot_bytes);
        float4* lo = hi + nelem;
        const float* prow = pbase + (int64_t)(strip.ty + q) * job.pitch;
        if constexpr (BF) {
          // R == 8: lane handles positions c = lane + 32k; hi as two tf32 quads,
          // lo as 8 bf16 (16 B) per position, one zero position past the row
          uint4* lo16 = reinterpret_cast<uint4*>(sA + slot * slot_bytes + hi_bytes);
          constexpr int PP = (TC_M + (FW > 0 ? FW : 1) + 31) / 32;
          float v8[PP][8];
#pragma unroll
          for (int k = 0; k < PP; ++k) {
            const int c = lane + 32 * k, x = x0 + c;
            const bool ok = c < tcols && x < job.W;
#pragma unroll
            for (int r = 0; r < 8; ++r) v8[k][r] = ok ? __ldg(prow + (int64_t)r * plane + x) : 0.f;
          }
#pragma unroll
          for (int k = 0; k < PP; ++k) {
            const int c = lane + 32 * k;
            if (c > tcols) continue;
            float h8[8], l8[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              h8[r] = tf32_hi(v8[k][r]);
              l8[r] = v8[k][r] - h8[r];
            }
            if (c < tcols) {
              hi[c] = make_float4(h8[0], h8[1], h8[2], h8[3]);
              hi[tcols + c] = make_float4(h8[4], h8[5], h8[6], h8[7]);
            }
            lo16[c] = make_uint4(bf16x2_rn(l8[0], l8[1]), bf16x2_rn(l8[2], l8[3]),
                                 bf16x2_rn(l8[4], l8[5]), bf16x2_rn(l8[6], l8[7]));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(full + slot);
          continue;
        }
        // batches of 32 * PQ quad-columns (R > 8: more than one batch per row)
        for (int e0 = 0; e0 < nelem; e0 += 32 * PQ) {
          float4 v[PQ];
#pragma unroll
          for (int k = 0; k < PQ; ++k) {
            const int e = e0 + lane + 32 * k;
            v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < nelem) {
              const int quad = e / tcols, c = e - quad * tcols;
              const int x = x0 + c;
              if (x < job.W) {
                const float* p = prow + (int64_t)(4 * quad) * plane + x;
                v[k].x = __ldg(p);
                v[k].y = __ldg(p + plane);
                v[k].z = __ldg(p + 2 * plane);
                v[k].w = __ldg(p + 3 * plane);
              }
            }
          }
#pragma unroll
          for (int k = 0; k < PQ; ++k) {
            const int e = e0 + lane + 32 * k;
            if (e < nelem) {
              const float4 h = make_float4(tf32_hi(v[k].x), tf32_hi(v[k].y), tf32_hi(v[k].z),
                                           tf32_hi(v[k].w));
              hi[e] = h;
              lo[e] = make_float4(v[k].x - h.x, v[k].y - h.y, v[k].z - h.z, v[k].w - h.w);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(full + slot);
      }
      q_glob += hs;
    }
  } else {
    // =================== epilogue ===================
    const int quarter = warp & 3;  // TMEM lanes 32*quarter ..
    // input-row slots are freed here, after the MMAs that last read them
    // completed (tfull), by one thread of the first epilogue warp
    const bool releaser = warp == 1 + TC_PRODUCERS && lane == 0;
    uint32_t eslot = 0;  // ring slot of the current strip's next unreleased row
    auto release = [&](int nrows) {
      for (int k = 0; k < nrows; ++k) {
        if (releaser) mbar_arrive(empty + eslot);
        if (++eslot == (uint32_t)a.ring) eslot = 0;
      }
    };
    if constexpr (KS > 1) {
      uint32_t row_glob = 0;
      for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
        const dpm_corr_tile strip = a.strips[st];
        const dpm_corr_job job = a.jobs[strip.job];
        const int ho = job.H - FH + 1, wo = job.W - FW + 1, wp = s_pitch(wo);
        const int x = strip.tx * TC_M + quarter * 32 + lane;
        float vmax[8], vmin[8];
#pragma unroll
        for (int f = 0; f < 8; ++f) { vmax[f] = -INFINITY; vmin[f] = INFINITY; }
        int y = 0;
        for (; y < ho; y += KS, ++row_glob) {
          const int b = row_glob & (TC_MAX_ACC - 1);
          mbar_wait(tfull + b, (row_glob / TC_MAX_ACC) & 1);
          tc_fence_after();
          release(min(KS, job.H - y));  // rows y .. y+KS-1: no later group reads them
          const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * a.acc_cols);
#pragma unroll
          for (int k = 0; k < KS; ++k) {
            if (y + k >= ho) break;
            float v[16];  // hi 0..7 | lo 8..15 of row y+k
            tmem_ld16(taddr + 16 * k, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float* dst = a.S + job.s_off + (int64_t)(y + k) * wp + x;
#pragma unroll
            for (int f = 0; f < 8; ++f) {
              if (f < job.nf && x < wo) {
                const float sv = v[f] + v[8 + f];
                dst[(int64_t)f * ho * wp] = sv;
                vmax[f] = fmaxf(vmax[f], sv);
                vmin[f] = fminf(vmin[f], sv);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty + b);
        }
        if (y < job.H) release(job.H - y);  // rows past the last group's first KS
        if (a.ranges != nullptr && job.range_idx >= 0) {
#pragma unroll
          for (int f = 0; f < 8; ++f) {
            if (f >= job.nf) continue;
            float mx = vmax[f], mn = vmin[f];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
              mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            }
            if (lane == 0 && mx >= mn) {
              atomicMax(a.ranges + 2 * (job.range_idx + f), float_key(mx));
              atomicMin(a.ranges + 2 * (job.range_idx + f) + 1, float_key(mn));
            }
          }
        }
      }
    } else {
    constexpr int SPLIT = EPI / 4;                       // warps per quarter
    constexpr int CW = SPLIT == 2 ? 8 : 16;              // TMEM columns per chunk
    constexpr int LOC = ((NMAX / CW + SPLIT - 1) / SPLIT) * CW;  // filters per warp
    const int half = (warp - 1 - TC_PRODUCERS) / 4;      // which column chunks
    uint32_t row_glob = 0;
    for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
      const dpm_corr_tile strip = a.strips[st];
      const dpm_corr_job job = a.jobs[strip.job];
      const int ho = job.H - a.h + 1, wo = job.W - a.w + 1;
      const int nout = seg_out_rows(strip, ho), hs = seg_in_rows(strip, job.H, a.h);
      const int x = strip.tx * TC_M + quarter * 32 + lane;
      float vmax[LOC], vmin[LOC];  // this warp's chunks only (chunk c -> local c / SPLIT)
#pragma unroll
      for (int f = 0; f < LOC; ++f) { vmax[f] = -INFINITY; vmin[f] = INFINITY; }
      const int wp = s_pitch(wo);
      const int64_t plane = (int64_t)ho * wp;
      const bool xin = x < wo;
      // N is a compile-time constant for the fixed DPM shapes (N == NMAX)
      const int N = FH > 0 ? NMAX : a.N;
      for (int y = 0; y < nout; ++y, ++row_glob) {
        const uint32_t b = row_glob & (TC_MAX_ACC - 1);
        mbar_wait(tfull + b, (row_glob / TC_MAX_ACC) & 1);
        tc_fence_after();
        if constexpr (FH > 0) release(1);  // input row y: no later output row reads it
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + b * (uint32_t)a.acc_cols;
        float* dst = a.S + job.s_off + (int64_t)(strip.ty + y) * wp + x;
        // CW filters at a time: hi-half columns [fc, fc+CW) and lo-half [N+fc, ...)
#pragma unroll
        for (int fc = 0; fc < NMAX; fc += CW) {
          if (fc < N && (fc / CW) % SPLIT == half) {
            float vh[CW], vl[CW];
            if constexpr (CW == 16) {
              tmem_ld16(taddr + fc, vh);
              tmem_ld16(taddr + N + fc, vl);
            } else {
              tmem_ld8(taddr + fc, vh);
              tmem_ld8(taddr + N + fc, vl);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            {
#pragma unroll
              for (int k = 0; k < CW; ++k) {
                const int f = fc + k, li = (fc / CW / SPLIT) * CW + k;
                if (f < job.nf && xin) {
                  const float sv = vh[k] + vl[k];
                  dst[(int64_t)f * plane] = sv;
                  vmax[li] = fmaxf(vmax[li], sv);
                  vmin[li] = fminf(vmin[li], sv);
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + b);
      }
      if constexpr (FH > 0) release(hs - nout);  // rows never first of an output row
      if (a.ranges != nullptr && job.range_idx >= 0) {
#pragma unroll
        for (int li = 0; li < LOC; ++li) {
          const int f = ((li / CW) * SPLIT + half) * CW + li % CW;
          if (f >= job.nf) continue;
          float mx = vmax[li], mn = vmin[li];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          }
          if (lane == 0 && mx >= mn) {
            atomicMax(a.ranges + 2 * (job.range_idx + f), float_key(mx));
            atomicMin(a.ranges + 2 * (job.range_idx + f) + 1, float_key(mn));
          }
        }
      }
    }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

}  // namespace dpm

using namespace dpm;

// compile-time shapes of the launcher (DPM part / root filters at R = 8):
// they use the bf16 correction MMA and its smem layout
static bool tc_bf16(int h, int w, int R) { return R == 8 && h == 6 && (w == 6 || w == 11); }

// Rows stacked per accumulator group (1 = one output row per group).  Stacked
// groups (<= 8 filters, e.g. the DPM roots: 3 mirrored pairs) take the core as
// tap-row windows: per tap column j, NB = h + 2(KS-1) blocks of 16 N-rows
// [hi 8 filters | lo 8 filters] for tap rows i = h-1+KS-1 down to -(KS-1)
// (zero outside 0..h-1), K-major [j][quad][NB*16][4] fp32; then the bf16
// tap-pair blocks [pair][tap parity][NB*16][8] with rows 8..15 of each block 0.
// KS = 6 (measured sweep, roots 6x11 at config 4: KS 1/3/4/5/6 -> 1.54/1.00/
// 0.90/0.86/0.83 ms) is the deepest whose core + minimal ring fit 227 KB.
static int tc_stack(int h, int w, int R, int nf) { return tc_bf16(h, w, R) && nf <= 8 ? 6 : 1; }

static size_t tc_b_bytes(int h, int w, int R, int nf) {
  const int ks = tc_stack(h, w, R, nf);
  if (ks > 1) return ((size_t)w * (h + 2 * (ks - 1)) * 512 + 1023) & ~(size_t)1023;
  const int N = (nf + 15) & ~15;
  return ((size_t)h * w * (R / 4) * 2 * N * 16 + 1023) & ~(size_t)1023;
}

static size_t tc_b2_bytes(int h, int w, int R, int nf) {
  if (!tc_bf16(h, w, R)) return 0;
  const int ks = tc_stack(h, w, R, nf);
  if (ks > 1) return ((size_t)((w + 1) / 2) * (h + 2 * (ks - 1)) * 512 + 1023) & ~(size_t)1023;
  const int N = (nf + 15) & ~15;
  return ((size_t)h * ((w + 1) / 2) * 2 * N * 16 + 1023) & ~(size_t)1023;
}

static size_t tc_slot(int h, int w, int R) {
  const int nq = R / 4, tcols = TC_M + w - 1;
  if (tc_bf16(h, w, R))
    return ((size_t)nq * tcols * 16 + (size_t)(tcols + 1) * 16 + 127) & ~(size_t)127;
  return 2ull * nq * tcols * 16;
}

// Input-row ring depth: at least the rows one accumulator group reads plus
// slack (h + KS + 1), then as deep as shared memory allows (up to
// TC_MAX_RING), so the producers run further ahead of the MMA warp and hide
// row-load latency.
static int tc_ring(int h, int w, int R, int nf) {
  const size_t slot = tc_slot(h, w, R);
  const size_t fixed = tc_b_bytes(h, w, R, nf) + tc_b2_bytes(h, w, R, nf) +
                       (2 * TC_MAX_RING + 2 * TC_MAX_ACC) * 8 + 32 + 15;
  const int need = h + tc_stack(h, w, R, nf) + 1;
  int ring = need <= TC_MAX_RING ? need : TC_MAX_RING;
  while (ring < TC_MAX_RING && fixed + (ring + 1) * slot <= 227 * 1024) ++ring;
  return ring;
}

// CTA-pair kernel for the part shape (corr_tc2.cu, "K2
// on CTA pairs"): by default for launches of at least 2 strips per SM;
// DPM_TC_PAIR=0 always selects the one-CTA kernel (bit-identical maps),
// DPM_TC_PAIR=1 pairs whatever the strip count (tests; the strips must be
// whole: DPM_TC_SEGMENT=0 for small pyramids)
static int tc_pairs_mode() {
  const char* e = getenv("DPM_TC_PAIR");
  return e && e[0] == '0' ? 0 : e && e[0] == '1' ? 1 : 2;
}

extern "C" int dpm_correlate_tc_stack(int h, int w, int R, int nf) { return tc_stack(h, w, R, nf); }

extern "C" size_t dpm_correlate_tc_smem(int h, int w, int R, int nf) {
  if (tc16_shape(h, w, R, (nf + 15) & ~15)) return tc16_smem(nullptr);
  const int ring = tc_ring(h, w, R, nf);
  const size_t slot = tc_slot(h, w, R);
  return tc_b_bytes(h, w, R, nf) + tc_b2_bytes(h, w, R, nf) + ((ring * slot + 15) & ~(size_t)15) +
         (2 * TC_MAX_RING + 2 * TC_MAX_ACC) * 8 + 32;
}

extern "C" size_t dpm_correlate_tc_core_floats(int h, int w, int R, int nf) {
  if (tc16_shape(h, w, R, (nf + 15) & ~15)) return tc16_core_floats();
  const int ks = tc_stack(h, w, R, nf);
  if (ks > 1) {
    const size_t nb = (size_t)h + 2 * (ks - 1);
    return (size_t)w * nb * 128 + (size_t)((w + 1) / 2) * nb * 128;  // 512 B per block
  }
  const int N = (nf + 15) & ~15;
  size_t f = (size_t)h * w * (R / 4) * 2 * N * 4;
  if (tc_bf16(h, w, R)) f += (size_t)h * ((w + 1) / 2) * 2 * N * 8 / 2;  // bf16 block
  return f;
}

static int tc_launch(const float* P, const float* Gtc, const int64_t* tc_off, float* S,
                     const dpm_corr_job* jobs, const dpm_corr_tile* strips, int nstrips, int h,
                     int w, int R, int nf, uint32_t* ranges, void* stream) {
  DPM_REQUIRE(P && Gtc && S && jobs && strips, "dpm_correlate_tc: null pointer");
  DPM_REQUIRE(R % 8 == 0 && R >= 8, "dpm_correlate_tc: R=%d must be a multiple of 8", R);
  DPM_REQUIRE(R <= 32 && w <= 64, "dpm_correlate_tc: R=%d w=%d outside the staged row", R, w);
  DPM_REQUIRE(nf >= 1 && nf <= 64, "dpm_correlate_tc: nf=%d outside [1, 64]", nf);
  DPM_REQUIRE(h >= 1 && w >= 1 && h + 2 <= TC_MAX_RING, "dpm_correlate_tc: filter %dx%d", h, w);
  if (nstrips == 0) return DPM_OK;
  const int N = (nf + 15) & ~15;
  const size_t smem = dpm_correlate_tc_smem(h, w, R, nf);
  DPM_REQUIRE(smem <= 227 * 1024, "dpm_correlate_tc: needs %zu B shared memory", smem);
  int dev = 0, sms = 148;
  DPM_CUDA(cudaGetDevice(&dev));
  DPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  TcArgs a{P, Gtc, S, jobs, strips, nstrips, h, w, R, N, tc_ring(h, w, R, nf), 0, 0, ranges, tc_off};
  a.acc_cols = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 256;
  a.nacc = 512 / a.acc_cols > TC_MAX_ACC ? TC_MAX_ACC : 512 / a.acc_cols;
  void (*fn)(const TcArgs) = N <= 16 ? corr_tc_kernel<16, 0, 0>
                             : N <= 32 ? corr_tc_kernel<32, 0, 0>
                             : N <= 48 ? corr_tc_kernel<48, 0, 0>
                                       : corr_tc_kernel<64, 0, 0>;
  int threads = TC_THREADS;
  const int ks = tc_stack(h, w, R, nf);
  if (tc16_shape(h, w, R, N)) {
    return launch_tc16(a, as_stream(stream));  // 6 x 6 at R = 16: compile-time kernel
  } else if (tc_off != nullptr) {
    // several groups per launch: the generic-shape kernel (runtime taps, B
    // reloaded per group by one bulk copy)
  } else if (ks > 1) {  // <= 8 filters (DPM roots: 3 mirrored pairs): rows stacked 6 per group
    a.N = 8;
    a.acc_cols = 16 * ks;
    a.nacc = 512 / a.acc_cols > TC_MAX_ACC ? TC_MAX_ACC : 512 / a.acc_cols;
    fn = w == 11 ? corr_tc_kernel<8, 6, 11, 4, 6> : corr_tc_kernel<8, 6, 6, 4, 6>;
  } else if (h == 6 && w == 6 && R == 8 &&
             (tc_pairs_mode() == 1 || (tc_pairs_mode() == 2 && nstrips >= 2 * sms))) {
    // DPM part filters: cta_group::2 pairs, on whole strips only.  The planner
    // (engine._segment_strips) splits strips only below 2 strips per SM and
    // keeps the segments below 2 per SM, so segmented lists never reach it.
    return launch_tc_pair(a, as_stream(stream));
  } else if (h == 6 && w == 6 && R == 8) {  // DPM part filters: 8 epilogue warps (12 measured slower)
    fn = N <= 16 ? corr_tc_kernel<16, 6, 6, 8>
       : N <= 32 ? corr_tc_kernel<32, 6, 6, 8>
       : N <= 48 ? corr_tc_kernel<48, 6, 6, 8>
                 : corr_tc_kernel<64, 6, 6, 8>;
    threads = 32 * (1 + TC_PRODUCERS + 8);
  }
  else if (h == 6 && w == 11 && R == 8 && N <= 16)  // DPM root filters (3 mirrored pairs)
    fn = corr_tc_kernel<16, 6, 11>;
  // the kernel indexes accumulators as row & 3 (N <= 64 keeps 4 buffers in TMEM)
  DPM_REQUIRE(a.nacc == TC_MAX_ACC, "dpm_correlate_tc: %d accumulator buffers", a.nacc);
  DPM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = nstrips < sms ? nstrips : sms;
  fn<<<grid, threads, smem, as_stream(stream)>>>(a);
  DPM_LAUNCHED("corr_tc_kernel");
  return DPM_OK;
}

extern "C" int dpm_correlate_tc(const float* P, const float* Gtc, float* S, const dpm_corr_job* jobs,
                                const dpm_corr_tile* strips, int nstrips, int h, int w, int R,
                                int nf, uint32_t* ranges, void* stream) {
  return tc_launch(P, Gtc, nullptr, S, jobs, strips, nstrips, h, w, R, nf, ranges, stream);
}

extern "C" int dpm_correlate_tc_groups(const float* P, const float* Gtc, const int64_t* tc_off,
                                       float* S, const dpm_corr_job* jobs,
                                       const dpm_corr_tile* strips, int nstrips, int h, int w,
                                       int R, int nf, uint32_t* ranges, void* stream) {
  DPM_REQUIRE(tc_off, "dpm_correlate_tc_groups: null tc_off");
  DPM_REQUIRE(!tc_bf16(h, w, R),
              "dpm_correlate_tc_groups: %dx%d at R=%d has a compile-time kernel; launch its "
              "groups with dpm_correlate_tc", h, w, R);
  return tc_launch(P, Gtc, tc_off, S, jobs, strips, nstrips, h, w, R, nf, ranges, stream);
}

#ifdef DPM_TC_PROBE
extern "C" int dpm_tc_probe_read(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, dpm_tc_probe, sizeof(unsigned long long) * 4);
  const unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(dpm_tc_probe, z, sizeof(z));
  return 0;
}
#endif
