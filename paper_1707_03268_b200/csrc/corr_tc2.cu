// K2 for the DPM part filters (6 x 6 taps, R = 8) on CTA pairs:
// tcgen05.mma.cta_group::2 with M = 256.
//
// Same computation and numerics as corr_tc_kernel<N, 6, 6, 8> (corr_tc.cu):
// per output row and tap (i, j) the tf32 MMA A_hi x [B_hi | B_lo] and per
// tap pair the bf16 correction A_lo x B_hi, accumulated in TMEM, summed
// hi + lo in the epilogue.  What changes is who reads the operands.  The
// one-CTA kernel is bound by shared-memory operand reads (per tap 4 KB of A
// and 3 KB of B for 128 x 96 x 8 MACs: ~56 cycles against the tensor floor's
// 48).  A pair of CTAs on one TPC issues each MMA once for 256 positions:
// CTA 0 supplies output row y, CTA 1 row y + 1 (A from each CTA's own ring,
// same shared offset), and B is split by columns -- CTA 0 holds the hi
// filters, CTA 1 the lo filters (bf16 block: the first / second half of the
// filters) -- so each SM reads its A and HALF of B per MMA.  The tf32 MMA
// drops to the tensor floor and the bf16 MMA from ~43 to ~37 cycles.
//
// Measured (config 4 part group, N = 48): the MMAs do
// get cheaper -- 2.70 ms with the epilogue's S stores switched off -- but the
// S stores (5 GB per launch) then bind: 3.50 ms against 3.42 ms for the
// one-CTA kernel, and on some boxes 12 ms, with the leader's epilogue the
// slow side (per-pair clock probes).  So the launcher keeps the one-CTA
// kernel and this one is opt-in (DPM_TC_PAIR=1); the maps are bit-identical
// either way (tests/test_gpu_parity.py).
//
// Row split.  The strip's ho output rows are halved: CTA r computes output
// rows r*np .. r*np + np - 1 (np = ceil(ho / 2)), and its ring position k
// holds input row k + r*np (rows past the level are zero), so tap row i of
// output pair p (rows p and np + p) is ring position p + i in BOTH CTAs: one
// descriptor addresses both.  Each CTA stages np + h - 1 rows per strip, so
// the pair stages each row about once (an earlier split -- CTA r taking rows
// 2p + r -- made BOTH CTAs stage every row of the strip, twice the staging of
// the one-CTA kernel).
//
// Synchronisation (rank 0 = leader issues every MMA):
//   full[s]   leader's barrier, 2 arrivals: each CTA's producer after staging
//             position s (the peer arrives remotely);
//   empty[s]  per CTA, its epilogue frees positions 2p, 2p + 1 once output
//             pair p's MMAs completed (tfull);
//   tfull[b]  per CTA, multicast tcgen05.commit of the pair's MMAs;
//   tempty[b] leader's barrier, 2 x 8 epilogue warps (peer remotely) after
//             draining accumulator b.
#include "tc_common.cuh"

namespace dpm {
namespace tc2 {

constexpr int FH = 6, FW = 6;
constexpr int NPAIR = (FW + 1) / 2;         // bf16 tap-pair blocks per tap row
constexpr int PRODUCERS = 4;                // warps 1..4
constexpr int EPI = 8;                      // warps 5..12 (two per TMEM lane quarter)
constexpr int THREADS = 32 * (1 + PRODUCERS + EPI);
constexpr int TCOLS = TC_M + FW - 1;        // staged positions of a row
constexpr uint32_t HI_BYTES = 2u * TCOLS * 16u;  // two tf32 rank quads
constexpr uint32_t SLOT_BYTES = (HI_BYTES + (TCOLS + 1u) * 16u + 127u) & ~127u;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// arrive on the barrier at the same shared offset in CTA `rank` of the pair.
// Default semantics (release at CTA scope, as CUTLASS's 2-SM producer
// commit): the staged rows were made visible to the tensor core's async
// proxy by fence.proxy.async before the arrive.  A .release.cluster arrive
// compiles to MEMBAR.ALL.GPU, which waits for every outstanding global store.
__device__ __forceinline__ void mbar_arrive_at(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// relaxed remote arrive: the epilogue's accumulator release, ordered after
// its TMEM loads by tcgen05.wait::ld + tcgen05.fence::before_thread_sync --
// no memory fence (the S stores need not be visible to the MMA warp)
__device__ __forceinline__ void mbar_arrive_relaxed_at(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

__device__ __forceinline__ void mma2_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma2_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc));
}

// MMA completion -> the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int N>
constexpr uint32_t b_bytes() { return (uint32_t)FH * FW * 2u * N * 16u; }  // half of [hi | lo]
template <int N>
constexpr uint32_t b2_bytes() { return (uint32_t)FH * NPAIR * 2u * (N / 2) * 16u; }
template <int N>
constexpr uint32_t fixed_bytes() {
  return ((b_bytes<N>() + 1023u) & ~1023u) + ((b2_bytes<N>() + 1023u) & ~1023u) +
         (2 * TC_MAX_RING + 2 * TC_MAX_ACC) * 8 + 16;
}

// N: padded filter count (16..64, multiple of 16) -- the MMA is 256 x 2N
// (tf32) and 256 x N (bf16), legal for cta_group::2 (N multiple of 16).
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    corr_tc2_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  constexpr int HN = N / 2;
  unsigned char* sB = smem;
  unsigned char* sB2 = smem + ((b_bytes<N>() + 1023u) & ~1023u);
  unsigned char* sA = sB2 + ((b2_bytes<N>() + 1023u) & ~1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + a.ring * SLOT_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + TC_MAX_RING;
  uint64_t* tfull = bars + 2 * TC_MAX_RING;
  uint64_t* tempty = tfull + TC_MAX_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + TC_MAX_ACC);
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  // ---- setup: this CTA's half of the core, barriers, TMEM (both CTAs)
  {
    // tf32 block [tap][quad][2N][4]: rank r keeps rows [rN, rN + N)
    const float4* src = reinterpret_cast<const float4*>(a.Gtc);
    float4* dst = reinterpret_cast<float4*>(sB);
    for (int e = threadIdx.x; e < FH * FW * 2 * N; e += THREADS) {
      const int tq = e / N, row = e - tq * N;
      dst[e] = __ldg(src + (int64_t)tq * 2 * N + rank * N + row);
    }
    // bf16 block [i][pair][parity][N][16 B] after it: rank r keeps rows [r N/2, ...)
    const float4* src2 = src + FH * FW * 2 * 2 * N;
    float4* dst2 = reinterpret_cast<float4*>(sB2);
    for (int e = threadIdx.x; e < FH * NPAIR * 2 * HN; e += THREADS) {
      const int blk = e / HN, row = e - blk * HN;
      dst2[e] = __ldg(src2 + (int64_t)blk * N + rank * HN + row);
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.ring; ++s) {
      mbar_init(full + s, 2);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < TC_MAX_ACC; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 2 * EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // core visible to the tensor core
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrival
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ring = (uint32_t)a.ring;

  if (warp == 0) {
    if (rank == 0) {
      // =================== MMA issuer (leader) ===================
      constexpr uint32_t idesc1 = idesc_tf32(2 * N, 2 * TC_M);
      constexpr uint32_t idescbf = idesc_bf16(N, 2 * TC_M);
      constexpr uint32_t TAPB = (2u * N * 16u) >> 4;     // tap stride of the tf32 half (>> 4)
      constexpr uint32_t PAIRB = (2u * HN * 16u) >> 4;   // tap-pair stride of the bf16 half
      constexpr uint32_t SLOT4 = SLOT_BYTES >> 4;
      const uint64_t dA0 = umma_desc(smem_u32(sA), TCOLS * 16u, 128);
      const uint64_t dAlo0 = umma_desc(smem_u32(sA) + HI_BYTES, 16u, 128u);
      const uint64_t dB0 = umma_desc(smem_u32(sB), N * 16u, 128);
      const uint64_t dB20 = umma_desc(smem_u32(sB2), HN * 16u, 128u);
      uint32_t qs = 0, qph = 0;   // ring slot / phase of the strip's position 0
      uint32_t acc = 0, aph = 0;  // accumulator / phase of the current output pair
      for (int st = cluster; st < a.nstrips; st += nclusters) {
        const dpm_corr_job job = a.jobs[a.strips[st].job];
        const int ho = job.H - FH + 1, np = (ho + 1) >> 1;
        for (int p = 0; p < np; ++p) {
          uint32_t sl[FH], ph[FH];  // slots / phases of positions p .. p + FH - 1
          sl[0] = qs;
          ph[0] = qph;
#pragma unroll
          for (int i = 1; i < FH; ++i) {
            sl[i] = sl[i - 1] + 1;
            ph[i] = ph[i - 1];
            if (sl[i] == ring) { sl[i] = 0; ph[i] ^= 1; }
          }
          mbar_wait(tempty + acc, aph ^ 1);
#pragma unroll
          for (int i = 0; i < FH; ++i)
            if (p == 0 || i == FH - 1) mbar_wait(full + sl[i], ph[i]);
          tc_fence_after();
          const uint32_t d = tmem_base + acc * (uint32_t)a.acc_cols;
          uint64_t bB = dB0, bB2 = dB20;
          asm volatile("" : "+l"(bB), "+l"(bB2));
          if (elect_one()) {
#pragma unroll
            for (int i = 0; i < FH; ++i) {
              const uint64_t da = dA0 + sl[i] * SLOT4;
#pragma unroll
              for (int j = 0; j < FW; ++j)
                mma2_tf32(d, da + (uint32_t)j, bB + (uint32_t)(i * FW + j) * TAPB, idesc1,
                          (i | j) != 0);
            }
#pragma unroll
            for (int i = 0; i < FH; ++i) {
              const uint64_t dl = dAlo0 + sl[i] * SLOT4;
#pragma unroll
              for (int jp = 0; jp < NPAIR; ++jp)
                mma2_bf16(d, dl + (uint32_t)(2 * jp), bB2 + (uint32_t)(i * NPAIR + jp) * PAIRB,
                          idescbf);
            }
            commit_pair(tfull + acc);
          }
          __syncwarp();
          qs = sl[1];
          qph = ph[1];
          if (++acc == TC_MAX_ACC) { acc = 0; aph ^= 1; }
        }
        for (int rr = np; rr < np + FH - 1; ++rr)  // positions no pair starts at
          if (++qs == ring) { qs = 0; qph ^= 1; }
      }
    }
  } else if (warp <= PRODUCERS) {
    // =================== producers (both CTAs) ===================
    // warp p stages positions k = p, p + 4, ... of every strip: input row
    // k + rank as hi tf32 quads + lo bf16, like corr_tc_kernel's R == 8 path
    const int pw = warp - 1;
    uint32_t q_glob = 0;
    for (int st = cluster; st < a.nstrips; st += nclusters) {
      const dpm_corr_tile strip = a.strips[st];
      const dpm_corr_job job = a.jobs[strip.job];
      const int x0 = strip.tx * TC_M;
      const int64_t plane = (int64_t)job.H * job.pitch;
      const float* pbase = a.P + job.p_off + (int64_t)job.chan_off * plane;
      const int np = (job.H - FH + 2) >> 1;  // output rows per CTA: ceil(ho / 2)
      DPM_CHECK(strip.pad == 0, "CTA-pair strips are never segmented");
      for (int k = pw; k < np + FH - 1; k += PRODUCERS) {
        const uint32_t qg = q_glob + k;
        const uint32_t slot = qg % ring;
        mbar_wait(empty + slot, ((qg / ring) & 1) ^ 1);
        const int q = k + (int)rank * np;
        float4* hi = reinterpret_cast<float4*>(sA + slot * SLOT_BYTES);
        uint4* lo16 = reinterpret_cast<uint4*>(sA + slot * SLOT_BYTES + HI_BYTES);
        const float* prow = pbase + (int64_t)q * job.pitch;
        constexpr int PP = (TC_M + FW + 31) / 32;
        float v8[PP][8];
#pragma unroll
        for (int kk = 0; kk < PP; ++kk) {
          const int c = lane + 32 * kk, x = x0 + c;
          const bool ok = c < TCOLS && x < job.W && q < job.H;
#pragma unroll
          for (int r = 0; r < 8; ++r) v8[kk][r] = ok ? __ldg(prow + (int64_t)r * plane + x) : 0.f;
        }
#pragma unroll
        for (int kk = 0; kk < PP; ++kk) {
          const int c = lane + 32 * kk;
          if (c > TCOLS) continue;
          float h8[8], l8[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            h8[r] = tf32_hi(v8[kk][r]);
            l8[r] = v8[kk][r] - h8[r];
          }
          if (c < TCOLS) {
            hi[c] = make_float4(h8[0], h8[1], h8[2], h8[3]);
            hi[TCOLS + c] = make_float4(h8[4], h8[5], h8[6], h8[7]);
          }
          lo16[c] = make_uint4(bf16x2_rn(l8[0], l8[1]), bf16x2_rn(l8[2], l8[3]),
                               bf16x2_rn(l8[4], l8[5]), bf16x2_rn(l8[6], l8[7]));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(full + slot);
          else mbar_arrive_at(full + slot, 0);
        }
      }
      q_glob += np + FH - 1;
    }
  } else {
    // =================== epilogue (both CTAs) ===================
    // output row p + rank * np of pair p from this CTA's TMEM (lanes = positions)
    constexpr int CW = 8;                               // TMEM columns per chunk
    constexpr int LOC = ((N / CW + 1) / 2) * CW;        // filters per warp
    const int quarter = warp & 3;
    const int half = (warp - 1 - PRODUCERS) / 4;        // which column chunks
    const bool releaser = warp == 1 + PRODUCERS && lane == 0;
    uint32_t eslot = 0;
    auto release = [&](int n) {
      for (int k = 0; k < n; ++k) {
        if (releaser) mbar_arrive(empty + eslot);
        if (++eslot == ring) eslot = 0;
      }
    };
    uint32_t row_glob = 0;
    for (int st = cluster; st < a.nstrips; st += nclusters) {
      const dpm_corr_tile strip = a.strips[st];
      const dpm_corr_job job = a.jobs[strip.job];
      const int ho = job.H - FH + 1, wo = job.W - FW + 1;
      const int np = (ho + 1) >> 1;
      const int x = strip.tx * TC_M + quarter * 32 + lane;
      float vmax[LOC], vmin[LOC];
#pragma unroll
      for (int f = 0; f < LOC; ++f) { vmax[f] = -INFINITY; vmin[f] = INFINITY; }
      const int wp = s_pitch(wo);
      const int64_t plane = (int64_t)ho * wp;
      const bool xin = x < wo;
      for (int p = 0; p < np; ++p, ++row_glob) {
        const uint32_t b = row_glob & (TC_MAX_ACC - 1);
        mbar_wait(tfull + b, (row_glob / TC_MAX_ACC) & 1);
        tc_fence_after();
        release(1);  // position p: no later pair reads it
        const int y = p + (int)rank * np;
        if (y < ho) {
          const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + b * (uint32_t)a.acc_cols;
          float* dst = a.S + job.s_off + (int64_t)y * wp + x;
          // all of this warp's chunks in flight, then one wait
          constexpr int NCH = LOC / CW;
          float vh[NCH][CW], vl[NCH][CW];
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const int fc = (2 * c + half) * CW;
            if (fc < N) {
              tmem_ld8(taddr + fc, vh[c]);
              tmem_ld8(taddr + N + fc, vl[c]);
            }
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (xin && job.nf >= N) {  // every filter of the padded group is real: no predicates
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              const int fc = (2 * c + half) * CW;
              if (fc >= N) continue;
              float* d = dst + (int64_t)fc * plane;
#pragma unroll
              for (int k = 0; k < CW; ++k, d += plane) {
                const int li = c * CW + k;
                const float sv = vh[c][k] + vl[c][k];
                *d = sv;
                vmax[li] = fmaxf(vmax[li], sv);
                vmin[li] = fminf(vmin[li], sv);
              }
            }
          } else if (xin) {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              const int fc = (2 * c + half) * CW;
#pragma unroll
              for (int k = 0; k < CW; ++k) {
                const int f = fc + k, li = c * CW + k;
                if (fc < N && f < job.nf) {
                  const float sv = vh[c][k] + vl[c][k];
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
        if (lane == 0) {
          if (rank == 0) mbar_arrive(tempty + b);
          else mbar_arrive_relaxed_at(tempty + b, 0);
        }
      }
      release(FH - 1);  // positions no pair starts at
      if (a.ranges != nullptr && job.range_idx >= 0) {
#pragma unroll
        for (int li = 0; li < LOC; ++li) {
          const int f = ((li / CW) * 2 + half) * CW + li % CW;
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

  // both CTAs done (the peer's smem and barriers are no longer addressed,
  // every accumulator drained) before the pair frees its TMEM
  tc_fence_before();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

template <int N>
int launch(TcArgs a, cudaStream_t stream) {
  const size_t fixed = fixed_bytes<N>();
  int ring = TC_MAX_RING;
  while (ring > FH + 2 && fixed + (size_t)ring * SLOT_BYTES > 227 * 1024) --ring;
  const size_t smem = fixed + (size_t)ring * SLOT_BYTES;
  DPM_REQUIRE(smem <= 227 * 1024, "dpm_correlate_tc (pairs): needs %zu B shared memory", smem);
  a.ring = ring;
  a.acc_cols = 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 256;
  DPM_REQUIRE(512 / a.acc_cols >= TC_MAX_ACC, "dpm_correlate_tc (pairs): N=%d", N);
  auto fn = corr_tc2_kernel<N>;
  DPM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  cfg.gridDim = dim3(2 * (a.nstrips < 74 ? a.nstrips : 74));
  DPM_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, fn, &cfg));
  DPM_REQUIRE(max_clusters >= 1, "dpm_correlate_tc (pairs): no CTA pair fits an SM pair");
  const int pairs = a.nstrips < max_clusters ? a.nstrips : max_clusters;
  cfg.gridDim = dim3(2 * pairs);
  DPM_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  DPM_LAUNCHED("corr_tc2_kernel");
  return DPM_OK;
}

}  // namespace tc2

// Launcher for the part shape (h = w = 6, R = 8, nf <= 64); a.N = padded
// filter count.
int launch_tc_pair(const TcArgs& a, cudaStream_t stream) {
  switch (a.N) {
    case 16: return tc2::launch<16>(a, stream);
    case 32: return tc2::launch<32>(a, stream);
    case 48: return tc2::launch<48>(a, stream);
    case 64: return tc2::launch<64>(a, stream);
  }
  DPM_REQUIRE(false, "dpm_correlate_tc (pairs): N=%d", a.N);
  return DPM_OK;
}

}  // namespace dpm
