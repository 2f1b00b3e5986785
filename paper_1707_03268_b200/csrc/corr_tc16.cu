// K2 on tcgen05 for 6 x 6 filters over a rank-16 basis, 16 filters per
// group, any number of groups per launch (config 3's part filters: 60 groups
// of one shared R = 16 basis).
//
// Same scheme as the R = 8 part kernel (corr_tc.cu): M = 128 output
// positions of one row, N = filters, the A operand of tap (i, j) is the
// staged input row y+i shifted by j positions (+16 j bytes on the smem
// descriptor), accumulators in TMEM.  At R = 16 a tap is K = 16 ranks:
//   MMA1 (kind::tf32, N = 32 = [B_hi | B_lo]) twice, rank quads 0-1 and 2-3;
//   MMA2 (kind::f16, bf16 A_lo x bf16 B_hi, N = 16) once -- K = 16 is
//   exactly the tap's 16 ranks, staged as two 8-rank bf16 planes;
// so D = A_hi B_hi + A_hi B_lo + A_lo B_hi in FP32 accumulation (the dropped
// A_lo B_lo is ~2^-22 relative, the bf16 rounding of the correction ~2^-19).
//
// Groups: the core (tf32 block [36 taps][4 quads][32][4] then bf16 block
// [36 taps][2][16][8], 90 KB) is resident in shared memory; with several
// groups per launch (tc_off != NULL) the MMA warp reloads it with bulk
// copies when a strip's group differs from the resident one, after a
// commit has drained every MMA that read the old core.  Persistent CTAs walk
// 128-wide strips top to bottom; every input row is staged once per strip.
//
// Warp roles: 0 MMA issue (one elected lane), 1-4 producers (input rows ->
// hi tf32 quads + lo bf16 planes in a ring, mbarrier full / empty), 5-8
// epilogue (tcgen05.ld of the row's accumulator, hi + lo, S stores, extrema).
#include "tc_common.cuh"

namespace dpm {
namespace tc16 {

constexpr int FH = 6, FW = 6, TAPS = FH * FW;
constexpr int N = 16;                       // filters per group (padded)
constexpr int PRODUCERS = 4;
constexpr int EPI = 4;
constexpr int THREADS = 32 * (1 + PRODUCERS + EPI);
constexpr int TCOLS = TC_M + FW - 1;        // staged positions of a row
constexpr uint32_t HI_BYTES = 4u * TCOLS * 16u;            // 4 tf32 rank quads
constexpr uint32_t LO_PLANE = (TCOLS + 1u) * 16u;          // one 8-rank bf16 plane
constexpr uint32_t SLOT_BYTES = (HI_BYTES + 2u * LO_PLANE + 127u) & ~127u;
constexpr uint32_t B_BYTES = TAPS * 4u * (2u * N) * 16u;   // tf32 hi|lo block
constexpr uint32_t B2_BYTES = TAPS * 2u * N * 16u;         // bf16 block
constexpr uint32_t FIXED = ((B_BYTES + 1023u) & ~1023u) + ((B2_BYTES + 1023u) & ~1023u) +
                           (2 * TC_MAX_RING + 2 * TC_MAX_ACC) * 8 + 32;
constexpr int ACC_COLS = 2 * N;             // hi | lo columns per accumulator

__global__ void __launch_bounds__(THREADS, 1) corr_tc16_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  unsigned char* sB = smem;
  unsigned char* sB2 = smem + ((B_BYTES + 1023u) & ~1023u);
  unsigned char* sA = sB2 + ((B2_BYTES + 1023u) & ~1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + a.ring * SLOT_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + TC_MAX_RING;
  uint64_t* tfull = bars + 2 * TC_MAX_RING;
  uint64_t* tempty = tfull + TC_MAX_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + TC_MAX_ACC);
  uint64_t* bdone = tempty + TC_MAX_ACC + 1;
  uint64_t* bload = bdone + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.ring; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < TC_MAX_ACC; ++b) {
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
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ring = (uint32_t)a.ring;

  if (warp == 0) {
    // =================== MMA issuer ===================
    constexpr uint32_t idesc1 = idesc_tf32(2 * N), idescbf = idesc_bf16(N);
    constexpr uint32_t LBOA = TCOLS * 16u;                 // between rank quads
    constexpr uint32_t QP_A = (2u * LBOA) >> 4;            // quads 2-3 (>> 4)
    constexpr uint32_t TAP_B = (4u * 2u * N * 16u) >> 4;   // tf32 block per tap
    constexpr uint32_t QP_B = (2u * 2u * N * 16u) >> 4;    // quads 2-3 within a tap
    constexpr uint32_t TAP_B2 = (2u * N * 16u) >> 4;       // bf16 block per tap
    constexpr uint32_t SLOT4 = SLOT_BYTES >> 4;
    const uint64_t dA0 = umma_desc(smem_u32(sA), LBOA, 128);
    const uint64_t dAlo0 = umma_desc(smem_u32(sA) + HI_BYTES, LO_PLANE, 128);
    const uint64_t dB0 = umma_desc(smem_u32(sB), 2u * N * 16u, 128);
    const uint64_t dB20 = umma_desc(smem_u32(sB2), N * 16u, 128);
    uint32_t qs = 0, qph = 0, acc = 0, aph = 0, bdone_ph = 0, bload_ph = 0;
    int64_t b_res = -1;
    bool issued = false;
    for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
      const int jid = a.strips[st].job;
      const dpm_corr_job job = a.jobs[jid];
      const int64_t off = a.tc_off != nullptr ? a.tc_off[jid] : 0;
      if (off != b_res) {
        // the old core is no longer read once every issued MMA completed
        if (issued) {
          if (elect_one()) tc_commit(bdone);
          __syncwarp();
          mbar_wait(bdone, bdone_ph);
          bdone_ph ^= 1;
        }
        if (elect_one()) {
          const unsigned char* src = reinterpret_cast<const unsigned char*>(a.Gtc + off);
          mbar_expect_tx(bload, B_BYTES + B2_BYTES);
          for (uint32_t o = 0; o < B_BYTES; o += 32768u)
            bulk_g2s(sB + o, src + o, min(32768u, B_BYTES - o), bload);
          bulk_g2s(sB2, src + B_BYTES, B2_BYTES, bload);
        }
        __syncwarp();
        mbar_wait(bload, bload_ph);
        bload_ph ^= 1;
        b_res = off;
      }
      const int ho = job.H - FH + 1;
      for (int y = 0; y < ho; ++y) {
        uint32_t sl[FH], ph[FH];
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
          if (y == 0 || i == FH - 1) mbar_wait(full + sl[i], ph[i]);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * (uint32_t)ACC_COLS;
        uint64_t bB = dB0, bB2 = dB20;
        asm volatile("" : "+l"(bB), "+l"(bB2));
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < FH; ++i) {
            const uint64_t da = dA0 + sl[i] * SLOT4;
#pragma unroll
            for (int j = 0; j < FW; ++j) {
              const uint64_t bt = bB + (uint32_t)(i * FW + j) * TAP_B;
              mma_tf32(d, da + (uint32_t)j, bt, idesc1, (i | j) != 0);
              mma_tf32(d, da + (uint32_t)j + QP_A, bt + QP_B, idesc1, 1);
            }
          }
#pragma unroll
          for (int i = 0; i < FH; ++i) {
            const uint64_t dl = dAlo0 + sl[i] * SLOT4;
#pragma unroll
            for (int j = 0; j < FW; ++j)
              mma_bf16(d, dl + (uint32_t)j, bB2 + (uint32_t)(i * FW + j) * TAP_B2, idescbf);
          }
          tc_commit(tfull + acc);
        }
        __syncwarp();
        issued = true;
        qs = sl[1];
        qph = ph[1];
        if (++acc == TC_MAX_ACC) { acc = 0; aph ^= 1; }
      }
      for (int rr = ho; rr < job.H; ++rr)  // rows never first of an output row
        if (++qs == ring) { qs = 0; qph ^= 1; }
    }
  } else if (warp <= PRODUCERS) {
    // =================== producers ===================
    // warp p stages rows q = p, p + 4, ...: per position 16 ranks as four tf32
    // hi quads and two 8-rank bf16 lo planes, in two halves of 8 ranks (all
    // of a half's loads in flight before converting)
    const int pw = warp - 1;
    uint32_t q_glob = 0;
    for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
      const dpm_corr_tile strip = a.strips[st];
      const dpm_corr_job job = a.jobs[strip.job];
      const int x0 = strip.tx * TC_M;
      const int64_t plane = (int64_t)job.H * job.pitch;
      const float* pbase = a.P + job.p_off + (int64_t)job.chan_off * plane;
      for (int q = pw; q < job.H; q += PRODUCERS) {
        const uint32_t qg = q_glob + q;
        const uint32_t slot = qg % ring;
        mbar_wait(empty + slot, ((qg / ring) & 1) ^ 1);
        float4* hi = reinterpret_cast<float4*>(sA + slot * SLOT_BYTES);
        uint4* lo16 = reinterpret_cast<uint4*>(sA + slot * SLOT_BYTES + HI_BYTES);
        const float* prow = pbase + (int64_t)q * job.pitch;
        constexpr int PP = (TCOLS + 31) / 32;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float v8[PP][8];
#pragma unroll
          for (int k = 0; k < PP; ++k) {
            const int c = lane + 32 * k, x = x0 + c;
            const bool ok = c < TCOLS && x < job.W;
#pragma unroll
            for (int r = 0; r < 8; ++r)
              v8[k][r] = ok ? __ldg(prow + (int64_t)(8 * hh + r) * plane + x) : 0.f;
          }
#pragma unroll
          for (int k = 0; k < PP; ++k) {
            const int c = lane + 32 * k;
            if (c >= TCOLS) continue;
            float h8[8], l8[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              h8[r] = tf32_hi(v8[k][r]);
              l8[r] = v8[k][r] - h8[r];
            }
            hi[(2 * hh) * TCOLS + c] = make_float4(h8[0], h8[1], h8[2], h8[3]);
            hi[(2 * hh + 1) * TCOLS + c] = make_float4(h8[4], h8[5], h8[6], h8[7]);
            lo16[hh * (TCOLS + 1) + c] =
                make_uint4(bf16x2_rn(l8[0], l8[1]), bf16x2_rn(l8[2], l8[3]),
                           bf16x2_rn(l8[4], l8[5]), bf16x2_rn(l8[6], l8[7]));
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(full + slot);
      }
      q_glob += job.H;
    }
  } else {
    // =================== epilogue ===================
    const int quarter = warp & 3;  // TMEM lanes 32 * quarter ..
    const bool releaser = warp == 1 + PRODUCERS && lane == 0;
    uint32_t eslot = 0;
    auto release = [&](int nrows) {
      for (int k = 0; k < nrows; ++k) {
        if (releaser) mbar_arrive(empty + eslot);
        if (++eslot == ring) eslot = 0;
      }
    };
    uint32_t row_glob = 0;
    for (int st = blockIdx.x; st < a.nstrips; st += gridDim.x) {
      const dpm_corr_tile strip = a.strips[st];
      const dpm_corr_job job = a.jobs[strip.job];
      const int ho = job.H - FH + 1, wo = job.W - FW + 1, wp = s_pitch(wo);
      const int x = strip.tx * TC_M + quarter * 32 + lane;
      const int64_t plane = (int64_t)ho * wp;
      const bool xin = x < wo;
      float vmax[N], vmin[N];
#pragma unroll
      for (int f = 0; f < N; ++f) { vmax[f] = -INFINITY; vmin[f] = INFINITY; }
      for (int y = 0; y < ho; ++y, ++row_glob) {
        const uint32_t b = row_glob & (TC_MAX_ACC - 1);
        mbar_wait(tfull + b, (row_glob / TC_MAX_ACC) & 1);
        tc_fence_after();
        release(1);  // input row y: no later output row reads it
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + b * (uint32_t)ACC_COLS;
        float vh[N], vl[N];
        tmem_ld16(taddr, vh);
        tmem_ld16(taddr + N, vl);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + b);  // accumulator drained
        float* dst = a.S + job.s_off + (int64_t)y * wp + x;
#pragma unroll
        for (int f = 0; f < N; ++f) {
          if (f < job.nf && xin) {
            const float sv = vh[f] + vl[f];
            dst[(int64_t)f * plane] = sv;
            vmax[f] = fmaxf(vmax[f], sv);
            vmin[f] = fminf(vmin[f], sv);
          }
        }
      }
      release(job.H - ho);  // rows never first of an output row
      if (a.ranges != nullptr && job.range_idx >= 0) {
#pragma unroll
        for (int f = 0; f < N; ++f) {
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
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(128));
}

}  // namespace tc16

bool tc16_shape(int h, int w, int R, int N) { return h == 6 && w == 6 && R == 16 && N == 16; }

size_t tc16_core_floats() { return (tc16::B_BYTES + tc16::B2_BYTES) / 4; }

size_t tc16_smem(int* ring_out) {
  int ring = TC_MAX_RING;
  while (ring > tc16::FH + 2 && tc16::FIXED + (size_t)ring * tc16::SLOT_BYTES > 227 * 1024) --ring;
  if (ring_out) *ring_out = ring;
  return tc16::FIXED + (size_t)ring * tc16::SLOT_BYTES;
}

int launch_tc16(TcArgs a, cudaStream_t stream) {
  int ring = 0;
  const size_t smem = tc16_smem(&ring);
  DPM_REQUIRE(smem <= 227 * 1024, "dpm_correlate_tc (R = 16): needs %zu B shared memory", smem);
  a.ring = ring;
  DPM_CUDA(cudaFuncSetAttribute(tc16::corr_tc16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  int dev = 0, sms = 148;
  DPM_CUDA(cudaGetDevice(&dev));
  DPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = a.nstrips < sms ? a.nstrips : sms;
  tc16::corr_tc16_kernel<<<grid, tc16::THREADS, smem, stream>>>(a);
  DPM_LAUNCHED("corr_tc16_kernel");
  return DPM_OK;
}

}  // namespace dpm
