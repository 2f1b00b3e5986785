// tcgen05 plumbing shared by the K2 tensor-core kernels (corr_tc.cu: one
// CTA per SM; corr_tc2.cu: CTA pairs on cta_group::2): constants, the
// kernel arguments, mbarrier / TMEM / UMMA descriptor helpers.
#pragma once
#include "common.cuh"

namespace dpm {

constexpr int TC_M = 128;
constexpr int TC_THREADS = 256;
constexpr int TC_PRODUCERS = 3;  // warps 1..3
constexpr int TC_MAX_RING = 16;
constexpr int TC_MAX_ACC = 4;

struct TcArgs {
  const float* P;
  const float* Gtc;  // [h*w][R/4][2N][4] fp32: rows < N hi, rows >= N lo
  float* S;
  const dpm_corr_job* jobs;
  const dpm_corr_tile* strips;  // (job, -, strip index)
  int nstrips;
  int h, w, R, N;               // N: padded filter count (multiple of 16)
  int ring, acc_cols, nacc;
  uint32_t* ranges;
  // several filter groups in one launch (generic-shape kernel only): the
  // float offset in Gtc of the core of each job's group, indexed by job; the
  // MMA warp reloads B whenever a strip's group differs from the resident one
  const int64_t* tc_off;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait for the phase with parity `parity`; traps (instead of hanging the GPU)
// if it has not completed after ~20 s, which can only be a pipeline bug.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (int spin = 0; spin < 2000 && !done; ++spin) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t"
        "}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(10000000u)
        : "memory");
  }
  if (!done) asm volatile("trap;");
}

// global -> shared bulk copy (async proxy), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// K-major, no-swizzle smem matrix descriptor (SM100 UMMA):
// start >> 4 in [0,14), LBO >> 4 in [16,30), SBO >> 4 in [32,46), version 1 at 46.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M rows
// (128; 256 for a cta_group::2 pair).
__host__ __device__ constexpr uint32_t idesc_tf32(int n, int m = TC_M) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// kind::f16 with bf16 A/B, f32 D, K-major, M rows
__host__ __device__ constexpr uint32_t idesc_bf16(int n, int m = TC_M) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t"
      ".reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t"
      "}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ float tf32_hi(float a) {
  return __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
}

// corr_tc2.cu: the part shape (6 x 6 taps, R = 8) on CTA pairs
int launch_tc_pair(const TcArgs& a, cudaStream_t stream);
// corr_tc16.cu: 6 x 6 taps at R = 16, 16 filters per group, multi-group
bool tc16_shape(int h, int w, int R, int N);
size_t tc16_core_floats();
size_t tc16_smem(int* ring_out);
int launch_tc16(TcArgs a, cudaStream_t stream);

// A strip is a 128-column band of one job's output rows, walked top to
// bottom.  tile.pad > 0 makes it a segment: output rows [ty, ty + pad) (the
// planner splits the tall strips of small pyramids this way so that every SM
// gets work); pad == 0 is the whole strip.  Input rows staged for a segment:
// [ty, min(ty + pad + fh - 1, H)).
__device__ __forceinline__ int seg_out_rows(const dpm_corr_tile& st, int ho) {
  return st.pad > 0 ? st.pad : ho;
}
__device__ __forceinline__ int seg_in_rows(const dpm_corr_tile& st, int H, int fh) {
  return st.pad > 0 ? min(st.ty + st.pad + fh - 1, H) - st.ty : H;
}

}  // namespace dpm
