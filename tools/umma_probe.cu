// Microbenchmark: cycles per tcgen05.mma (M = 128) by A-operand layout and N.
//
// One CTA per SM; one thread issues `iters` MMAs into one TMEM accumulator,
// commits, waits, and reports clock64 cycles / MMA.  Operand contents are
// irrelevant (timing only).  Modes:
//   0  kind::tf32, A K-major no-swizzle, start shifted 16 B per tap (the
//      K2 kernel's tap shift: core matrices not 128 B aligned)
//   1  kind::tf32, A K-major no-swizzle, start shifted 128 B per tap (aligned)
//   2  kind::tf32, A K-major SWIZZLE_128B, start stepping 32 B (K) in the atom
//   3  kind::f16 (bf16), A no-swizzle with LBO 16 B (the tap-pair correction)
//   4  kind::f16 (bf16), A K-major SWIZZLE_128B
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_probe tools/umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
               : "=r"(pred));
  return pred != 0;
}

template <bool BF>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (BF)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// MODE as above; NACC accumulators rotated (128 TMEM columns apart)
template <int MODE, int NACC>
__global__ void __launch_bounds__(128, 1) probe(int n, int iters, long long* out) {
  constexpr bool BF = MODE >= 3, SW = MODE == 2 || MODE == 4;
  constexpr uint32_t STEP = MODE == 0 ? 1 : MODE == 1 ? 8 : 2;
  constexpr int CYC = SW ? 4 : 6;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  unsigned char* A = sm;               // 96 KB
  unsigned char* B = sm + 96 * 1024;   // 64 KB
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f800000u, 0x3f800000u, 0x3f800000u, 0x3f800000u);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t d = tslot;
  if (threadIdx.x < 32) {  // warp 0 walks the loop (warp-uniform descriptors), one lane issues
    const uint32_t idesc = (1u << 4) | ((BF ? 1u : 2u) << 7) | ((BF ? 1u : 2u) << 10) |
                           ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t a0 = SW ? desc(s32(A), 16u, 1024u, 2)
                      : MODE == 3 ? desc(s32(A), 16u, 128u, 0) : desc(s32(A), 138u * 16u, 128u, 0);
    const uint64_t bdesc = SW ? desc(s32(B), 16u, 1024u, 2) : desc(s32(B), (uint32_t)n * 16u, 128u, 0);
    __syncwarp();
    long long t0 = clock64();
    if (elect_one())
#pragma unroll
      for (int k = 0; k < NACC; ++k) mma<BF>(d + 128u * k, a0, bdesc, idesc, 0u);
    __syncwarp();
    for (int i = 0; i < iters; i += 12) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 12; ++k)
          mma<BF>(d + 128u * (k % NACC), a0 + (uint64_t)((k % CYC) * STEP), bdesc, idesc, 1u);
      }
      __syncwarp();
    }
    if (elect_one()) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       s32(&bar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, P;\n\t}" : "=r"(done) : "r"(s32(&bar)) : "memory");
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
}

// The K2 part kernel's MMA sequence for one output row, replayed without
// producers or epilogue: 6 x 6 tf32 MMAs (N = 96 = [B_hi | B_lo] of 48 filters)
// over 6 ring slots, then 6 x 3 bf16 tap-pair MMAs (N = 48).  Same descriptors,
// strides and smem footprint as corr_tc_kernel<48, 6, 6, 8>.
// extra: 0 none, 1 per-row fence::after_thread_sync, 2 per-row commits (2),
// 3 per-row wait on an already-completed mbarrier + fence, 4 all of them
__global__ void __launch_bounds__(128, 1) parts_row(int rows, int fill, int extra, long long* out) {
  constexpr int N = 48, FH = 6, FW = 6, TCOLS = 128 + FW - 1, RING = 8;
  constexpr uint32_t HI = 2 * TCOLS * 16, SLOT = (HI + (TCOLS + 1) * 16 + 127) & ~127u;
  constexpr uint32_t BB = FH * FW * 2 * (2 * N) * 16, B2 = FH * 3 * 2 * N * 16;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar, bar2[4];
  __shared__ uint32_t tslot;
  unsigned char* sB = sm;
  unsigned char* sB2 = sm + ((BB + 1023) & ~1023u);
  unsigned char* sA = sB2 + ((B2 + 1023) & ~1023u);
  // operand contents: 0 = zeros, 1 = pseudo-random values of HOG / filter magnitude
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 97u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    const float v = fill ? ((float)(h & 0xFFFFFF) / 16777216.0f - 0.5f) * 0.4f : 0.f;
    reinterpret_cast<float*>(sm)[i] = v;
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    for (int k = 0; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar2[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tslot;
  uint32_t dummy_phase = 0;
  if (threadIdx.x < 32) {
    const uint32_t lboA = TCOLS * 16, lboB = 2 * N * 16;
    const uint64_t dA0 = desc(s32(sA), lboA, 128, 0), dB0 = desc(s32(sB), lboB, 128, 0);
    const uint64_t dAlo0 = desc(s32(sA) + HI, 16, 128, 0), dB2 = desc(s32(sB2), N * 16, 128, 0);
    const uint32_t i1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(2 * N >> 3) << 17) | (8u << 24);
    const uint32_t ib = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    long long t0 = clock64();
    for (int y = 0; y < rows; ++y) {
      const uint32_t d = tb + (uint32_t)((y & 3) * 128);
      if (extra == 3 || extra == 4) {  // wait for the commit of 4 rows ago (completes long before)
        if (y >= 4) {
          uint32_t done = 0;
          while (!done)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, P;\n\t}" : "=r"(done) : "r"(s32(&bar2[y & 3])), "r"(((y >> 2) - 1) & 1) : "memory");
        }
      }
      if (extra == 1 || extra >= 3) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint64_t da[FH], dl[FH];
#pragma unroll
      for (int i = 0; i < FH; ++i) {
        da[i] = dA0 + ((y + i) % RING) * (SLOT >> 4);
        dl[i] = dAlo0 + ((y + i) % RING) * (SLOT >> 4);
      }
      if (elect_one()) {
#pragma unroll
        for (int i = 0; i < FH; ++i)
#pragma unroll
          for (int j = 0; j < FW; ++j)
            mma<false>(d, da[i] + (uint32_t)j, dB0 + (uint32_t)((i * FW + j) * 2) * (lboB >> 4), i1,
                       (i | j) != 0);
#pragma unroll
        for (int i = 0; i < FH; ++i)
#pragma unroll
          for (int jp = 0; jp < 3; ++jp)
            mma<true>(d, dl[i] + (uint32_t)(2 * jp), dB2 + (uint32_t)((i * 3 + jp) * (2 * N * 16 >> 4)), ib, 1u);
        if (extra == 2 || extra >= 3) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           s32(&bar2[y & 3])) : "memory");
          if (extra == 2 || extra == 4)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             s32(&bar)) : "memory");
        }
      }
      __syncwarp();
    }
    if (elect_one()) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       s32(&bar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, P;\n\t}" : "=r"(done) : "r"(s32(&bar)) : "memory");
      out[blockIdx.x] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

typedef void (*Probe)(int, int, long long*);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMalloc(&out, sms * sizeof(long long));
  struct Cfg { const char* name; Probe f1, f4; };
  Cfg cfgs[] = {{"tf32 noswz +16B", probe<0, 1>, probe<0, 4>},
                {"tf32 noswz +128B", probe<1, 1>, probe<1, 4>},
                {"tf32 sw128", probe<2, 1>, probe<2, 4>},
                {"bf16 noswz lbo16", probe<3, 1>, probe<3, 4>},
                {"bf16 sw128", probe<4, 1>, probe<4, 4>}};
  const int ns[] = {16, 32, 48, 64, 96, 128, 192, 256};
  const int iters = 4104;
  printf("cycles per MMA (M=128, %d back-to-back MMAs per SM, %d SMs)\n", iters, sms);
  printf("%-24s", "mode \\ N");
  for (int n : ns) printf("%8d", n);
  printf("\n");
  for (const Cfg& c : cfgs) {
    for (int na : {1, 4}) {
      printf("%-18s x%d acc", c.name, na);
      for (int n : ns) {
        Probe f = (na == 4 && n <= 128) ? c.f4 : c.f1;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        f<<<sms, 128, 160 * 1024>>>(n, iters, out);  // warm
        f<<<sms, 128, 160 * 1024>>>(n, iters, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("  error %s\n", cudaGetErrorString(e)); return 1; }
        long long h[256];
        cudaMemcpy(h, out, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%8.1f", (double)mx / iters);
      }
      printf("\n");
    }
  }
  {
    const int rows = 4096;
    for (int extra = 0; extra < 5; ++extra) {
    const int fill = 1;
    cudaFuncSetAttribute(parts_row, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    parts_row<<<sms, 128, 200 * 1024>>>(rows, fill, extra, out);
    parts_row<<<sms, 128, 200 * 1024>>>(rows, fill, extra, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("parts_row error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[256];
    cudaMemcpy(h, out, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const char* ex[] = {"none", "fence::after_thread_sync", "2 commits", "wait(done)+fence+commit",
                        "wait+fence+2 commits"};
    printf("K2 part-kernel MMA sequence, per-row extra = %-26s: %.0f cycles per output row\n",
           ex[extra], (double)mx / rows);
    }
  }
  return 0;
}
