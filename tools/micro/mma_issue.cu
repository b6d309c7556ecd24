// Micro-benchmark: tcgen05.mma issue rate (kind::f16, M = 128, K = 16, N = 64 or
// 128, both operands in shared memory, no-swizzle K-major) from one issuing warp
// vs two warps issuing into separate TMEM accumulators at the same time.
// One CTA per SM; prints cycles per MMA (per issuing warp and aggregate).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_issue mma_issue.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_plain(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  return d;
}

template <int N, bool TS>
__global__ void __launch_bounds__(128) probe(int nmma, int two, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = slot;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const bool issuer = (warp == 1) || (two && warp == 2);
  long long t0 = 0, t1 = 0;
  if (issuer && (threadIdx.x & 31) == 0) {
    const int w = warp - 1;
    const uint32_t a0 = su32(smem), b0 = su32(smem + 32768);
    const uint64_t ad = desc_plain(a0, 16, 128 * 2), bd = desc_plain(b0, 16, 128 * 2);
    const uint32_t d = tbase + (uint32_t)(w * (TS ? 128 : 256));
    const uint32_t at = tbase + 256u + (uint32_t)(w * 64);   // TS: A (128 x 16 bf16) in TMEM columns
    t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint64_t aa = ad + (uint64_t)((i & 3) * 2), bb = bd + (uint64_t)((i & 3) * 2);
      if constexpr (TS)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(at + (uint32_t)((i & 3) * 8)), "l"(bb), "r"(IDESC), "r"(i > 0 ? 1 : 0)
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(aa), "l"(bb), "r"(IDESC), "r"(i > 0 ? 1 : 0)
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[w]))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
            su32(&bar[w]))
        : "memory");
    t1 = clock64();
    out[(blockIdx.x * 2 + w) * 2] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

template <int N, bool TS = false>
static void run(int nmma, int two) {
  long long* d;
  const int ctas = 148;
  cudaMalloc(&d, ctas * 4 * sizeof(long long));
  cudaMemset(d, 0, ctas * 4 * sizeof(long long));
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int r = 0; r < 2; ++r) probe<N, TS><<<ctas, 128, 65536>>>(nmma, two, d);
  cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  int c = 0;
  for (int i = 0; i < ctas * 2; ++i)
    if (h[i * 2] > 0) { s += h[i * 2]; ++c; }
  const double per = s / c / nmma;
  printf("%s N=%3d %s: %.1f cycles per MMA per warp, %.1f per MMA aggregate (%s)\n", TS ? "TS" : "SS", N, two ? "two warps" : "one warp ",
         per, two ? per / 2 : per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64>(512, 0);
  run<64>(512, 1);
  run<128>(512, 0);
  run<128>(512, 1);
  run<64, true>(512, 0);
  run<64, true>(512, 1);
  run<128, true>(512, 0);
  run<128, true>(512, 1);
  return 0;
}
