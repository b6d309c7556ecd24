// Micro-benchmark: period of a chain of dependent launches (PDL, one CUDA graph)
// for kernels that add, one at a time, the fixed parts of a batch-1 conv launch:
//   0 empty                         1 + griddepcontrol.wait / launch_dependents
//   2 + tcgen05.alloc/dealloc       3 + 8 KB of y stores per CTA
//   4 + a 4 KB global read per CTA  5 = 2 + 3 + 4 (all of them)
//   6 = 5 with the TMEM allocation before the PDL wait (as the conv kernels do)
//   7 = 6 with the dealloc before the y stores
//   8 = 5 with alloc and dealloc both before the PDL wait (TMEM not held in the body)
//   9 = 5 with the dealloc before the y stores
//  10 = 3 with the 8 KB written by one bulk copy (cp.async.bulk smem -> global), wait_group.read
//  11 = 10 with wait_group 0 (writes complete) before the exit
//  12 = 3 with 2 KB per CTA, 13 = 3 with 32 KB per CTA
//  P  = 1 with a 1 KB __grid_constant__ parameter block (the conv kernels pass ~0.9 KB)
// usage: launch_gap [ctas=100] [threads=256]     Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o launch_gap launch_gap.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int V>
__global__ void __launch_bounds__(256) k(const uint4* __restrict__ x, uint4* __restrict__ y) {
  __shared__ uint32_t slot;
  __shared__ __align__(128) uint4 stg[512];
  const bool tmem = V == 2 || V == 5 || V == 6 || V == 7 || V == 9;
  if ((V == 6 || V == 7 || V == 8) && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (V == 8) {
    __syncwarp();
    if (threadIdx.x < 32) {
      const uint32_t base = slot;
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(base) : "memory");
    }
  }
  if (V >= 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if ((V == 2 || V == 5 || V == 9) && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  uint4 acc = make_uint4(0, 0, 0, 0);
  if (V >= 4) {   // 4 KB per CTA: 256 threads x 16 B
    acc = x[(size_t)blockIdx.x * blockDim.x + threadIdx.x];
  }
  __syncthreads();
  if ((V == 7 || V == 9) && threadIdx.x < 32) {
    const uint32_t base = slot;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(base) : "memory");
  }
  if (V == 10 || V == 11) {
    stg[threadIdx.x] = acc;
    stg[threadIdx.x + blockDim.x] = acc;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      uint4* yp = y + (size_t)blockIdx.x * blockDim.x * 2;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 8192;" ::"l"(yp), "r"(su32(stg)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (V == 10) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  if (V == 12) {   // 2 KB per CTA
    if (threadIdx.x < 128) y[(size_t)blockIdx.x * 128 + threadIdx.x] = acc;
  }
  if (V == 13) {   // 32 KB per CTA
    uint4* yp = y + (size_t)blockIdx.x * blockDim.x * 8;
    for (int j = 0; j < 8; ++j) yp[threadIdx.x + j * blockDim.x] = acc;
  }
  if (V == 3 || (V >= 5 && V <= 9)) {   // 8 KB per CTA
    uint4* yp = y + (size_t)blockIdx.x * blockDim.x * 2;
    yp[threadIdx.x] = acc;
    yp[threadIdx.x + blockDim.x] = acc;
  }
  if (tmem && V != 7 && V != 9) {
    __syncthreads();
    if (threadIdx.x < 32) {
      const uint32_t base = slot;
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(base) : "memory");
    }
  }
}

struct Big { unsigned char b[1024]; };

__global__ void __launch_bounds__(256) kbig(const __grid_constant__ Big p, uint4* __restrict__ y) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.b[threadIdx.x] == 0xAB && threadIdx.x == 1023) y[0] = make_uint4(1, 1, 1, 1);
}

static float period_big(int ctas, int threads, uint4* y, cudaStream_t st, int n) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  Big p = {};
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, kbig, p, y);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return best * 1000.0f / n;
}

template <int V>
static float period(int ctas, int threads, const uint4* x, uint4* y, cudaStream_t st, int n) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = V >= 1 ? 1 : 0;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k<V>, x, y);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return best * 1000.0f / n;
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 100, threads = argc > 2 ? atoi(argv[2]) : 256;
  uint4 *x, *y;
  cudaMalloc(&x, (size_t)ctas * threads * 16);
  cudaMalloc(&y, (size_t)ctas * threads * 128);
  cudaMemset(x, 0, (size_t)ctas * threads * 16);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int n = 200;
  printf("ctas %d threads %d: us per launch in a chain of %d\n", ctas, threads, n);
  printf("0 empty                 %.3f\n", period<0>(ctas, threads, x, y, st, n));
  printf("1 + PDL wait/trigger    %.3f\n", period<1>(ctas, threads, x, y, st, n));
  printf("2 + TMEM alloc/dealloc  %.3f\n", period<2>(ctas, threads, x, y, st, n));
  printf("3 + 8 KB stores / CTA   %.3f\n", period<3>(ctas, threads, x, y, st, n));
  printf("4 + 4 KB load / CTA     %.3f\n", period<4>(ctas, threads, x, y, st, n));
  printf("5 = 2 + 3 + 4           %.3f\n", period<5>(ctas, threads, x, y, st, n));
  printf("6 = 5, alloc before wait %.3f\n", period<6>(ctas, threads, x, y, st, n));
  printf("7 = 6, dealloc early    %.3f\n", period<7>(ctas, threads, x, y, st, n));
  printf("8 = TMEM before wait only %.3f\n", period<8>(ctas, threads, x, y, st, n));
  printf("9 = 5, dealloc early    %.3f\n", period<9>(ctas, threads, x, y, st, n));
  printf("10 = 8 KB bulk, read    %.3f\n", period<10>(ctas, threads, x, y, st, n));
  printf("11 = 8 KB bulk, done    %.3f\n", period<11>(ctas, threads, x, y, st, n));
  printf("12 = 2 KB stores        %.3f\n", period<12>(ctas, threads, x, y, st, n));
  printf("13 = 32 KB stores       %.3f\n", period<13>(ctas, threads, x, y, st, n));
  printf("P = 1 + 1 KB params     %.3f\n", period_big(ctas, threads, y, st, n));
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
