// Micro-benchmark: latency of TMA tiled loads (box = 64 bf16 x ROWS rows) vs row pitch,
// number of loads in flight, L2-warm vs first touch.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_latency tma_latency.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void warm(const uint4* p, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    acc.x ^= v.x;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

// One CTA per SM (grid = ctas): thread 0 issues `nops` loads (consecutive row blocks), waits, records cycles.
__global__ void probe(const __grid_constant__ CUtensorMap tm, int rows, int nops, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm) : "memory");
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    long long t0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(nops * rows * 128)
                 : "memory");
    for (int i = 0; i < nops; ++i) {
      int row0 = ((blockIdx.x * nops + i) * rows) % 4096;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(su32(smem + i * rows * 128)), "l"((uint64_t)&tm), "r"(0), "r"(row0), "r"(su32(&bar))
          : "memory");
    }
    long long t1 = clock64();
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            su32(&bar)),
        "r"(phase)
        : "memory");
    phase ^= 1;
    long long t2 = clock64();
    if (blockIdx.x == 0 && rep < 4) { out[rep * 2] = t1 - t0; out[rep * 2 + 1] = t2 - t0; }
  }
}

int main() {
  const size_t bytes = 64ull << 20;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  uint4* sink;
  cudaMalloc(&sink, 16);
  long long* d_out;
  cudaMalloc(&d_out, 64 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("pitch_B rows nops ctas | issue_cyc  land_cyc(first) land_cyc(rep2,rep3)\n");
  for (int pitch : {128, 256, 2048, 9216}) {
    for (int rows : {32, 64}) {
      for (int nops : {1, 4, 8}) {
        for (int ctas : {1, 64, 148}) {
          if (nops * rows * 128 > 190 * 1024) continue;
          CUtensorMap tm;
          cuuint64_t dims[2] = {(cuuint64_t)(pitch / 2), 4096 + 64 * 8};
          cuuint64_t strides[1] = {(cuuint64_t)pitch};
          cuuint32_t box[2] = {64, (cuuint32_t)rows};
          cuuint32_t es[2] = {1, 1};
          if (pitch < 128) continue;
          if ((size_t)pitch * dims[1] > bytes) continue;
          CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
          warm<<<296, 512>>>((const uint4*)buf, (size_t)pitch * dims[1] / 16, sink);
          probe<<<ctas, 32, nops * rows * 128>>>(tm, rows, nops, 4, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          long long h[8];
          cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
          printf("%7d %4d %4d %4d | %6lld %8lld %8lld %8lld %s\n", pitch, rows, nops, ctas, h[0], h[1], h[3], h[5],
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
      }
    }
  }
  return 0;
}
