// Micro-benchmark: issue cost of TMA loads per op -- tiled 2D vs im2col 4D, box rows 32/64/128,
// one vs two issuing warps.  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_issue tma_issue.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: tiled 2D box {64, rows}; mode 1: im2col 4D (C=512, W=H=14) box 64 ch x rows pixels, tap (1,1).
// nwarps issuing warps, each issues nops loads into its own region, own barrier.
__global__ void probe(const __grid_constant__ CUtensorMap tm, int mode, int rows, int nops, int nwarps,
                      long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm) : "memory");
  }
  __syncthreads();
  if (warp >= nwarps || lane != 0) return;
  uint32_t phase = 0;
  for (int rep = 0; rep < 3; ++rep) {
    long long t0 = clock64();
    uint8_t* base = smem + warp * nops * rows * 128;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp])),
                 "r"(nops * rows * 128)
                 : "memory");
    for (int i = 0; i < nops; ++i) {
      const int op = warp * nops + i;
      if (mode == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(base + i * rows * 128)),
            "l"((uint64_t)&tm), "r"((op % 8) * 64), "r"((op / 8) * rows), "r"(su32(&bar[warp]))
            : "memory");
      } else {
        // im2col: coordinates (c, w, h, n) of the window origin; offsets (s, r)
        const int c = (op % 8) * 64;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5}], [%6], {%7, %8};" ::"r"(su32(base + i * rows * 128)),
            "l"((uint64_t)&tm), "r"(c), "r"(-1), "r"(-1), "r"(0), "r"(su32(&bar[warp])), "h"((uint16_t)1),
            "h"((uint16_t)1)
            : "memory");
      }
    }
    long long t1 = clock64();
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            su32(&bar[warp])),
        "r"(phase)
        : "memory");
    phase ^= 1;
    long long t2 = clock64();
    if (blockIdx.x == 0 && rep == 2) { out[warp * 2] = t1 - t0; out[warp * 2 + 1] = t2 - t0; }
  }
}

int main() {
  const int N = 8, H = 14, W = 14, C = 512;
  void* buf;
  cudaMalloc(&buf, 64 << 20);
  cudaMemset(buf, 1, 64 << 20);
  long long* d_out;
  cudaMalloc(&d_out, 64 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("mode rows nops nwarps | issue(w0) land(w0) issue(w1) land(w1)\n");
  for (int mode : {0, 1})
    for (int rows : {32, 64, 128})
      for (int nops : {2, 4, 8})
        for (int nw : {1, 2}) {
          if (nw * nops * rows * 128 > 192 * 1024) continue;
          CUtensorMap tm;
          CUresult r;
          cuuint32_t es4[4] = {1, 1, 1, 1};
          if (mode == 0) {
            cuuint64_t dims[2] = {(cuuint64_t)C, 65536};
            cuuint64_t strides[1] = {(cuuint64_t)C * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)rows};
            r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es4,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          } else {
            cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
            int lower[2] = {-1, -1}, upper[2] = {-1, -1};
            r = cuTensorMapEncodeIm2col(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, lower, upper, 64,
                                        (cuuint32_t)rows, es4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          }
          if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
          cudaMemset(d_out, 0, 64 * 8);
          probe<<<1, 128, nw * nops * rows * 128>>>(tm, mode, rows, nops, nw, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          long long h[4];
          cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
          printf("%4s %4d %4d %6d | %8lld %8lld %8lld %8lld %s\n", mode ? "i2c" : "tile", rows, nops, nw, h[0], h[1],
                 h[2], h[3], e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
  return 0;
}
