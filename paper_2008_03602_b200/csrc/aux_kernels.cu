// aux_kernels.cu -- support kernels of the hot path (
// 2.3 K7): layout transposes (NCHW <-> NHWC pre/post pass, reading C6),
// operand packing (fp32 -> bf16 RNE, KCRS -> KRSC), the sampled-output gather
// of the correctness gate, the %smid partition probe, a STREAM-copy kernel
// for the per-partition HBM roofline and an L2 flush for cold-cache timing.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <algorithm>
#include <cstdint>

#include "tp_kernels.h"

namespace tp {

// 32x32 tiled transpose of [N][A][B] -> [N][B][A] on 2- or 4-byte elements.
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ src, T* __restrict__ dst, int A, int B) {
  __shared__ T tile[32][33];
  const int n = blockIdx.z;
  const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
  const T* s = src + (int64_t)n * A * B;
  T* d = dst + (int64_t)n * A * B;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int a = a0 + i, b = b0 + threadIdx.x;
    if (a < A && b < B) tile[i][threadIdx.x] = s[(int64_t)a * B + b];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int b = b0 + i, a = a0 + threadIdx.x;
    if (a < A && b < B) d[(int64_t)b * A + a] = tile[threadIdx.x][i];
  }
}

template <typename T>
static cudaError_t transpose(const void* src, void* dst, int N, int A, int B, cudaStream_t st) {
  dim3 grid((B + 31) / 32, (A + 31) / 32, N), block(32, 8);
  transpose_kernel<T><<<grid, block, 0, st>>>(reinterpret_cast<const T*>(src), reinterpret_cast<T*>(dst), A, B);
  return cudaGetLastError();
}

cudaError_t launch_nchw_to_nhwc(const void* src, void* dst, int N, int C, int H, int W, int eb, cudaStream_t st) {
  return eb == 2 ? transpose<uint16_t>(src, dst, N, C, H * W, st) : transpose<uint32_t>(src, dst, N, C, H * W, st);
}
cudaError_t launch_nhwc_to_nchw(const void* src, void* dst, int N, int C, int H, int W, int eb, cudaStream_t st) {
  return eb == 2 ? transpose<uint16_t>(src, dst, N, H * W, C, st) : transpose<uint32_t>(src, dst, N, H * W, C, st);
}

// fp32 NCHW -> (NHWC | NCHW) x (bf16 RNE | fp32); one thread per output element.
__global__ void pack_input_kernel(const float* __restrict__ x, void* out, int N, int C, int H, int W, int to_nhwc,
                                  int bf16) {
  const int64_t total = (int64_t)N * C * H * W;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t src;
    if (to_nhwc) {
      int64_t t = o;
      const int c = (int)(t % C); t /= C;
      const int w = (int)(t % W); t /= W;
      const int h = (int)(t % H); const int n = (int)(t / H);
      src = (((int64_t)n * C + c) * H + h) * W + w;
    } else {
      src = o;
    }
    const float v = x[src];
    if (bf16) reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(out)[o] = v;
  }
}

// fp32 KCRS -> KRSC in bf16 RNE or fp32.
__global__ void pack_weights_kernel(const float* __restrict__ w, void* out, int K, int Cg, int R, int S, int bf16) {
  const int64_t total = (int64_t)K * Cg * R * S;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = o;
    const int c = (int)(t % Cg); t /= Cg;
    const int s = (int)(t % S); t /= S;
    const int r = (int)(t % R); const int k = (int)(t / R);
    const float v = w[(((int64_t)k * Cg + c) * R + r) * S + s];
    if (bf16) reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(out)[o] = v;
  }
}

cudaError_t launch_pack_input(const float* x, void* out, int N, int C, int H, int W, int to_nhwc, int bf16,
                              cudaStream_t st) {
  const int64_t total = (int64_t)N * C * H * W;
  const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  pack_input_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(x, out, N, C, H, W, to_nhwc, bf16);
  return cudaGetLastError();
}

cudaError_t launch_pack_weights(const float* w, void* out, int K, int Cg, int R, int S, int bf16, cudaStream_t st) {
  const int64_t total = (int64_t)K * Cg * R * S;
  const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  pack_weights_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(w, out, K, Cg, R, S, bf16);
  return cudaGetLastError();
}

// y at flat logical NKPQ indices -> fp64.
__global__ void gather_kernel(const void* y, int nhwc, int out_f32, int N, int K, int P, int Q,
                              const int64_t* __restrict__ idx, int n, double* vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t t = idx[i];
  const int q = (int)(t % Q); t /= Q;
  const int p = (int)(t % P); t /= P;
  const int k = (int)(t % K); const int nn = (int)(t / K);
  const int64_t off = nhwc ? (((int64_t)nn * P + p) * Q + q) * K + k : idx[i];
  vals[i] = out_f32 ? (double)reinterpret_cast<const float*>(y)[off]
                    : (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(y)[off]);
}

cudaError_t launch_gather(const void* y, int nhwc, int out_f32, int N, int K, int P, int Q, const int64_t* idx, int n,
                          double* vals, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  gather_kernel<<<(n + 255) / 256, 256, 0, st>>>(y, nhwc, out_f32, N, K, P, Q, idx, n, vals);
  return cudaGetLastError();
}

// %smid probe: each CTA records the SM it ran on, and lingers briefly so CTAs spread.
__global__ void smid_kernel(int* smids) {
  if (threadIdx.x == 0) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    smids[blockIdx.x] = (int)s;
    const long long t0 = clock64();
    while (clock64() - t0 < 20000) {}
  }
}

cudaError_t launch_smid_probe(int ctas, int* smids, cudaStream_t st) {
  smid_kernel<<<ctas, 32, 0, st>>>(smids);
  return cudaGetLastError();
}

// STREAM copy, 16-byte vectors, grid-stride.
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

cudaError_t launch_copy(const void* src, void* dst, size_t bytes, int grid, cudaStream_t st) {
  copy_kernel<<<grid, 512, 0, st>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), bytes / 16);
  return cudaGetLastError();
}

__global__ void flush_kernel(uint4* buf, size_t n16, uint32_t salt) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_uint4(salt, (uint32_t)i, 0u, 0u);
}

cudaError_t launch_l2_flush(void* buf, size_t bytes, int grid, cudaStream_t st) {
  static uint32_t salt = 0;
  flush_kernel<<<grid, 512, 0, st>>>(reinterpret_cast<uint4*>(buf), bytes / 16, ++salt);
  return cudaGetLastError();
}

// Empty kernel with the same PDL protocol as the conv kernels: the measured
// per-launch floor of the timing protocol (SURVEY 8(d) "empty-kernel floor").
__global__ void empty_kernel(int* sink) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (sink && threadIdx.x == 0 && blockIdx.x == 0x7fffffff) *sink = 1;   // never taken
}

// Strip-kind pre-pass (TP_KIND_IGEMM_TC_STRIP): x NHWC with C <= 8 channels ->
// x8 NHWC with 8 (zero padded, 16-byte pixels); w KRSC -> w8 [R][S][K][8].
// One 16-byte store per pixel / weight row; waits for the producer of x (PDL).
__global__ void pad_c8_kernel(const uint16_t* __restrict__ x, uint4* __restrict__ x8, int64_t npix, int C,
                              const uint16_t* __restrict__ w, uint4* __restrict__ w8, int K, int R, int S) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t nw = (int64_t)K * R * S;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix + nw; i += (int64_t)gridDim.x * blockDim.x) {
    const uint16_t* src;
    uint4* dst;
    if (i < npix) {
      src = x + i * C;
      dst = x8 + i;
    } else {
      const int64_t j = i - npix;                     // (k, r, s) in KRS order
      const int k = (int)(j / (R * S)), rs = (int)(j - (int64_t)k * R * S);
      src = w + j * C;
      dst = w8 + (int64_t)rs * K + k;                 // [r][s][k]
    }
    uint32_t v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = c < C ? src[c] : 0u;
    *dst = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16));
  }
}

cudaError_t launch_pad_c8(const void* x, void* x8, int64_t npix, int C, const void* w, void* w8, int K, int R, int S,
                          int pdl, cudaStream_t st) {
  const int64_t total = npix + (int64_t)K * R * S;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::min<int64_t>((total + 255) / 256, 148 * 8));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, pad_c8_kernel, reinterpret_cast<const uint16_t*>(x), reinterpret_cast<uint4*>(x8),
                            npix, C, reinterpret_cast<const uint16_t*>(w), reinterpret_cast<uint4*>(w8), K, R, S);
}

cudaError_t launch_empty(int ctas, int threads, int pdl, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
}

}  // namespace tp
