// direct_conv.cu -- CUDA-core direct conv2d (fp32 accumulate) for sm_100a.
//
// Computes the same operator as igemm_tc ("2D convolution",
// P:388 ReLU; SURVEY 8(a) a7 + a9) for the layers the tensor-core path does
// not take: every fp32 layer (north_star's 1e-5 path -- FFMA only, reading C8:
// no TF32), depthwise layers (g = C, MobileNet's even ops) and
// small-channel stems (C < 8).
//
// Schedule knobs: threads per CTA, tile_q (outputs per thread along
// Q), vec_k (output channels per thread), tile_p (output rows per CTA) and
// smem_stage (stage the input halo + weights in shared memory, "caching").
// Thread layout: tid = tk + lanes_k * (tq + lanes_q * tp); lanes_k is a power
// of two so consecutive lanes own consecutive channel vectors (coalesced NHWC
// stores).  Each thread keeps a tile_q x vec_k fp32 accumulator in registers.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "tp_kernels.h"

namespace tp {

template <typename T>
__device__ __forceinline__ float ld_f(const T* p);
template <>
__device__ __forceinline__ float ld_f<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }

// Load VK consecutive elements (16-byte aligned when VK * sizeof(T) >= 16 and
// the start is a multiple of VK; guaranteed for depthwise by C % vec_k == 0).
template <typename T, int VK>
__device__ __forceinline__ void ld_vec(const T* p, float (&o)[VK]) {
  if constexpr (sizeof(T) == 4 && VK % 4 == 0) {
#pragma unroll
    for (int j = 0; j < VK; j += 4) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(p + j));
      o[j] = f.x; o[j + 1] = f.y; o[j + 2] = f.z; o[j + 3] = f.w;
    }
  } else if constexpr (sizeof(T) == 2 && VK == 8) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) { const float2 f = __bfloat1622float2(b[j]); o[2 * j] = f.x; o[2 * j + 1] = f.y; }
  } else {
#pragma unroll
    for (int j = 0; j < VK; ++j) o[j] = ld_f<T>(p + j);
  }
}

__device__ __forceinline__ void st_out(void* y, int64_t off, float v, int out_f32) {
  if (out_f32) reinterpret_cast<float*>(y)[off] = v;
  else reinterpret_cast<__nv_bfloat16*>(y)[off] = __float2bfloat16_rn(v);
}

// Depthwise 3x3, compile-time stride: the 3 x VK weights of a filter row and
// the (TQ-1)*SW+3 input columns of an input row are loaded once per row, with
// every load of the row issued before the FMAs (one memory latency per filter
// row instead of one per tap).
template <typename T, int TQ, int VK, int SW>
__device__ __forceinline__ void dw3x3_rows(const DirectArgs& a, const T* __restrict__ x, const T* __restrict__ w,
                                           int n, int p, int q0, int k0, float (&acc)[TQ][VK]) {
  constexpr int NC = (TQ - 1) * SW + 3;
  const int H = a.H, W = a.W, C = a.C;
  const int wbase = q0 * SW - a.pw;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int hi = p * a.sh - a.ph + r;
    if ((unsigned)hi >= (unsigned)H) continue;
    const T* xrow = x + ((int64_t)n * H + hi) * W * C + k0;
    float wv[3][VK];
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
      for (int j = 0; j < VK; ++j) wv[s][j] = ld_f<T>(w + (int64_t)(k0 + j) * 9 + r * 3 + s);
    float xc[NC][VK];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int wi = wbase + c;
      if ((unsigned)wi < (unsigned)W) {
        ld_vec<T, VK>(xrow + (int64_t)wi * C, xc[c]);
      } else {
#pragma unroll
        for (int j = 0; j < VK; ++j) xc[c][j] = 0.0f;
      }
    }
#pragma unroll
    for (int i = 0; i < TQ; ++i)
#pragma unroll
      for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int j = 0; j < VK; ++j) acc[i][j] = fmaf(xc[i * SW + s][j], wv[s][j], acc[i][j]);
  }
}

template <typename T, int TQ, int VK, bool DW, bool SMEM>
__global__ void __launch_bounds__(512) direct_conv_kernel(DirectArgs a) {
  extern __shared__ float dsm[];
  const int tid = threadIdx.x;
  const int tk = tid & (a.lanes_k - 1);
  const int tq = (tid / a.lanes_k) % a.lanes_q;
  const int tp = tid / (a.lanes_k * a.lanes_q);
  const int QT = a.lanes_q * TQ, KT = a.lanes_k * VK;
  const int qb = blockIdx.x % a.n_qb, pb = blockIdx.x / a.n_qb;
  const int n = blockIdx.z;
  const int p = pb * a.tile_p + tp;
  const int q0 = qb * QT + tq * TQ;
  const int k0 = blockIdx.y * KT + tk * VK;
  const T* __restrict__ x = reinterpret_cast<const T*>(a.x);
  const T* __restrict__ w = reinterpret_cast<const T*>(a.w);
  const int C = a.C, H = a.H, W = a.W, K = a.K, R = a.R, S = a.S;
  // Programmatic dependent launch: let the next kernel get scheduled, and wait
  // for the previous one before reading memory.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  float acc[TQ][VK];
#pragma unroll
  for (int i = 0; i < TQ; ++i)
#pragma unroll
    for (int j = 0; j < VK; ++j) acc[i][j] = 0.0f;

  // Depthwise 3x3 with stride 1 or 2 (every MobileNet depthwise layer): the
  // unrolled row-at-a-time path.
  const bool dw33 = DW && !SMEM && R == 3 && S == 3 && (a.sw == 1 || a.sw == 2);
  if (dw33) {
    if (p < a.P && k0 < K) {
      if (a.sw == 1) dw3x3_rows<T, TQ, VK, 1>(a, x, w, n, p, q0, k0, acc);
      else dw3x3_rows<T, TQ, VK, 2>(a, x, w, n, p, q0, k0, acc);
    }
  } else if constexpr (!SMEM) {
    if (p < a.P) {
      for (int r = 0; r < R; ++r) {
        const int hi = p * a.sh - a.ph + r;
        if (hi < 0 || hi >= H) continue;
        const T* xrow = x + ((int64_t)n * H + hi) * W * C;
        for (int s = 0; s < S; ++s) {
          int wi[TQ];
          bool ok[TQ];
#pragma unroll
          for (int i = 0; i < TQ; ++i) {
            wi[i] = (q0 + i) * a.sw - a.pw + s;
            ok[i] = (q0 + i) < a.Q && wi[i] >= 0 && wi[i] < W;
          }
          if constexpr (DW) {
            if (k0 < K) {
              float wv[VK];
#pragma unroll
              for (int j = 0; j < VK; ++j) wv[j] = ld_f<T>(w + ((int64_t)(k0 + j) * R + r) * S + s);
#pragma unroll
              for (int i = 0; i < TQ; ++i) {
                if (!ok[i]) continue;
                float xv[VK];
                ld_vec<T, VK>(xrow + (int64_t)wi[i] * C + k0, xv);
#pragma unroll
                for (int j = 0; j < VK; ++j) acc[i][j] = fmaf(xv[j], wv[j], acc[i][j]);
              }
            }
          } else {
            for (int c = 0; c < C; ++c) {
              float xv[TQ], wv[VK];
#pragma unroll
              for (int i = 0; i < TQ; ++i) xv[i] = ok[i] ? ld_f<T>(xrow + (int64_t)wi[i] * C + c) : 0.0f;
#pragma unroll
              for (int j = 0; j < VK; ++j)
                wv[j] = (k0 + j < K) ? ld_f<T>(w + (((int64_t)(k0 + j) * R + r) * S + s) * C + c) : 0.0f;
#pragma unroll
              for (int i = 0; i < TQ; ++i)
#pragma unroll
                for (int j = 0; j < VK; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);
            }
          }
        }
      }
    }
  } else {
    const int rows_in = (a.tile_p - 1) * a.sh + R;
    const int cols_in = (QT - 1) * a.sw + S;
    const int h_base = pb * a.tile_p * a.sh - a.ph;
    const int w_base = qb * QT * a.sw - a.pw;
    const int k_base = blockIdx.y * KT;
    const int nthr = blockDim.x;
    if constexpr (DW) {
      // xs[rows_in][cols_in][KT], ws[R][S][KT]
      float* xs = dsm;
      float* wsm = dsm + rows_in * cols_in * KT;
      const int nx = rows_in * cols_in * KT;
      for (int e = tid; e < nx; e += nthr) {
        const int kt = e % KT, t = e / KT, col = t % cols_in, row = t / cols_in;
        const int hi = h_base + row, wi = w_base + col, k = k_base + kt;
        xs[e] = (hi >= 0 && hi < H && wi >= 0 && wi < W && k < K)
                    ? ld_f<T>(x + (((int64_t)n * H + hi) * W + wi) * C + k) : 0.0f;
      }
      for (int e = tid; e < R * S * KT; e += nthr) {
        const int kt = e % KT, rs = e / KT, k = k_base + kt;
        wsm[e] = k < K ? ld_f<T>(w + (int64_t)k * R * S + rs) : 0.0f;
      }
      __syncthreads();
      if (p < a.P) {
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s) {
            float wv[VK];
#pragma unroll
            for (int j = 0; j < VK; ++j) wv[j] = wsm[(r * S + s) * KT + tk * VK + j];
#pragma unroll
            for (int i = 0; i < TQ; ++i) {
              const float* xp = xs + ((tp * a.sh + r) * cols_in + (tq * TQ + i) * a.sw + s) * KT + tk * VK;
#pragma unroll
              for (int j = 0; j < VK; ++j) acc[i][j] = fmaf(xp[j], wv[j], acc[i][j]);
            }
          }
      }
    } else {
      // per channel chunk: xs[rows_in][cols_in][CC], ws[R][S][CC][KT]
      const int CC = a.cc;
      float* xs = dsm;
      float* wsm = dsm + rows_in * cols_in * CC;
      for (int c0 = 0; c0 < C; c0 += CC) {
        const int ccn = min(CC, C - c0);
        const int nx = rows_in * cols_in * CC;
        for (int e = tid; e < nx; e += nthr) {
          const int cc = e % CC, t = e / CC, col = t % cols_in, row = t / cols_in;
          const int hi = h_base + row, wi = w_base + col;
          xs[e] = (cc < ccn && hi >= 0 && hi < H && wi >= 0 && wi < W)
                      ? ld_f<T>(x + (((int64_t)n * H + hi) * W + wi) * C + c0 + cc) : 0.0f;
        }
        const int nw = R * S * CC * KT;
        for (int e = tid; e < nw; e += nthr) {   // read order: cc fastest (contiguous in KRSC)
          const int cc = e % CC, t = e / CC, s = t % S, t2 = t / S, r = t2 % R, kt = t2 / R;
          const int k = k_base + kt;
          wsm[((r * S + s) * CC + cc) * KT + kt] =
              (cc < ccn && k < K) ? ld_f<T>(w + (((int64_t)k * R + r) * S + s) * C + c0 + cc) : 0.0f;
        }
        __syncthreads();
        if (p < a.P) {
          for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) {
              const float* xb = xs + ((tp * a.sh + r) * cols_in + tq * TQ * a.sw + s) * CC;
              const float* wb = wsm + (r * S + s) * CC * KT + tk * VK;
              for (int cc = 0; cc < ccn; ++cc) {
                float xv[TQ], wv[VK];
#pragma unroll
                for (int i = 0; i < TQ; ++i) xv[i] = xb[i * a.sw * CC + cc];
#pragma unroll
                for (int j = 0; j < VK; ++j) wv[j] = wb[cc * KT + j];
#pragma unroll
                for (int i = 0; i < TQ; ++i)
#pragma unroll
                  for (int j = 0; j < VK; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);
              }
            }
        }
        __syncthreads();
      }
    }
  }

  if (p >= a.P) return;
#pragma unroll
  for (int i = 0; i < TQ; ++i) {
    const int q = q0 + i;
    if (q >= a.Q) continue;
    const int64_t base = (((int64_t)n * a.P + p) * a.Q + q) * K;
#pragma unroll
    for (int j = 0; j < VK; ++j) {
      const int k = k0 + j;
      if (k >= K) continue;
      float v = acc[i][j];
      if (a.has_bias) v += __ldg(a.bias + k);
      if (a.relu) v = fmaxf(v, 0.0f);
      st_out(a.y, base + k, v, a.out_f32);
    }
  }
}

// ------------------------------------------------------------- dispatch
using DirectFn = void (*)(DirectArgs);

template <typename T, int TQ, int VK>
static DirectFn pick3(bool dw, bool sm) {
  if (dw) return sm ? direct_conv_kernel<T, TQ, VK, true, true> : direct_conv_kernel<T, TQ, VK, true, false>;
  return sm ? direct_conv_kernel<T, TQ, VK, false, true> : direct_conv_kernel<T, TQ, VK, false, false>;
}
template <typename T, int TQ>
static DirectFn pick2(int vk, bool dw, bool sm) {
  switch (vk) {
    case 1: return pick3<T, TQ, 1>(dw, sm);
    case 2: return pick3<T, TQ, 2>(dw, sm);
    case 4: return pick3<T, TQ, 4>(dw, sm);
    case 8: return pick3<T, TQ, 8>(dw, sm);
  }
  return nullptr;
}
template <typename T>
static DirectFn pick1(int tq, int vk, bool dw, bool sm) {
  switch (tq) {
    case 1: return pick2<T, 1>(vk, dw, sm);
    case 2: return pick2<T, 2>(vk, dw, sm);
    case 4: return pick2<T, 4>(vk, dw, sm);
  }
  return nullptr;
}

tp_status direct_prepare(const Layer& L, const tp_schedule& s, const void* x, const void* w, const float* bias,
                         void* y, DirectPlan* plan) {
  DirectArgs& a = plan->args;
  const tp_conv_desc& d = L.d;
  a.x = x; a.w = w; a.bias = bias; a.y = y;
  a.N = d.n; a.C = d.c; a.H = d.h; a.W = d.w; a.K = d.k; a.R = d.r; a.S = d.s;
  a.sh = d.stride_h; a.sw = d.stride_w; a.ph = d.pad_h; a.pw = d.pad_w; a.P = L.P; a.Q = L.Q;
  a.tile_p = s.tile_p;
  direct_lanes(L, s.threads, s.tile_q, s.vec_k, s.tile_p, &a.lanes_k, &a.lanes_q);
  a.n_qb = (int)cdiv(L.Q, (int64_t)a.lanes_q * s.tile_q);
  a.cc = d.c < 16 ? d.c : 16;
  a.relu = (d.epilogue & TP_EPI_RELU) ? 1 : 0;
  a.has_bias = (d.epilogue & TP_EPI_BIAS) ? 1 : 0;
  a.out_f32 = d.out_dtype == TP_DTYPE_FP32;
  const bool dw = L.depthwise, sm = s.smem_stage != 0;
  DirectFn fn = d.dtype == TP_DTYPE_FP32 ? pick1<float>(s.tile_q, s.vec_k, dw, sm)
                                         : pick1<__nv_bfloat16>(s.tile_q, s.vec_k, dw, sm);
  if (!fn) { set_error("no direct_conv instantiation for this schedule"); return TP_EINVALID_CONFIG; }
  plan->fn = reinterpret_cast<const void*>(fn);
  tp_schedule g = s;
  if (!g.grid_x) fill_geometry(L, &g);
  plan->grid = dim3(g.grid_x, g.grid_y, g.grid_z);
  plan->block = dim3(s.threads);
  plan->smem = sm ? (size_t)direct_smem_bytes(L, s.threads, s.tile_q, s.vec_k, s.tile_p) : 0;
  if (plan->smem > 48 * 1024) {
    cudaError_t e = ensure_smem_attr(plan->fn, plan->smem);
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return TP_ECUDA;
    }
  }
  return TP_OK;
}

cudaError_t direct_launch(const DirectPlan& plan, cudaStream_t stream) {
  DirectFn fn = reinterpret_cast<DirectFn>(const_cast<void*>(plan.fn));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = plan.grid;
  cfg.blockDim = plan.block;
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, plan.args);
}

int direct_occupancy(const DirectPlan& plan) {
  return cached_occupancy(plan.fn, plan.block.x, plan.smem);
}

}  // namespace tp
