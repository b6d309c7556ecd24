// igemm_tc.cu -- implicit-GEMM conv2d on 5th-gen tensor cores (sm_100a).
//
// What it computes: the "2D convolution" operator the paper tunes (PAPER.md
// P:254) as D[M x K] = sum_k A_im2col[M x (R S C)] * W[K x (R S C)]^T with
// M = N*P*Q output pixels, then bias + ReLU (a9; the "RELU
// operator" of P:388), split-K partial sums reduced in-kernel (a8).
// Schedule knobs ("loop tiles ... CUDA threading"): BM x BN output tile
// (template), BK channel chunk per filter tap, pipeline depth, threads per CTA,
// split-K (runtime).
//
// B200 design:
//  * warp 0 / lane 0: TMA producer.  A tiles come from an im2col-mode tensor
//    map over NHWC x (box = BM consecutive output pixels x BK channels, one
//    filter tap (r, s) per load, conv padding = out-of-bounds zero fill);
//    B tiles from a tiled 4-D map over KRSC weights.  SWIZZLE_{32,64,128}B.
//  * warp 1 / lane 0: tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32)
//    issuer; accumulator in TMEM; tcgen05.commit releases smem stages.
//  * all warps: epilogue tcgen05.ld (32x32b) -> +bias -> ReLU -> bf16/fp32
//    NHWC stores; with split-K the last CTA of a tile sums the fp32 partials
//    in split order (deterministic).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "tp_kernels.h"

namespace tp {

// ------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TP_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_im2col_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c,
                                                   int32_t w, int32_t h, int32_t n, uint16_t off_w,
                                                   uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h)
      : "memory");
}
__device__ __forceinline__ void tma_load_tile_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                 int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor, K-major, swizzled (sm100 format: start>>4
// [0,14), LBO>>4 [16,30) (unused for swizzled K-major, =1), SBO>>4 [32,46) =
// 8 rows * row pitch, version 1 at [46,48), layout type at [61,64)).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t swz_bytes) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(((8u * swz_bytes) >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  const uint64_t layout = swz_bytes == 128 ? 2 : (swz_bytes == 64 ? 4 : 6);
  d |= layout << 61;
  return d;
}

__device__ __forceinline__ float apply_epi(float v, int n, const float* __restrict__ bias, int has_bias,
                                           int relu) {
  if (has_bias) v += __ldg(bias + n);
  if (relu) v = fmaxf(v, 0.0f);
  return v;
}

// Store 16 consecutive output channels [n0, n0+16) of row m.
__device__ __forceinline__ void store16(void* y, int64_t m, int K, int n0, const float (&v)[16], int out_f32) {
  if (out_f32) {
    float* p = reinterpret_cast<float*>(y) + m * K + n0;
#pragma unroll
    for (int g = 0; g < 16; g += 8) {
      if (n0 + g + 8 <= K) {
        reinterpret_cast<float4*>(p + g)[0] = make_float4(v[g], v[g + 1], v[g + 2], v[g + 3]);
        reinterpret_cast<float4*>(p + g)[1] = make_float4(v[g + 4], v[g + 5], v[g + 6], v[g + 7]);
      }
    }
  } else {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(y) + m * K + n0;
#pragma unroll
    for (int g = 0; g < 16; g += 8) {
      if (n0 + g + 8 <= K) {
        uint4 u;
        __nv_bfloat162 b0 = __floats2bfloat162_rn(v[g], v[g + 1]);
        __nv_bfloat162 b1 = __floats2bfloat162_rn(v[g + 2], v[g + 3]);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[g + 4], v[g + 5]);
        __nv_bfloat162 b3 = __floats2bfloat162_rn(v[g + 6], v[g + 7]);
        u.x = *reinterpret_cast<uint32_t*>(&b0);
        u.y = *reinterpret_cast<uint32_t*>(&b1);
        u.z = *reinterpret_cast<uint32_t*>(&b2);
        u.w = *reinterpret_cast<uint32_t*>(&b3);
        *reinterpret_cast<uint4*>(p + g) = u;
      }
    }
  }
}

template <int BM, int BN>
__global__ void __launch_bounds__(256) igemm_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bk = a.bk, stages = a.stages;
  const int sub_k = bk < 64 ? bk : 64;             // channels per swizzle row
  const int nsub = bk / sub_k;                     // 1, or 2 for BK = 128
  const uint32_t swz = (uint32_t)sub_k * 2;        // 32 / 64 / 128 bytes
  const uint32_t a_sub_bytes = BM * sub_k * 2, b_sub_bytes = BN * sub_k * 2;
  const uint32_t a_stage_bytes = a_sub_bytes * nsub, b_stage_bytes = b_sub_bytes * nsub;

  uint8_t* a_tiles = smem_raw;
  uint8_t* b_tiles = a_tiles + (size_t)stages * a_stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(b_tiles + (size_t)stages * b_stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  const int kb0 = (int)(((int64_t)split * a.kblocks) / a.split_k);
  const int kb1 = (int)(((int64_t)(split + 1) * a.kblocks) / a.split_k);
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;

  if (threadIdx.x == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0) __trap();   // swizzle atoms need 1 KiB alignment
    for (int i = 0; i < stages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Output-pixel origin of this M tile -> im2col base coordinate (lower corner = -pad).
  const int64_t m0 = (int64_t)m_tile * BM;
  const int q0 = (int)(m0 % a.Q);
  const int64_t t0 = m0 / a.Q;
  const int p0 = (int)(t0 % a.P);
  const int n0 = (int)(t0 / a.P);
  const int cw = q0 * a.sw - a.pw, ch = p0 * a.sh - a.ph;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(empty + stage, phase ^ 1u);
      mbar_arrive_expect_tx(full + stage, a_stage_bytes + b_stage_bytes);
      const int rs = kb / a.cblocks, cbi = kb - rs * a.cblocks;
      const int r = rs / a.S, s = rs - r * a.S;
      const int c0 = cbi * bk;
      for (int sb = 0; sb < nsub; ++sb) {
        tma_load_im2col_4d(a_tiles + (size_t)stage * a_stage_bytes + sb * a_sub_bytes, &tmA, full + stage,
                           c0 + sb * sub_k, cw, ch, n0, (uint16_t)s, (uint16_t)r);
        tma_load_tile_4d(b_tiles + (size_t)stage * b_stage_bytes + sb * b_sub_bytes, &tmB, full + stage,
                         c0 + sb * sub_k, s, r, n_tile * BN);
      }
      if (++stage == stages) { stage = 0; phase ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread) ----------------
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(full + stage, phase);
      tc_fence_after();
      const uint32_t a_base = smem_u32(a_tiles + (size_t)stage * a_stage_bytes);
      const uint32_t b_base = smem_u32(b_tiles + (size_t)stage * b_stage_bytes);
      for (int kk = 0; kk < bk / 16; ++kk) {
        const int sb = (kk * 16) / sub_k;
        const uint32_t koff = (uint32_t)((kk * 16) % sub_k) * 2;
        const uint64_t ad = make_sdesc(a_base + sb * a_sub_bytes + koff, swz);
        const uint64_t bd = make_sdesc(b_base + sb * b_sub_bytes + koff, swz);
        tc_mma(tmem_base, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
      }
      tc_commit(empty + stage);
      if (++stage == stages) { stage = 0; phase ^= 1u; }
    }
    tc_commit(tmem_full);
  }

  // ---------------- epilogue (all warps) ----------------
  __syncwarp();
  mbar_wait(tmem_full, 0);
  tc_fence_after();
  const int quad = warp & 3, ngroups = blockDim.x >> 7, cgroup = warp >> 2;
  const int cols = BN / ngroups;
  const int row = (BM == 128) ? quad * 32 + lane : quad * 16 + lane;
  const bool row_ok = (BM == 128 || lane < 16);
  const int64_t m = m0 + row;
  const bool m_ok = row_ok && m < a.M;
  const int64_t tile = (int64_t)m_tile * gridDim.y + n_tile;
  const int64_t n_tiles = (int64_t)gridDim.x * gridDim.y;

  for (int c = cgroup * cols; c < (cgroup + 1) * cols; c += 16) {
    uint32_t raw[16];
    tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)c, raw);
    const int nb = n_tile * BN + c;
    if (a.split_k == 1) {
      if (m_ok && nb < a.K) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = nb + i < a.K ? nb + i : a.K - 1;
          v[i] = apply_epi(__uint_as_float(raw[i]), n, a.bias, a.has_bias, a.relu);
        }
        store16(a.y, m, a.K, nb, v, a.out_f32);
      }
    } else if (row_ok) {
      float* part = a.ws_partial + (((int64_t)split * n_tiles + tile) * BM + row) * BN + c;
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        __stcg(reinterpret_cast<float4*>(part + i), make_float4(__uint_as_float(raw[i]), __uint_as_float(raw[i + 1]),
                                                                __uint_as_float(raw[i + 2]),
                                                                __uint_as_float(raw[i + 3])));
    }
  }

  if (a.split_k > 1) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int old = atomicAdd(a.ws_counters + tile, 1);
      *last_flag = (old == a.split_k - 1);
    }
    __syncthreads();
    if (*last_flag) {
      __threadfence();
      for (int c = cgroup * cols; c < (cgroup + 1) * cols; c += 16) {
        const int nb = n_tile * BN + c;
        if (!m_ok || nb >= a.K) continue;
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.0f;
        for (int sp = 0; sp < a.split_k; ++sp) {   // fixed order -> deterministic
          const float* part = a.ws_partial + (((int64_t)sp * n_tiles + tile) * BM + row) * BN + c;
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 f = __ldcg(reinterpret_cast<const float4*>(part + i));
            v[i] += f.x; v[i + 1] += f.y; v[i + 2] += f.z; v[i + 3] += f.w;
          }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = nb + i < a.K ? nb + i : a.K - 1;
          v[i] = apply_epi(v[i], n, a.bias, a.has_bias, a.relu);
        }
        store16(a.y, m, a.K, nb, v, a.out_f32);
      }
      if (threadIdx.x == 0) a.ws_counters[tile] = 0;   // leave the workspace zeroed
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------------------- host side
using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, TcArgs);

static KernelFn pick_tc(int bm, int bn) {
#define TP_TC_CASE(M_, N_) \
  if (bm == M_ && bn == N_) return igemm_tc_kernel<M_, N_>;
  TP_TC_CASE(64, 32) TP_TC_CASE(64, 64) TP_TC_CASE(64, 128) TP_TC_CASE(64, 256)
  TP_TC_CASE(128, 32) TP_TC_CASE(128, 64) TP_TC_CASE(128, 128) TP_TC_CASE(128, 256)
#undef TP_TC_CASE
  return nullptr;
}

size_t tc_dyn_smem(int bm, int bn, int bk, int stages) {
  return (size_t)stages * (bm + bn) * bk * 2 + 1024;
}

tp_status tc_prepare(const TcProblem& pb, TcPlan* plan) {
  const DriverApi& drv = driver();
  const int sub_k = pb.bk < 64 ? pb.bk : 64;
  const CUtensorMapSwizzle swz = sub_k == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                             : (sub_k == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  // A: im2col over NHWC x, dims (C, W, H, N).
  cuuint64_t a_dims[4] = {(cuuint64_t)pb.C, (cuuint64_t)pb.W, (cuuint64_t)pb.H, (cuuint64_t)pb.N};
  cuuint64_t a_strides[3] = {(cuuint64_t)pb.C * 2, (cuuint64_t)pb.W * pb.C * 2, (cuuint64_t)pb.H * pb.W * pb.C * 2};
  int lower[2] = {-pb.pw, -pb.ph};
  int upper[2] = {pb.pw - (pb.S - 1), pb.ph - (pb.R - 1)};
  cuuint32_t a_estr[4] = {1, (cuuint32_t)pb.sw, (cuuint32_t)pb.sh, 1};
  CUresult r = drv.encodeIm2col(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pb.x), a_dims,
                                a_strides, lower, upper, (cuuint32_t)sub_k, (cuuint32_t)pb.bm, a_estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
    return TP_ECUDA;
  }
  // B: tiled over KRSC weights, dims (C, S, R, K).
  cuuint64_t b_dims[4] = {(cuuint64_t)pb.C, (cuuint64_t)pb.S, (cuuint64_t)pb.R, (cuuint64_t)pb.K};
  cuuint64_t b_strides[3] = {(cuuint64_t)pb.C * 2, (cuuint64_t)pb.S * pb.C * 2, (cuuint64_t)pb.R * pb.S * pb.C * 2};
  cuuint32_t b_box[4] = {(cuuint32_t)sub_k, 1, 1, (cuuint32_t)pb.bn};
  cuuint32_t b_estr[4] = {1, 1, 1, 1};
  r = drv.encodeTiled(&plan->tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pb.w), b_dims, b_strides,
                      b_box, b_estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return TP_ECUDA;
  }
  TcArgs& a = plan->args;
  a.M = pb.M; a.K = pb.K; a.P = pb.P; a.Q = pb.Q; a.S = pb.S;
  a.sh = pb.sh; a.sw = pb.sw; a.ph = pb.ph; a.pw = pb.pw;
  a.bk = pb.bk; a.stages = pb.stages; a.split_k = pb.split_k;
  a.cblocks = (pb.C + pb.bk - 1) / pb.bk;
  a.kblocks = pb.R * pb.S * a.cblocks;
  a.bias = pb.bias; a.y = pb.y; a.out_f32 = pb.out_f32; a.relu = pb.relu; a.has_bias = pb.has_bias;
  a.ws_partial = pb.ws_partial; a.ws_counters = pb.ws_counters;
  plan->fn = reinterpret_cast<const void*>(pick_tc(pb.bm, pb.bn));
  if (!plan->fn) { set_error("no igemm_tc instantiation for this BM x BN"); return TP_EINVALID_CONFIG; }
  plan->grid = dim3((unsigned)((pb.M + pb.bm - 1) / pb.bm), (unsigned)((pb.K + pb.bn - 1) / pb.bn),
                    (unsigned)pb.split_k);
  if (pb.grid_x) plan->grid = dim3(pb.grid_x, pb.grid_y, pb.grid_z);
  plan->block = dim3(pb.threads);
  plan->smem = tc_dyn_smem(pb.bm, pb.bn, pb.bk, pb.stages);
  cudaError_t e = cudaFuncSetAttribute(plan->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan->smem);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return TP_ECUDA;
  }
  return TP_OK;
}

cudaError_t tc_launch(const TcPlan& plan, cudaStream_t stream) {
  KernelFn fn = reinterpret_cast<KernelFn>(const_cast<void*>(plan.fn));
  fn<<<plan.grid, plan.block, plan.smem, stream>>>(plan.tmA, plan.tmB, plan.args);
  return cudaGetLastError();
}

int tc_occupancy(const TcPlan& plan) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, plan.fn, plan.block.x, plan.smem) != cudaSuccess) return 1;
  return n < 1 ? 1 : n;
}

}  // namespace tp
