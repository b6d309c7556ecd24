// igemm_tf32.cu -- fp32 implicit-GEMM conv2d on 5th-gen tensor cores with a
// 3xTF32 split (north_star fp32 tolerance 1e-5).
//
// What it computes: the same "2D convolution" operator as
// igemm_tc.cu, D[M x K] = sum_k A_im2col[M x (R S C)] * W[K x (R S C)]^T, for
// fp32 layers, then bias + ReLU and an fp32 (or bf16) NHWC store.
// tcgen05 kind::tf32 reads only the top 10 mantissa bits of each fp32 operand,
// which alone gives ~1e-3 relative error (reading C8).  Each operand is split
// exactly into a = a_hi + a_lo (a_hi = a with the low 13 mantissa bits cleared,
// a_lo = a - a_hi, exact in fp32) and the product is accumulated in fp32 TMEM as
//     a_hi*b_hi + a_hi*b_lo + a_lo*b_hi          (a_lo*b_lo ~ 2^-22 |ab| dropped)
// so every product carries ~2^-21 relative error instead of ~2^-11.
//
// B200 design (one CTA per BM x BN output tile, 256 threads):
//  * warp 0: TMA producer -- per k-block (32-channel block cb, filter tap (r, s))
//    one im2col box of BM pixels x 32 fp32 channels over NHWC x (conv padding =
//    out-of-bounds zero fill; a tiled [M][C] box for 1x1/s1/p0 layers) and one
//    tiled box of BN filters x 32 channels over KRSC w; 128-B swizzle.
//  * warps 4..7: split -- once a stage lands they rewrite its tiles in place as
//    hi parts and write the lo parts to a twin ring (the swizzle is a byte
//    permutation inside each tile, so the elementwise split ignores it), then
//    fence the generic proxy against the async proxy and arrive on `ready`.
//  * warp 1: one elected lane issues 3 tcgen05.mma.kind::tf32 per 8-channel
//    k-step into one TMEM accumulator and commits each stage back to `empty`.
//  * warp 2: TMEM allocation; all warps: epilogue (tcgen05.ld -> bias -> ReLU ->
//    16-byte NHWC stores).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "tp_kernels.h"
#include "tc_ptx.cuh"

namespace tp {

template <int BM, int BN>
__global__ void __launch_bounds__(256) igemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB,
                                                         const __grid_constant__ CUtensorMap, TcArgs a) {
  constexpr uint32_t A_T = BM * 128, B_T = BN * 128;   // one k-block tile: rows x 32 fp32 channels
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  // kind::tf32: D = F32 (bit 4), A = B = TF32 (format 2 at bits 7 and 10), K-major A and B.
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
  constexpr int kSplitWarps = 4;                       // warps 4..7

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stages = a.stages;
  uint8_t* a_hi = smem_raw;
  uint8_t* b_hi = a_hi + (size_t)stages * A_T;
  uint8_t* a_lo = b_hi + (size_t)stages * B_T;
  uint8_t* b_lo = a_lo + (size_t)stages * A_T;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + a.bar_off);
  uint64_t* ready = full + stages;
  uint64_t* empty = ready + stages;
  uint64_t* tmem_full = empty + stages;
  uint64_t* red_bar = tmem_full + 1;   // split-K: every peer's partial rows landed in this CTA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_bar + 1);

  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  const int m0 = m_tile * BM;
  const int q0 = m0 % a.Q, t0 = m0 / a.Q;
  const int p0 = t0 % a.P, n0 = t0 / a.P;
  const int cw = q0 * a.sw - a.pw, ch = p0 * a.sh - a.ph;
  const int nbase = n_tile * BN;
  // This split's k-blocks (a k-block = 32-channel block cb of filter tap (r, s), cb fastest).
  const int kb0 = (split * a.kblocks) / a.split_k, kb1 = ((split + 1) * a.kblocks) / a.split_k;
  const int rows_per = BM / a.split_k;   // split-K: output rows this CTA owns and reduces

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0) __trap();   // swizzle atoms need 1 KiB alignment
    for (int i = 0; i < stages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(ready + i, kSplitWarps);
      mbar_init(empty + i, 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(red_bar, 1);
    if (a.split_k > 1) mbar_arrive_expect_tx(red_bar, (uint32_t)((a.split_k - 1) * rows_per * BN * 4));
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
  // Publish the reduction barrier to the cluster (waited on before the first remote store).
  if (a.split_k > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // Every warp sleeps in the PDL wait (no operand is touched before it).
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    const uint32_t lead = elect_one();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int rs = kb0 / a.cblocks;
    int cb = kb0 - rs * a.cblocks, s = rs % a.S, r = rs / a.S, stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(empty + stage, phase ^ 1u);
      mbar_arrive_expect_tx_p(full + stage, A_T + B_T, lead);
      if (a.a_tiled)
        tma_load_tile_2d_p(a_hi + (size_t)stage * A_T, &tmA, full + stage, cb * 32, m0, lead);
      else
        tma_load_im2col_4d_p(a_hi + (size_t)stage * A_T, &tmA, full + stage, cb * 32, cw, ch, n0, (uint16_t)s,
                             (uint16_t)r, lead);
      tma_load_tile_4d_p(b_hi + (size_t)stage * B_T, &tmB, full + stage, cb * 32, s, r, nbase, lead);
      if (++cb == a.cblocks) {
        cb = 0;
        if (++s == a.S) { s = 0; ++r; }
      }
      if (++stage == stages) { stage = 0; phase ^= 1u; }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t lead = elect_one();
    const uint64_t ahi0 = make_sdesc(smem_u32(a_hi), 128), bhi0 = make_sdesc(smem_u32(b_hi), 128);
    const uint64_t alo0 = make_sdesc(smem_u32(a_lo), 128), blo0 = make_sdesc(smem_u32(b_lo), 128);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(ready + stage, phase);
      tc_fence_after();
      const uint32_t oa = (uint32_t)(stage * A_T) >> 4, ob = (uint32_t)(stage * B_T) >> 4;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {   // 4 k-steps of 8 tf32 (32 B) per 128-B row
        const uint32_t ko = (uint32_t)(kk * 32) >> 4;
        tc_mma_tf32_p(tmem_base, ahi0 + oa + ko, bhi0 + ob + ko, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u, lead);
        if (!(a.dbg & 8)) {   // dbg bit3 (experiments only): 1xTF32
          tc_mma_tf32_p(tmem_base, ahi0 + oa + ko, blo0 + ob + ko, IDESC, 1u, lead);
          tc_mma_tf32_p(tmem_base, alo0 + oa + ko, bhi0 + ob + ko, IDESC, 1u, lead);
        }
      }
      tc_commit_p(empty + stage, lead);
      if (++stage == stages) { stage = 0; phase ^= 1u; }
    }
    tc_commit_p(tmem_full, lead);
  } else if (warp >= 4) {
    // ---------------- hi/lo split of each landed stage ----------------
    const int t = threadIdx.x - 128;
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(full + stage, phase);
      uint4* ah = reinterpret_cast<uint4*>(a_hi + (size_t)stage * A_T);
      uint4* al = reinterpret_cast<uint4*>(a_lo + (size_t)stage * A_T);
      uint4* bh = reinterpret_cast<uint4*>(b_hi + (size_t)stage * B_T);
      uint4* bl = reinterpret_cast<uint4*>(b_lo + (size_t)stage * B_T);
      // Thread t owns chunks t + 128 J, J < PER; chunk J is in A iff J < BM / 16
      // (BM * 8 chunks of A, a multiple of 128).  Batches of loads are issued
      // before any store (the compiler cannot prove hi/lo stores do not alias
      // the next loads).
      if (!(a.dbg & 4)) {   // dbg bit2 (experiments only): no split work
        constexpr int PER = (BM + BN) / 16, BATCH = PER < 8 ? PER : 8;
#pragma unroll
        for (int j0 = 0; j0 < PER; j0 += BATCH) {
          uint4 v[BATCH];
#pragma unroll
          for (int j = 0; j < BATCH; ++j) {
            const int J = j0 + j;
            if (J < PER) v[j] = J < BM / 16 ? ah[t + J * 128] : bh[t + (J - BM / 16) * 128];
          }
#pragma unroll
          for (int j = 0; j < BATCH; ++j) {
            const int J = j0 + j;
            if (J >= PER) break;
            uint4 h, l;
            h.x = v[j].x & 0xFFFFE000u; h.y = v[j].y & 0xFFFFE000u;
            h.z = v[j].z & 0xFFFFE000u; h.w = v[j].w & 0xFFFFE000u;
            l.x = __float_as_uint(__uint_as_float(v[j].x) - __uint_as_float(h.x));
            l.y = __float_as_uint(__uint_as_float(v[j].y) - __uint_as_float(h.y));
            l.z = __float_as_uint(__uint_as_float(v[j].z) - __uint_as_float(h.z));
            l.w = __float_as_uint(__uint_as_float(v[j].w) - __uint_as_float(h.w));
            if (J < BM / 16) {
              ah[t + J * 128] = h;
              al[t + J * 128] = l;
            } else {
              bh[t + (J - BM / 16) * 128] = h;
              bl[t + (J - BM / 16) * 128] = l;
            }
          }
        }
      }
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(ready + stage);
      if (++stage == stages) { stage = 0; phase ^= 1u; }
    }
  }

  // ---------------- epilogue (all 8 warps: TMEM lane quadrant = warp % 4, column half = warp / 4) ----------------
  const int quad = warp & 3, cgroup = warp >> 2;
  const int cols = BN / 2;
  const int c_begin = cgroup * cols, c_end = c_begin + cols;
  const int row = (BM == 128) ? quad * 32 + lane : quad * 16 + lane;
  const bool row_ok = (BM == 128 || lane < 16);
  const int64_t m = m0 + row;
  const bool m_ok = row_ok && m < a.M;
  __syncwarp();
  mbar_wait(tmem_full, 0);
  tc_fence_after();
  auto bias_relu = [&](int nb, float (&v)[16]) {
#pragma unroll
    for (int g = 0; g < 16; g += 4) {
      float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (a.has_bias && nb + g + 4 <= a.K) bv = __ldg(reinterpret_cast<const float4*>(a.bias + nb + g));
      const float b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float t = v[g + j] + b4[j];
        v[g + j] = a.relu ? fmaxf(t, 0.0f) : t;
      }
    }
  };
  if (a.split_k == 1) {
    for (int c = c_begin; c < c_end; c += 16) {
      uint32_t raw[16];
      tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)c, raw);
      const int nb = nbase + c;
      if (m_ok && nb < a.K) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(raw[j]);
        bias_relu(nb, v);
        store16(a.y, m, a.K, nb, v, a.out_f32);
      }
    }
  } else {
    // Split-K through DSMEM (as igemm_tc.cu): every row segment goes to the
    // CTA of the cluster that owns the row (st.async completing bytes on the
    // owner's red_bar; a plain shared store for own rows); the owner sums the
    // split_k slices in split order (deterministic), adds bias, applies ReLU.
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    float* recv = reinterpret_cast<float*>(smem_raw + a.recv_off);
    for (int c = c_begin; c < c_end; c += 16) {
      uint32_t raw[16];
      tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)c, raw);
      if (row_ok) {
        const int owner = row / rows_per;
        float* slot = recv + (split * rows_per + (row - owner * rows_per)) * (BN + 4) + c;
        if (owner == split) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<uint4*>(slot + i) = make_uint4(raw[i], raw[i + 1], raw[i + 2], raw[i + 3]);
        } else {
          const uint32_t rdst = mapa_u32(smem_u32(slot), (uint32_t)owner);
          const uint32_t rbar = mapa_u32(smem_u32(red_bar), (uint32_t)owner);
#pragma unroll
          for (int i = 0; i < 16; i += 4) st_async_v4(rdst + i * 4, raw[i], raw[i + 1], raw[i + 2], raw[i + 3], rbar);
        }
      }
    }
    const bool owns = row_ok && (row / rows_per) == split;
    mbar_wait(red_bar, 0);
    __syncthreads();   // own-row plain stores of the other warps are visible
    if (owns && m < a.M) {
      const float* mine = recv + (row - split * rows_per) * (BN + 4);
      for (int c = c_begin; c < c_end; c += 16) {
        const int nb = nbase + c;
        if (nb >= a.K) continue;
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.0f;
        for (int j = 0; j < a.split_k; ++j) {
          const float* sl = mine + j * rows_per * (BN + 4) + c;
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 t = *reinterpret_cast<const float4*>(sl + i);
            v[i] += t.x; v[i + 1] += t.y; v[i + 2] += t.z; v[i + 3] += t.w;
          }
        }
        bias_relu(nb, v);
        store16(a.y, m, a.K, nb, v, a.out_f32);
      }
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

const void* pick_tf32(int bm, int bn) {
#define TP_TF32_CASE(M_, N_) \
  if (bm == M_ && bn == N_) return reinterpret_cast<const void*>(igemm_tf32_kernel<M_, N_>);
  TP_TF32_CASE(64, 32) TP_TF32_CASE(64, 64) TP_TF32_CASE(64, 128) TP_TF32_CASE(64, 256)
  TP_TF32_CASE(128, 32) TP_TF32_CASE(128, 64) TP_TF32_CASE(128, 128) TP_TF32_CASE(128, 256)
#undef TP_TF32_CASE
  return nullptr;
}

}  // namespace tp
