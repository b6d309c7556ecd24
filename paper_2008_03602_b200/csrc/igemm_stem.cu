// igemm_stem.cu -- tensor-core conv2d for the small-channel stems (C < 8:
// ResNet-50 conv1, VGG-19 conv1_1, MobileNetV2 conv0), kind TP_KIND_IGEMM_TC_STEM.
//
// What it computes: the same operator as igemm_tc.cu (bias +
// ReLU of P:388), D[M x K] = A_im2col[M x K_g] W[K x K_g]^T with the reduction
// axis k = (r, s, c) flattened (c fastest, KRSC weights), K_g = R S C <= 256
// padded with zeros to KP = 64 ceil(K_g / 64).
//
// Why a separate kind: a C = 3 pixel row is 6 bytes, so neither TMA mode can
// feed it, and gathering the im2col tile element by element from global memory
// (the gathered kind) is bound by the L1 wavefront rate of scattered 2-byte
// loads (~2 elements / cycle / SM measured, ~4000 cycles per 128-pixel VGG
// tile).  Here a tile is BM output pixels of ONE output row, whose input patch
// (R rows x ((BM-1) s_w + S) pixels x C channels) is a set of R contiguous
// global segments: three producer warps copy it into shared memory with
// coalesced loads, then expand it into the 128-B-swizzled K-major im2col tile
// with shared-memory reads (a k table maps k -> patch offset).  The BN x KP
// weight tile is staged once per CTA and stays resident for tiles_per_cta
// tiles; two TMEM accumulators let the epilogue of tile i overlap the MMAs of
// tile i+1.
//
// Warp roles (256 threads): warps 0-2 producers (patch + im2col tile, named
// barrier 1), warp 3 MMA issuer (one elected lane), warps 4-7 epilogue (TMEM
// lane quadrant = warp % 4), warp 2 also allocates TMEM.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "tp_kernels.h"
#include "tc_ptx.cuh"

namespace tp {

template <int BM, int BN>
__global__ void __launch_bounds__(256) igemm_stem_kernel(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                                         const __grid_constant__ CUtensorMap tmY, TcArgs a) {   // (no tensor maps: same launch signature as igemm_tc)
  constexpr uint32_t A_SUB = BM * 128, B_SUB = BN * 128;   // one 64-element (128-B) k column block
  constexpr uint32_t kTmemCols = 2 * BN;                   // two accumulators
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);   // bf16 x bf16 -> f32, K-major A and B
  constexpr int kProd = 96;                                 // producer threads (warps 0-2)

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KP = a.bk, NSUB = KP >> 6, CH = KP >> 3;        // 16-byte chunks per row
  uint8_t* b_s = smem_raw;
  uint8_t* a_s = smem_raw + (size_t)NSUB * B_SUB;
  uint16_t* patch0 = reinterpret_cast<uint16_t*>(smem_raw + a.patch_off);   // pdist + 1 buffers of a.pbuf bytes
  int* ktab = reinterpret_cast<int*>(smem_raw + a.tab_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + a.bar_off);
  uint64_t* b_full = bars;        // weights staged (3 producer warps)
  uint64_t* a_full = bars + 1;    // [2] im2col tile ready (3 producer warps)
  uint64_t* a_empty = bars + 3;   // [2] MMAs of the tile done (commit)
  uint64_t* t_full = bars + 5;    // [2] accumulator ready (commit)
  uint64_t* t_empty = bars + 7;   // [2] accumulator drained (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

  int tile0, ntl;
  tile_span(a.ntiles, a.tpc, a.slots, tile0, ntl);
  if (ntl <= 0) return;   // past the resident slots (whole CTA, before any barrier)
  const int nbase = blockIdx.y * BN;
  // Patch row r of a tile holds input elements e0 - sh1 .. e0 - sh1 + prow - 1 of
  // input row h0 + r (e0 = (q0 s_w - p_w) C; sh1 = a.psh = (p_w C) & 1 makes the row
  // start on a 4-byte word, since q0 s_w C is even).
  const int C = a.C, prow = a.prow, sh1 = a.psh;   // (16-byte mode: a 16-byte boundary, psh = (-p_w C) mod 8)

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
    mbar_init(b_full, 3);
    for (int i = 0; i < 2; ++i) {
      mbar_init(a_full + i, 3);
      mbar_init(a_empty + i, 1);
      mbar_init(t_full + i, 1);
      mbar_init(t_empty + i, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // k table: k = (r, s, c) -> offset of x[r][s + m s_w][c] in the patch for pixel m = 0; -1 = padding.
  for (int k = threadIdx.x; k < KP; k += blockDim.x) {
    int v = -1;
    if (k < a.Kg) {
      const int c = k % C, rs = k / C, s = rs % a.S, r = rs / a.S;
      v = r * prow + sh1 + s * C + c;
    }
    ktab[k] = v;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp < 3) {
    // ---------------- producers ----------------
    const int pt = threadIdx.x;
    if (warp == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint16_t* xg = reinterpret_cast<const uint16_t*>(a.xg);
    const uint16_t* wg = reinterpret_cast<const uint16_t*>(a.wg);
    // Weights once per CTA: row n of B = W[nbase + n][0..KP) (zero past K_g / K).
    for (int idx = pt; idx < BN * CH; idx += kProd) {
      const int n = idx % BN, ch = idx / BN, k0 = ch * 8, kn = nbase + n;
      uint32_t v[4];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        uint32_t lo = 0, hi = 0;
        if (kn < a.K && k0 + j < a.Kg) lo = __ldg(wg + (int64_t)kn * a.Kg + k0 + j);
        if (kn < a.K && k0 + j + 1 < a.Kg) hi = __ldg(wg + (int64_t)kn * a.Kg + k0 + j + 1);
        v[j / 2] = lo | (hi << 16);
      }
      const uint32_t off = (uint32_t)n * 128 + ((uint32_t)(((k0 & 63) >> 3) ^ (n & 7)) << 4);
      *reinterpret_cast<uint4*>(b_s + (size_t)(k0 >> 6) * B_SUB + off) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(b_full);

    const int WC = a.W * C;
    const int nw = prow >> 1;   // 4-byte words per patch row
    // Stream tile t's patch into buffer pb: with cp.async (4-byte words, zero
    // fill outside the image) when the input rows are whole words, else by
    // plain loads.
    // Tiles are staged in order tile0, tile0 + 1, ...: their (q-block, row,
    // image) advance as a counter instead of two divisions per tile.
    int s_qb = tile0 % a.nqb, s_p = (tile0 / a.nqb) % a.P, s_n = (tile0 / a.nqb) / a.P;
    const int v_nv = prow >> 3, v_r0 = pt / v_nv, v_vi0 = pt % v_nv, v_dr = kProd / v_nv, v_dv = kProd % v_nv;
    auto stage_patch = [&](int pbi) {
      const int qb = s_qb, p = s_p, n = s_n;
      if (++s_qb == a.nqb) {
        s_qb = 0;
        if (++s_p == a.P) { s_p = 0; ++s_n; }
      }
      const int e0 = (qb * BM * a.sw - a.pw) * C - sh1;
      const int h0 = p * a.sh - a.ph;
      uint16_t* pbase = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(patch0) + (size_t)pbi * a.pbuf);
      const uint16_t* ximg = xg + (int64_t)n * a.H * WC;
      if (a.pc_async == 2) {
        // The R x (prow / 8) chunks of the patch as one flat range over the
        // 96 producer threads (a row alone has fewer chunks than threads).
        for (int r = v_r0, vi = v_vi0; r < a.R;) {
          const int h = h0 + r, g = e0 + 8 * vi;
          const bool ok = (unsigned)h < (unsigned)a.H && g >= 0 && g < WC;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(pbase + r * prow + 8 * vi)),
                       "l"(ok ? ximg + (int64_t)h * WC + g : ximg), "r"(ok ? 16 : 0)
                       : "memory");
          vi += v_dv;
          r += v_dr;
          if (vi >= v_nv) { vi -= v_nv; ++r; }
        }
      }
      for (int r = 0; r < a.R && a.pc_async != 2; ++r) {
        const int h = h0 + r;
        const bool hv = (unsigned)h < (unsigned)a.H;
        const uint16_t* xr = ximg + (int64_t)(hv ? h : 0) * WC;
        uint16_t* pr = pbase + r * prow;
        if (a.pc_async) {
          for (int wi = pt; wi < nw; wi += kProd) {
            const int g = e0 + 2 * wi;
            const bool ok = hv && g >= 0 && g < WC;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(pr + 2 * wi)),
                         "l"(ok ? xr + g : xr), "r"(ok ? 4 : 0)
                         : "memory");
          }
        } else {
          for (int e = pt; e < prow; e += kProd) {
            const int g = e0 + e;
            pr[e] = (hv && (unsigned)g < (unsigned)WC) ? __ldg(xr + g) : (uint16_t)0;
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // Patches run a.pdist tiles ahead through pdist + 1 buffers (one cp.async
    // group per tile, empty past the last tile, so that "wait until pdist
    // groups are pending" always means "tile i's patch has landed").
    const int PD = a.pdist;
    for (int j = 0; j < PD; ++j) {
      if (j < ntl) stage_patch(j);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int i = 0; i < ntl; ++i) {
      const int b = i & 1;
      const uint16_t* patch = reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(patch0) +
                                                                (size_t)(i % (PD + 1)) * a.pbuf);
      if (i + PD < ntl) stage_patch((i + PD) % (PD + 1));
      else asm volatile("cp.async.commit_group;" ::: "memory");
      if (PD == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else asm volatile("cp.async.wait_group 1;" ::: "memory");
      asm volatile("bar.sync 1, 96;" ::: "memory");
      // Expand into the swizzled im2col tile b (after the MMAs of tile i-2 released it).
      mbar_wait(a_empty + b, ((uint32_t)(i >> 1) & 1u) ^ 1u);
      uint8_t* at = a_s + (size_t)b * NSUB * A_SUB;
      // Chunk columns past K_g are all padding: when the count of real chunk
      // columns divides 96 they are zeroed on the first use of each of the two
      // tile buffers and skipped afterwards.  Thread pt owns chunk column
      // pt % CHn for rows pt / CHn + j (96 / CHn); its 8 k-table entries stay in
      // registers (CH = KP / 8 in {8, 16, 24, 32} divides 96).
      const int mstep = a.sw * C;
      const int CHv = (a.Kg + 7) >> 3;
      const int CHn = (i >= 2 && kProd % CHv == 0) ? CHv : CH;
      const int myc = pt % CHn, rstep = kProd / CHn, k0 = myc * 8;
      // Per k: the shared-memory address of its element for pixel 0 (padding
      // k reads element 0 and is masked to zero), so a row costs 8 adds, 8
      // 2-byte loads, 4 byte-permutes and 4 masks (no per-element predicates).
      uint32_t pa[8], mk[4];
      const uint32_t pbase_s = smem_u32(patch);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int oj = ktab[k0 + j];
        pa[j] = pbase_s + 2u * (uint32_t)(oj >= 0 ? oj : 0);
        if (j & 1) mk[j >> 1] |= oj >= 0 ? 0xFFFF0000u : 0u;
        else mk[j >> 1] = oj >= 0 ? 0x0000FFFFu : 0u;
      }
      uint8_t* colb = at + (size_t)(k0 >> 6) * A_SUB;
      const uint32_t cpos = (uint32_t)((k0 & 63) >> 3);
      for (int m = pt / CHn; m < BM; m += rstep) {
        const uint32_t mo2 = 2u * (uint32_t)(m * mstep);
        uint32_t e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint16_t h;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(pa[j] + mo2));
          e[j] = h;
        }
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = __byte_perm(e[2 * q], e[2 * q + 1], 0x5410) & mk[q];
        const uint32_t off = (uint32_t)m * 128 + ((cpos ^ (uint32_t)(m & 7)) << 4);
        *reinterpret_cast<uint4*>(colb + off) = make_uint4(v[0], v[1], v[2], v[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + b);
      asm volatile("bar.sync 1, 96;" ::: "memory");   // tile i's patch buffer is refilled next iteration
    }
  } else if (warp == 3) {
    // ---------------- MMA issuer ----------------
    const uint32_t lead = elect_one();
    mbar_wait(b_full, 0);
    const uint64_t bdesc0 = make_sdesc(smem_u32(b_s), 128);
    for (int i = 0; i < ntl; ++i) {
      const int b = i & 1;
      mbar_wait(a_full + b, (uint32_t)(i >> 1) & 1u);
      if (i >= 2) mbar_wait(t_empty + b, (uint32_t)((i - 2) >> 1) & 1u);
      tc_fence_after();
      const uint64_t adesc0 = make_sdesc(smem_u32(a_s + (size_t)b * NSUB * A_SUB), 128);
      const uint32_t d = tmem_base + (uint32_t)(b * BN);
      for (int kk = 0; kk < KP / 16; ++kk) {
        const uint32_t sb = (uint32_t)(kk >> 2), ko = (uint32_t)((kk & 3) * 32);
        tc_mma_p(d, adesc0 + ((sb * A_SUB + ko) >> 4), bdesc0 + ((sb * B_SUB + ko) >> 4), IDESC, kk > 0 ? 1u : 0u,
                 lead);
      }
      tc_commit_p(a_empty + b, lead);
      tc_commit_p(t_full + b, lead);
    }
  } else {
    // ---------------- epilogue (warps 4-7) ----------------
    // y_tma: the tile is staged in its own buffer in the swizzled box layout of
    // a 3-D [N P][Q][K] map (q >= Q clipped by the store) and written by one
    // 2-D-per-column-block TMA store; else 16-byte row stores.
    const int quad = warp & 3;
    const int row = (BM == 128) ? quad * 32 + lane : quad * 16 + lane;
    const bool row_ok = (BM == 128 || lane < 16);
    uint8_t* stg = smem_raw + a.recv_off;
    const uint32_t EB = a.out_f32 ? 4u : 2u;
    const uint32_t IB = BN * EB < 128u ? BN * EB : 128u;
    // Bias of the CTA's BN columns staged once (zero past K and without a
    // bias); ReLU as a max against 0 (or -inf without ReLU).
    float* bias_s = reinterpret_cast<float*>(smem_raw + a.bar_off + 128);
    for (int j = (int)threadIdx.x - 128; j < BN; j += 128)
      bias_s[j] = (a.has_bias && nbase + j < a.K) ? __ldg(a.bias + nbase + j) : 0.0f;
    asm volatile("bar.sync 2, 128;" ::: "memory");
    const float lo = a.relu ? 0.0f : __int_as_float(0xff800000u);
    int e_qb = tile0 % a.nqb, e_prw = tile0 / a.nqb;   // tile (q-block, output row), advanced per tile
    for (int i = 0; i < ntl; ++i) {
      const int b = i & 1;
      const int qb = e_qb, prw = e_prw;
      if (++e_qb == a.nqb) { e_qb = 0; ++e_prw; }
      const int q = qb * BM + row;
      __syncwarp();
      mbar_wait(t_full + b, (uint32_t)(i >> 1) & 1u);
      tc_fence_after();
      if (a.y_tma) {
        // the previous tile's store must have read the staging buffer
        if (threadIdx.x == 128) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("bar.sync 2, 128;" ::: "memory");
      }
      for (int c = 0; c < BN; c += 16) {
        uint32_t raw[16];
        tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * BN + c), raw);
        const int nb = nbase + c;
        float v[16];
#pragma unroll
        for (int g = 0; g < 16; g += 4) {
          const float4 bv = *reinterpret_cast<const float4*>(bias_s + c + g);
          const float b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) v[g + j] = fmaxf(__uint_as_float(raw[g + j]) + b4[j], lo);
        }
        if (a.y_tma) {
          if (row_ok) {
            const uint32_t cb = (uint32_t)c * EB, j = cb / IB, cin = cb % IB;
            uint8_t* sub = stg + (size_t)j * BM * IB;
            const uint32_t swm = IB / 16 - 1;
            for (uint32_t qq = 0; qq < 16 * EB / 16; ++qq) {
              uint32_t off = (uint32_t)row * IB + cin + qq * 16;
              off ^= ((off >> 7) & swm) << 4;
              uint4 u;
              if (a.out_f32) {
                u = make_uint4(__float_as_uint(v[4 * qq]), __float_as_uint(v[4 * qq + 1]),
                               __float_as_uint(v[4 * qq + 2]), __float_as_uint(v[4 * qq + 3]));
              } else {
                __nv_bfloat162 b0 = __floats2bfloat162_rn(v[8 * qq], v[8 * qq + 1]);
                __nv_bfloat162 b1 = __floats2bfloat162_rn(v[8 * qq + 2], v[8 * qq + 3]);
                __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * qq + 4], v[8 * qq + 5]);
                __nv_bfloat162 b3 = __floats2bfloat162_rn(v[8 * qq + 6], v[8 * qq + 7]);
                u = make_uint4(*reinterpret_cast<uint32_t*>(&b0), *reinterpret_cast<uint32_t*>(&b1),
                               *reinterpret_cast<uint32_t*>(&b2), *reinterpret_cast<uint32_t*>(&b3));
              }
              *reinterpret_cast<uint4*>(sub + off) = u;
            }
          }
        } else if (row_ok && q < a.Q && nb < a.K) {
          store16(a.y, (int64_t)prw * a.Q + q, a.K, nb, v, a.out_f32);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_empty + b);
      if (a.y_tma) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (threadIdx.x == 128) {
          for (uint32_t j = 0; j < BN * EB / IB; ++j)
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                             reinterpret_cast<uint64_t>(&tmY)),
                         "r"(smem_u32(stg + (size_t)j * BM * IB)), "r"((int)(nbase + j * (IB / EB))),
                         "r"(qb * BM), "r"(prw)
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (a.y_tma && threadIdx.x == 128) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
}

const void* pick_stem(int bm, int bn) {
#define TP_STEM_CASE(M_, N_) \
  if (bm == M_ && bn == N_) return reinterpret_cast<const void*>(igemm_stem_kernel<M_, N_>);
  TP_STEM_CASE(64, 32) TP_STEM_CASE(64, 64) TP_STEM_CASE(64, 128)
  TP_STEM_CASE(128, 32) TP_STEM_CASE(128, 64) TP_STEM_CASE(128, 128)
#undef TP_STEM_CASE
  return nullptr;
}

}  // namespace tp
