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
#include <type_traits>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <climits>

#include "tp_kernels.h"
#include "tc_ptx.cuh"

namespace tp {

// Timeline slots per CTA when tracing (SM clock64 cycles): 0 entry, 1 prologue
// done, 2 epilogue start (tmem_full seen), 3 end, 4.. MMA-thread full-barrier
// completions of the first kTraceK k-blocks; slot 31 = %globaltimer (ns) at
// entry and slot 30 = %smid, for cross-CTA skew.
constexpr int kTraceSlots = 96, kTraceK = 16;   // 4..19 MMA full-wait done, 20..35 producer
                                                   // after empty-wait, 36..51 MMA after commit
__device__ __forceinline__ unsigned long long gtimer() { return (unsigned long long)clock64(); }

// GATHER = false: A by TMA im2col per filter tap, B by TMA tiled (C % 8 == 0).
// GATHER = true : the reduction axis is (r, s, c) flattened (c fastest) and
//   every warp but the MMA warp gathers the A (im2col) and B (weight) tiles
//   element by element into the same swizzled K-major shared-memory layout the
//   TMA would produce (the C = 3 stems, where a pixel row is 6 bytes and
//   neither TMA mode applies).
template <int BM, int BN, int BK, int MODE>
__global__ void __launch_bounds__(256, MODE == 1 ? 3 : 2) igemm_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB,
                                                       const __grid_constant__ CUtensorMap tmY, TcArgs a) {
  constexpr bool GATHER = MODE == 1;
  static_assert(MODE == 0 || MODE == 1 || MODE == 6, "modes 2-5 are igemm_mt_kernel");
  // MODE 0 / 6: TMA-fed split_k == 1 / split_k > 1 instantiations (each launch runs
  // only its own epilogue; smaller code per launch), MODE 1 (gathered): either.
  const bool sk1 = MODE == 0 ? true : (MODE == 6 ? false : a.split_k == 1);
  // Compile-time tile geometry: one swizzle row holds SUBK channels (32/64/128 B).
  constexpr int SUBK = BK < 64 ? BK : 64;
  constexpr int NSUB = BK / SUBK;
  constexpr uint32_t SWZ = SUBK * 2;
  constexpr uint32_t A_SUB = BM * SUBK * 2, B_SUB = BN * SUBK * 2;
  constexpr uint32_t A_STAGE = A_SUB * NSUB, B_STAGE = B_SUB * NSUB;
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);   // bf16 x bf16 -> f32, K-major A and B

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stages = a.stages;
  uint8_t* a_tiles = smem_raw;
  uint8_t* b_tiles = a_tiles + (size_t)stages * A_STAGE;
  // Barriers live after max(pipeline ring, split-K reduction buffer) (a.bar_off).
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + a.bar_off);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;
  uint64_t* red_bar = tmem_full + 1;   // split-K DSMEM reduction: all peers' slices landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_bar + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  unsigned long long* trace =
      a.trace ? a.trace + ((size_t)(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * kTraceSlots
              : nullptr;
  // Entry stamps stay in registers until the prologue is done: a global store
  // here would make the release fence below wait for it.
  unsigned long long tr_entry = 0, tr_gt = 0;
  if (trace && threadIdx.x == 0) {
    tr_entry = gtimer();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_gt));
  }
  const int kb0 = (split * a.kblocks) / a.split_k;   // 32-bit: M, k-blocks < 2^31 (checked on the host)
  const int kb1 = ((split + 1) * a.kblocks) / a.split_k;
  const int nkb = kb1 - kb0;

  // Output-pixel origin of this M tile -> im2col base coordinate (lower corner = -pad).
  const int m0 = m_tile * BM;
  const int q0 = m0 % a.Q;
  const int t0 = m0 / a.Q;
  const int p0 = t0 % a.P;
  const int n0 = t0 / a.P;
  const int cw = q0 * a.sw - a.pw, ch = p0 * a.sh - a.ph;
  const int nbase = n_tile * BN;

  // Producer state: filter tap (r, s) and channel block of the next k-block,
  // advanced incrementally (no divisions in the loop).
  int p_cb = 0, p_s = 0, p_r = 0, p_stage = 0, p_kb = kb0;
  uint32_t p_phase = 0;
  // Move the producer state `step` k-blocks ahead (step <= stages).
  auto advance = [&](int step) {
    for (int t = 0; t < step; ++t) {
      if (++p_cb == a.cblocks) {
        p_cb = 0;
        if (++p_s == a.S) { p_s = 0; ++p_r; }
      }
    }
    p_stage += step;
    if (p_stage >= stages) { p_stage -= stages; p_phase ^= 1u; }
    p_kb += step;
  };
  // parts: bit0 A (im2col) boxes, bit1 B (weight) boxes, bit2 the stage's expect_tx.
  // The producer warps (up to four, see is_prod below) take k-blocks round
  // robin (step = nprod): a TMA issue costs ~90 cycles of the issuing thread
  // (measured, tools/micro/tma_issue.cu) and independent threads issue in parallel.
  auto produce = [&](uint32_t lead, int parts, int step) {
    uint8_t* sa = a_tiles + (size_t)p_stage * A_STAGE;
    uint8_t* sbp = b_tiles + (size_t)p_stage * B_STAGE;
    if (parts & 4)
      mbar_arrive_expect_tx_p(full + p_stage, ((a.dbg & 1) ? 0u : A_STAGE) + ((a.dbg & 2) ? 0u : B_STAGE), lead);
    const int c0 = p_cb * BK;
#pragma unroll
    for (int sb = 0; sb < NSUB; ++sb) {
      if (!(a.dbg & 1) && (parts & 1)) {
        if (a.a_tiled)   // 1x1 / s1 / p0: A is the plain [M x C] matrix (tiled box, cheaper than im2col)
          tma_load_tile_2d_p(sa + sb * A_SUB, &tmA, full + p_stage, c0 + sb * SUBK, m0, lead);
        else
          tma_load_im2col_4d_p(sa + sb * A_SUB, &tmA, full + p_stage, c0 + sb * SUBK, cw, ch, n0, (uint16_t)p_s,
                               (uint16_t)p_r, lead);
      }
      if (!(a.dbg & 2) && (parts & 2))
        tma_load_tile_4d_p(sbp + sb * B_SUB, &tmB, full + p_stage, c0 + sb * SUBK, p_s, p_r, nbase, lead);
    }
    advance(step);
  };

  // TMA producer warps (k-block j goes to producer j mod nprod): warp 0, 3, 2, 4
  // in rank order, at most one per ring stage.  A TMA issue costs the issuing
  // thread ~50-90 cycles (tools/micro/tma_issue.cu) and threads issue in parallel.
  const int nprod_hw = blockDim.x == 256 ? 4 : 3;
  const int nprod = nprod_hw < stages ? (nprod_hw < a.nprod ? nprod_hw : a.nprod)
                                      : (stages < a.nprod ? stages : a.nprod);
  const int prank = warp == 0 ? 0 : (warp == 3 ? 1 : (warp == 2 ? 2 : (warp == 4 ? 3 : 99)));
  const bool is_prod = !GATHER && prank < nprod;
  if (is_prod) {
    const int rs = kb0 / a.cblocks;
    p_cb = kb0 - rs * a.cblocks;
    p_s = rs % a.S;
    p_r = rs / a.S;
  }
  if (warp == 0) {
    if (lane == 0) {
      if ((smem_u32(smem_raw) & 1023u) != 0) __trap();   // swizzle atoms need 1 KiB alignment
      // GATHER: every producer warp arrives once per stage.
      const uint32_t full_count = GATHER ? (blockDim.x >> 5) - 1 : 1;
      for (int i = 0; i < stages; ++i) { mbar_init(full + i, full_count); mbar_init(empty + i, 1); }
      mbar_init(tmem_full, 1);
      mbar_init(red_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if constexpr (!GATHER) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
      }
      // This CTA owns BM/split_k rows of the tile and receives them from the
      // split_k - 1 other splits of the cluster.
      if (a.cluster_red) mbar_arrive_expect_tx(red_bar, (uint32_t)((a.split_k - 1) * (BM / a.split_k) * BN * 4));
      if (trace) trace[52] = gtimer();
    }
    __syncwarp();
    if constexpr (!GATHER) {
      const uint32_t lead = elect_one();
      // With w_early the weight boxes of the first ring pass go out before the
      // PDL wait (weights are layer constants; the runtime sets w_early only
      // when the preceding kernel is a launch of this same plan).  Everything
      // that depends on the previous grid is issued after the CTA-wide sync, so
      // the MMA warp waits on stage 0 instead of on the whole ring fill.
      if (a.w_early) {
        const int pre = nkb < stages ? nkb : stages;
        const int s_cb = p_cb, s_s = p_s, s_r = p_r, s_kb = p_kb;
        for (int i = 0; i < pre; ++i) produce(lead, 6, 1);
        p_cb = s_cb; p_s = s_s; p_r = s_r; p_kb = s_kb; p_stage = 0; p_phase = 0;
      }
    }
  }
  if constexpr (GATHER) {
    // Pixel table (rowbase, h0, w0) for the BM rows of this tile and k table
    // (offset of (r, s, c) relative to the row base, (r << 16) | s) over the
    // padded reduction extent; built once per CTA.  Rows past M and k past
    // R*S*C get coordinates that fail every bounds check (zero fill).
    int4* rowtab = reinterpret_cast<int4*>(smem_raw + a.tab_off);
    int2* ktab = reinterpret_cast<int2*>(smem_raw + a.tab_off + BM * 16);
    for (int r = threadIdx.x; r < BM; r += blockDim.x) {
      const int m = (int)m0 + r;
      int4 e = make_int4(0, -(1 << 20), -(1 << 20), 0);
      if (m < (int)a.M) {
        const int q = m % a.Q, t = m / a.Q, pp = t % a.P, n = t / a.P;
        const int h0 = pp * a.sh - a.ph, w0 = q * a.sw - a.pw;
        e = make_int4(((n * a.H + h0) * a.W + w0) * a.C, h0, w0, 0);
      }
      rowtab[r] = e;
    }
    for (int k = threadIdx.x; k < a.kblocks * BK; k += blockDim.x) {
      int2 e = make_int2(0, 0x7FFF7FFF);
      if (k < a.Kg) {
        const int c = k % a.C, rs = k / a.C, ss = rs % a.S, rr = rs / a.S;
        e = make_int2((rr * a.W + ss) * a.C + c, (rr << 16) | ss);
      }
      ktab[k] = e;
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    if (trace && lane == 0) trace[58] = gtimer();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Publish the initialised reduction barrier to the cluster; the matching
  // wait sits just before the first remote store, long after every peer arrived.
  // (relaxed: the mbarrier init is already ordered by fence.mbarrier_init.release.cluster;
  // a release arrive would also wait for this thread's outstanding memory operations)
  if (a.cluster_red) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);   // provably warp-uniform
  if (trace && threadIdx.x == 0) {
    trace[1] = gtimer();
    trace[0] = tr_entry;
    trace[63] = tr_gt;
    unsigned sm, ncta;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
    trace[62] = sm;
    trace[61] = ncta;
    trace[60] = (unsigned long long)a.cluster_red;
  }
  // Every warp sleeps in the PDL wait rather than spinning on an mbarrier while
  // the previous grid may still run on this SM (co-resident CTAs).
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (GATHER && warp != 1) {
    // ---------------- gather producers (all warps but the MMA warp) ----------------
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int pt = warp == 0 ? lane : (int)threadIdx.x - 32;
    const int np = (int)blockDim.x - 32;
    const int4* rowtab = reinterpret_cast<const int4*>(smem_raw + a.tab_off);
    const int2* ktab = reinterpret_cast<const int2*>(smem_raw + a.tab_off + BM * 16);
    const uint16_t* xg = reinterpret_cast<const uint16_t*>(a.xg);
    const uint16_t* wg = reinterpret_cast<const uint16_t*>(a.wg);
    constexpr int CPR = BK / 8;                 // 16-byte chunks per tile row
    constexpr uint32_t SWM = SWZ / 16 - 1;      // swizzle: chunk ^= (offset >> 7) & SWM
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(empty + stage, phase ^ 1u);
      if (trace && threadIdx.x == 0 && kb - kb0 < 8) trace[84 + kb - kb0] = gtimer();
      uint8_t* sa = a_tiles + (size_t)stage * A_STAGE;
      uint8_t* sbt = b_tiles + (size_t)stage * B_STAGE;
      const int kbase = kb * BK;
      // np is a multiple of 32 and CPR divides 32, so this thread's 16-byte
      // chunk column kc is the same for every row it fills: its 8 k-table
      // entries are read once per k-block, and the rows (pixel rows of A, then
      // weight rows of B) are visited 4 at a time with all 32 element loads
      // issued before any shared-memory store.
      const int kc = pt % CPR, rstep = np / CPR;
      const int k0 = kbase + kc * 8;
      int2 kt[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) kt[j] = ktab[k0 + j];
      const int sub = (kc * 8) / SUBK, ch = ((kc * 8) % SUBK) / 8;
      for (int row0 = pt / CPR; row0 < BM + BN; row0 += 4 * rstep) {
        uint32_t v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = row0 + u * rstep;
          if (rr < BM) {
            const int4 rt = rowtab[rr];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              uint32_t lo = 0, hi = 0;
              if ((unsigned)(rt.y + (kt[j].y >> 16)) < (unsigned)a.H &&
                  (unsigned)(rt.z + (kt[j].y & 0xFFFF)) < (unsigned)a.W)
                lo = __ldg(xg + rt.x + kt[j].x);
              if ((unsigned)(rt.y + (kt[j + 1].y >> 16)) < (unsigned)a.H &&
                  (unsigned)(rt.z + (kt[j + 1].y & 0xFFFF)) < (unsigned)a.W)
                hi = __ldg(xg + rt.x + kt[j + 1].x);
              v[u][j / 2] = lo | (hi << 16);
            }
          } else if (rr < BM + BN) {
            const int kn = nbase + rr - BM;
            const uint16_t* wr = wg + (int64_t)kn * a.Kg + k0;
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              uint32_t lo = 0, hi = 0;
              if (kn < a.K && k0 + j < a.Kg) lo = __ldg(wr + j);
              if (kn < a.K && k0 + j + 1 < a.Kg) hi = __ldg(wr + j + 1);
              v[u][j / 2] = lo | (hi << 16);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = row0 + u * rstep;
          if (rr >= BM + BN) break;
          const bool is_a = rr < BM;
          const int row = is_a ? rr : rr - BM;
          uint32_t off = (uint32_t)row * SWZ + (uint32_t)ch * 16;
          off ^= ((off >> 7) & SWM) << 4;
          uint8_t* dst = (is_a ? sa + sub * A_SUB : sbt + sub * B_SUB) + off;
          *reinterpret_cast<uint4*>(dst) = make_uint4(v[u][0], v[u][1], v[u][2], v[u][3]);
        }
      }
      if (trace && threadIdx.x == 0 && kb - kb0 < 8) trace[68 + kb - kb0] = gtimer();
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (trace && threadIdx.x == 0 && kb - kb0 < 8) trace[76 + kb - kb0] = gtimer();
      __syncwarp();
      if (lane == 0) mbar_arrive(full + stage);
      if (trace && threadIdx.x == 0 && kb - kb0 < kTraceK) trace[20 + kb - kb0] = gtimer();
      if (++stage == stages) { stage = 0; phase ^= 1u; }
    }
  } else if (is_prod) {
    // ---------------- TMA producers: k-blocks j = prank (mod nprod), one elected lane each ----------------
    const uint32_t lead = elect_one();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // Every operand this grid reads is now final: the next kernel in the
    // stream may be scheduled (programmatic dependent launch).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (trace && warp == 0 && lane == 0) trace[53] = gtimer();
    const int pre = a.w_early ? (nkb < stages ? nkb : stages) : 0;   // weight boxes already in flight
    if (prank > 0) advance(prank);
    while (p_kb < kb1) {
      const int j = p_kb - kb0;
      mbar_wait(empty + p_stage, p_phase ^ 1u);   // free on the first ring pass
      if (trace && warp == 0 && lane == 0 && j < kTraceK) trace[20 + j] = gtimer();
      produce(lead, j < pre ? 1 : 7, nprod);
      if (trace && warp == 0 && lane == 0 && j < 8) trace[54 + j / 2] = gtimer();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one elected lane of warp 1) ----------------
    const uint32_t lead = elect_one();
    const uint64_t adesc0 = make_sdesc(smem_u32(a_tiles), SWZ);
    const uint64_t bdesc0 = make_sdesc(smem_u32(b_tiles), SWZ);
    int stage = 0;
    uint32_t phase = 0, soff_a = 0, soff_b = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(full + stage, phase);
      tc_fence_after();
      if (trace && lane == 0 && kb - kb0 < kTraceK) trace[4 + kb - kb0] = gtimer();
      const uint64_t ad = adesc0 + soff_a, bd = bdesc0 + soff_b;
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        constexpr int kPerSub = SUBK / 16;
        const uint32_t sb = kk / kPerSub, koff = (kk % kPerSub) * 32;   // compile-time after unroll
        tc_mma_p(tmem_base, ad + ((sb * A_SUB + koff) >> 4), bd + ((sb * B_SUB + koff) >> 4), IDESC,
                 (kb > kb0 || kk > 0) ? 1u : 0u, lead);
      }
      tc_commit_p(empty + stage, lead);
      if (trace && lane == 0 && kb - kb0 < kTraceK) trace[36 + kb - kb0] = gtimer();
      soff_a += A_STAGE >> 4;
      soff_b += B_STAGE >> 4;
      if (++stage == stages) { stage = 0; phase ^= 1u; soff_a = 0; soff_b = 0; }
    }
    tc_commit_p(tmem_full, lead);
  }

  // ---------------- epilogue (all warps) ----------------
  const int quad = warp & 3, ngroups = blockDim.x >> 7, cgroup = warp >> 2;
  const int cols = BN / ngroups;
  const int c_begin = cgroup * cols, c_end = c_begin + cols;
  const int row = (BM == 128) ? quad * 32 + lane : quad * 16 + lane;
  const bool row_ok = (BM == 128 || lane < 16);
  const int64_t m = m0 + row;
  const bool m_ok = row_ok && m < a.M;
  const int64_t tile = (int64_t)m_tile * gridDim.y + n_tile;
  const int64_t n_tiles = (int64_t)gridDim.x * gridDim.y;

  // Bias for a 16-column chunk (vector loads, broadcast across the warp).
  auto load_bias16 = [&](int nb, float (&bv)[16]) {
#pragma unroll
    for (int g = 0; g < 16; g += 4) {
      if (a.has_bias && nb + g + 4 <= a.K) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(a.bias + nb + g));
        bv[g] = f.x; bv[g + 1] = f.y; bv[g + 2] = f.z; bv[g + 3] = f.w;
      } else {
        bv[g] = bv[g + 1] = bv[g + 2] = bv[g + 3] = 0.0f;
      }
    }
  };
  float bias_next[16];
  load_bias16(nbase + c_begin, bias_next);   // prefetch while the mainloop runs

  __syncwarp();
  mbar_wait(tmem_full, 0);
  tc_fence_after();
  if (trace && threadIdx.x == 0) trace[2] = gtimer();
  if (a.cluster_red) {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (trace && threadIdx.x == 0) trace[65] = gtimer();
  }

  // split_k == 1, bf16 row stores, at most 4 chunks per thread: pack every
  // chunk first, release TMEM, then issue the stores (a dealloc after the
  // stores' issue cost ~0.1 us per launch in a dependent chain).
  const int nch = (c_end - c_begin) >> 4;
  if (sk1 && !a.y_tma && !a.out_f32 && nch <= 4) {
    auto drain = [&](auto n_c) {
      constexpr int NCH = decltype(n_c)::value;
      uint32_t pk[NCH][8];
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        uint32_t raw[16];
        tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(c_begin + 16 * j), raw);
        float bv[16];
        if (j == 0) {
#pragma unroll
          for (int i = 0; i < 16; ++i) bv[i] = bias_next[i];
        } else {
          load_bias16(nbase + c_begin + 16 * j, bv);
        }
        if (a.relu) bias_pack16<true>(raw, bv, pk[j]);
        else bias_pack16<false>(raw, bv, pk[j]);
      }
      if (!GATHER && trace && threadIdx.x == 0) trace[69] = gtimer();
      tc_fence_before();
      __syncthreads();
      if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
      }
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int nb = nbase + c_begin + 16 * j;
        if (m_ok && nb < a.K) store16_pk(a.y, m, a.K, nb, pk[j]);
      }
    };
    if (nch == 1) drain(std::integral_constant<int, 1>());
    else if (nch == 2) drain(std::integral_constant<int, 2>());
    else if (nch == 3) drain(std::integral_constant<int, 3>());
    else drain(std::integral_constant<int, 4>());
    if (trace && threadIdx.x == 0) trace[3] = gtimer();
    return;
  }

  for (int c = c_begin; c < c_end; c += 16) {
    uint32_t raw[16];
    tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)c, raw);
    if (!GATHER && trace && threadIdx.x == 0 && c == c_begin) trace[68] = gtimer();
    const int nb = nbase + c;
    float bv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) bv[i] = bias_next[i];
    if (c + 16 < c_end) load_bias16(nb + 16, bias_next);
    if (sk1 && a.y_tma) {
      // Stage the tile in the (now idle) ring in the swizzled layout of the y
      // tensor map's box (IB-byte rows, BN / (IB / EB) boxes side by side); rows
      // past M and columns past K are clipped by the TMA store.
      if (row_ok && !a.out_f32) {
        // bf16: paired bias adds and one RNE pack per pair, ReLU in the conversion
        constexpr uint32_t IBf = BN * 2 < 128 ? BN * 2 : 128, SWM = IBf / 16 - 1;
        uint32_t pk[8];
        if (a.relu) bias_pack16<true>(raw, bv, pk);
        else bias_pack16<false>(raw, bv, pk);
        const uint32_t xr = ((((uint32_t)row * IBf) >> 7) & SWM) << 4;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint32_t cb = (uint32_t)(c + 8 * q) * 2u, j = cb / IBf, cin = cb % IBf;
          *reinterpret_cast<uint4*>(smem_raw + (size_t)j * BM * IBf + (size_t)row * IBf + (cin ^ xr)) =
              make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      } else if (row_ok) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float t = __uint_as_float(raw[i]) + bv[i];
          v[i] = a.relu ? fmaxf(t, 0.0f) : t;
        }
        const uint32_t EB = a.out_f32 ? 4u : 2u;
        const uint32_t IB = BN * EB < 128u ? BN * EB : 128u;
        const uint32_t cb = (uint32_t)c * EB, j = cb / IB, cin = cb % IB;
        uint8_t* sub = smem_raw + (size_t)j * BM * IB;
        const uint32_t swm = IB / 16 - 1;
        if (a.out_f32) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t off = (uint32_t)row * IB + cin + q * 16;
            off ^= ((off >> 7) & swm) << 4;
            *reinterpret_cast<float4*>(sub + off) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t off = (uint32_t)row * IB + cin + q * 16;
            off ^= ((off >> 7) & swm) << 4;
            uint4 u;
            __nv_bfloat162 b0 = __floats2bfloat162_rn(v[8 * q], v[8 * q + 1]);
            __nv_bfloat162 b1 = __floats2bfloat162_rn(v[8 * q + 2], v[8 * q + 3]);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * q + 4], v[8 * q + 5]);
            __nv_bfloat162 b3 = __floats2bfloat162_rn(v[8 * q + 6], v[8 * q + 7]);
            u.x = *reinterpret_cast<uint32_t*>(&b0);
            u.y = *reinterpret_cast<uint32_t*>(&b1);
            u.z = *reinterpret_cast<uint32_t*>(&b2);
            u.w = *reinterpret_cast<uint32_t*>(&b3);
            *reinterpret_cast<uint4*>(sub + off) = u;
          }
        }
      }
    } else if (sk1) {
      if (m_ok && nb < a.K && !a.out_f32) {
        uint32_t pk[8];
        if (a.relu) bias_pack16<true>(raw, bv, pk);
        else bias_pack16<false>(raw, bv, pk);
        store16_pk(a.y, m, a.K, nb, pk);
      } else if (m_ok && nb < a.K) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float t = __uint_as_float(raw[i]) + bv[i];
          v[i] = a.relu ? fmaxf(t, 0.0f) : t;
        }
        store16(a.y, m, a.K, nb, v, a.out_f32);
      }
    } else if (a.cluster_red) {
      // Row segment -> the owner CTA's receive slot [split][row - owner_r0]:
      // st.async into a peer (completes on the peer's red_bar), a plain
      // shared store for the rows this CTA owns.  Every row is sent, so the
      // byte count each owner expects is fixed.
      if (row_ok) {
        const int rows_per = BM / a.split_k;
        const int owner = row / rows_per;
        float* slot = reinterpret_cast<float*>(smem_raw + a.recv_off) +
                      (split * rows_per + (row - owner * rows_per)) * (BN + 4) + c;
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
    } else if (row_ok) {
      float* part = a.ws_partial + (((int64_t)split * n_tiles + tile) * BM + row) * BN + c;
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        __stcg(reinterpret_cast<float4*>(part + i), make_float4(__uint_as_float(raw[i]), __uint_as_float(raw[i + 1]),
                                                                __uint_as_float(raw[i + 2]),
                                                                __uint_as_float(raw[i + 3])));
    }
  }

  if (!GATHER && trace && threadIdx.x == 0) trace[69] = gtimer();
  // Every warp's last tcgen05.ld is done: release TMEM now, before the TMA
  // store, the split-K reduction and the exit (in a chain of dependent launches
  // a dealloc issued after the output stores cost ~0.1 us per launch:
  // tools/micro/launch_gap.cu, variants 6 and 7).
  if (sk1 && a.y_tma)   // generic-proxy smem writes -> visible to the TMA engine
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
  if (sk1 && a.y_tma) {
    // one thread stores the staged tile
    if (threadIdx.x == 0) {
      const int EB = a.out_f32 ? 4 : 2;
      const int IB = BN * EB < 128 ? BN * EB : 128;
      for (int j = 0; j < BN * EB / IB; ++j)
        tma_store_2d(&tmY, smem_raw + (size_t)j * BM * IB, nbase + j * (IB / EB), m0);
      tma_store_commit_wait();
    }
  }
  if (!sk1 && a.cluster_red) {
    // Owner side: the threads whose row this CTA owns wait for the other
    // splits' slices, sum all split_k slices in split order (deterministic),
    // add bias, ReLU, store.  Same thread <-> row mapping as the send pass.
    if (trace && threadIdx.x == 0) trace[64] = gtimer();
    const int rows_per = BM / a.split_k;
    const bool owns = row_ok && (row / rows_per) == split;
    float bv[16];
    if (owns) load_bias16(nbase + c_begin, bv);
    mbar_wait(red_bar, 0);
    if (trace && threadIdx.x == 0) trace[66] = gtimer();
    if (owns && m < a.M) {
      const float* recv = reinterpret_cast<const float*>(smem_raw + a.recv_off) + (row - split * rows_per) * (BN + 4);
      for (int c = c_begin; c < c_end; c += 16) {
        const int nb = nbase + c;
        if (c > c_begin) load_bias16(nb, bv);
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.0f;
        for (int j = 0; j < a.split_k; ++j) {
          const float* sl = recv + j * rows_per * (BN + 4) + c;
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 t = *reinterpret_cast<const float4*>(sl + i);
            v[i] += t.x; v[i + 1] += t.y; v[i + 2] += t.z; v[i + 3] += t.w;
          }
        }
        if (nb < a.K && !a.out_f32) {
          uint32_t raw[16], pk[8];
#pragma unroll
          for (int i = 0; i < 16; ++i) raw[i] = __float_as_uint(v[i]);
          if (a.relu) bias_pack16<true>(raw, bv, pk);
          else bias_pack16<false>(raw, bv, pk);
          store16_pk(a.y, m, a.K, nb, pk);
        } else if (nb < a.K) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float t = v[i] + bv[i];
            v[i] = a.relu ? fmaxf(t, 0.0f) : t;
          }
          store16(a.y, m, a.K, nb, v, a.out_f32);
        }
      }
    }
    if (trace && threadIdx.x == 0) trace[67] = gtimer();
  } else if (!sk1) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int old = atomicAdd(a.ws_counters + tile, 1);
      *last_flag = (old == a.split_k - 1);
    }
    __syncthreads();
    if (*last_flag) {
      __threadfence();
      for (int c = c_begin; c < c_end; c += 16) {
        const int nb = nbase + c;
        if (!m_ok || nb >= a.K) continue;
        float v[16], bv[16];
        load_bias16(nb, bv);
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
          const float t = v[i] + bv[i];
          v[i] = a.relu ? fmaxf(t, 0.0f) : t;
        }
        store16(a.y, m, a.K, nb, v, a.out_f32);
      }
      if (threadIdx.x == 0) a.ws_counters[tile] = 0;   // leave the workspace zeroed
    }
  }

  if (!GATHER && trace && threadIdx.x == 0) trace[70] = gtimer();
  if (trace && threadIdx.x == 0) trace[3] = gtimer();
}

// ------------------------------------------------------------- multi-tile kernel
// TP_KIND_IGEMM_TC_ROW (ROW = true) and TP_KIND_IGEMM_TC_MT (ROW = false).
// ROW: a tile is BM pixels of one output row (q0 .. q0+BM-1
// of row p, image n); a k-block is (64-channel block cb, filter row r): one
// tiled TMA box brings the input strip of BM+2 pixels (padding = out-of-bounds
// zero fill) and three boxes bring the taps' BN x 64 weight tiles; the MMA
// reads tap s as the strip shifted by s rows of 128 B (descriptor start
// address + s*128; the 128-B swizzle is applied on absolute address bits, so
// the base-offset field stays 0 -- measured).  Each CTA handles `tpc`
// consecutive tiles: the producer ring runs across tiles, the MMA alternates
// between two TMEM accumulators, and (tpc > 1) warps 2..7 drain one
// accumulator while the MMA fills the other (tmem_full / tmem_empty pairs).
// MT (ROW = false) runs the same multi-tile pipeline with the im2col k-blocks
// of the TMA kind: tile = BM consecutive pixels, k-block = (channel block,
// tap), one im2col box + one weight box per k-block.
//
// STRIP (KM = 2, TP_KIND_IGEMM_TC_STRIP): x and w padded to 8 channels (16-byte
// pixels); tile = BM pixels of one output row as in ROW; a k-block is a filter
// row r: one tiled box per column phase f < s_w (element stride s_w) brings
// the strip of a.strip_px pixels starting at input column q0 s_w - p_w + f.
// Tap s = f + s_w t of phase f is that strip shifted by t pixels, and ONE MMA
// (K = 16) covers taps t and t + 1: no-swizzle K-major descriptors with the two
// core matrices along K 16 B apart (A) and s_w BN 16 B apart (weights laid out
// [r][s][n][8] in shared memory, loaded once; the s_w zero taps after each
// row's S taps pair with an odd tap count).
#ifndef TP_MT_WAIT
#define TP_MT_WAIT mbar_wait_sleep
#endif
template <int BM, int BN, int BK, int KM>
__global__ void __launch_bounds__(KM == 1 ? 352 : 320) igemm_mt_kernel(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB,
                                                       const __grid_constant__ CUtensorMap tmY, TcArgs a) {
  // KM 3 = the row-halo kind's CTA-pair form: a separate instantiation, since a kernel
  // containing cta_group::2 instructions must be launched with clusters of 2.
  constexpr bool ROW = KM == 1 || KM == 3, STRIP = KM == 2, PAIR = KM == 3;
  static_assert(!ROW || BK == 64, "row-halo k-blocks are 64 channels");
  constexpr int SUBK = BK < 64 ? BK : 64;
  constexpr int NSUB = BK / SUBK;
  constexpr uint32_t SWZ = ROW ? 128 : SUBK * 2;
  constexpr uint32_t A_SUB = BM * SUBK * 2, B_SUB = BN * SUBK * 2;
  constexpr uint32_t A_STRIP = ((BM + 2) * 128 + 1023) / 1024 * 1024;
  constexpr uint32_t B_TAP = BN * 128;
  // STRIP: runtime stage size (phase boxes only; the weights are resident)
  const uint32_t A_STAGE = STRIP ? (uint32_t)a.strip_stage : (ROW ? A_STRIP : A_SUB * NSUB);
  const uint32_t B_STAGE = (STRIP || (ROW && a.roww)) ? 0u : (ROW ? 3 * B_TAP : B_SUB * NSUB);
  const uint32_t A_BYTES = STRIP ? (a.sw == 1 ? (uint32_t)a.strip_stage : (uint32_t)(a.sw * a.strip_px * 16))
                                 : (ROW ? (BM + 2) * 128 : A_SUB * NSUB);   // expect_tx of the A part
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
  // CTA pair (ROW + roww + a.pair2): one cta_group::2 MMA of 2 BM rows x BN over the
  // (2, 1, 1) cluster -- each CTA holds its own tile's strips (A rows) and half of
  // the weight rows (BN / 2 per tap); rank 0 issues, both TMEMs receive their rows.
  constexpr uint32_t IDESC2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                              ((uint32_t)((2 * BM) >> 4) << 24);
  constexpr uint32_t B_TAP_HALF = (BN / 2) * 128;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stages = a.stages;
  constexpr bool pair = PAIR;
  const uint32_t prank = pair ? cluster_ctarank() : 0u;
  const uint32_t w_tap = pair ? B_TAP_HALF : B_TAP;   // resident weight bytes per tap in this CTA
  uint8_t* a_tiles = smem_raw;
  uint8_t* b_tiles = a_tiles + (size_t)stages * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + a.bar_off);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;     // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint64_t* wfull = tempty + 2;         // STRIP: resident weights landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfull + 1);
  uint8_t* w_res = smem_raw + a.strip_woff;   // STRIP: [r][S + s_w taps][BN][16 B]; ROW + roww: [r][s][BN][128 B]
  const uint32_t w_row = STRIP ? (uint32_t)((a.S + a.sw) * BN * 16) : 0u;

  const int tpc = a.tpc;
  const bool split_roles = tpc > 1;     // warps 2..7 drain while warps 0/1 run ahead
  int tile0, ntl;
  if (pair) {
    // cluster c runs pair steps u in [c tpc, c tpc + tpc); step u = tiles 2u (rank 0), 2u + 1 (rank 1);
    // both CTAs of a cluster get the same count (they return together or not at all)
    const int npairs = (a.ntiles + 1) / 2, u0 = (int)(blockIdx.x >> 1) * tpc;
    ntl = npairs - u0 < tpc ? npairs - u0 : tpc;
    tile0 = 2 * u0 + (int)prank;
  } else {
    tile_span(a.ntiles, tpc, a.slots, tile0, ntl);
  }
  if (ntl <= 0) return;                 // past the resident slots (whole CTA, before any barrier)
  const int nbase = blockIdx.y * BN;
  const int kpt = a.kblocks;            // k-blocks per tile = (C / 64) * 3
  const uint32_t ncols = (uint32_t)(split_roles ? 2 * BN : BN) <= 32 ? 32u : (uint32_t)(split_roles ? 2 * BN : BN);
  // tpc > 1: warps 2.. drain -- 8 of them (two per TMEM lane quadrant) when the
  // block has 320 threads, else 6 (quadrants 2 and 3 get two warps, 0 and 1 one).
  const bool epi8 = blockDim.x >= 320;
  // 352 threads (N = 64 tiles): warp 10 is a second MMA issuer taking the odd
  // tiles -- one thread issues an N = 64 MMA every ~52-56 cycles, two reach the
  // shared-memory operand rate (~48; tools/micro/mma_issue.cu).
  const bool mma2 = blockDim.x == 352;
  const int n_epi_warps = split_roles ? (epi8 ? 8 : 6) : (int)(blockDim.x >> 5);
  unsigned long long* trace =
      a.trace ? a.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots : nullptr;
  if (trace && threadIdx.x == 0) {
    trace[0] = gtimer();
    unsigned long long g;
    unsigned sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    trace[63] = g;
    trace[62] = sm;
  }

  // ROW / STRIP: tile = BM pixels of one output row (q-block t % nqb of row t / nqb);
  // im2col: tile = BM consecutive output pixels m0 = t * BM (rows past M masked).
  // A CTA's tiles are consecutive: the cursor is set once (divisions) and then
  // advanced with compares (ncu: the per-tile divisions were ~6% of the strip
  // kernel's instructions).
  struct TileCursor { int qb, p, n, m0; };
  auto cursor_at = [&](int t) {
    TileCursor c{0, 0, 0, 0};
    if constexpr (ROW || STRIP) {
      const int row = t / a.nqb;
      c.qb = t - row * a.nqb;
      c.p = row % a.P;
      c.n = row / a.P;
    } else {
      c.m0 = t * BM;
    }
    return c;
  };
  auto cursor_next = [&](TileCursor& c) {
    if constexpr (ROW || STRIP) {
      if (++c.qb == a.nqb) {
        c.qb = 0;
        if (++c.p == a.P) { c.p = 0; ++c.n; }
      }
    } else {
      c.m0 += BM;
    }
  };
  auto tile_coords = [&](const TileCursor& c, int& q0, int& p0, int& n0, int& mrow0, int& mvalid) {
    if constexpr (ROW || STRIP) {
      q0 = c.qb * BM;
      p0 = c.p;
      n0 = c.n;
      mrow0 = (n0 * a.P + p0) * a.Q + q0;
      mvalid = a.Q - q0 < BM ? a.Q - q0 : BM;
    } else {
      const int m0 = c.m0;
      q0 = m0 % a.Q;
      const int t0 = m0 / a.Q;
      p0 = t0 % a.P;
      n0 = t0 / a.P;
      mrow0 = m0;
      mvalid = (int)a.M - m0 < BM ? (int)a.M - m0 : BM;
    }
  };

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
    for (int i = 0; i < stages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    // pair: the leader's tempty counts both CTAs' drain warps (they arrive remotely)
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, (uint32_t)(pair ? 2 * n_epi_warps : n_epi_warps));
    }
    mbar_init(wfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if constexpr (STRIP) {
    // The s_w zero taps after each filter row's S taps (never written by TMA).
    const int zwords = a.sw * BN;       // 16-byte words of one row's zero taps (s_w x BN x 16 B)
    for (int i = threadIdx.x; i < a.R * zwords; i += blockDim.x) {
      const int r = i / zwords, j = i - r * zwords;
      *reinterpret_cast<uint4*>(w_res + (size_t)r * w_row + (size_t)a.S * BN * 16 + (size_t)j * 16) =
          make_uint4(0u, 0u, 0u, 0u);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    if (pair) {   // the same warp of both CTAs, the same columns
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(ncols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(ncols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (pair) cluster_sync_all();   // both CTAs' barriers exist before any cross-CTA signal
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  if (trace && threadIdx.x == 0) trace[1] = gtimer();

  if (warp == 0) {
    // ---------------- TMA producer: strips + tap weights, ring across tiles ----------------
    const uint32_t lead = elect_one();
    // One k-block of a tile: parts bit0 = A box(es), bit1 = weight boxes, bit2 = expect_tx.
    auto issue = [&](int stage, int cb, int r, int sx, int q0, int p0, int n0, int m0, int parts) {
      uint8_t* sa = a_tiles + (size_t)stage * A_STAGE;
      uint8_t* sb = b_tiles + (size_t)stage * B_STAGE;
      if (parts & 4) {
        if (!pair)
          mbar_arrive_expect_tx_p(full + stage, A_BYTES + ((parts & 2) ? B_STAGE : 0u), lead);
        else if (prank == 0)   // the leader's barrier counts both CTAs' strips
          mbar_arrive_expect_tx_p(full + stage, 2 * A_BYTES, lead);
      }
      if constexpr (STRIP) {
        // filter row r: one strip per column phase (the weights are resident).
        // s_w = 1: the strip is contiguous in the padded row, loaded as 512-byte
        // boxes of a (W*8, H, N) view -- a box of 16-byte rows costs the TMA
        // engine one request per row (measured: the ring then starves the MMA).
        if (parts & 1) {
          if (a.sw == 1) {
            for (int j = 0; j < a.strip_px; j += 32)
              tma_load_tile_3d_p(sa + j * 16, &tmA, full + stage, (q0 - a.pw + j) * 8, p0 * a.sh - a.ph + r, n0, lead);
          } else {
            const uint32_t pb = (uint32_t)a.strip_stage / (uint32_t)a.sw;
            for (int f = 0; f < a.sw; ++f)
              tma_load_tile_4d_p(sa + f * pb, &tmA, full + stage, 0, q0 * a.sw - a.pw + f, p0 * a.sh - a.ph + r, n0,
                                 lead);
          }
        }
      } else if constexpr (ROW) {
        // (channel block cb, filter row r): the input strip + the three taps
        if (parts & 1) {
          if (pair)
            tma_load_tile_4d_pair_p(sa, &tmA, full + stage, cb * 64, q0 - 1, p0 + r - 1, n0, lead);
          else
            tma_load_tile_4d_p(sa, &tmA, full + stage, cb * 64, q0 - 1, p0 + r - 1, n0, lead);
        }
        if ((parts & 2) && !a.roww) {
#pragma unroll
          for (int ss = 0; ss < 3; ++ss)
            tma_load_tile_4d_p(sb + ss * B_TAP, &tmB, full + stage, cb * 64, ss, r, nbase, lead);
        }
      } else {
        // (channel block cb, tap (r, sx)): one im2col box + the weight box
        const int cw = q0 * a.sw - a.pw, chh = p0 * a.sh - a.ph;
#pragma unroll
        for (int sb2 = 0; sb2 < NSUB; ++sb2) {
          if (parts & 1) {
            if (a.a_tiled)
              tma_load_tile_2d_p(sa + sb2 * A_SUB, &tmA, full + stage, cb * BK + sb2 * SUBK, m0, lead);
            else
              tma_load_im2col_4d_p(sa + sb2 * A_SUB, &tmA, full + stage, cb * BK + sb2 * SUBK, cw, chh, n0,
                                   (uint16_t)sx, (uint16_t)r, lead);
          }
          if (parts & 2)
            tma_load_tile_4d_p(sb + sb2 * B_SUB, &tmB, full + stage, cb * BK + sb2 * SUBK, sx, r, nbase, lead);
        }
      }
    };
    auto advance = [&](int& cb, int& r, int& sx) {
      if constexpr (STRIP) {
        ++r;
      } else if constexpr (ROW) {
        if (++r == 3) { r = 0; ++cb; }
      } else if (++cb == a.cblocks) {
        cb = 0;
        if (++sx == a.S) { sx = 0; ++r; }
      }
    };
    // w_early: the weight boxes of the first tile's first ring pass go out
    // before the PDL wait (weights are layer constants; see TcArgs::w_early).
    const int npre = (!STRIP && !(ROW && a.roww) && a.w_early && ntl > 0) ? (kpt < stages ? kpt : stages) : 0;
    {
      int cb = 0, r = 0, sx = 0;
      for (int kb = 0; kb < npre; ++kb) {
        issue(kb, cb, r, sx, 0, 0, 0, 0, 6);
        advance(cb, r, sx);
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if constexpr (STRIP) {
      // resident weights: one box (8 channels, BN rows, S taps) per filter row
      mbar_arrive_expect_tx_p(wfull, (uint32_t)(a.R * a.S * BN * 16), lead);
      for (int r = 0; r < a.R; ++r) tma_load_tile_4d_p(w_res + (size_t)r * w_row, &tmB, wfull, 0, nbase, 0, r, lead);
    } else if constexpr (ROW) {
      if (a.roww) {   // resident weights (C = 64): the nine taps, once
        if (!pair) {
          mbar_arrive_expect_tx_p(wfull, 9u * B_TAP, lead);
          for (int r = 0; r < 3; ++r)
            for (int ss = 0; ss < 3; ++ss)
              tma_load_tile_4d_p(w_res + (size_t)(r * 3 + ss) * B_TAP, &tmB, wfull, 0, ss, r, nbase, lead);
        } else {      // each CTA its half of the weight rows, counted on the leader's barrier
          if (prank == 0) mbar_arrive_expect_tx_p(wfull, 9u * B_TAP, lead);
          for (int r = 0; r < 3; ++r)
            for (int ss = 0; ss < 3; ++ss)
              tma_load_tile_4d_pair_p(w_res + (size_t)(r * 3 + ss) * B_TAP_HALF, &tmB, wfull, 0, ss, r,
                                      nbase + (int)prank * (BN / 2), lead);
        }
      }
    }
    int stage = 0;
    uint32_t phase = 0;
    TileCursor cur = cursor_at(tile0);
    for (int i = 0; i < ntl; ++i) {
      int q0, p0, n0, mrow0, mvalid;
      tile_coords(cur, q0, p0, n0, mrow0, mvalid);
      cursor_next(cur);
      if (pair) cursor_next(cur);
      int cb = 0, r = 0, sx = 0;
      for (int kb = 0; kb < kpt; ++kb) {
        TP_MT_WAIT(empty + stage, phase ^ 1u);
        // Resident weights: when the ring has exactly one stage per k-block of a
        // tile, k-block kb always lands in stage kb, so the weight boxes of the
        // first tile stay valid and later tiles load the input side only
        // (row-halo kind with C = 64: 123 -> 50 KB of L2 -> SMEM traffic per tile).
        const bool w_resident = !STRIP && stages == kpt && i > 0;
        issue(stage, cb, r, sx, q0, p0, n0, mrow0, (i == 0 && kb < npre) ? 1 : (w_resident ? 5 : 7));
        advance(cb, r, sx);
        if (++stage == stages) { stage = 0; phase ^= 1u; }
      }
      if (trace && lane == 0 && i < 8) trace[4 + i] = gtimer();    // tile i's loads issued
    }
  } else if ((warp == 1 || (mma2 && warp == 10)) && prank == 0) {
    // ---------------- MMA issuer: two accumulators, alternating per tile ----------------
    // (mma2: warp 1 issues the even tiles into accumulator 0, warp 10 the odd
    // tiles into accumulator 1; each finds its ring position from the tile index)
    const uint32_t lead = elect_one();
    const int i_first = (mma2 && warp == 10) ? 1 : 0, i_step = mma2 ? 2 : 1;
    const uint64_t adesc0 = STRIP ? make_sdesc_plain(smem_u32(a_tiles), 16u, 128u) : make_sdesc(smem_u32(a_tiles), SWZ);
    const bool wres = STRIP || (ROW && a.roww);
    const uint64_t bdesc0 = STRIP ? make_sdesc_plain(smem_u32(w_res), (uint32_t)(a.sw * BN * 16), 128u)
                                  : make_sdesc(smem_u32(wres ? w_res : b_tiles), SWZ);
    int stage = 0;
    uint32_t phase = 0;
    if (wres) {
      TP_MT_WAIT(wfull, 0);
      tc_fence_after();
    }
    for (int i = i_first; i < ntl; i += i_step) {
      const int buf = i & 1;
      if (mma2) {
        const int g = i * kpt;
        stage = g % stages;
        phase = (uint32_t)((g / stages) & 1);
      }
      if (i >= 2) {
        TP_MT_WAIT(tempty + buf, (uint32_t)(((i - 2) >> 1) & 1));
        tc_fence_after();
      }
      const uint32_t dcol = tmem_base + (uint32_t)(buf * BN);
      for (int kb = 0; kb < kpt; ++kb) {
        TP_MT_WAIT(full + stage, phase);
        tc_fence_after();
        const uint64_t ad = adesc0 + ((uint32_t)(stage * A_STAGE) >> 4);
        // roww: the weights of filter row kb (C = 64: one channel block) are resident
        const uint64_t bd = (ROW && a.roww) ? bdesc0 + ((uint32_t)(kb * 3 * w_tap) >> 4)
                                            : bdesc0 + ((uint32_t)(stage * B_STAGE) >> 4);
        if constexpr (STRIP) {
          // filter row kb: per phase f, tap pairs (t, t + 1), t even; tap s = f + s_w t
          const uint32_t pb = (uint32_t)a.strip_stage / (uint32_t)a.sw;
          const uint64_t bdr = bdesc0 + ((uint32_t)kb * w_row >> 4);
          for (int f = 0; f < a.sw; ++f) {
            const int taps = (a.S - f + a.sw - 1) / a.sw;
            for (int t = 0; t < taps; t += 2)
              tc_mma_p(dcol, ad + ((f * pb + (uint32_t)t * 16) >> 4),
                       bdr + ((uint32_t)(f + a.sw * t) * BN * 16 >> 4), IDESC, (kb > 0 || f > 0 || t > 0) ? 1u : 0u,
                       lead);
          }
        } else if constexpr (ROW) {
          const uint32_t tap = a.roww ? w_tap : B_TAP;
          if (pair) {
#pragma unroll
            for (int ss = 0; ss < 3; ++ss)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                tc_mma_pair_p(dcol, ad + ((uint32_t)(ss * 128 + kk * 32) >> 4),
                              bd + ((uint32_t)(ss * tap + kk * 32) >> 4), IDESC2,
                              (kb > 0 || ss > 0 || kk > 0) ? 1u : 0u, lead);
          } else {
#pragma unroll
            for (int ss = 0; ss < 3; ++ss)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                tc_mma_p(dcol, ad + ((uint32_t)(ss * 128 + kk * 32) >> 4),
                         bd + ((uint32_t)(ss * tap + kk * 32) >> 4), IDESC, (kb > 0 || ss > 0 || kk > 0) ? 1u : 0u,
                         lead);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            constexpr int kPerSub = SUBK / 16;
            const uint32_t sb2 = kk / kPerSub, koff = (kk % kPerSub) * 32;
            tc_mma_p(dcol, ad + ((sb2 * A_SUB + koff) >> 4), bd + ((sb2 * B_SUB + koff) >> 4), IDESC,
                     (kb > 0 || kk > 0) ? 1u : 0u, lead);
          }
        }
        if (pair) tc_commit_pair_p(empty + stage, lead); else tc_commit_p(empty + stage, lead);
        if (++stage == stages) { stage = 0; phase ^= 1u; }
      }
      if (pair) tc_commit_pair_p(tfull + buf, lead); else tc_commit_p(tfull + buf, lead);
      if (trace && lane == 0 && i < 8) trace[12 + i] = gtimer();   // tile i's MMAs issued
    }
  }

  // ---------------- epilogue ----------------
  if (!split_roles || (warp >= 2 && !(mma2 && warp == 10))) {
    const int quad = warp & 3;
    int c_begin, c_end;
    if (split_roles) {               // warps 2..7 -> quadrants 2,3,0,1,2,3 (+ 8,9 -> 0,1 with epi8)
      const int twin = (epi8 || quad >= 2) ? 2 : 1;
      const int half = (warp >= 6) ? 1 : 0;
      c_begin = half * (BN / twin);
      c_end = c_begin + BN / twin;
    } else {
      const int ngroups = blockDim.x >> 7;
      c_begin = (warp >> 2) * (BN / ngroups);
      c_end = c_begin + BN / ngroups;
    }
    const int row = (BM == 128) ? quad * 32 + lane : quad * 16 + lane;
    const bool row_ok = (BM == 128 || lane < 16);
    // y_tma: stage each tile in its own buffer (after the barriers) in the box
    // layout of the y map -- 3-D [N P][Q][K] for row tiles (q >= Q clipped), 2-D
    // [M][K] for multi-tile im2col tiles -- and store it with TMA from one thread.
    const int n_epi = n_epi_warps * 32;
    const int issuer = split_roles ? 64 : 0;
    // Bias of the CTA's BN columns staged once in shared memory (inside the
    // barrier block: BN <= 128 floats fit after the barriers), read after this
    // grid's PDL wait like every other operand; BN = 256 keeps per-chunk loads.
    constexpr bool kBiasSmem = BN <= 128;
    float* sbias = reinterpret_cast<float*>(smem_raw + a.bar_off + 256);
    if constexpr (kBiasSmem) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int j = (int)threadIdx.x - (split_roles ? 64 : 0); j < BN; j += n_epi)
        sbias[j] = (a.has_bias && nbase + j < a.K) ? __ldg(a.bias + nbase + j) : 0.0f;
      asm volatile("bar.sync 3, %0;" ::"r"(n_epi) : "memory");
    }
    uint8_t* stg = smem_raw + a.recv_off;
    const uint32_t EB = a.out_f32 ? 4u : 2u;
    const uint32_t IB = BN * EB < 128u ? BN * EB : 128u;
    const uint32_t ystage = (uint32_t)BM * BN * EB;   // bytes of one staged tile
    TileCursor cur = cursor_at(tile0);
    for (int i = 0; i < ntl; ++i) {
      const int buf = i & 1;
      int q0, p0, n0, mrow0, mvalid;
      tile_coords(cur, q0, p0, n0, mrow0, mvalid);
      cursor_next(cur);
      if (pair) {
        cursor_next(cur);
        if (tile0 + 2 * i >= a.ntiles) mvalid = 0;   // odd tile count: rank 1's last tile is empty
      }
      // a.ystage2: two staging buffers alternate, so only the store of tile i - 2
      // must have read this one (one bulk group may stay in flight)
      uint8_t* stg_t = stg + (a.ystage2 ? (size_t)buf * ystage : 0);
      float bv[16];
      const int nb0 = nbase + c_begin;
      if constexpr (kBiasSmem) {
#pragma unroll
        for (int g = 0; g < 16; g += 4) {
          const float4 f = *reinterpret_cast<const float4*>(sbias + c_begin + g);
          bv[g] = f.x; bv[g + 1] = f.y; bv[g + 2] = f.z; bv[g + 3] = f.w;
        }
      } else {
#pragma unroll
        for (int g = 0; g < 16; g += 4) {
          if (a.has_bias && nb0 + g + 4 <= a.K) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(a.bias + nb0 + g));
            bv[g] = f.x; bv[g + 1] = f.y; bv[g + 2] = f.z; bv[g + 3] = f.w;
          } else {
            bv[g] = bv[g + 1] = bv[g + 2] = bv[g + 3] = 0.0f;
          }
        }
      }
      __syncwarp();
      // The issuer's warp polls the accumulator barrier (its issuer thread also
      // makes sure the store that last used this staging buffer has read it);
      // the named barrier releases the other drain warps, which would otherwise
      // spend issue slots polling.
      if (((int)threadIdx.x >> 5) == (issuer >> 5)) {
        if (a.y_tma && (int)threadIdx.x == issuer) {
          if (a.ystage2)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        TP_MT_WAIT(tfull + buf, (uint32_t)((i >> 1) & 1));
      }
      asm volatile("bar.sync 2, %0;" ::"r"(n_epi) : "memory");
      tc_fence_after();
      if (trace && (int)threadIdx.x == issuer && i < 8) trace[28 + i] = gtimer();   // tile i's accumulator ready
      if constexpr (kBiasSmem) {
        if (!a.out_f32 && a.y_tma) {
          // bf16 + TMA store: compile-time staging geometry, ReLU chosen once per tile
          constexpr uint32_t IBf = BN * 2 < 128 ? BN * 2 : 128, SWM = IBf / 16 - 1;
          const uint32_t xr = ((((uint32_t)row * IBf) >> 7) & SWM) << 4;
          uint8_t* rowp = stg_t + (size_t)row * IBf;
          const uint32_t tb = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN);
          auto drain = [&](auto relu_c) {
            constexpr bool RELU = decltype(relu_c)::value;
            for (int c = c_begin; c < c_end; c += 16) {
              uint32_t raw[16];
              tmem_ld16(tb + (uint32_t)c, raw);
              float bw[16];
#pragma unroll
              for (int g = 0; g < 16; g += 4) {
                const float4 f = *reinterpret_cast<const float4*>(sbias + c + g);
                bw[g] = f.x; bw[g + 1] = f.y; bw[g + 2] = f.z; bw[g + 3] = f.w;
              }
              uint32_t pk[8];
              bias_pack16<RELU>(raw, bw, pk);
              if (row_ok) {
#pragma unroll
                for (int qq = 0; qq < 2; ++qq) {
                  const uint32_t cb = (uint32_t)(c + 8 * qq) * 2u, j = cb / IBf, cin = cb % IBf;
                  *reinterpret_cast<uint4*>(rowp + (size_t)j * BM * IBf + (cin ^ xr)) =
                      make_uint4(pk[4 * qq], pk[4 * qq + 1], pk[4 * qq + 2], pk[4 * qq + 3]);
                }
              }
            }
          };
          if (a.relu) drain(std::integral_constant<bool, true>());
          else drain(std::integral_constant<bool, false>());
        }
      }
      const bool fast_done = kBiasSmem && !a.out_f32 && a.y_tma;
      for (int c = c_begin; c < c_end && !fast_done; c += 16) {
        uint32_t raw[16];
        tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + c), raw);
        const int nb = nbase + c;
        if (c > c_begin) {
#pragma unroll
          for (int g = 0; g < 16; g += 4) {
            if constexpr (kBiasSmem) {
              const float4 f = *reinterpret_cast<const float4*>(sbias + c + g);
              bv[g] = f.x; bv[g + 1] = f.y; bv[g + 2] = f.z; bv[g + 3] = f.w;
            } else if (a.has_bias && nb + g + 4 <= a.K) {
              const float4 f = __ldg(reinterpret_cast<const float4*>(a.bias + nb + g));
              bv[g] = f.x; bv[g + 1] = f.y; bv[g + 2] = f.z; bv[g + 3] = f.w;
            } else {
              bv[g] = bv[g + 1] = bv[g + 2] = bv[g + 3] = 0.0f;
            }
          }
        }
        if (a.y_tma) {
          if (row_ok) {
            const uint32_t cb = (uint32_t)c * EB, jb = cb / IB, cin = cb % IB;
            uint8_t* sub = stg_t + (size_t)jb * BM * IB;
            const uint32_t swm = IB / 16 - 1;
            if (!a.out_f32) {
              // bf16: packed bias add (FADD2), one RNE pack per pair, ReLU on the packed pair
              // (max(rne(x), 0) == rne(max(x, 0)): rounding is monotone and keeps 0).
              uint32_t pk[8];
              const __nv_bfloat162 zero2 = __floats2bfloat162_rn(0.0f, 0.0f);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float2 t = __fadd2_rn(make_float2(__uint_as_float(raw[2 * j]), __uint_as_float(raw[2 * j + 1])),
                                            make_float2(bv[2 * j], bv[2 * j + 1]));
                __nv_bfloat162 h = __float22bfloat162_rn(t);
                if (a.relu) h = __hmax2(h, zero2);
                pk[j] = *reinterpret_cast<uint32_t*>(&h);
              }
#pragma unroll
              for (uint32_t qq = 0; qq < 2; ++qq) {
                uint32_t off = (uint32_t)row * IB + cin + qq * 16;
                off ^= ((off >> 7) & swm) << 4;
                *reinterpret_cast<uint4*>(sub + off) = make_uint4(pk[4 * qq], pk[4 * qq + 1], pk[4 * qq + 2], pk[4 * qq + 3]);
              }
            } else {
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float t = __uint_as_float(raw[j]) + bv[j];
              v[j] = a.relu ? fmaxf(t, 0.0f) : t;
            }
            for (uint32_t qq = 0; qq < EB; ++qq) {   // 16 values = EB 16-byte pieces
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
          }
        } else if (row_ok && row < mvalid && nb < a.K) {
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float t = __uint_as_float(raw[j]) + bv[j];
            v[j] = a.relu ? fmaxf(t, 0.0f) : t;
          }
          store16(a.y, (int64_t)mrow0 + row, a.K, nb, v, a.out_f32);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (pair)
          mbar_arrive_remote(tempty + buf, 0);   // the leader's MMA thread waits for both CTAs
        else
          mbar_arrive(tempty + buf);
      }
      if (trace && (int)threadIdx.x == issuer && i < 8) trace[20 + i] = gtimer();   // tile i drained (issuer warp)
      if (a.y_tma) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"r"(n_epi) : "memory");
        if ((int)threadIdx.x == issuer) {
          for (uint32_t jb = 0; jb < BN * EB / IB; ++jb) {
            const int ncol = nbase + (int)(jb * (IB / EB));
            if constexpr (ROW || STRIP)
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                               reinterpret_cast<uint64_t>(&tmY)),
                           "r"(smem_u32(stg_t + (size_t)jb * BM * IB)), "r"(ncol), "r"(q0), "r"(n0 * a.P + p0)
                           : "memory");
            else
              tma_store_2d(&tmY, stg_t + (size_t)jb * BM * IB, ncol, mrow0);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[3] = gtimer();
  if (pair) {
    // the leader's MMAs wrote this CTA's TMEM and its drain warps arrived on the
    // leader's barriers: both CTAs are done with each other before the free
    cluster_sync_all();
    if (warp == 2) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols) : "memory");
    }
  } else if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols) : "memory");
  }
  // the last tile's store must have read the staging buffer before the CTA
  // exits (waited after the TMEM release, which it does not need)
  if (a.y_tma && (int)threadIdx.x == (split_roles ? 64 : 0))
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ------------------------------------------------------------- host side
using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, TcArgs);

template <int BM, int BN, int MODE>
static KernelFn pick_bk(int bk) {
  if constexpr (MODE == 4) {
    if constexpr (BN <= 128) return bk == 16 ? igemm_mt_kernel<BM, BN, 16, 2> : nullptr;
    return nullptr;
  } else if constexpr (MODE == 5) {   // row-halo, resident weights, CTA pair (BM = 128)
    if constexpr (BM == 128 && BN <= 128) return bk == 64 ? igemm_mt_kernel<BM, BN, 64, 3> : nullptr;
    return nullptr;
  } else if constexpr (MODE == 2) {
    return bk == 64 ? igemm_mt_kernel<BM, BN, 64, 1> : nullptr;
  } else if constexpr (MODE == 3) {
    switch (bk) {
      case 16: return igemm_mt_kernel<BM, BN, 16, 0>;
      case 32: return igemm_mt_kernel<BM, BN, 32, 0>;
      case 64: return igemm_mt_kernel<BM, BN, 64, 0>;
      case 128: return igemm_mt_kernel<BM, BN, 128, 0>;
    }
  } else {
    static_assert(MODE == 0 || MODE == 1 || MODE == 6, "igemm_tc_kernel modes");
    switch (bk) {
      case 16: return igemm_tc_kernel<BM, BN, 16, MODE>;
      case 32: return igemm_tc_kernel<BM, BN, 32, MODE>;
      case 64: return igemm_tc_kernel<BM, BN, 64, MODE>;
      case 128: return igemm_tc_kernel<BM, BN, 128, MODE>;
    }
  }
  return nullptr;
}

static KernelFn pick_tc(int bm, int bn, int bk, int mode) {
#define TP_TC_CASE(M_, N_)                                                                       \
  if (bm == M_ && bn == N_)                                                                      \
    return mode == 6 ? pick_bk<M_, N_, 6>(bk)                                                    \
                     : mode == 5 ? pick_bk<M_, N_, 5>(bk)                                        \
                     : mode == 4 ? pick_bk<M_, N_, 4>(bk)                                        \
                     : mode == 3 ? pick_bk<M_, N_, 3>(bk)                                        \
                     : (mode == 2 ? pick_bk<M_, N_, 2>(bk)                                       \
                                  : (mode == 1 ? pick_bk<M_, N_, 1>(bk) : pick_bk<M_, N_, 0>(bk)));
  TP_TC_CASE(64, 32) TP_TC_CASE(64, 64) TP_TC_CASE(64, 128) TP_TC_CASE(64, 256)
  TP_TC_CASE(128, 32) TP_TC_CASE(128, 64) TP_TC_CASE(128, 128) TP_TC_CASE(128, 256)
#undef TP_TC_CASE
  return nullptr;
}

size_t tc_dyn_smem(int bm, int bn, int bk, int stages) {
  return (size_t)stages * (bm + bn) * bk * 2 + 1024;
}

// Shared-memory layout: [ring] [split-K receive buffer (cluster path)] [barriers, 1 KiB].
// The receive buffer must not alias the ring: peers push their slices while
// this CTA may still be in its mainloop.
static size_t tc_ring_bytes(int bm, int bn, int bk, int stages, bool row) {
  if (row) return (size_t)stages * ((((size_t)(bm + 2) * 128) + 1023) / 1024 * 1024 + 3 * (size_t)bn * 128);
  return (size_t)stages * (bm + bn) * bk * 2;
}
static size_t tc_bar_off(int bm, int bn, int bk, int stages, bool cluster_red, bool row) {
  size_t off = tc_ring_bytes(bm, bn, bk, stages, row);
  if (cluster_red) off += (size_t)bm * (bn + 4) * 4;
  return (off + 1023) & ~(size_t)1023;
}

// L2 promotion of the A (activation) tensor maps (TP_A_PROMO = 0 / 64 / 128 / 256 bytes; default 128)
static CUtensorMapL2promotion a_promotion() {
  static const int v = getenv("TP_A_PROMO") ? atoi(getenv("TP_A_PROMO")) : 128;
  return v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                  : (v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                             : (v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B));
}

static bool ystage2_enabled() {
  static const bool on = !(getenv("TP_YSTAGE2") && atoi(getenv("TP_YSTAGE2")) == 0);
  return on;
}

static bool roww_pair_enabled() {
  static const bool on = getenv("TP_ROWW2") && atoi(getenv("TP_ROWW2")) != 0;
  return on;
}

static bool mt_epi8() {
  static const bool on = !(getenv("TP_EPI8") && atoi(getenv("TP_EPI8")) == 0);
  return on;
}

// Strip kind (C <= 8 stems): pb.x = x padded to NHWC with 8 channels, pb.w =
// weights padded and laid out [R][S][K][8] (both written by the pre-pass into the
// workspace).  A: tiled map (8, W, H, N), box (8, s_w px, 1, 1) with element
// stride s_w along W (px pixels land), no swizzle; B: tiled map (8, K, S, R),
// box (8, BN, S, 1) -> shared [s][n][16 B] per filter row.  Shared memory:
// [ring: stages x s_w phase boxes][resident weights][barriers][y staging].
static tp_status strip_prepare(const TcProblem& pb, TcPlan* plan) {
  const DriverApi& drv = driver();
  const int sw = pb.sw;
  const int t0 = (pb.S + sw - 1) / sw;
  const int px = pb.bm + 2 * ((t0 + 1) / 2) - 1;
  // s_w = 1: whole 512-byte boxes (32 pixels each); s_w = 2: one strided box per phase
  const int phase_bytes = sw == 1 ? (px * 16 + 511) / 512 * 512 : (px * 16 + 127) / 128 * 128;
  {
    CUresult r;
    if (sw == 1) {   // padded rows as (W*8, H, N): 256-element (512-byte) boxes along the row
      cuuint64_t dims[3] = {(cuuint64_t)pb.W * 8, (cuuint64_t)pb.H, (cuuint64_t)pb.N};
      cuuint64_t strides[2] = {(cuuint64_t)pb.W * 16, (cuuint64_t)pb.H * pb.W * 16};
      cuuint32_t box[3] = {256, 1, 1};
      cuuint32_t es[3] = {1, 1, 1};
      r = drv.encodeTiled(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(pb.x), dims, strides, box,
                          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[4] = {8, (cuuint64_t)pb.W, (cuuint64_t)pb.H, (cuuint64_t)pb.N};
      cuuint64_t strides[3] = {16, (cuuint64_t)pb.W * 16, (cuuint64_t)pb.H * pb.W * 16};
      cuuint32_t box[4] = {8, (cuuint32_t)(sw * px), 1, 1};
      cuuint32_t es[4] = {1, (cuuint32_t)sw, 1, 1};
      r = drv.encodeTiled(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pb.x), dims, strides, box,
                          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
      set_error("tensor map (strip A) failed (" + std::to_string((int)r) + ")");
      return TP_ECUDA;
    }
  }
  {
    cuuint64_t dims[4] = {8, (cuuint64_t)pb.K, (cuuint64_t)pb.S, (cuuint64_t)pb.R};
    cuuint64_t strides[3] = {16, (cuuint64_t)pb.K * 16, (cuuint64_t)pb.S * pb.K * 16};
    cuuint32_t box[4] = {8, (cuuint32_t)pb.bn, (cuuint32_t)pb.S, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = drv.encodeTiled(&plan->tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pb.w), dims,
                                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("tensor map (strip weights) failed (" + std::to_string((int)r) + ")");
      return TP_ECUDA;
    }
  }
  TcArgs& a = plan->args;
  std::memset(&a, 0, sizeof(a));
  a.M = pb.M; a.K = pb.K; a.P = pb.P; a.Q = pb.Q; a.S = pb.S; a.R = pb.R;
  a.sh = pb.sh; a.sw = pb.sw; a.ph = pb.ph; a.pw = pb.pw;
  a.bk = 16; a.stages = pb.stages; a.split_k = 1;
  a.kblocks = pb.R;
  a.H = pb.H; a.W = pb.W; a.C = 8;
  a.nqb = (pb.Q + pb.bm - 1) / pb.bm;
  a.ntiles = pb.N * pb.P * a.nqb;
  a.tpc = pb.tpc > 1 ? pb.tpc : 1;
  a.bias = pb.bias; a.y = pb.y; a.out_f32 = pb.out_f32; a.relu = pb.relu; a.has_bias = pb.has_bias;
  a.trace = pb.trace;
  a.strip_px = px;
  a.strip_stage = sw * phase_bytes;
  const size_t ring = (size_t)pb.stages * a.strip_stage;
  a.strip_woff = (int)((ring + 1023) / 1024 * 1024);
  const size_t wbytes = ((size_t)pb.R * (pb.S + sw) * pb.bn * 16 + 1023) / 1024 * 1024;
  a.bar_off = a.strip_woff + (int)wbytes;
  plan->fn = reinterpret_cast<const void*>(pick_tc(pb.bm, pb.bn, 16, 4));
  if (!plan->fn) { set_error("no strip instantiation for this BM x BN"); return TP_EINVALID_CONFIG; }
  plan->grid = dim3((unsigned)((a.ntiles + a.tpc - 1) / a.tpc), (unsigned)((pb.K + pb.bn - 1) / pb.bn), 1u);
  if (pb.grid_x) plan->grid = dim3(pb.grid_x, pb.grid_y, pb.grid_z);
  plan->block = dim3(a.tpc > 1 && pb.bn >= 128 && mt_epi8() ? 320 : 256);   // + two drain warps (two per quadrant)
  plan->cluster_z = 1;
  plan->smem = (size_t)a.bar_off + 1024;
  // TMA-store epilogue through a staging buffer after the barriers, when it fits
  // (3-D [N P][Q][K] map as in the row kind: q >= Q is clipped).
  static const bool no_ytma = getenv("TP_NO_YTMA") && atoi(getenv("TP_NO_YTMA")) != 0;
  const int eb = pb.out_f32 ? 4 : 2;
  const int ib = pb.bn * eb < 128 ? pb.bn * eb : 128;
  const size_t stage_bytes = (size_t)pb.bm * pb.bn * eb;
  a.y_tma = 0;
  if (!no_ytma && plan->smem + stage_bytes <= 232448 && ((size_t)pb.K * eb) % 16 == 0) {
    cuuint64_t dims[3] = {(cuuint64_t)pb.K, (cuuint64_t)pb.Q, (cuuint64_t)pb.N * pb.P};
    cuuint64_t strides[2] = {(cuuint64_t)pb.K * eb, (cuuint64_t)pb.Q * pb.K * eb};
    cuuint32_t box[3] = {(cuuint32_t)(ib / eb), (cuuint32_t)pb.bm, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapSwizzle swz = ib == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                             : (ib == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    CUresult ry = drv.encodeTiled(&plan->tmY, pb.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                         : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                  3, pb.y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (ry == CUDA_SUCCESS) {
      a.y_tma = 1;
      a.recv_off = (int)plan->smem;
      a.ystage2 = (a.tpc > 1 && ystage2_enabled() && plan->smem + 2 * stage_bytes <= 232448) ? 1 : 0;
      plan->smem += (a.ystage2 ? 2 : 1) * stage_bytes;
    }
  }
  if (!a.y_tma) std::memset(&plan->tmY, 0, sizeof(plan->tmY));
  cudaError_t e = ensure_smem_attr(plan->fn, plan->smem);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return TP_ECUDA;
  }
  return TP_OK;
}

// 3xTF32 kind: fp32 maps (32-channel boxes = 128-B rows, 128-B swizzle), ring of
// hi tiles + twin ring of lo tiles, barriers (full, ready, empty) after the rings.
static tp_status tf32_prepare(const TcProblem& pb, bool a_tiled, TcPlan* plan) {
  const DriverApi& drv = driver();
  CUresult r;
  if (a_tiled) {
    cuuint64_t dims[2] = {(cuuint64_t)pb.C, (cuuint64_t)pb.M};
    cuuint64_t strides[1] = {(cuuint64_t)pb.C * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)pb.bm};
    cuuint32_t es[2] = {1, 1};
    r = drv.encodeTiled(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(pb.x), dims, strides, box,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)pb.C, (cuuint64_t)pb.W, (cuuint64_t)pb.H, (cuuint64_t)pb.N};
    cuuint64_t strides[3] = {(cuuint64_t)pb.C * 4, (cuuint64_t)pb.W * pb.C * 4, (cuuint64_t)pb.H * pb.W * pb.C * 4};
    int lower[2] = {-pb.pw, -pb.ph};
    int upper[2] = {pb.pw - (pb.S - 1), pb.ph - (pb.R - 1)};
    cuuint32_t es[4] = {1, (cuuint32_t)pb.sw, (cuuint32_t)pb.sh, 1};
    r = drv.encodeIm2col(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(pb.x), dims, strides, lower,
                         upper, 32, (cuuint32_t)pb.bm, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    set_error("tensor map (tf32 A) failed (" + std::to_string((int)r) + ")");
    return TP_ECUDA;
  }
  {
    cuuint64_t dims[4] = {(cuuint64_t)pb.C, (cuuint64_t)pb.S, (cuuint64_t)pb.R, (cuuint64_t)pb.K};
    cuuint64_t strides[3] = {(cuuint64_t)pb.C * 4, (cuuint64_t)pb.S * pb.C * 4, (cuuint64_t)pb.R * pb.S * pb.C * 4};
    cuuint32_t box[4] = {32, 1, 1, (cuuint32_t)pb.bn};
    cuuint32_t es[4] = {1, 1, 1, 1};
    r = drv.encodeTiled(&plan->tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(pb.w), dims, strides, box,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("tensor map (tf32 B) failed (" + std::to_string((int)r) + ")");
      return TP_ECUDA;
    }
  }
  TcArgs& a = plan->args;
  std::memset(&a, 0, sizeof(a));
  a.M = pb.M; a.K = pb.K; a.P = pb.P; a.Q = pb.Q; a.S = pb.S;
  a.sh = pb.sh; a.sw = pb.sw; a.ph = pb.ph; a.pw = pb.pw;
  a.bk = 32; a.stages = pb.stages; a.split_k = pb.split_k > 1 ? pb.split_k : 1;
  a.cblocks = (pb.C + 31) / 32;
  a.kblocks = pb.R * pb.S * a.cblocks;
  a.H = pb.H; a.W = pb.W; a.C = pb.C; a.Kg = pb.R * pb.S * pb.C;
  a.bias = pb.bias; a.y = pb.y; a.out_f32 = pb.out_f32; a.relu = pb.relu; a.has_bias = pb.has_bias;
  a.a_tiled = a_tiled ? 1 : 0;
  static const int dbg_env = getenv("TP_DEBUG_TC") ? atoi(getenv("TP_DEBUG_TC")) : 0;
  a.dbg = dbg_env;   // experiments only (bit2: no hi/lo split work, bit3: 1xTF32)
  // [hi rings][lo rings][split-K receive buffer BM x (BN + 4) fp32][barriers]; all 1 KiB multiples.
  a.recv_off = (int)((size_t)pb.stages * (pb.bm + pb.bn) * 256);
  a.bar_off = a.recv_off + (a.split_k > 1 ? pb.bm * (pb.bn + 4) * 4 : 0);
  a.cluster_red = a.split_k > 1 ? 1 : 0;
  plan->fn = pick_tf32(pb.bm, pb.bn);
  if (!plan->fn) { set_error("no igemm_tf32 instantiation for this BM x BN"); return TP_EINVALID_CONFIG; }
  plan->grid = dim3((unsigned)((pb.M + pb.bm - 1) / pb.bm), (unsigned)((pb.K + pb.bn - 1) / pb.bn),
                    (unsigned)a.split_k);
  if (pb.grid_x) plan->grid = dim3(pb.grid_x, pb.grid_y, pb.grid_z);
  plan->block = dim3(256);
  plan->cluster_z = a.split_k;
  plan->smem = (size_t)a.bar_off + 1024;
  cudaError_t e = ensure_smem_attr(plan->fn, plan->smem);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return TP_ECUDA;
  }
  // Split-K reduces only through DSMEM: the (1, 1, split_k) cluster must be
  // co-schedulable in the current context (green contexts may not be able to).
  if (a.split_k > 1 && (plan->grid.z % (unsigned)a.split_k != 0 ||
                        cached_max_clusters(plan->fn, 256, plan->smem, a.split_k) <= 0)) {
    set_error("3xTF32 split-K cluster cannot be co-scheduled in this context");
    return TP_EUNSUPPORTED;
  }
  return TP_OK;
}

// Stem kind: no tensor maps; smem = [weights NSUB x BN x 128 B][2 im2col tiles NSUB x BM x 128 B]
// [input patch, 1 KiB multiple][k table KP x 4 B][barriers] (matches space.cpp stem_smem_bytes).
static tp_status stem_prepare(const TcProblem& pb, TcPlan* plan) {
  std::memset(&plan->tmA, 0, sizeof(plan->tmA));
  std::memset(&plan->tmB, 0, sizeof(plan->tmB));
  std::memset(&plan->tmY, 0, sizeof(plan->tmY));
  TcArgs& a = plan->args;
  std::memset(&a, 0, sizeof(a));
  const int kg = pb.R * pb.S * pb.C;
  const int kp = (kg + 63) / 64 * 64;
  a.M = pb.M; a.K = pb.K; a.P = pb.P; a.Q = pb.Q; a.S = pb.S; a.R = pb.R;
  a.sh = pb.sh; a.sw = pb.sw; a.ph = pb.ph; a.pw = pb.pw;
  a.H = pb.H; a.W = pb.W; a.C = pb.C; a.Kg = kg; a.bk = kp; a.stages = 2; a.split_k = 1;
  a.xg = pb.x; a.wg = pb.w;
  a.bias = pb.bias; a.y = pb.y; a.out_f32 = pb.out_f32; a.relu = pb.relu; a.has_bias = pb.has_bias;
  a.pcols = (pb.bm - 1) * pb.sw + pb.S;
  a.nqb = (pb.Q + pb.bm - 1) / pb.bm;
  a.ntiles = pb.N * pb.P * a.nqb;
  a.tpc = pb.tpc > 1 ? pb.tpc : 1;
  // Two patch buffers of R rows x prow elements (prow = pcols C + 2: a row starts on a 4-byte word).
  a.prow = (a.pcols * pb.C + 3) & ~1;   // even pitch >= pcols C + 1 (row shifted by (pw C) & 1)
  a.pbuf = (int)(((size_t)pb.R * a.prow * 2 + 1023) / 1024 * 1024);
  a.pc_async = ((pb.W * pb.C) % 2 == 0) ? 1 : 0;   // cp.async 4-byte words need even rows
  a.psh = (pb.pw * pb.C) & 1;
  {
    // 16-byte mode: shift each patch row by psh = (-pw C) mod 8 elements so that
    // every tile's row segment starts on a 16-byte boundary (needs BM s_w C and
    // W C multiples of 8, so no 16-byte chunk straddles the image border), with
    // a pitch that is a multiple of 8 -- only when the patch buffer size (and
    // so the validated shared-memory budget) stays the same.
    static const bool no_v16 = getenv("TP_STEM_V16") && atoi(getenv("TP_STEM_V16")) == 0;
    const int sh8 = (8 - (pb.pw * pb.C) % 8) % 8;
    const int prow8 = (a.pcols * pb.C + sh8 + 7) / 8 * 8;
    const int pbuf8 = (int)(((size_t)pb.R * prow8 * 2 + 1023) / 1024 * 1024);
    if (!no_v16 && (pb.bm * pb.sw * pb.C) % 8 == 0 && (pb.W * pb.C) % 8 == 0 && pbuf8 == a.pbuf) {
      a.pc_async = 2;
      a.psh = sh8;
      a.prow = prow8;
    }
  }
  a.patch_off = (int)((size_t)pb.bn * kp * 2 + 2 * (size_t)pb.bm * kp * 2);
  // Output staging for the TMA-store epilogue (the space budgets it at fp32
  // size and two patch buffers; a bf16 output allocates half, which can fit
  // one more CTA per SM, or a third patch buffer: patches run two tiles ahead).
  static const int pdist_env = getenv("TP_STEM_PDIST") ? atoi(getenv("TP_STEM_PDIST")) : 2;
  const size_t budget = (size_t)a.patch_off + 2 * (size_t)a.pbuf + (size_t)(kp * 4 + 1023) / 1024 * 1024 +
                        (size_t)pb.bm * pb.bn * 4;
  const size_t stg = (size_t)pb.bm * pb.bn * (pb.out_f32 ? 4 : 2);
  a.pdist = (pdist_env >= 2 && (size_t)a.patch_off + 3 * (size_t)a.pbuf + (size_t)(kp * 4 + 1023) / 1024 * 1024 +
                                       stg <= budget) ? 2 : 1;
  a.tab_off = a.patch_off + (int)((size_t)(a.pdist + 1) * a.pbuf);
  a.recv_off = (a.tab_off + kp * 4 + 1023) / 1024 * 1024;
  a.bar_off = a.recv_off + (int)stg;
  {
    // Wide path (TcArgs::wide): when s_w C_w = 8 for some C_w in {2, 4, 8} >= C,
    // input row segments are widened to C_w-element (16 / s_w-byte) pixels in a
    // ring of NS = R + 2 s_h slots and read by the MMAs in place.  Layout:
    // [B, K_P' = 64 ceil(R K_r / 64)][ring slots, output staging -- or the raw
    // weights while they are repacked][4 R raw row buffers][barriers | bias at +512].
    static const int dbg = getenv("TP_STEM_DBG") ? atoi(getenv("TP_STEM_DBG")) : 0;
    a.dbg = dbg;
    // Used for spans of >= 4 tiles (TP_STEM_WIDE: 0 never, 2 always): the ring
    // pays off once consecutive tiles share input rows; for 1-2 tiles per CTA
    // the im2col tile starts sooner (ResNet-50 conv1 at 100%: 7.9 us im2col vs
    // 11.6 us ring; VGG-19 conv1_1 b16 at 25%, 16 tiles per CTA: 131 vs 89-92 us).
    static const int wide_env = getenv("TP_STEM_WIDE") ? atoi(getenv("TP_STEM_WIDE")) : 1;
    const int cw = (pb.sw == 1 || pb.sw == 2 || pb.sw == 4) ? 8 / pb.sw : 0;
    a.wide = 0;
    const int ns = pb.R + 2 * pb.sh;
    if ((wide_env == 2 || (wide_env == 1 && a.tpc >= 4)) && cw > 0 && pb.C <= cw && ns <= 16) {
      const int spad = (pb.S * cw + 15) / 16 * 16 / cw;
      const int kr = spad * cw, kpn = (pb.R * kr + 63) / 64 * 64;
      const int pcolsw = (pb.bm - 1) * pb.sw + spad;
      const int wrow = (pcolsw * cw * 2 + 15) / 16 * 16;
      const size_t ring = ((size_t)ns * wrow + 1023) / 1024 * 1024;
      const size_t stg = (size_t)pb.bm * pb.bn * (pb.out_f32 ? 4 : 2);
      const size_t wreg = std::max(ring + stg, ((size_t)pb.bn * kg * 2 + 1023) / 1024 * 1024);
      const size_t bbytes = (size_t)pb.bn * kpn * 2;
      const int rrow = (a.prow * 2 + 15) / 16 * 16;
      const int nraw = 4 * pb.R;   // raw rows of the tiles being widened and copied ahead (kPDT = 2)
      const size_t raw = ((size_t)nraw * rrow + 1023) / 1024 * 1024;
      const size_t total = bbytes + wreg + raw + 512 + (size_t)pb.bn * 4;
      if (kpn <= 256 && total <= 232448) {
        a.wide = cw; a.kr = kr; a.pcolsw = pcolsw; a.wrow = wrow; a.nslots = ns; a.rrow = rrow; a.nraw = nraw;
        static const bool no_fold = getenv("TP_STEM_FOLD") && atoi(getenv("TP_STEM_FOLD")) == 0;
        a.bias_mma = (!no_fold && cw == 8 && pb.C <= 5 && !pb.out_f32) ? 1 : 0;
        a.bk = kpn;
        a.recv_off = (int)(bbytes + ring);
        a.patch_off = (int)(bbytes + wreg);
        a.tab_off = a.patch_off + (int)raw;
        a.bar_off = a.tab_off;
      }
    }
  }
  {
    static const bool no_ytma = getenv("TP_NO_YTMA") && atoi(getenv("TP_NO_YTMA")) != 0;
    const int eb = pb.out_f32 ? 4 : 2;
    const int ib = pb.bn * eb < 128 ? pb.bn * eb : 128;
    cuuint64_t dims[3] = {(cuuint64_t)pb.K, (cuuint64_t)pb.Q, (cuuint64_t)pb.N * pb.P};
    cuuint64_t strides[2] = {(cuuint64_t)pb.K * eb, (cuuint64_t)pb.Q * pb.K * eb};
    cuuint32_t box[3] = {(cuuint32_t)(ib / eb), (cuuint32_t)pb.bm, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = ib == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                            : (ib == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    a.y_tma = 0;
    if (!no_ytma && ((size_t)pb.K * eb) % 16 == 0 &&
        driver().encodeTiled(&plan->tmY, pb.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                             3, pb.y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      a.y_tma = 1;
  }
  plan->fn = pick_stem(pb.bm, pb.bn, a.wide != 0);
  if (!plan->fn) { set_error("no igemm_stem instantiation for this BM x BN"); return TP_EINVALID_CONFIG; }
  plan->grid = dim3((unsigned)((a.ntiles + a.tpc - 1) / a.tpc), (unsigned)((pb.K + pb.bn - 1) / pb.bn), 1u);
  if (pb.grid_x) plan->grid = dim3(pb.grid_x, pb.grid_y, pb.grid_z);
  plan->block = dim3(256);
  plan->cluster_z = 1;
  plan->smem = (size_t)a.bar_off + (a.wide ? 512 : 128) + (size_t)pb.bn * 4;   // + the staged bias
  cudaError_t e = ensure_smem_attr(plan->fn, plan->smem);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return TP_ECUDA;
  }
  return TP_OK;
}

tp_status tc_prepare(const TcProblem& pb, TcPlan* plan) {
  const DriverApi& drv = driver();
  if (pb.stem) return stem_prepare(pb, plan);
  if (pb.strip) return strip_prepare(pb, plan);
  const int sub_k = pb.bk < 64 ? pb.bk : 64;
  static const bool no_atile = getenv("TP_NO_ATILE") && atoi(getenv("TP_NO_ATILE")) != 0;
  const bool a_tiled = !pb.gather && !pb.row && !no_atile && pb.R == 1 && pb.S == 1 && pb.sh == 1 && pb.sw == 1 &&
                       pb.ph == 0 && pb.pw == 0;
  if (pb.tf32) return tf32_prepare(pb, a_tiled, plan);
  if (pb.M > INT32_MAX / 2 || (int64_t)pb.N * pb.H * pb.W * pb.C > INT32_MAX) {
    set_error("tensor too large for 32-bit tile indexing");
    return TP_EUNSUPPORTED;
  }
  if (pb.gather) {
    // Gathered kind: no tensor maps (the kernel never touches tmA / tmB).
    std::memset(&plan->tmA, 0, sizeof(plan->tmA));
    std::memset(&plan->tmB, 0, sizeof(plan->tmB));
  } else if (pb.row) {
    // Row-halo kind: A = tiled map over NHWC x, box (64 channels, BM+2 pixels,
    // 1 row, 1 image), 128-B swizzle; out-of-bounds pixels/rows are zero (pad 1).
    cuuint64_t dims[4] = {(cuuint64_t)pb.C, (cuuint64_t)pb.W, (cuuint64_t)pb.H, (cuuint64_t)pb.N};
    cuuint64_t strides[3] = {(cuuint64_t)pb.C * 2, (cuuint64_t)pb.W * pb.C * 2, (cuuint64_t)pb.H * pb.W * pb.C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)(pb.bm + 2), 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = drv.encodeTiled(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pb.x), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (row strip) failed (" + std::to_string((int)r) + ")");
      return TP_ECUDA;
    }
    cuuint64_t b_dims[4] = {(cuuint64_t)pb.C, (cuuint64_t)pb.S, (cuuint64_t)pb.R, (cuuint64_t)pb.K};
    cuuint64_t b_strides[3] = {(cuuint64_t)pb.C * 2, (cuuint64_t)pb.S * pb.C * 2,
                               (cuuint64_t)pb.R * pb.S * pb.C * 2};
    // CTA pair (resident-weight row kind): each CTA loads half of the BN weight rows
    const bool pair2 = pb.roww && pb.bm == 128 && pb.bn <= 128 && roww_pair_enabled();
    cuuint32_t b_box[4] = {64, 1, 1, (cuuint32_t)(pair2 ? pb.bn / 2 : pb.bn)};
    r = drv.encodeTiled(&plan->tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pb.w), b_dims, b_strides,
                        b_box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (row weights) failed (" + std::to_string((int)r) + ")");
      return TP_ECUDA;
    }
  } else {
  const CUtensorMapSwizzle swz = sub_k == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                             : (sub_k == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUresult r;
  if (a_tiled) {
    // 1x1 / stride 1 / pad 0: im2col is the identity, A = NHWC x viewed as [M][C]
    // (a tiled box issues ~3x faster than an im2col box; rows past M are zero fill).
    cuuint64_t a_dims[2] = {(cuuint64_t)pb.C, (cuuint64_t)pb.M};
    cuuint64_t a_strides[1] = {(cuuint64_t)pb.C * 2};
    cuuint32_t a_box[2] = {(cuuint32_t)sub_k, (cuuint32_t)pb.bm};
    cuuint32_t a_estr[2] = {1, 1};
    r = drv.encodeTiled(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pb.x), a_dims, a_strides,
                        a_box, a_estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, a_promotion(),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (1x1 A) failed (" + std::to_string((int)r) + ")");
      return TP_ECUDA;
    }
  } else {
  // A: im2col over NHWC x, dims (C, W, H, N).
  cuuint64_t a_dims[4] = {(cuuint64_t)pb.C, (cuuint64_t)pb.W, (cuuint64_t)pb.H, (cuuint64_t)pb.N};
  cuuint64_t a_strides[3] = {(cuuint64_t)pb.C * 2, (cuuint64_t)pb.W * pb.C * 2, (cuuint64_t)pb.H * pb.W * pb.C * 2};
  int lower[2] = {-pb.pw, -pb.ph};
  int upper[2] = {pb.pw - (pb.S - 1), pb.ph - (pb.R - 1)};
  cuuint32_t a_estr[4] = {1, (cuuint32_t)pb.sw, (cuuint32_t)pb.sh, 1};
  r = drv.encodeIm2col(&plan->tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pb.x), a_dims,
                       a_strides, lower, upper, (cuuint32_t)sub_k, (cuuint32_t)pb.bm, a_estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, swz, a_promotion(),
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
    return TP_ECUDA;
  }
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
  }
  // TMA-store epilogue (igemm_tc_kernel, split 1): y viewed as [M][K], box
  // (IB / EB columns, BM rows) with the swizzle of IB-byte rows; the tile is
  // staged in the ring, so it must fit there.
  int y_tma = 0;
  {
    static const bool no_ytma = getenv("TP_NO_YTMA") && atoi(getenv("TP_NO_YTMA")) != 0;
    const int eb = pb.out_f32 ? 4 : 2;
    const int ib = pb.bn * eb < 128 ? pb.bn * eb : 128;
    const size_t ring = (size_t)pb.stages * (pb.bm + pb.bn) * pb.bk * 2;
    if (!no_ytma && !pb.row && !pb.mt && pb.split_k == 1 && (size_t)pb.bm * pb.bn * eb <= ring &&
        ((size_t)pb.K * eb) % 16 == 0) {
      cuuint64_t dims[2] = {(cuuint64_t)pb.K, (cuuint64_t)pb.M};
      cuuint64_t strides[1] = {(cuuint64_t)pb.K * eb};
      cuuint32_t box[2] = {(cuuint32_t)(ib / eb), (cuuint32_t)pb.bm};
      cuuint32_t es[2] = {1, 1};
      const CUtensorMapSwizzle sw = ib == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                              : (ib == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
      CUresult ry = drv.encodeTiled(&plan->tmY, pb.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                           : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                    2, pb.y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      y_tma = ry == CUDA_SUCCESS ? 1 : 0;
    }
    if (!y_tma) std::memset(&plan->tmY, 0, sizeof(plan->tmY));
  }
  TcArgs& a = plan->args;
  a.M = pb.M; a.K = pb.K; a.P = pb.P; a.Q = pb.Q; a.S = pb.S;
  a.sh = pb.sh; a.sw = pb.sw; a.ph = pb.ph; a.pw = pb.pw;
  a.bk = pb.bk; a.stages = pb.stages; a.split_k = pb.split_k;
  a.cblocks = (pb.C + pb.bk - 1) / pb.bk;
  a.kblocks = pb.R * pb.S * a.cblocks;
  a.xg = pb.x; a.wg = pb.w;
  a.H = pb.H; a.W = pb.W; a.C = pb.C; a.Kg = pb.R * pb.S * pb.C;
  if (pb.gather) a.kblocks = (a.Kg + pb.bk - 1) / pb.bk;
  a.nqb = 1;
  a.ntiles = 0;
  a.tpc = 1;
  if (pb.mt) {
    a.ntiles = (int)((pb.M + pb.bm - 1) / pb.bm);
    a.tpc = pb.tpc > 1 ? pb.tpc : 1;
  }
  if (pb.row) {
    a.kblocks = (pb.C / 64) * 3;
    a.nqb = (pb.Q + pb.bm - 1) / pb.bm;
    a.ntiles = pb.N * pb.P * a.nqb;
    a.tpc = pb.tpc > 1 ? pb.tpc : 1;
  }
  a.bias = pb.bias; a.y = pb.y; a.out_f32 = pb.out_f32; a.relu = pb.relu; a.has_bias = pb.has_bias;
  a.ws_partial = pb.ws_partial; a.ws_counters = pb.ws_counters;
  a.trace = pb.trace;
  {
    static const int dbg = getenv("TP_DEBUG_TC") ? atoi(getenv("TP_DEBUG_TC")) : 0;
    a.dbg = dbg;
  }
  {
    static const int nprod_env = getenv("TP_NPROD") ? atoi(getenv("TP_NPROD")) : 4;
    a.nprod = nprod_env < 1 ? 1 : nprod_env;   // producer warps cap (experiments: TP_NPROD)
  }
  a.w_early = 0;   // set per launch sequence by the runtime (time_plan / tuner phase B)
  a.ystage2 = 0;
  a.strip_px = a.strip_stage = a.strip_woff = 0;
  a.a_tiled = a_tiled ? 1 : 0;
  a.y_tma = y_tma;
  plan->fn = reinterpret_cast<const void*>(
      pick_tc(pb.bm, pb.bn, pb.bk, pb.mt ? 3 : (pb.row ? 2 : (pb.gather ? 1 : (pb.split_k > 1 ? 6 : 0)))));
  if (!plan->fn) { set_error("no igemm_tc instantiation for this BM x BN x BK"); return TP_EINVALID_CONFIG; }
  plan->grid = (pb.row || pb.mt)
                   ? dim3((unsigned)((a.ntiles + a.tpc - 1) / a.tpc), (unsigned)((pb.K + pb.bn - 1) / pb.bn), 1u)
                      : dim3((unsigned)((pb.M + pb.bm - 1) / pb.bm), (unsigned)((pb.K + pb.bn - 1) / pb.bn),
                             (unsigned)pb.split_k);
  if (pb.grid_x) plan->grid = dim3(pb.grid_x, pb.grid_y, pb.grid_z);
  plan->block = dim3(pb.threads);
  plan->cluster_x = 1;
  // Multi-tile kinds with tiles_per_cta > 1: two more drain warps, so each TMEM
  // lane quadrant has two (the knob stays 256 threads; TP_EPI8=0 turns it off).
  // (BN = 64 with two CTAs per SM lost a CTA to the extra registers; the resident-weight
  //  row kind runs one CTA per SM, so it always takes the eight drain warps.)
  if ((pb.row || pb.mt) && a.tpc > 1 && pb.threads == 256 && (pb.bn >= 128 || pb.roww) && mt_epi8())
    plan->block = dim3(320);
  // N = 64 resident-weight row tiles: a second MMA-issuing warp (TP_MMA2=0: off)
  {
    static const bool no_mma2 = getenv("TP_MMA2") && atoi(getenv("TP_MMA2")) == 0;
    // the two issuers wait on the ring by phase parity: each one's stages must
    // stay within one ring pass of the oldest unfinished fill (stages >= 2 k-blocks per tile)
    if (!no_mma2 && plan->block.x == 320 && pb.row && pb.roww && pb.bn == 64 && !roww_pair_enabled() &&
        a.stages >= 2 * a.kblocks)
      plan->block = dim3(352);
  }
  // Split-K reduces through DSMEM inside a (1, 1, split_k) cluster when the
  // context can co-schedule such clusters; otherwise (e.g. a green context
  // split without SM co-scheduling) through the global workspace.
  a.cluster_red = 0;
  plan->cluster_z = 1;
  if (pb.split_k > 1 && plan->grid.z % (unsigned)pb.split_k == 0 && !getenv("TP_NO_CLUSTER")) {
    const size_t tabs = pb.gather ? (size_t)pb.bm * 16 + (size_t)a.kblocks * pb.bk * 8 : 0;
    const size_t smem_c = tc_bar_off(pb.bm, pb.bn, pb.bk, pb.stages, true, pb.row != 0) + 1024 + tabs;
    if (smem_c <= 232448 && ensure_smem_attr(plan->fn, smem_c) == cudaSuccess &&
        cached_max_clusters(plan->fn, plan->block.x, smem_c, pb.split_k) > 0) {
      a.cluster_red = 1;
      plan->cluster_z = pb.split_k;
    }
  }
  a.bar_off = (int)tc_bar_off(pb.bm, pb.bn, pb.bk, pb.stages, a.cluster_red != 0, pb.row != 0);
  a.recv_off = (int)tc_ring_bytes(pb.bm, pb.bn, pb.bk, pb.stages, pb.row != 0);
  a.roww = 0;
  a.pair2 = 0;
  if (pb.roww) {   // [strip ring][nine resident weight taps][barriers]
    a.roww = 1;
    a.pair2 = (pb.bm == 128 && pb.bn <= 128 && roww_pair_enabled()) ? 1 : 0;   // CTA pair: half the weight rows each
    a.strip_woff = (int)((size_t)pb.stages * (((size_t)(pb.bm + 2) * 128 + 1023) / 1024 * 1024));
    a.bar_off = a.strip_woff + 9 * pb.bn * (a.pair2 ? 64 : 128);
    a.recv_off = a.strip_woff;
    if (a.pair2) {   // (2, 1, 1) clusters; cluster c runs tile pairs [c tpc, c tpc + tpc)
      const int npairs = (a.ntiles + 1) / 2;
      plan->grid.x = 2u * (unsigned)((npairs + a.tpc - 1) / a.tpc);
      plan->cluster_x = 2;
      plan->fn = reinterpret_cast<const void*>(pick_tc(pb.bm, pb.bn, 64, 5));
      if (!plan->fn) { set_error("no CTA-pair row instantiation for this BM x BN"); return TP_EINVALID_CONFIG; }
    }
  }
  a.tab_off = a.bar_off + 1024;
  plan->smem = (size_t)a.tab_off + (pb.gather ? (size_t)pb.bm * 16 + (size_t)a.kblocks * pb.bk * 8 : 0);
  if (pb.row || pb.mt) {
    // Multi-tile kinds: TMA-store epilogue from a staging buffer after the
    // barriers, when it fits in shared memory (a launch-time choice; the space
    // is unchanged).  The ring stays busy with the next tile meanwhile.
    static const bool no_ytma = getenv("TP_NO_YTMA") && atoi(getenv("TP_NO_YTMA")) != 0;
    const int eb = pb.out_f32 ? 4 : 2;
    const int ib = pb.bn * eb < 128 ? pb.bn * eb : 128;
    const size_t stage_bytes = (size_t)pb.bm * pb.bn * eb;
    a.y_tma = 0;
    if (!no_ytma && plan->smem + stage_bytes <= 232448 && ((size_t)pb.K * eb) % 16 == 0) {
      const CUtensorMapSwizzle sw = ib == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                              : (ib == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
      const CUtensorMapDataType dt = pb.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
      CUresult ry;
      if (pb.row) {
        cuuint64_t dims[3] = {(cuuint64_t)pb.K, (cuuint64_t)pb.Q, (cuuint64_t)pb.N * pb.P};
        cuuint64_t strides[2] = {(cuuint64_t)pb.K * eb, (cuuint64_t)pb.Q * pb.K * eb};
        cuuint32_t box[3] = {(cuuint32_t)(ib / eb), (cuuint32_t)pb.bm, 1};
        cuuint32_t es[3] = {1, 1, 1};
        ry = drv.encodeTiled(&plan->tmY, dt, 3, pb.y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[2] = {(cuuint64_t)pb.K, (cuuint64_t)pb.M};
        cuuint64_t strides[1] = {(cuuint64_t)pb.K * eb};
        cuuint32_t box[2] = {(cuuint32_t)(ib / eb), (cuuint32_t)pb.bm};
        cuuint32_t es[2] = {1, 1};
        ry = drv.encodeTiled(&plan->tmY, dt, 2, pb.y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (ry == CUDA_SUCCESS) {
        a.y_tma = 1;
        a.recv_off = (int)((plan->smem + 1023) / 1024 * 1024);
        plan->smem = (size_t)a.recv_off + stage_bytes;
        if (plan->smem > 232448) { a.y_tma = 0; plan->smem = (size_t)a.tab_off; }
        // (a second staging buffer for the row / multi-tile im2col kinds was measured slower:
        //  VGG conv1_2 at 25% 232.7 -> 262.4 us, the extra 16 KiB costs a resident CTA)
      }
    }
  }
  cudaError_t e = ensure_smem_attr(plan->fn, plan->smem);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return TP_ECUDA;
  }
  return TP_OK;
}

cudaError_t tc_launch(const TcPlan& plan, cudaStream_t stream) {
  KernelFn fn = reinterpret_cast<KernelFn>(const_cast<void*>(plan.fn));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = plan.grid;
  cfg.blockDim = plan.block;
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (plan.cluster_x > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = (unsigned)plan.cluster_x;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  } else if (plan.cluster_z > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = (unsigned)plan.cluster_z;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, fn, plan.tmA, plan.tmB, plan.tmY, plan.args);
}

int tc_occupancy(const TcPlan& plan) {
  return cached_occupancy(plan.fn, plan.block.x, plan.smem);
}

}  // namespace tp
