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
#include <type_traits>

#include "tp_kernels.h"
#include "tc_ptx.cuh"

namespace tp {

// Wide path helpers (C_w = 8 / s_w channels per widened pixel, compile-time).
// One widened pixel u of a raw row (elements u C + c, c < C; zero past C and
// past the raw columns).
template <int CW, int CC, bool ONES>   // CC: compile-time C (0: runtime C); ONES: TcArgs::bias_mma
__device__ __forceinline__ void widen_px(const uint16_t* raw, uint8_t* wrow, int u, int pcols, int sh1, int C_rt) {
  const int C = CC > 0 ? CC : C_rt;
  uint32_t wv[CW / 2];
#pragma unroll
  for (int q = 0; q < CW / 2; ++q) {   // bf16 1.0 on the bias channels C..C+2
    uint32_t w = 0u;
    if (ONES && 2 * q >= C && 2 * q < C + 3) w |= 0x3F80u;
    if (ONES && 2 * q + 1 >= C && 2 * q + 1 < C + 3) w |= 0x3F800000u;
    wv[q] = w;
  }
  if (u < pcols) {
    const uint16_t* src = raw + sh1 + u * C;
#pragma unroll
    for (int c = 0; c < (CC > 0 ? CC : CW); ++c)
      if (c < C) wv[c >> 1] |= (uint32_t)src[c] << ((c & 1) * 16);
  }
  uint8_t* dst = wrow + (size_t)u * (CW * 2);
  if constexpr (CW == 8) *reinterpret_cast<uint4*>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  else if constexpr (CW == 4) *reinterpret_cast<uint2*>(dst) = make_uint2(wv[0], wv[1]);
  else *reinterpret_cast<uint32_t*>(dst) = wv[0];
}

// One 8-element chunk of a B row in the wide order: pixels s0 .. s0 + 8 / CW - 1
// of filter row r (src = W[n][r][0][0]), CW channels each.
template <int CW>
__device__ __forceinline__ void wide_wchunk(const uint16_t* src, uint32_t (&v)[4], int s0, int S, int C, bool ok) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int s = s0 + j / CW, c = j % CW;
    if (ok && s < S && c < C) v[j >> 1] |= (uint32_t)src[s * C + c] << ((j & 1) * 16);
  }
}

template <int BM, int BN, bool WIDE>   // WIDE: the ring path (TcArgs::wide), else the im2col tile
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
  uint64_t* slot_full = bars + 10;   // wide path: [nslots] input row slot widened (3 producer warps)
  uint64_t* slot_free = bars + 26;   // wide path: [nslots] MMAs reading the slot done (commit)

  int tile0, ntl;
  tile_span(a.ntiles, a.tpc, a.slots, tile0, ntl);
  if (ntl <= 0) return;   // past the resident slots (whole CTA, before any barrier)
  // tp_conv2d_trace (slots as tools/mt_trace.py reads them): 0 entry, 1 after the
  // PDL wait, 2 weights staged, 4+i patch of tile i landed, 36+i im2col tile i
  // built, 12+i MMAs issued, 28+i accumulator ready, 20+i drained, 3 end.
  constexpr int kSlots = 96;
  unsigned long long* trace = a.trace ? a.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * kSlots : nullptr;
  if (trace && threadIdx.x == 0) {
    trace[0] = (unsigned long long)clock64();
    unsigned long long g;
    unsigned sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    trace[63] = g;
    trace[62] = sm;
  }
  const int nbase = blockIdx.y * BN;
  // Patch row r of a tile holds input elements e0 - sh1 .. e0 - sh1 + prow - 1 of
  // input row h0 + r (e0 = (q0 s_w - p_w) C; sh1 = a.psh = (p_w C) & 1 makes the row
  // start on a 4-byte word, since q0 s_w C is even).
  const int C = a.C, prow = a.prow, sh1 = a.psh;   // (16-byte mode: a 16-byte boundary, psh = (-p_w C) mod 8)

  // ring path: the raw copy goes to the output staging buffer (unused until
  // the first drain) when it fits, and the epilogue warps repack it too.
  const bool wraw_b1 = !WIDE && (size_t)BN * a.Kg * 2 <= (size_t)NSUB * A_SUB;
  const bool wraw_stg = WIDE && (size_t)BN * a.Kg * 2 <= (size_t)BM * BN * (a.out_f32 ? 4 : 2);
  uint8_t* wraw = WIDE ? (wraw_stg ? smem_raw + a.recv_off : a_s) : (a_s + (wraw_b1 ? (size_t)NSUB * A_SUB : 0));
  const bool w_epi = !WIDE || wraw_stg;   // who copies and repacks: warps 4-7, else the producer warp(s)
  // (one producer warp for the ring path was tried: VGG conv1_1 86.9 -> 105 us,
  // the per-row copy + widen chain is latency-bound, three warps overlap it)
  constexpr int kProdR = kProd;
  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem_raw) & 1023u) != 0) __trap();
    mbar_init(b_full, w_epi ? 4 : 3);
    for (int i = 0; i < 2; ++i) {
      mbar_init(a_full + i, 3);
      mbar_init(a_empty + i, 1);
      mbar_init(t_full + i, 1);
      mbar_init(t_empty + i, 4);
    }
    for (int i = 0; i < a.nslots; ++i) {
      mbar_init(slot_full + i, 3);
      mbar_init(slot_free + i, 1);
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
  for (int k = threadIdx.x; k < KP && !WIDE; k += blockDim.x) {
    int v = -1;
    if (k < a.Kg) {
      const int c = k % C, rs = k / C, s = rs % a.S, r = rs / a.S;
      v = r * prow + sh1 + s * C + c;
    }
    ktab[k] = v;
  }
  // Raw weights W[nbase, nbase + BN) x [0, K_g) are one contiguous range of
  // global memory: 16-byte cp.async copies into the (not yet used) im2col tile
  // buffers, repacked into the swizzled B tile below.  In repeated launches of
  // one plan (w_early: weights are layer constants) they go out before the PDL wait.
  // im2col path: the raw copy lands in the second tile buffer when it fits and
  // is repacked by the epilogue warps (idle until the first accumulator), so the
  // producers start on the patches at once; the ring path repacks in the producers.
  auto issue_weights = [&](int tid, int nthr) {
    const int nrows = min(BN, a.K - nbase);
    const int64_t wbytes = (int64_t)nrows * a.Kg * 2;
    const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(a.wg) + (int64_t)nbase * a.Kg * 2;
    for (int64_t c = tid; c * 16 < wbytes; c += nthr) {
      const int nb = (int)min((int64_t)16, wbytes - c * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(wraw + c * 16)), "l"(wsrc + c * 16),
                   "r"(nb)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // Raw weights landed (the caller waited for their cp.async group and synced
  // the participating warps): row n of B = W[nbase + n] in reduction order k
  // (zero past K_g / K and in the padding); each participating warp arrives on b_full.
  auto repack_weights = [&](int tid, int nthr) {
    const uint16_t* wst = reinterpret_cast<const uint16_t*>(wraw);
    const int nrows = min(BN, a.K - nbase);
    for (int idx = tid; idx < BN * CH && !(a.dbg & 2); idx += nthr) {
      const int n = idx % BN, ch = idx / BN, k0 = ch * 8;
      uint32_t v[4] = {0u, 0u, 0u, 0u};
      if constexpr (WIDE) {
        // k = r K_r + s C_w + c (K_r = S_pad C_w): zero for s >= S, c >= C
        const int r = k0 / a.kr, s0 = (k0 - r * a.kr) >> (a.wide == 8 ? 3 : (a.wide == 4 ? 2 : 1));
        if (a.wide == 8) wide_wchunk<8>(wst + n * a.Kg + r * a.S * C, v, s0, a.S, C, n < nrows && r < a.R);
        else if (a.wide == 4) wide_wchunk<4>(wst + n * a.Kg + r * a.S * C, v, s0, a.S, C, n < nrows && r < a.R);
        else wide_wchunk<2>(wst + n * a.Kg + r * a.S * C, v, s0, a.S, C, n < nrows && r < a.R);
        if (a.bias_mma && k0 == 0) {
          // bias = b1 + b2 + b3 exactly (three bf16 parts of the fp32 value) on
          // pixel s = 0, channels C..C+2 (C_w = 8: chunk 0 is that pixel)
          const float bf = (a.has_bias && n < nrows) ? __ldg(a.bias + nbase + n) : 0.0f;
          const __nv_bfloat16 b1 = __float2bfloat16_rn(bf);
          const float r1 = bf - __bfloat162float(b1);
          const __nv_bfloat16 b2 = __float2bfloat16_rn(r1);
          const __nv_bfloat16 b3 = __float2bfloat16_rn(r1 - __bfloat162float(b2));
          const uint32_t p1 = __bfloat16_as_ushort(b1), p2 = __bfloat16_as_ushort(b2), p3 = __bfloat16_as_ushort(b3);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int j = c - C;
            const uint32_t pv = j == 0 ? p1 : (j == 1 ? p2 : p3);
            if (j >= 0 && j < 3) v[c >> 1] |= pv << ((c & 1) * 16);
          }
        }
      } else {
        const int lim = n < nrows ? a.Kg - k0 : 0;   // elements j < lim of the chunk are W[n][k0 + j]
        const uint16_t* src = wst + n * a.Kg + k0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < lim) v[j >> 1] |= (uint32_t)src[j] << ((j & 1) * 16);
      }
      const uint32_t off = (uint32_t)n * 128 + ((uint32_t)(((k0 & 63) >> 3) ^ (n & 7)) << 4);
      *reinterpret_cast<uint4*>(b_s + (size_t)(k0 >> 6) * B_SUB + off) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(b_full);
  };
  if (a.w_early) {
    if (w_epi && warp >= 4) issue_weights((int)threadIdx.x - 128, 128);
    else if (!w_epi && warp < 3) issue_weights((int)threadIdx.x, kProdR);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (trace && threadIdx.x == 0) trace[1] = (unsigned long long)clock64();

  if (warp < 3) {
    // ---------------- producers ----------------
    const int pt = threadIdx.x;
    if (warp == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (trace && pt == 0) trace[54] = (unsigned long long)clock64();
    const uint16_t* xg = reinterpret_cast<const uint16_t*>(a.xg);
    if (!w_epi && !a.w_early) issue_weights(pt, kProdR);

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
      if (a.dbg & 1) {
      } else if (a.pc_async == 2) {
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
      for (int r = 0; r < a.R && a.pc_async != 2 && !(a.dbg & 1); ++r) {
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
    if constexpr (WIDE) {
      // ---- wide path: a ring of widened input rows ----
      // Tiles run column-major (q-block outer, output row inner), so tile i + 1
      // (next output row, same q-block) shares R - s_h input rows with tile i:
      // each input row segment (pcolsw pixels of the q-block) is copied and
      // widened once, into ring slot g % NS (g = the CTA's row sequence number),
      // and read in place by the MMAs of every tile that needs it.
      const int NP = a.ntiles / a.nqb, NS = a.nslots;
      uint8_t* slots = a_s;
      uint8_t* rawb = reinterpret_cast<uint8_t*>(patch0);
      struct RowCur { int i, rw, qb, k, nnew, h, n; };
      auto cur_tile = [&](RowCur& c, bool first) {
        const int n = c.rw / a.P, p = c.rw - n * a.P;
        const bool reset = first || p == 0 || a.sh >= a.R;
        c.nnew = reset ? a.R : a.sh;
        c.h = p * a.sh - a.ph + (reset ? 0 : a.R - a.sh);
        c.n = n;
        c.k = 0;
      };
      // Raw copy of one input row segment into raw buffer rb (zero outside the image).
      auto stage_row = [&](int rb, int qb, int n, int h) {
        const int e0 = (qb * BM * a.sw - a.pw) * C - sh1;
        const bool hv = (unsigned)h < (unsigned)a.H;
        const uint16_t* xr = xg + ((int64_t)n * a.H + (hv ? h : 0)) * WC;
        uint16_t* pr = reinterpret_cast<uint16_t*>(rawb + (size_t)rb * a.rrow);
        if (a.pc_async == 2) {
          for (int vi = pt; vi < (prow >> 3); vi += kProdR) {
            const int g = e0 + 8 * vi;
            const bool ok = hv && g >= 0 && g < WC;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(pr + 8 * vi)),
                         "l"(ok ? xr + g : xr), "r"(ok ? 16 : 0)
                         : "memory");
          }
        } else if (a.pc_async == 1) {
          for (int wi = pt; wi < nw; wi += kProdR) {
            const int g = e0 + 2 * wi;
            const bool ok = hv && g >= 0 && g < WC;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(pr + 2 * wi)),
                         "l"(ok ? xr + g : xr), "r"(ok ? 4 : 0)
                         : "memory");
          }
        } else {
          for (int e = pt; e < prow; e += kProdR) {
            const int g = e0 + e;
            pr[e] = (hv && (unsigned)g < (unsigned)WC) ? __ldg(xr + g) : (uint16_t)0;
          }
        }
      };
      // Tile-granular copies: tile i's new input rows (R after a reset, s_h
      // otherwise) are copied as one cp.async group kPDT tiles ahead, then
      // widened together; raw row g lives in raw buffer g % RB.
      constexpr int kPDT = 2;
      const int RB = a.nraw;
      RowCur fc;
      fc.i = 0; fc.qb = tile0 / NP; fc.rw = tile0 - fc.qb * NP;
      cur_tile(fc, true);
      RowCur pc = fc;
      int frb = 0;   // raw buffer of the next row to copy
      auto stage_tile = [&](RowCur& c) {   // copy the new rows of tile c.i, advance c to the next tile
        for (int k = 0; k < c.nnew; ++k) {
          stage_row(frb, c.qb, c.n, c.h + k);
          if (++frb == RB) frb = 0;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (++c.i < ntl) {
          if (++c.rw == NP) { c.rw = 0; ++c.qb; }
          cur_tile(c, false);
        }
      };
      for (int j = 0; j < kPDT; ++j) {
        if (fc.i < ntl) stage_tile(fc);
        else asm volatile("cp.async.commit_group;" ::: "memory");
      }
      if (trace && pt == 0) trace[52] = (unsigned long long)clock64();
      if (!w_epi) {
        asm volatile("cp.async.wait_group 2;" ::: "memory");   // the weights (older than the kPDT tiles)
        asm volatile("bar.sync 1, 96;" ::: "memory");
        repack_weights(pt, kProdR);
      }
      int sl = 0, rbi = 0;             // ring slot / raw buffer of the next row to widen
      uint32_t freeph = 0xFFFFFFFFu;   // bit s: parity that passes slot s's next free wait (first: free)
      const int pw8 = a.pcolsw;
      for (int i = 0; i < ntl; ++i) {
        if (fc.i < ntl) stage_tile(fc);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 2;" ::: "memory");   // tile i's rows landed
        if (trace && pt == 0 && i < 8) trace[4 + i] = (unsigned long long)clock64();
        const int nnew = pc.nnew;
        if (warp == 0) {
          int s2 = sl;
          for (int k = 0; k < nnew; ++k) {
            mbar_wait(slot_free + s2, (freeph >> s2) & 1u);
            if (++s2 == NS) s2 = 0;
          }
        }
        {
          int s2 = sl;
          for (int k = 0; k < nnew; ++k) {
            freeph ^= 1u << s2;
            if (++s2 == NS) s2 = 0;
          }
        }
        asm volatile("bar.sync 1, 96;" ::: "memory");   // every thread's row copies landed, the slots are free
        // widen rows k < nnew: pixel u of row k -> slot (sl + k) % NS
        int k = 0, u = pt;
        while (u >= pw8 && k < nnew) { u -= pw8; ++k; }
        while (k < nnew) {
          int sk = sl + k, rk = rbi + k;
          if (sk >= NS) sk -= NS;
          if (rk >= RB) rk -= RB;
          const uint16_t* rawr = reinterpret_cast<const uint16_t*>(rawb + (size_t)rk * a.rrow);
          uint8_t* wr = slots + (size_t)sk * a.wrow;
          if (a.wide == 8) {
            if (C == 3) {
              if (a.bias_mma) widen_px<8, 3, true>(rawr, wr, u, a.pcols, sh1, C);
              else widen_px<8, 3, false>(rawr, wr, u, a.pcols, sh1, C);
            } else {
              if (a.bias_mma) widen_px<8, 0, true>(rawr, wr, u, a.pcols, sh1, C);
              else widen_px<8, 0, false>(rawr, wr, u, a.pcols, sh1, C);
            }
          } else if (a.wide == 4) {
            if (C == 3) widen_px<4, 3, false>(rawr, wr, u, a.pcols, sh1, C);
            else widen_px<4, 0, false>(rawr, wr, u, a.pcols, sh1, C);
          } else {
            widen_px<2, 0, false>(rawr, wr, u, a.pcols, sh1, C);
          }
          u += kProdR;
          while (u >= pw8 && k < nnew) { u -= pw8; ++k; }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          int s2 = sl;
          for (int k2 = 0; k2 < nnew; ++k2) {
            mbar_arrive(slot_full + s2);
            if (++s2 == NS) s2 = 0;
          }
        }
        if (trace && pt == 0 && i < 8) trace[36 + i] = (unsigned long long)clock64();
        sl += nnew;
        if (sl >= NS) sl -= NS;
        rbi += nnew;
        if (rbi >= RB) rbi -= RB;
        if (pc.i + 1 < ntl) {
          ++pc.i;
          if (++pc.rw == NP) { pc.rw = 0; ++pc.qb; }
          cur_tile(pc, false);
        }
      }
    } else {
    const int PD = a.pdist;
    if (trace && pt == 0) trace[55] = (unsigned long long)clock64();
    for (int j = 0; j < PD; ++j) {
      if (j < ntl) stage_patch(j);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      if (trace && pt == 0) trace[56 + j] = (unsigned long long)clock64();
    }
    if (trace && pt == 0) trace[52] = (unsigned long long)clock64();
    for (int i = 0; i < ntl; ++i) {
      const int b = i & 1;
      const uint16_t* patch = reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(patch0) +
                                                                (size_t)(i % (PD + 1)) * a.pbuf);
      if (i + PD < ntl) stage_patch((i + PD) % (PD + 1));
      else asm volatile("cp.async.commit_group;" ::: "memory");
      if (PD == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else asm volatile("cp.async.wait_group 1;" ::: "memory");
      if (trace && pt == 0 && i < 8) trace[4 + i] = (unsigned long long)clock64();
      // Tile buffer b is free once the MMAs of tile i-2 are done: warp 0 polls,
      // the named barrier releases the other producer warps (and publishes
      // every thread's landed patch copies).
      if (warp == 0) {
        mbar_wait(a_empty + b, ((uint32_t)(i >> 1) & 1u) ^ 1u);
        if (i == (wraw_b1 ? 1 : 0)) mbar_wait(b_full, 0);   // the raw weights in this buffer are repacked
      }
      asm volatile("bar.sync 1, 96;" ::: "memory");
      if (trace && pt == 0 && i < 8) trace[44 + i] = (unsigned long long)clock64();
      uint8_t* at = a_s + (size_t)b * NSUB * A_SUB;
      const int mstep = a.sw * C;
      // Chunk columns past K_g are all padding: when the count of real chunk
      // columns divides 96 they are zeroed on the first use of each of the two
      // tile buffers and skipped afterwards.  Thread pt owns chunk column
      // pt % CHn for rows pt / CHn + j (96 / CHn); its 8 k-table entries stay in
      // registers (CH = KP / 8 in {8, 16, 24, 32} divides 96).
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
      // two rows per pass (sixteen loads in flight before the first use)
      for (int m = pt / CHn; m < BM; m += 2 * rstep) {
        const int m2 = m + rstep;
        const bool two = m2 < BM;
        const uint32_t mo2 = 2u * (uint32_t)(m * mstep), mo2b = 2u * (uint32_t)(m2 * mstep);
        uint32_t e[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint16_t h;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(pa[j] + mo2));
          e[j] = h;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint16_t h = 0;
          if (two) asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(pa[j] + mo2b));
          e[8 + j] = h;
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int mm = hh ? m2 : m;
          if (hh && !two) break;
          uint32_t v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = __byte_perm(e[8 * hh + 2 * q], e[8 * hh + 2 * q + 1], 0x5410) & mk[q];
          const uint32_t off = (uint32_t)mm * 128 + ((cpos ^ (uint32_t)(mm & 7)) << 4);
          *reinterpret_cast<uint4*>(colb + off) = make_uint4(v[0], v[1], v[2], v[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + b);
      if (trace && pt == 0 && i < 8) trace[36 + i] = (unsigned long long)clock64();
      asm volatile("bar.sync 1, 96;" ::: "memory");   // tile i's patch buffer is refilled next iteration
    }
    }
  } else if (warp == 3) {
    // ---------------- MMA issuer ----------------
    const uint32_t lead = elect_one();
    const bool slp = !(a.dbg & 8);
    if (slp) mbar_wait_sleep(b_full, 0); else mbar_wait(b_full, 0);
    const uint64_t bdesc0 = make_sdesc(smem_u32(b_s), 128);
    if constexpr (WIDE) {
      // Wide path: tile i (column-major order) reads input rows gstart .. gstart + R - 1
      // of the ring; A for MMA kk = (filter row r, half h) is a no-swizzle K-major
      // view of slot (gstart + r) % NS at byte 32 h of the q-block's segment --
      // rows 16 B apart (SBO 128 B per 8 rows), the second core matrix 16 B on (LBO).
      const int NP = a.ntiles / a.nqb, NS = a.nslots, hpr = a.kr >> 4;
      const uint32_t slots = smem_u32(a_s), wrow = (uint32_t)a.wrow;
      // ring bookkeeping without divisions: sl0 = gstart % NS, slot parities in a bit mask
      int rw = tile0 % NP, sl0 = 0, slend = 0;   // slend = gend % NS
      uint32_t fullph = 0u;                      // bit s: parity of slot s's next fill
      for (int i = 0; i < ntl; ++i) {
        const int b = i & 1;
        const bool reset = i == 0 || rw % a.P == 0 || a.sh >= a.R;
        int nnew;
        if (reset) { sl0 = slend; nnew = a.R; }
        else { sl0 += a.sh; if (sl0 >= NS) sl0 -= NS; nnew = a.sh; }
        // wait for the new rows (the last nnew of the window)
        int sl = sl0 + a.R - nnew;
        if (sl >= NS) sl -= NS;
        for (int j = 0; j < nnew; ++j) {
          mbar_wait(slot_full + sl, (fullph >> sl) & 1u);
          fullph ^= 1u << sl;
          if (++sl == NS) sl = 0;
        }
        slend = sl;
        if (i >= 2) mbar_wait(t_empty + b, (uint32_t)((i - 2) >> 1) & 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(b * BN);
        uint32_t abase = slots + (uint32_t)sl0 * wrow;
        const uint32_t aend = slots + (uint32_t)NS * wrow;
        int kk = 0;
        for (int r = 0; r < a.R; ++r) {
          for (int h = 0; h < hpr; ++h, ++kk) {
            const uint64_t ad = make_sdesc_plain(abase + 32u * (uint32_t)h, 16u, 128u);
            const uint32_t sb = (uint32_t)(kk >> 2), ko = (uint32_t)((kk & 3) * 32);
            tc_mma_p(d, ad, bdesc0 + ((sb * B_SUB + ko) >> 4), IDESC, kk > 0 ? 1u : 0u, lead);
          }
          abase += wrow;
          if (abase == aend) abase = slots;
        }
        tc_commit_p(t_full + b, lead);
        // rows the next tile does not read go back to the producers
        if (++rw == NP) rw = 0;
        const bool nreset = i + 1 >= ntl || rw % a.P == 0 || a.sh >= a.R;
        const int nfree = nreset ? a.R : a.sh;
        int fs = sl0;
        for (int j = 0; j < nfree; ++j) {
          tc_commit_p(slot_free + fs, lead);
          if (++fs == NS) fs = 0;
        }
        if (trace && lane == 0 && i < 8) trace[12 + i] = (unsigned long long)clock64();
      }
    }
    for (int i = 0; i < ntl && !WIDE; ++i) {
      const int b = i & 1;
      if (slp) mbar_wait_sleep(a_full + b, (uint32_t)(i >> 1) & 1u);
      else mbar_wait(a_full + b, (uint32_t)(i >> 1) & 1u);
      if (i >= 2) {
        if (slp) mbar_wait_sleep(t_empty + b, (uint32_t)((i - 2) >> 1) & 1u);
        else mbar_wait(t_empty + b, (uint32_t)((i - 2) >> 1) & 1u);
      }
      tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)(b * BN);
      const uint64_t adesc0 = make_sdesc(smem_u32(a_s + (size_t)b * NSUB * A_SUB), 128);
      for (int kk = 0; kk < KP / 16; ++kk) {
        const uint32_t sb = (uint32_t)(kk >> 2), ko = (uint32_t)((kk & 3) * 32);
        tc_mma_p(d, adesc0 + ((sb * A_SUB + ko) >> 4), bdesc0 + ((sb * B_SUB + ko) >> 4), IDESC, kk > 0 ? 1u : 0u,
                 lead);
      }
      tc_commit_p(a_empty + b, lead);
      tc_commit_p(t_full + b, lead);
      if (trace && lane == 0 && i < 8) trace[12 + i] = (unsigned long long)clock64();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (warps 4-7) ----------------
    // y_tma: the tile is staged in its own buffer in the swizzled box layout of
    // a 3-D [N P][Q][K] map (q >= Q clipped by the store) and written by one
    // 2-D-per-column-block TMA store; else 16-byte row stores.
    if (w_epi) {
      if (!a.w_early) issue_weights((int)threadIdx.x - 128, 128);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("bar.sync 2, 128;" ::: "memory");
      repack_weights((int)threadIdx.x - 128, 128);
      if (trace && threadIdx.x == 128) trace[2] = (unsigned long long)clock64();
    }
    const int quad = warp & 3;
    const int row = (BM == 128) ? quad * 32 + lane : quad * 16 + lane;
    const bool row_ok = (BM == 128 || lane < 16);
    uint8_t* stg = smem_raw + a.recv_off;
    const uint32_t EB = a.out_f32 ? 4u : 2u;
    const uint32_t IB = BN * EB < 128u ? BN * EB : 128u;
    // Bias of the CTA's BN columns staged once (zero past K and without a
    // bias); ReLU as a max against 0 (or -inf without ReLU).
    float* bias_s = reinterpret_cast<float*>(smem_raw + a.bar_off + (WIDE ? 512 : 128));
    for (int j = (int)threadIdx.x - 128; j < BN; j += 128)
      bias_s[j] = (a.has_bias && nbase + j < a.K) ? __ldg(a.bias + nbase + j) : 0.0f;
    asm volatile("bar.sync 2, 128;" ::: "memory");
    const float lo = a.relu ? 0.0f : __int_as_float(0xff800000u);
    // tile (q-block, output row), advanced per tile: q-block fastest, or (wide
    // path) column-major -- output row fastest
    const int NPe = a.ntiles / a.nqb;
    int e_qb = WIDE ? tile0 / NPe : tile0 % a.nqb;
    int e_prw = WIDE ? tile0 - e_qb * NPe : tile0 / a.nqb;
    for (int i = 0; i < ntl; ++i) {
      const int b = i & 1;
      const int qb = e_qb, prw = e_prw;
      if constexpr (WIDE) {
        if (++e_prw == NPe) { e_prw = 0; ++e_qb; }
      } else if (++e_qb == a.nqb) {
        e_qb = 0;
        ++e_prw;
      }
      const int q = qb * BM + row;
      __syncwarp();
      // One warp polls the accumulator barrier (its lane 0 also retires the
      // previous tile's store of the staging buffer); the other three wait in
      // the named barrier without issuing (ncu: polling warps took ~20% of the
      // issue slots of this issue-bound kernel).
      if (warp == 4) {
        if (a.y_tma && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (a.dbg & 8) mbar_wait(t_full + b, (uint32_t)(i >> 1) & 1u);
        else mbar_wait_sleep(t_full + b, (uint32_t)(i >> 1) & 1u);
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      tc_fence_after();
      if (trace && threadIdx.x == 128 && i < 8) trace[28 + i] = (unsigned long long)clock64();
      if (!a.out_f32 && a.y_tma) {
        // bf16 + TMA store (the stems' case): compile-time staging geometry, ReLU
        // and the bias-in-MMA form chosen once per tile.
        constexpr uint32_t IBf = BN * 2 < 128 ? BN * 2 : 128, SWM = IBf / 16 - 1;
        const uint32_t xr = ((((uint32_t)row * IBf) >> 7) & SWM) << 4;
        uint8_t* rowp = stg + (size_t)row * IBf;
        const uint32_t tb = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * BN);
        auto drain = [&](auto relu_c, auto fold_c) {
          constexpr bool RELU = decltype(relu_c)::value, FOLD = decltype(fold_c)::value;
#pragma unroll
          for (int c = 0; c < BN; c += 16) {
            uint32_t raw[16], pk[8];
            tmem_ld16(tb + (uint32_t)c, raw);
            if constexpr (FOLD) {
              pack16<RELU>(raw, pk);
            } else {
              float bv[16];
#pragma unroll
              for (int g = 0; g < 16; g += 4) {
                const float4 f = *reinterpret_cast<const float4*>(bias_s + c + g);
                bv[g] = f.x; bv[g + 1] = f.y; bv[g + 2] = f.z; bv[g + 3] = f.w;
              }
              bias_pack16<RELU>(raw, bv, pk);
            }
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
        using T = std::integral_constant<bool, true>;
        using F = std::integral_constant<bool, false>;
        if (WIDE && a.bias_mma) {
          if constexpr (WIDE) {
            if (a.relu) drain(T(), T()); else drain(F(), T());
          }
        } else {
          if (a.relu) drain(T(), F()); else drain(F(), F());
        }
      }
#pragma unroll
      for (int c = 0; c < BN && !(!a.out_f32 && a.y_tma); c += 16) {
        uint32_t raw[16];
        tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * BN + c), raw);
        const int nb = nbase + c;
        if (!a.out_f32) {
          // bf16: paired bias adds, one RNE pack per pair with the ReLU fused (cvt .relu)
          float bv[16];
#pragma unroll
          for (int g = 0; g < 16; g += 4) {
            const float4 f = *reinterpret_cast<const float4*>(bias_s + c + g);
            bv[g] = f.x; bv[g + 1] = f.y; bv[g + 2] = f.z; bv[g + 3] = f.w;
          }
          uint32_t pk[8];
          if (a.relu) bias_pack16<true>(raw, bv, pk);
          else bias_pack16<false>(raw, bv, pk);
          if (a.y_tma) {
            if (row_ok) {
              const uint32_t cb = (uint32_t)c * 2u, j = cb / IB, cin = cb % IB;
              uint8_t* sub = stg + (size_t)j * BM * IB;
              const uint32_t swm = IB / 16 - 1;
#pragma unroll
              for (uint32_t qq = 0; qq < 2; ++qq) {
                uint32_t off = (uint32_t)row * IB + cin + qq * 16;
                off ^= ((off >> 7) & swm) << 4;
                *reinterpret_cast<uint4*>(sub + off) = make_uint4(pk[4 * qq], pk[4 * qq + 1], pk[4 * qq + 2], pk[4 * qq + 3]);
              }
            }
          } else if (row_ok && q < a.Q && nb < a.K) {
            uint4* yp = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.y) + ((int64_t)prw * a.Q + q) * a.K + nb);
            if (nb + 8 <= a.K) yp[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            if (nb + 16 <= a.K) yp[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
          continue;
        }
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
      if (trace && threadIdx.x == 128 && i < 8) trace[20 + i] = (unsigned long long)clock64();
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
  }
  tc_fence_before();
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[3] = (unsigned long long)clock64();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
  // the last tile's store must have read the staging buffer before the CTA
  // exits (waited after the TMEM release, which it does not need)
  if (a.y_tma && threadIdx.x == 128) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

const void* pick_stem(int bm, int bn, bool wide) {
#define TP_STEM_CASE(M_, N_) \
  if (bm == M_ && bn == N_)    \
    return wide ? reinterpret_cast<const void*>(igemm_stem_kernel<M_, N_, true>) \
                : reinterpret_cast<const void*>(igemm_stem_kernel<M_, N_, false>);
  TP_STEM_CASE(64, 32) TP_STEM_CASE(64, 64) TP_STEM_CASE(64, 128)
  TP_STEM_CASE(128, 32) TP_STEM_CASE(128, 64) TP_STEM_CASE(128, 128)
#undef TP_STEM_CASE
  return nullptr;
}

}  // namespace tp
