// tc_ptx.cuh -- inline-PTX wrappers shared by the tensor-core conv kernels
// (mbarriers, TMA tiled / im2col loads, tcgen05 MMA / commit / ld, shared-
// memory matrix descriptors, vector NHWC stores).  sm_100a only.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace tp {

// ------------------------------------------------------------- PTX wrappers
static __device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
static __device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
static __device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
static __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TP_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Same wait with a suspend-time hint: the thread sleeps until the phase
// completes (or the hint elapses) instead of re-issuing try_wait, leaving the
// issue slots to the warps doing work (multi-tile kinds: ncu showed ~30% of the
// stall samples and a large share of the instructions in spin loops).
static __device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TP_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TP_WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
static __device__ __forceinline__ void tma_load_im2col_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c,
                                                   int32_t w, int32_t h, int32_t n, uint16_t off_w,
                                                   uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h)
      : "memory");
}
static __device__ __forceinline__ void tma_load_tile_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                 int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// Warp-uniform issue: the whole warp executes these (uniform control flow, so
// descriptors/coordinates stay in uniform registers and no per-instruction
// ELECT loop is generated); only the lane with lead != 0 issues.
static __device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, e;\n\t}"
      : "=r"(pred));
  return pred;
}
static __device__ __forceinline__ void mbar_arrive_expect_tx_p(uint64_t* bar, uint32_t bytes, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes), "r"(lead)
      : "memory");
}
static __device__ __forceinline__ void tma_load_im2col_4d_p(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c,
                                                     int32_t w, int32_t h, int32_t n, uint16_t off_w, uint16_t off_h,
                                                     uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %9, 0;\n\t"
      "@q cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h), "r"(lead)
      : "memory");
}
static __device__ __forceinline__ void tma_load_tile_4d_p(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                   int32_t c1, int32_t c2, int32_t c3, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %7, 0;\n\t"
      "@q cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(lead)
      : "memory");
}
static __device__ __forceinline__ void tma_load_tile_2d_p(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                   int32_t c1, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(lead)
      : "memory");
}
static __device__ __forceinline__ void tma_load_tile_3d_p(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                   int32_t c1, int32_t c2, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %6, 0;\n\t"
      "@q cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(lead)
      : "memory");
}
static __device__ __forceinline__ void tc_mma_p(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(lead)
      : "memory");
}
static __device__ __forceinline__ void tc_mma_tf32_p(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                     uint32_t accumulate, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(lead)
      : "memory");
}
// TMA 2-D tile store shared -> global (bulk group), commit and wait until the
// shared-memory source has been read (the global writes complete with the grid,
// before any dependent grid's griddepcontrol.wait returns).
static __device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
static __device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
static __device__ __forceinline__ void tc_commit_p(uint64_t* bar, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar)),
      "r"(lead)
      : "memory");
}
// ---- CTA pair (cta_group::2): one 256-row MMA over two SMs of a TPC ----
// Both CTAs of the (2, 1, 1) cluster load their own half; the TMA completes its
// bytes on CTA 0's mbarrier (bit 24 of the shared::cluster address selects the
// peer; cleared = rank 0), which the leader's MMA thread waits on.
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
static __device__ __forceinline__ void tma_load_tile_4d_pair_p(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                               int32_t c0, int32_t c1, int32_t c2, int32_t c3,
                                                               uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %7, 0;\n\t"
      "@q cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(lead)
      : "memory");
}
static __device__ __forceinline__ void tc_mma_pair_p(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                     uint32_t accumulate, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(lead)
      : "memory");
}
// Commit the leader's MMAs to the barrier at the same offset in both CTAs.
static __device__ __forceinline__ void tc_commit_pair_p(uint64_t* bar, uint32_t lead) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %2;\n\t}"
      ::"r"(smem_u32(bar)), "r"(lead), "h"((uint16_t)3)
      : "memory");
}
// Arrive on the barrier at this offset in cluster CTA `rank` (release, cluster scope).
static __device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
static __device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
static __device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

static __device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  return remote;
}
// 16-byte store into a peer CTA's shared memory that completes `bytes` on the
// peer's mbarrier (both addresses in the shared::cluster window).
static __device__ __forceinline__ void st_async_v4(uint32_t dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(dst), "r"(a), "r"(b), "r"(c), "r"(d), "r"(bar)
               : "memory");
}
// Store 4 consecutive output channels of row m.
static __device__ __forceinline__ void store4(void* y, int64_t m, int K, int n0, float4 v, int out_f32) {
  if (out_f32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + m * K + n0) = v;
  } else {
    __nv_bfloat162 b0 = __floats2bfloat162_rn(v.x, v.y), b1 = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&b0);
    u.y = *reinterpret_cast<uint32_t*>(&b1);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(y) + m * K + n0) = u;
  }
}
static __device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
static __device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
static __device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
static __device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 consecutive TMEM columns of this warp's lane quadrant, one load + one wait.
static __device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[16], uint32_t (&u)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor, K-major, swizzled (sm100 format: start>>4
// [0,14), LBO>>4 [16,30) (unused for swizzled K-major, =1), SBO>>4 [32,46) =
// 8 rows * row pitch, version 1 at [46,48), layout type at [61,64)).
static __device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t swz_bytes) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(((8u * swz_bytes) >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  const uint64_t layout = swz_bytes == 128 ? 2 : (swz_bytes == 64 ? 4 : 6);
  d |= layout << 61;
  return d;
}

// No-swizzle K-major descriptor (canonical layout ((8, m), (8, 2k)) of 8-row x
// 16-byte core matrices): LBO = byte distance between the two core matrices
// along K, SBO = byte distance between 8-row groups along M / N.  The strip
// kind sets LBO = 16 B on A (tap t + 1 = the strip one pixel later).
static __device__ __forceinline__ uint64_t make_sdesc_plain(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;   // layout type 0 (no swizzle) at [61, 64)
  return d;
}

// Two fp32 values -> packed bf16x2 (RNE, lo in the low half), ReLU fused into the
// conversion (cvt .relu: max(rne(x), 0) == rne(max(x, 0)), rounding is monotone).
template <bool RELU>
static __device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  if constexpr (RELU)
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  else
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// 16 fp32 accumulator words + bias -> 8 packed bf16x2 words (paired adds, FADD2).
template <bool RELU>
static __device__ __forceinline__ void bias_pack16(const uint32_t (&raw)[16], const float (&bv)[16], uint32_t (&pk)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 t = __fadd2_rn(make_float2(__uint_as_float(raw[2 * j]), __uint_as_float(raw[2 * j + 1])),
                                make_float2(bv[2 * j], bv[2 * j + 1]));
    pk[j] = cvt_bf16x2<RELU>(t.x, t.y);
  }
}

// 16 fp32 accumulator words -> 8 packed bf16x2 words (bias already in the accumulator).
template <bool RELU>
static __device__ __forceinline__ void pack16(const uint32_t (&raw)[16], uint32_t (&pk)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) pk[j] = cvt_bf16x2<RELU>(__uint_as_float(raw[2 * j]), __uint_as_float(raw[2 * j + 1]));
}

// Store 16 packed bf16 output channels [n0, n0+16) of row m (two 16-byte stores).
static __device__ __forceinline__ void store16_pk(void* y, int64_t m, int K, int n0, const uint32_t (&pk)[8]) {
  uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(y) + m * K + n0);
  if (n0 + 8 <= K) p[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  if (n0 + 16 <= K) p[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
}

// Store 16 consecutive output channels [n0, n0+16) of row m.
static __device__ __forceinline__ void store16(void* y, int64_t m, int K, int n0, const float (&v)[16], int out_f32) {
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


// Tiles of one CTA in the multi-tile kinds.  Default: `tpc` consecutive tiles
// from blockIdx.x * tpc.  With slots > 0 (fewer resident CTA columns than
// grid.x, see TcArgs::slots) CTA x < slots takes the balanced span
// [x ntiles / slots, (x + 1) ntiles / slots) and the rest get none, so the
// last wave is not a partial one (the grid itself stays the frozen geometry).
static __device__ __forceinline__ void tile_span(int ntiles, int tpc, int slots, int& tile0, int& ntl) {
  const int x = (int)blockIdx.x;
  if (slots > 0) {
    if (x >= slots) { tile0 = ntiles; ntl = 0; return; }
    tile0 = (int)((int64_t)x * ntiles / slots);
    ntl = (int)((int64_t)(x + 1) * ntiles / slots) - tile0;
    return;
  }
  tile0 = x * tpc;
  ntl = ntiles - tile0 < tpc ? ntiles - tile0 : tpc;
}

}  // namespace tp
