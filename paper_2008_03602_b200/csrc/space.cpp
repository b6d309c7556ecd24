// space.cpp -- host-only schedule space of libtp.
//
// The paper's tuner searches "loop tiles and ordering, caching, and loop
// unrolling ... CUDA threading", picks random candidates when
// it has no data, profiles them and keeps the best per
// operator.  The v0 knob table and validity predicate are DESIGN.md
// "Schedule space v0"; this file and oracle/space.py implement that table
// independently and tests/test_space.py checks them bit-exactly.
#include <algorithm>
#include <unordered_set>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tp_internal.h"

namespace tp {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
const std::string& get_error() { return g_err; }

static int32_t out_dim(int32_t in, int32_t k, int32_t st, int32_t pad, int32_t dil) {
  const int32_t span = in + 2 * pad - dil * (k - 1) - 1;
  if (span < 0 || st < 1) return 0;
  return span / st + 1;
}

int32_t layer_kind(const tp_conv_desc& d) {
  if (d.dtype == TP_DTYPE_BF16 && d.groups == 1 && d.k % 8 == 0 && d.dil_h == 1 && d.dil_w == 1)
    return d.c % 8 == 0 ? TP_KIND_IGEMM_TC : TP_KIND_IGEMM_TC_GATHER;
  return TP_KIND_DIRECT;
}

tp_status make_layer(const tp_conv_desc* d, Layer* L) {
  if (!d) { set_error("null descriptor"); return TP_EINVAL; }
  const tp_conv_desc& x = *d;
  if (x.n < 1 || x.c < 1 || x.h < 1 || x.w < 1 || x.k < 1 || x.r < 1 || x.s < 1 ||
      x.stride_h < 1 || x.stride_w < 1 || x.pad_h < 0 || x.pad_w < 0 || x.dil_h < 1 ||
      x.dil_w < 1 || x.groups < 1) {
    set_error("descriptor has a non-positive extent or negative padding");
    return TP_EINVAL;
  }
  if (x.c % x.groups || x.k % x.groups) { set_error("groups must divide C and K"); return TP_EINVAL; }
  if ((x.in_layout != TP_LAYOUT_NHWC && x.in_layout != TP_LAYOUT_NCHW) ||
      (x.dtype != TP_DTYPE_BF16 && x.dtype != TP_DTYPE_FP32) ||
      (x.out_dtype != TP_DTYPE_BF16 && x.out_dtype != TP_DTYPE_FP32) || (x.epilogue & ~3)) {
    set_error("bad layout / dtype / epilogue code");
    return TP_EINVAL;
  }
  L->d = x;
  L->P = out_dim(x.h, x.r, x.stride_h, x.pad_h, x.dil_h);
  L->Q = out_dim(x.w, x.s, x.stride_w, x.pad_w, x.dil_w);
  if (L->P < 1 || L->Q < 1) { set_error("output size < 1 (reading C3)"); return TP_EINVAL; }
  L->M = (int64_t)x.n * L->P * L->Q;
  L->Cg = x.c / x.groups;
  L->Kg = x.k / x.groups;
  L->kind = layer_kind(x);
  L->depthwise = (x.groups > 1);
  if (x.dil_h != 1 || x.dil_w != 1) { set_error("dilation > 1 is not on the GPU path (C4)"); return TP_EUNSUPPORTED; }
  if (x.groups != 1 && !(x.groups == x.c && x.k == x.c)) {
    set_error("only groups in {1, C} with K == C are on the GPU path (C5)");
    return TP_EUNSUPPORTED;
  }
  return TP_OK;
}

// ---- knob table ----
static const int kTcBM[] = {64, 128};
static const int kTcBN[] = {32, 64, 128, 256};
static const int kTcBK[] = {16, 32, 64, 128};
static const int kTcStages[] = {2, 3, 4, 6};
static const int kTcThreads[] = {128, 256};
static const int kTcSplit[] = {1, 2, 4, 8};
static const int kDThreads[] = {64, 128, 256, 512};
static const int kDTileQ[] = {1, 2, 4};
static const int kDVecK[] = {1, 2, 4, 8};
static const int kDTileP[] = {1, 2, 4, 8};
static const int kDSmem[] = {0, 1};

int64_t tc_smem_bytes(int bm, int bn, int bk, int stages) {
  return (int64_t)stages * (bm + bn) * bk * 2 + 1024;
}

void direct_lanes(const Layer& L, int threads, int tile_q, int vec_k, int tile_p, int* lanes_k, int* lanes_q) {
  const int64_t kv = cdiv(L.d.k, vec_k);
  const int64_t lk = std::min<int64_t>(np2(kv), threads / tile_p);
  *lanes_k = (int)lk;
  *lanes_q = (int)(threads / (lk * tile_p));
}

int64_t direct_smem_bytes(const Layer& L, int threads, int tile_q, int vec_k, int tile_p) {
  int lk, lq;
  direct_lanes(L, threads, tile_q, vec_k, tile_p, &lk, &lq);
  const int64_t qt = (int64_t)lq * tile_q, kt = (int64_t)lk * vec_k;
  const int64_t rows_in = (int64_t)(tile_p - 1) * L.d.stride_h + L.d.r;
  const int64_t cols_in = (qt - 1) * L.d.stride_w + L.d.s;
  if (!L.depthwise) {
    const int64_t cc = std::min<int64_t>(L.d.c, 16);
    return 4 * (rows_in * cols_in * cc + (int64_t)L.d.r * L.d.s * cc * kt);
  }
  return 4 * (rows_in * cols_in * kt + (int64_t)L.d.r * L.d.s * kt);
}

// Gather kind: the reduction axis is R*S*C flattened (c fastest), cut into
// BK-wide k-blocks; the CTA also holds a pixel table (16 B per row) and a
// k table (8 B per padded k).
int64_t tcg_table_bytes(const Layer& L, int bm, int bk) {
  const int64_t kg = (int64_t)L.d.r * L.d.s * L.d.c;
  return (int64_t)bm * 16 + cdiv(kg, bk) * bk * 8;
}

static bool valid_tc(const Layer& L, int bm, int bn, int bk, int stages, int /*threads*/, int split) {
  const bool gather = L.kind == TP_KIND_IGEMM_TC_GATHER;
  const int64_t extra = gather ? tcg_table_bytes(L, bm, bk) : 0;
  if (tc_smem_bytes(bm, bn, bk, stages) + extra > kSmemLimit) return false;
  if (bn > std::max<int64_t>(32, np2(L.d.k))) return false;
  if (bm > std::max<int64_t>(64, np2(L.M))) return false;
  if (gather) {
    const int64_t kg = (int64_t)L.d.r * L.d.s * L.d.c;
    if (bk > std::max<int64_t>(16, np2(kg))) return false;
    return split <= cdiv(kg, bk);
  }
  if (bk > std::max<int64_t>(16, np2(L.d.c))) return false;
  return split <= (int64_t)L.d.r * L.d.s * cdiv(L.d.c, bk);
}

static bool valid_direct(const Layer& L, int threads, int tq, int vk, int tpp, int sm) {
  if (tq > L.Q || tpp > L.P || vk > L.d.k) return false;
  if (L.depthwise && L.d.c % vk) return false;
  if (sm && direct_smem_bytes(L, threads, tq, vk, tpp) > kSmemLimit) return false;
  return true;
}

// Row-halo kind (3x3, stride 1, pad 1, C % 64 == 0, Q >= 56): an output tile
// is BM pixels of ONE output row; per (64-channel block, filter row r) the
// producer loads one input-row strip of BM+2 pixels and the three taps'
// weight tiles, and the MMA reads the three taps as strips shifted by s.
bool row_kind_eligible(const Layer& L) {
  const tp_conv_desc& d = L.d;
  return L.kind == TP_KIND_IGEMM_TC && d.r == 3 && d.s == 3 && d.stride_h == 1 && d.stride_w == 1 &&
         d.pad_h == 1 && d.pad_w == 1 && d.c % 64 == 0 && L.Q >= 56;
}
int64_t row_stage_bytes(int bm, int bn) {
  const int64_t strip = (((int64_t)(bm + 2) * 128) + 1023) / 1024 * 1024;
  return strip + 3 * (int64_t)bn * 128;
}
// Multi-tile im2col kind (TMA-kind layers with >= 1024 tiles of 64 x 32): the
// TMA kind's k-blocks inside the multi-tile pipeline (two TMEM accumulators,
// epilogue of one tile overlapping the mainloop of the next), 256 threads,
// split_k = 1, BK = 64.
bool mt_kind_eligible(const Layer& L) {
  return L.kind == TP_KIND_IGEMM_TC && cdiv(L.M, 64) * cdiv(L.d.k, 32) >= 1024;
}
static const int kMtStages[] = {2, 3, 4};
static const int kMtTpc[] = {2, 4, 8};

static bool valid_mt(const Layer& L, int bm, int bn, int stages) {
  if (tc_smem_bytes(bm, bn, 64, stages) > kSmemLimit) return false;
  if (bn > std::max<int64_t>(32, np2(L.d.k))) return false;
  if (bm > std::max<int64_t>(64, np2(L.M))) return false;
  return 64 <= std::max<int64_t>(16, np2(L.d.c));
}

// Row-halo kind with resident weights (C = 64 layers): the 3 x 3 taps' BN x 64
// weight tiles are loaded once per CTA and the ring carries input strips only,
// so it can run several tiles ahead of the MMA (the strips of the large VGG
// layers come from HBM; weight reloads were most of the L2 -> SMEM traffic).
bool roww_kind_eligible(const Layer& L) { return row_kind_eligible(L) && L.d.c == 64; }
static const int kRowwStages[] = {2, 4, 6, 8};
static const int kRowwTpc[] = {2, 4, 8, 16};
int64_t row_strip_bytes(int bm) { return (((int64_t)(bm + 2) * 128) + 1023) / 1024 * 1024; }
static bool valid_roww(const Layer& L, int bm, int bn, int stages) {
  if ((int64_t)stages * row_strip_bytes(bm) + 9 * (int64_t)bn * 128 + 1024 > kSmemLimit) return false;
  if (bm > np2(L.Q)) return false;
  return bn <= std::max<int64_t>(32, np2(L.d.k));
}

static const int kRowBM[] = {64, 128};
static const int kRowStages[] = {1, 2, 3};
static const int kRowTpc[] = {1, 2, 4, 8, 16};

static bool valid_row(const Layer& L, int bm, int bn, int stages, int threads, int tpc) {
  if ((int64_t)stages * row_stage_bytes(bm, bn) + 1024 > kSmemLimit) return false;
  if (bm > np2(L.Q)) return false;
  if (tpc > 1 && threads != 256) return false;   // warps 2..7 drain while warps 0/1 run ahead
  return bn <= std::max<int64_t>(32, np2(L.d.k));
}

// 3xTF32 tensor-core kind for fp32 dense layers: fp32 NHWC x
// and KRSC w are TMA-loaded (32-channel k-blocks, 128-B rows), split in shared
// memory into tf32 hi/lo parts, and D += A_hi B_hi + A_hi B_lo + A_lo B_hi on
// tcgen05 kind::tf32; appended after the direct tuples; 256 threads.  Split-K
// (1, 2, 4, 8) reduces through DSMEM in a (1, 1, split_k) cluster: the fp32
// receive buffer (BM x (BN + 4) x 4 B) sits after the rings and counts toward
// the shared-memory limit; split_k <= k-blocks = R S ceil(C / 32).
bool tf32_kind_eligible(const Layer& L) {
  const tp_conv_desc& d = L.d;
  return L.kind == TP_KIND_DIRECT && d.dtype == TP_DTYPE_FP32 && d.groups == 1 && d.c % 4 == 0 && d.k % 8 == 0;
}
static const int kTf32Stages[] = {2, 3, 4};
int64_t tf32_smem_bytes(int bm, int bn, int stages, int split) {
  return (int64_t)stages * (bm + bn) * 128 * 2 + (split > 1 ? (int64_t)bm * (bn + 4) * 4 : 0) + 1024;
}
static bool valid_tf32(const Layer& L, int bm, int bn, int stages, int split) {
  if (tf32_smem_bytes(bm, bn, stages, split) > kSmemLimit) return false;
  if (bn > std::max<int64_t>(32, np2(L.d.k))) return false;
  if (bm > std::max<int64_t>(64, np2(L.M))) return false;
  return split <= (int64_t)L.d.r * L.d.s * cdiv(L.d.c, 32);
}

// Stem kind for the C < 8 gathered layers (ResNet-50 conv1, VGG-19 conv1_1,
// MobileNetV2 conv0): a tile is BM output pixels of one output row; three
// producer warps stage the tile's input patch (R rows x ((BM-1) s_w + S) pixels
// x C channels, coalesced) in shared memory and expand it into the swizzled
// im2col tile (k = (r, s, c) flattened, padded to KP = 64 ceil(R S C / 64));
// the BN x KP weight tile stays resident for tiles_per_cta tiles; two TMEM
// accumulators overlap the epilogue of one tile with the next tile's MMAs.
bool stem_kind_eligible(const Layer& L) {
  const tp_conv_desc& d = L.d;
  return L.kind == TP_KIND_IGEMM_TC_GATHER && d.c <= 8 && (int64_t)d.r * d.s * d.c <= 256 && L.Q >= 64;
}
static const int kStemBM[] = {64, 128};
static const int kStemBN[] = {32, 64, 128};
static const int kStemTpc[] = {2, 4, 8, 16};
int64_t stem_kp(const Layer& L) { return cdiv((int64_t)L.d.r * L.d.s * L.d.c, 64) * 64; }
// Two patch buffers (the next tile's patch streams in while this tile's im2col
// tile is built), rows padded by 2 elements (a row starts on a 4-byte word).
int64_t stem_patch_bytes(const Layer& L, int bm) {
  const int64_t cols = (int64_t)(bm - 1) * L.d.stride_w + L.d.s;
  const int64_t prow = (cols * L.d.c + 3) & ~(int64_t)1;   // even row pitch >= cols C + 1
  return 2 * cdiv((int64_t)L.d.r * prow * 2, 1024) * 1024;
}
int64_t stem_smem_bytes(const Layer& L, int bm, int bn) {
  const int64_t kp = stem_kp(L);
  // + the output staging of the TMA-store epilogue (BM x BN at fp32 size, 1 KiB aligned)
  return (int64_t)bn * kp * 2 + 2 * (int64_t)bm * kp * 2 + stem_patch_bytes(L, bm) + cdiv(kp * 4, 1024) * 1024 +
         (int64_t)bm * bn * 4 + 1024;
}
static bool valid_stem(const Layer& L, int bm, int bn) {
  if (stem_smem_bytes(L, bm, bn) > kSmemLimit) return false;
  if (bm > np2(L.Q)) return false;
  return bn <= std::max<int64_t>(32, np2(L.d.k));
}

// Strip kind for the C <= 8 gathered layers ("strip
// kind"): x and w are padded to 8 channels (16-byte pixel rows) by a pre-pass
// inside the call; a tile is BM output pixels of one output row; per filter
// row r one TMA box per column phase (stride s_w in {1, 2}) brings the input
// strip, and one MMA covers two taps of a phase: the no-swizzle K-major core
// matrices of taps t and t + 1 are the strip and the strip one pixel (16 B)
// later (LBO = 16 B).  Weights stay resident; two TMEM accumulators.
bool strip_kind_eligible(const Layer& L) {
  const tp_conv_desc& d = L.d;
  return L.kind == TP_KIND_IGEMM_TC_GATHER && d.c <= 8 && (d.stride_w == 1 || d.stride_w == 2) && d.s <= 8 &&
         d.r <= 8;
}
static const int kStripBM[] = {64, 128};
static const int kStripBN[] = {32, 64, 128};
static const int kStripStages[] = {2, 4, 6};
static const int kStripTpc[] = {1, 2, 4, 8, 16};
// Pixels of one phase box: BM + 2 ceil(T0 / 2) - 1 with T0 = ceil(S / s_w) taps
// in phase 0 (the MMA of the last tap pair reads one row past an odd tap count).
int64_t strip_box_px(const Layer& L, int bm) {
  const int64_t t0 = cdiv(L.d.s, L.d.stride_w);
  return bm + 2 * cdiv(t0, 2) - 1;
}
// s_w = 1: the strip is loaded as whole 512-byte boxes; s_w = 2: one box per
// column phase, each rounded up to 128 bytes.
int64_t strip_stage_bytes(const Layer& L, int bm) {
  if (L.d.stride_w == 1) return cdiv(strip_box_px(L, bm) * 16, 512) * 512;
  return (int64_t)L.d.stride_w * cdiv(strip_box_px(L, bm) * 16, 128) * 128;
}
// Resident weights: per filter row, S taps + s_w zero taps of BN x 16 B.
int64_t strip_weight_bytes(const Layer& L, int bn) {
  return cdiv((int64_t)L.d.r * (L.d.s + L.d.stride_w) * bn * 16, 1024) * 1024;
}
static bool valid_strip(const Layer& L, int bm, int bn, int stages) {
  if (bm > std::max<int64_t>(64, np2(L.Q))) return false;
  if (bn > std::max<int64_t>(32, np2(L.d.k))) return false;
  if ((int64_t)L.d.stride_w * strip_box_px(L, bm) > 256) return false;   // TMA box extent
  return (int64_t)stages * strip_stage_bytes(L, bm) + strip_weight_bytes(L, bn) + 1024 <= kSmemLimit;
}

void fill_geometry(const Layer& L, tp_schedule* s) {
  if (s->kind == TP_KIND_IGEMM_TC_STEM || s->kind == TP_KIND_IGEMM_TC_STRIP) {
    s->grid_x = (int32_t)cdiv((int64_t)L.d.n * L.P * cdiv(L.Q, s->bm), std::max(1, s->tiles_per_cta));
    s->grid_y = (int32_t)cdiv(L.d.k, s->bn);
    s->grid_z = 1;
    return;
  }
  if (s->kind == TP_KIND_IGEMM_TC_MT) {
    s->grid_x = (int32_t)cdiv(cdiv(L.M, s->bm), std::max(1, s->tiles_per_cta));
    s->grid_y = (int32_t)cdiv(L.d.k, s->bn);
    s->grid_z = 1;
  } else if (s->kind == TP_KIND_IGEMM_TC_ROW || s->kind == TP_KIND_IGEMM_TC_ROWW) {
    s->grid_x = (int32_t)cdiv((int64_t)L.d.n * L.P * cdiv(L.Q, s->bm), std::max(1, s->tiles_per_cta));
    s->grid_y = (int32_t)cdiv(L.d.k, s->bn);
    s->grid_z = 1;
  } else if (s->kind == TP_KIND_IGEMM_TC || s->kind == TP_KIND_IGEMM_TC_GATHER || s->kind == TP_KIND_IGEMM_TF32X3) {
    s->grid_x = (int32_t)cdiv(L.M, s->bm);
    s->grid_y = (int32_t)cdiv(L.d.k, s->bn);
    s->grid_z = s->split_k;
  } else {
    int lk, lq;
    direct_lanes(L, s->threads, s->tile_q, s->vec_k, s->tile_p, &lk, &lq);
    s->grid_x = (int32_t)(cdiv(L.Q, (int64_t)lq * s->tile_q) * cdiv(L.P, s->tile_p));
    s->grid_y = (int32_t)cdiv(L.d.k, (int64_t)lk * s->vec_k);
    s->grid_z = L.d.n;
  }
}

// Enumerate in lexicographic order; visit(schedule) returns false to stop.
template <class F>
static void enumerate(const Layer& L, F visit) {
  int64_t idx = 0;
  if (L.kind == TP_KIND_IGEMM_TC || L.kind == TP_KIND_IGEMM_TC_GATHER) {
    for (int bm : kTcBM) for (int bn : kTcBN) for (int bk : kTcBK) for (int st : kTcStages)
      for (int th : kTcThreads) for (int sk : kTcSplit) {
        if (!valid_tc(L, bm, bn, bk, st, th, sk)) continue;
        tp_schedule s; std::memset(&s, 0, sizeof(s));
        s.kind = L.kind; s.bm = bm; s.bn = bn; s.bk = bk; s.stages = st;
        s.threads = th; s.split_k = sk; s.space_index = idx++;
        if (!visit(s)) return;
      }
    // Eligible layers append the row-halo kind after every TMA-kind tuple
    // (BK is fixed at 64, split_k at 1).
    if (row_kind_eligible(L))
      for (int bm : kRowBM) for (int bn : kTcBN) for (int st : kRowStages) for (int th : kTcThreads)
        for (int tpc : kRowTpc) {
          if (!valid_row(L, bm, bn, st, th, tpc)) continue;
          tp_schedule s; std::memset(&s, 0, sizeof(s));
          s.kind = TP_KIND_IGEMM_TC_ROW; s.bm = bm; s.bn = bn; s.bk = 64; s.stages = st;
          s.threads = th; s.split_k = 1; s.tiles_per_cta = tpc; s.space_index = idx++;
          if (!visit(s)) return;
        }
    // ... then the row-halo kind with resident weights (C = 64).
    if (roww_kind_eligible(L))
      for (int bm : kRowBM) for (int bn : kTcBN) for (int st : kRowwStages) for (int tpc : kRowwTpc) {
        if (!valid_roww(L, bm, bn, st)) continue;
        tp_schedule s; std::memset(&s, 0, sizeof(s));
        s.kind = TP_KIND_IGEMM_TC_ROWW; s.bm = bm; s.bn = bn; s.bk = 64; s.stages = st;
        s.threads = 256; s.split_k = 1; s.tiles_per_cta = tpc; s.space_index = idx++;
        if (!visit(s)) return;
      }
    // Gathered stems append the stem kind (after every gathered tuple).
    if (stem_kind_eligible(L))
      for (int bm : kStemBM) for (int bn : kStemBN) for (int tpc : kStemTpc) {
        if (!valid_stem(L, bm, bn)) continue;
        tp_schedule s; std::memset(&s, 0, sizeof(s));
        s.kind = TP_KIND_IGEMM_TC_STEM; s.bm = bm; s.bn = bn; s.bk = (int32_t)stem_kp(L); s.stages = 2;
        s.threads = 256; s.split_k = 1; s.tiles_per_cta = tpc; s.space_index = idx++;
        if (!visit(s)) return;
      }
    // ... then the strip kind.
    if (strip_kind_eligible(L))
      for (int bm : kStripBM) for (int bn : kStripBN) for (int st : kStripStages) for (int tpc : kStripTpc) {
        if (!valid_strip(L, bm, bn, st)) continue;
        tp_schedule s; std::memset(&s, 0, sizeof(s));
        s.kind = TP_KIND_IGEMM_TC_STRIP; s.bm = bm; s.bn = bn; s.bk = 16; s.stages = st;
        s.threads = 256; s.split_k = 1; s.tiles_per_cta = tpc; s.space_index = idx++;
        if (!visit(s)) return;
      }
    // Layers with many tiles append the multi-tile im2col kind last.
    if (mt_kind_eligible(L))
      for (int bm : kTcBM) for (int bn : kTcBN) for (int st : kMtStages) for (int tpc : kMtTpc) {
        if (!valid_mt(L, bm, bn, st)) continue;
        tp_schedule s; std::memset(&s, 0, sizeof(s));
        s.kind = TP_KIND_IGEMM_TC_MT; s.bm = bm; s.bn = bn; s.bk = 64; s.stages = st;
        s.threads = 256; s.split_k = 1; s.tiles_per_cta = tpc; s.space_index = idx++;
        if (!visit(s)) return;
      }
  } else {
    for (int th : kDThreads) for (int tq : kDTileQ) for (int vk : kDVecK) for (int tpp : kDTileP)
      for (int sm : kDSmem) {
        if (!valid_direct(L, th, tq, vk, tpp, sm)) continue;
        tp_schedule s; std::memset(&s, 0, sizeof(s));
        s.kind = TP_KIND_DIRECT; s.threads = th; s.tile_q = tq; s.vec_k = vk; s.tile_p = tpp;
        s.smem_stage = sm; s.split_k = 1; s.space_index = idx++;
        if (!visit(s)) return;
      }
    if (tf32_kind_eligible(L))
      for (int bm : kTcBM) for (int bn : kTcBN) for (int st : kTf32Stages) for (int sk : kTcSplit) {
        if (!valid_tf32(L, bm, bn, st, sk)) continue;
        tp_schedule s; std::memset(&s, 0, sizeof(s));
        s.kind = TP_KIND_IGEMM_TF32X3; s.bm = bm; s.bn = bn; s.bk = 32; s.stages = st;
        s.threads = 256; s.split_k = sk; s.space_index = idx++;
        if (!visit(s)) return;
      }
  }
}

std::vector<tp_schedule> space_all(const Layer& L) {
  std::vector<tp_schedule> out;
  enumerate(L, [&](const tp_schedule& sc) {
    out.push_back(sc);
    fill_geometry(L, &out.back());
    return true;
  });
  return out;
}

int64_t space_size(const Layer& L) {
  int64_t n = 0;
  enumerate(L, [&](const tp_schedule&) { ++n; return true; });
  return n;
}

bool space_get(const Layer& L, int64_t idx, tp_schedule* out) {
  bool found = false;
  enumerate(L, [&](const tp_schedule& s) {
    if (s.space_index == idx) { *out = s; found = true; return false; }
    return true;
  });
  if (found) fill_geometry(L, out);
  return found;
}

bool schedule_in_space(const Layer& L, const tp_schedule& s) {
  auto in_ = [](int v, const int* a, int n) { return std::find(a, a + n, v) != a + n; };
  if (s.kind == TP_KIND_IGEMM_TC_MT)
    return mt_kind_eligible(L) && in_(s.bm, kTcBM, 2) && in_(s.bn, kTcBN, 4) && s.bk == 64 &&
           in_(s.stages, kMtStages, 3) && s.threads == 256 && s.split_k == 1 && in_(s.tiles_per_cta, kMtTpc, 3) &&
           valid_mt(L, s.bm, s.bn, s.stages);
  if (s.kind == TP_KIND_IGEMM_TC_ROW)
    return row_kind_eligible(L) && in_(s.bm, kRowBM, 2) && in_(s.bn, kTcBN, 4) && s.bk == 64 &&
           in_(s.stages, kRowStages, 3) && in_(s.threads, kTcThreads, 2) && s.split_k == 1 &&
           in_(s.tiles_per_cta, kRowTpc, 5) && valid_row(L, s.bm, s.bn, s.stages, s.threads, s.tiles_per_cta);
  if (s.kind == TP_KIND_IGEMM_TC_ROWW)
    return roww_kind_eligible(L) && in_(s.bm, kRowBM, 2) && in_(s.bn, kTcBN, 4) && s.bk == 64 &&
           in_(s.stages, kRowwStages, 4) && s.threads == 256 && s.split_k == 1 &&
           in_(s.tiles_per_cta, kRowwTpc, 4) && valid_roww(L, s.bm, s.bn, s.stages);
  if (s.kind == TP_KIND_IGEMM_TC_STEM)
    return stem_kind_eligible(L) && in_(s.bm, kStemBM, 2) && in_(s.bn, kStemBN, 3) && s.bk == stem_kp(L) &&
           s.stages == 2 && s.threads == 256 && s.split_k == 1 && in_(s.tiles_per_cta, kStemTpc, 4) &&
           valid_stem(L, s.bm, s.bn);
  if (s.kind == TP_KIND_IGEMM_TC_STRIP)
    return strip_kind_eligible(L) && in_(s.bm, kStripBM, 2) && in_(s.bn, kStripBN, 3) && s.bk == 16 &&
           in_(s.stages, kStripStages, 3) && s.threads == 256 && s.split_k == 1 &&
           in_(s.tiles_per_cta, kStripTpc, 5) && valid_strip(L, s.bm, s.bn, s.stages);
  if (s.kind == TP_KIND_IGEMM_TF32X3)
    return tf32_kind_eligible(L) && in_(s.bm, kTcBM, 2) && in_(s.bn, kTcBN, 4) && s.bk == 32 &&
           in_(s.stages, kTf32Stages, 3) && s.threads == 256 && in_(s.split_k, kTcSplit, 4) &&
           valid_tf32(L, s.bm, s.bn, s.stages, s.split_k);
  if (s.kind != L.kind) return false;
  if (s.kind == TP_KIND_IGEMM_TC || s.kind == TP_KIND_IGEMM_TC_GATHER) {
    auto in = [](int v, const int* a, int n) { return std::find(a, a + n, v) != a + n; };
    return in(s.bm, kTcBM, 2) && in(s.bn, kTcBN, 4) && in(s.bk, kTcBK, 4) && in(s.stages, kTcStages, 4) &&
           in(s.threads, kTcThreads, 2) && in(s.split_k, kTcSplit, 4) &&
           valid_tc(L, s.bm, s.bn, s.bk, s.stages, s.threads, s.split_k);
  }
  auto in = [](int v, const int* a, int n) { return std::find(a, a + n, v) != a + n; };
  return in(s.threads, kDThreads, 4) && in(s.tile_q, kDTileQ, 3) && in(s.vec_k, kDVecK, 4) &&
         in(s.tile_p, kDTileP, 4) && in(s.smem_stage, kDSmem, 2) &&
         valid_direct(L, s.threads, s.tile_q, s.vec_k, s.tile_p, s.smem_stage);
}

static uint64_t splitmix64_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Fallback check points of the consensus gate (a10, used when the caller
// passes no oracle points): n distinct flat NKPQ indices drawn uniformly
// without replacement (Floyd's algorithm over SplitMix64 seeded by the output
// size), sorted.  A fixed stride i*total/n is not used: on VGG-19 b16 it is a
// multiple of P*Q, so every point lands in output column q = 0.
std::vector<int64_t> gate_points(const Layer& L, int64_t n) {
  const int64_t total = L.M * L.d.k;
  std::vector<int64_t> out;
  if (total <= n) {
    out.resize(total);
    for (int64_t i = 0; i < total; ++i) out[i] = i;
    return out;
  }
  uint64_t state = 0x7470676174650000ull ^ (uint64_t)total;
  std::unordered_set<int64_t> seen;
  seen.reserve((size_t)n * 2);
  for (int64_t j = total - n; j < total; ++j) {
    const int64_t t = (int64_t)(splitmix64_next(state) % (uint64_t)(j + 1));
    seen.insert(seen.count(t) ? j : t);
  }
  out.assign(seen.begin(), seen.end());
  std::sort(out.begin(), out.end());
  return out;
}

}  // namespace tp

using namespace tp;

extern "C" {

const char* tp_status_str(tp_status s) {
  switch (s) {
    case TP_OK: return "ok";
    case TP_EINVAL: return "invalid argument";
    case TP_EINVALID_CONFIG: return "invalid_config";
    case TP_ECAPACITY: return "capacity";
    case TP_ECUDA: return "server_error";
    case TP_EMISMATCH: return "mismatch";
    case TP_EUNSUPPORTED: return "unsupported";
  }
  return "unknown";
}

const char* tp_last_error(void) { return get_error().c_str(); }

tp_status tp_output_shape(const tp_conv_desc* d, int32_t* p, int32_t* q) {
  Layer L;
  tp_status st = make_layer(d, &L);
  if (st == TP_EINVAL) return st;
  if (p) *p = L.P;
  if (q) *q = L.Q;
  return TP_OK;
}

tp_status tp_layer_kind(const tp_conv_desc* d, int32_t* kind) {
  Layer L;
  tp_status st = make_layer(d, &L);
  if (st != TP_OK) return st;
  *kind = L.kind;
  return TP_OK;
}

tp_status tp_space_size(const tp_conv_desc* d, int64_t* n_valid) {
  Layer L;
  tp_status st = make_layer(d, &L);
  if (st != TP_OK) return st;
  *n_valid = space_size(L);
  return TP_OK;
}

tp_status tp_space_get(const tp_conv_desc* d, int64_t idx, tp_schedule* out) {
  Layer L;
  tp_status st = make_layer(d, &L);
  if (st != TP_OK) return st;
  if (idx < 0 || !space_get(L, idx, out)) {
    set_error("space index out of range");
    return TP_EINVALID_CONFIG;
  }
  return TP_OK;
}

tp_status tp_space_sample(const tp_conv_desc* d, int32_t trials, uint64_t seed, int64_t* idx_out,
                          int32_t cap, int32_t* n_out) {
  Layer L;
  tp_status st = make_layer(d, &L);
  if (st != TP_OK) return st;
  if (trials < 0 || !idx_out || !n_out) { set_error("bad sample arguments"); return TP_EINVAL; }
  const int64_t n = space_size(L);
  const int64_t t = std::min<int64_t>(trials, n);
  if (t > cap) { set_error("sample output capacity too small"); return TP_EINVAL; }
  std::vector<int64_t> a(n);
  for (int64_t i = 0; i < n; ++i) a[i] = i;
  if (trials < n) {
    uint64_t state = seed;
    for (int64_t i = 0; i < t; ++i) {
      const int64_t j = i + (int64_t)(splitmix64_next(state) % (uint64_t)(n - i));
      std::swap(a[i], a[j]);
    }
  }
  for (int64_t i = 0; i < t; ++i) idx_out[i] = a[i];
  *n_out = (int32_t)t;
  return TP_OK;
}

tp_status tp_gate_points(const tp_conv_desc* d, int32_t n, int64_t* idx_out, int32_t cap, int32_t* n_out) {
  Layer L;
  tp_status st = make_layer(d, &L);
  if (st != TP_OK) return st;
  if (n < 0 || !idx_out || !n_out) { set_error("bad gate-point arguments"); return TP_EINVAL; }
  const std::vector<int64_t> v = gate_points(L, n);
  if ((int64_t)v.size() > cap) { set_error("gate-point output capacity too small"); return TP_EINVAL; }
  std::copy(v.begin(), v.end(), idx_out);
  *n_out = (int32_t)v.size();
  return TP_OK;
}

tp_status tp_select_best(const tp_measurement* r, int32_t n, int32_t* best) {
  if (!best || (n > 0 && !r)) { set_error("bad select arguments"); return TP_EINVAL; }
  int32_t b = -1;
  for (int32_t i = 0; i < n; ++i) {
    if (r[i].status != TP_OK) continue;
    if (b < 0 || r[i].median_us < r[b].median_us ||
        (r[i].median_us == r[b].median_us && r[i].space_index < r[b].space_index))
      b = i;
  }
  *best = b;
  return TP_OK;
}

}  // extern "C"
