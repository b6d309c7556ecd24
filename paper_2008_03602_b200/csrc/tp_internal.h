// tp_internal.h -- shared declarations inside libtp (not part of the ABI).
#pragma once
#include <cstdint>
#include <cstddef>
#include <string>
#include <vector>
#include "../../include/tp.h"

namespace tp {

// Thread-local error message (tp_last_error).
void set_error(const std::string& msg);
const std::string& get_error();

// Derived per-layer quantities.
struct Layer {
  tp_conv_desc d;
  int32_t P, Q;
  int64_t M;      // GEMM M = N*P*Q (output pixels)
  int32_t Cg, Kg; // channels per group
  int32_t kind;   // TP_KIND_*
  bool depthwise;
};

// Validate + derive.  Returns TP_OK, TP_EINVAL or TP_EUNSUPPORTED.
tp_status make_layer(const tp_conv_desc* d, Layer* L);
int32_t layer_kind(const tp_conv_desc& d);

// Space (space.cpp).
int64_t space_size(const Layer& L);
bool space_get(const Layer& L, int64_t idx, tp_schedule* out);
std::vector<tp_schedule> space_all(const Layer& L);   // the whole valid space in order, one pass
void fill_geometry(const Layer& L, tp_schedule* s);
void direct_lanes(const Layer& L, int threads, int tile_q, int vec_k, int tile_p, int* lanes_k, int* lanes_q);
int64_t direct_smem_bytes(const Layer& L, int threads, int tile_q, int vec_k, int tile_p);
int64_t tc_smem_bytes(int bm, int bn, int bk, int stages);
int64_t tcg_table_bytes(const Layer& L, int bm, int bk);   // gather kind: pixel + k tables
bool row_kind_eligible(const Layer& L);                     // row-halo kind applies
bool roww_kind_eligible(const Layer& L);                    // row-halo kind with resident weights (C = 64)
int64_t row_strip_bytes(int bm);                            // row-halo kinds: one input strip (1 KiB multiple)
bool mt_kind_eligible(const Layer& L);                      // multi-tile im2col kind applies
bool tf32_kind_eligible(const Layer& L);
bool stem_kind_eligible(const Layer& L);                    // stem kind applies (C < 8 gathered layers)
bool strip_kind_eligible(const Layer& L);                   // strip kind applies (C <= 8 gathered layers)
int64_t strip_box_px(const Layer& L, int bm);               // strip kind: pixels per phase box
int64_t strip_stage_bytes(const Layer& L, int bm);          // strip kind: one ring stage (all phase boxes)
int64_t strip_weight_bytes(const Layer& L, int bn);         // strip kind: resident weights
int64_t stem_kp(const Layer& L);                            // stem kind: reduction padded to 64 (R S C)
int64_t stem_patch_bytes(const Layer& L, int bm);                    // 3xTF32 tensor-core kind applies (fp32 dense)
int64_t tf32_smem_bytes(int bm, int bn, int stages, int split);
int64_t row_stage_bytes(int bm, int bn);                    // row-halo kind: one pipeline stage
bool schedule_in_space(const Layer& L, const tp_schedule& s);
std::vector<int64_t> gate_points(const Layer& L, int64_t n);   // consensus-gate fallback points (a10)

constexpr int64_t kSmemLimit = 232448;  // 227 KiB per CTA

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t np2(int64_t v) { int64_t p = 1; while (p < v) p *= 2; return p; }

}  // namespace tp
