// tp_kernels.h -- kernel argument blocks and launch plans (internal to libtp).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "tp_internal.h"

namespace tp {

// Driver entry points, resolved at run time through cudaGetDriverEntryPoint so
// that libtp.so loads (and its host-only functions run) without libcuda.
struct DriverApi {
  bool ok = false;
  CUresult (*encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
  CUresult (*encodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                           CUtensorMapFloatOOBfill) = nullptr;
  CUresult (*ctxPush)(CUcontext) = nullptr;
  CUresult (*ctxPop)(CUcontext*) = nullptr;
  CUresult (*ctxGetCurrent)(CUcontext*) = nullptr;
  CUresult (*deviceGet)(CUdevice*, int) = nullptr;
  CUresult (*devicePrimaryCtxRetain)(CUcontext*, CUdevice) = nullptr;
  CUresult (*deviceGetDevResource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*devSmResourceSplitByCount)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                                        unsigned int, unsigned int) = nullptr;
  CUresult (*devResourceGenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
  CUresult (*greenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
  CUresult (*greenCtxDestroy)(CUgreenCtx) = nullptr;
  CUresult (*ctxFromGreenCtx)(CUcontext*, CUgreenCtx) = nullptr;
  CUresult (*greenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
  CUresult (*greenCtxGetDevResource)(CUgreenCtx, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*streamDestroy)(CUstream) = nullptr;
};
const DriverApi& driver();

// Programmatic dependent launch (PDL) for back-to-back kernels in a stream:
// on unless TP_PDL=0.  Kernels call griddepcontrol.wait before reading memory.
bool pdl_enabled();
// Weight prefetch across the PDL wait (TcArgs::w_early) in repeated launches
// of one plan: on unless TP_W_EARLY=0.
bool w_early_enabled();

// Per-(function, context) caches of launch-time queries (host-side hot path of
// the tuner): the max-dynamic-smem attribute and the occupancy calculator.
cudaError_t ensure_smem_attr(const void* fn, size_t smem);
int cached_occupancy(const void* fn, int block, size_t smem);
// cudaOccupancyMaxActiveClusters for a (1, 1, cz) cluster in the current context (0 = cannot launch).
int cached_max_clusters(const void* fn, int block, size_t smem, int cz);

// ---------------------------------------------------------------- igemm_tc
struct TcArgs {
  int64_t M;
  int K, P, Q, S, sh, sw, ph, pw;
  int bk, stages, split_k, cblocks, kblocks;
  const float* bias;
  void* y;
  int out_f32, relu, has_bias;
  float* ws_partial;
  int* ws_counters;
  unsigned long long* trace;   // optional per-CTA timeline (tp_conv2d_trace), nullptr = off
  const void* xg;              // gathered kind: NHWC x and dense [K][R*S*C] weights
  const void* wg;
  int H, W, C, Kg;             // gathered kind: input extent, channels, reduction length R*S*C
  int tab_off;                 // gathered kind: byte offset of the pixel / k tables
  int nqb;                     // row-halo kind: q-blocks per output row, ceil(Q / BM)
  int ntiles, tpc;             // row-halo kind: N*P*nqb tiles, consecutive tiles per CTA
  int slots;                   // multi-tile kinds: > 0 = resident CTA columns of the tuned partition
                               //   (SMs x CTAs/SM / grid.y) when fewer than grid.x; the first `slots`
                               //   CTAs split the tiles into balanced spans, the rest exit (tile_span)
  int cluster_red;             // 1: split-K reduced through DSMEM in a (1,1,split_k) cluster
  int bar_off;                 // byte offset of the mbarriers in dynamic shared memory
  int recv_off;                // byte offset of the split-K receive buffer (cluster path)
  int dbg;                     // TP_DEBUG_TC env (experiments only): bit0 skip A TMA, bit1 skip B TMA;
                               //   stem kind (TP_STEM_DBG): bit0 no patch copies, bit1 no weight repack, bit2 no widening
  int a_tiled;                 // 1: A is a tiled [M][C] map (1x1 / stride 1 / pad 0 layers), not im2col
  int nprod;                   // igemm_tc: cap on TMA producer warps (4 = all available)
  int y_tma;                   // igemm_tc split 1: epilogue staged in the ring smem, TMA 2-D store of y
  int R, pcols, patch_off;     // stem kind: filter rows, patch pixels per row, patch offset in smem
  int prow, pbuf, pc_async;    // stem kind: patch row pitch (elements), bytes per patch buffer, cp.async path
  int pdist;                   // stem kind: patch prefetch distance in tiles (1 or 2; pdist + 1 buffers)
  int bias_mma;                // stem kind, wide path with C_w - C >= 3: the bias enters the MMA as three
                               //   bf16 parts (exact sum) on constant-one channels C..C+2 of the (r, s) =
                               //   (0, 0) tap; the epilogue only converts
  int wide, wrow, nslots, rrow, nraw, pcolsw, kr;   // stem kind, wide path (wide = C_w > 0, s_w C_w = 8):
                               //   input row segments widened to C_w-element pixels in a ring of nslots
                               //   slots (pitch wrow bytes, pcolsw pixels), nraw raw rows rrow bytes apart;
                               //   reduction order k = r K_r + s C_w + c, K_r = S_pad C_w a multiple of
                               //   16; tiles column-major; 0 = im2col tile, k = (r, s, c)
  int psh;                     // stem kind: elements a patch row starts before its first input
                               //   element ((pw C) & 1; (-pw C) mod 8 in the 16-byte mode pc_async = 2)
  int w_early;                 // 1: weight (B) boxes of the first ring pass are issued before
                               //    griddepcontrol.wait -- only when the preceding kernel in the
                               //    stream is a launch of this plan (weights are layer constants)
  int strip_px;                // strip kind: 16-byte pixels per phase box
  int strip_stage;             // strip kind: bytes of one ring stage (s_w phase boxes)
  int strip_woff;              // strip kind: byte offset of the resident weights
  int ystage2;                 // multi-tile kinds: two y staging buffers (TMA-store epilogue)
  int roww;                    // row-halo kind: weights resident at strip_woff (ring = strips only)
  int pair2;                   // roww, BM = 128: CTA pair, cta_group::2 MMAs of 256 rows ((2,1,1) cluster)
};

struct TcProblem {
  const void* x;   // NHWC bf16
  const void* w;   // KRSC bf16
  const float* bias;
  void* y;         // NHWC
  int N, C, H, W, K, R, S, P, Q, sh, sw, ph, pw;
  int64_t M;
  int bm, bn, bk, stages, threads, split_k;
  int grid_x, grid_y, grid_z;
  int out_f32, relu, has_bias;
  float* ws_partial;
  int* ws_counters;
  unsigned long long* trace;
  int gather;      // 1: TP_KIND_IGEMM_TC_GATHER (C % 8 != 0)
  int row;         // 1: TP_KIND_IGEMM_TC_ROW (row-halo strips)
  int tpc;         // row-halo / multi-tile: tiles per CTA
  int mt;          // 1: TP_KIND_IGEMM_TC_MT (im2col multi-tile)
  int tf32;        // 1: TP_KIND_IGEMM_TF32X3 (fp32 NHWC x, KRSC w; 3xTF32 split)
  int stem;        // 1: TP_KIND_IGEMM_TC_STEM (C < 8 stems: staged input patch, resident weights)
  int strip;       // 1: TP_KIND_IGEMM_TC_STRIP (x, w padded to 8 channels in the workspace)
  int roww;        // 1: TP_KIND_IGEMM_TC_ROWW (row-halo with resident weights; row = 1 too)
};

struct TcPlan {
  CUtensorMap tmA, tmB;
  CUtensorMap tmY;   // output [M][K] tiled map for the TMA-store epilogue (TcArgs::y_tma)
  TcArgs args;
  const void* fn = nullptr;
  dim3 grid, block;
  size_t smem = 0;
  int cluster_z = 1;
  int cluster_x = 1;   // roww CTA pairs: (2, 1, 1) clusters
};

tp_status tc_prepare(const TcProblem& pb, TcPlan* plan);
const void* pick_tf32(int bm, int bn);   // igemm_tf32.cu
const void* pick_stem(int bm, int bn, bool wide);   // igemm_stem.cu
cudaError_t tc_launch(const TcPlan& plan, cudaStream_t stream);
int tc_occupancy(const TcPlan& plan);
size_t tc_dyn_smem(int bm, int bn, int bk, int stages);

// ---------------------------------------------------------------- direct
struct DirectArgs {
  const void* x;   // NHWC, bf16 or fp32
  const void* w;   // KRSC
  const float* bias;
  void* y;         // NHWC
  int N, C, H, W, K, R, S, sh, sw, ph, pw, P, Q;
  int tile_p, lanes_k, lanes_q, n_qb, cc;
  int relu, has_bias, out_f32;
};

struct DirectPlan {
  DirectArgs args;
  const void* fn = nullptr;
  dim3 grid, block;
  size_t smem = 0;
};

tp_status direct_prepare(const Layer& L, const tp_schedule& s, const void* x, const void* w, const float* bias,
                         void* y, DirectPlan* plan);
cudaError_t direct_launch(const DirectPlan& plan, cudaStream_t stream);
int direct_occupancy(const DirectPlan& plan);

// ---------------------------------------------------------------- aux kernels
cudaError_t launch_nchw_to_nhwc(const void* src, void* dst, int N, int C, int H, int W, int elem_bytes,
                                cudaStream_t st);
cudaError_t launch_nhwc_to_nchw(const void* src, void* dst, int N, int C, int H, int W, int elem_bytes,
                                cudaStream_t st);
cudaError_t launch_pack_input(const float* x_nchw, void* out, int N, int C, int H, int W, int to_nhwc, int bf16,
                              cudaStream_t st);
cudaError_t launch_pack_weights(const float* w_kcrs, void* out, int K, int Cg, int R, int S, int bf16,
                                cudaStream_t st);
cudaError_t launch_gather(const void* y, int layout_nhwc, int out_f32, int N, int K, int P, int Q,
                          const int64_t* idx, int n, double* vals, cudaStream_t st);
cudaError_t launch_smid_probe(int ctas, int* smids, cudaStream_t st);
cudaError_t launch_copy(const void* src, void* dst, size_t bytes, int grid, cudaStream_t st);
cudaError_t launch_l2_flush(void* buf, size_t bytes, int grid, cudaStream_t st);
cudaError_t launch_pad_c8(const void* x, void* x8, int64_t npix, int C, const void* w, void* w8, int K, int R, int S,
                          int pdl, cudaStream_t st);
cudaError_t launch_empty(int ctas, int threads, int pdl, cudaStream_t st);

}  // namespace tp
