/*
 * tp.h -- C ABI of libtp: SM-share-aware conv2d autotuning on B200 (sm_100a).
 *
 * The three calls of the paper's problem statement (arXiv 2008.03602):
 *   - run a conv2d operator with a schedule under a GPU% limit
 *       PAPER.md P:175 (GPU% = number of SMs an application can use), P:378,
 *       P:388 (conv2d "operator"), P:254 (2D convolution)          -> tp_conv2d_run
 *   - tune an operator at a GPU% to its best configuration
 *       P:257-267 (select -> build -> profile -> search), P:586 (fixed trials
 *       per operator), P:841 (combine per-operator best results)     -> tp_tune / tp_tune_subset
 *   - infer with a schedule tuned at p% under a q% limit
 *       P:385-399 (tuned-at-p x inferred-at-q tables T1-T3),
 *       P:560-566 (thread counts frozen at tuning time)             -> tp_cross_eval
 * plus the spatial partitioner that gives each tuner a fixed SM share
 *       P:175, P:378, P:832-834 (TSI scaling with distinct GPU%)    -> tp_partition_*
 *
 * Conventions (all functions):
 *   - Every function returns tp_status; nothing throws or aborts across the ABI.
 *     On failure a thread-local message is available from tp_last_error().
 *   - Device pointers (x, w, bias, y, ws) are 16-byte aligned (tensor-core
 *     kinds; TP_EINVAL otherwise) device memory of the *primary*
 *     context of `device` (e.g. PyTorch allocations); the caller owns them.
 *     Host arrays (records, check_*, out structs) are owned by the caller.
 *   - libtp owns green contexts, their streams and events, TMA descriptors and
 *     the kernel instantiation table; tp_shutdown() frees them.
 *   - Host-only functions (tp_space_*, tp_output_shape, tp_select_best,
 *     tp_gate_points, tp_search_next, tp_search_should_stop, tp_status_str, tp_last_error) never
 *     touch the GPU and work without one.
 *   - Threading: one tuner thread per partition; calls on *different*
 *     partitions may run concurrently from different host threads (a green
 *     context may be current to one thread at a time, cuda.h cuGreenCtxCreate).
 *
 * Layouts:
 *   x : NHWC (in_layout = TP_LAYOUT_NHWC) or NCHW (TP_LAYOUT_NCHW; a transpose
 *       pre-pass into the workspace runs inside the call and is timed with it)
 *   w : KRSC = [K][R][S][C/groups], dtype = desc.dtype
 *   bias : fp32 [K] (read iff epilogue bit0)
 *   y : same layout as x, dtype = desc.out_dtype
 */
#ifndef TP_H_
#define TP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TP_OK = 0,
    TP_EINVAL = 1,            /* bad descriptor / argument (readings C3-C6)             */
    TP_EINVALID_CONFIG = 2,   /* schedule not in the layer's space          */
    TP_ECAPACITY = 3,         /* requested SM partition cannot be granted   */
    TP_ECUDA = 4,             /* driver / launch error ("server_error")      */
    TP_EMISMATCH = 5,         /* correctness gate failed        */
    TP_EUNSUPPORTED = 6       /* valid conv, not on the GPU path (e.g. dilation > 1)     */
} tp_status;

enum { TP_LAYOUT_NHWC = 0, TP_LAYOUT_NCHW = 1 };
enum { TP_DTYPE_BF16 = 0, TP_DTYPE_FP32 = 1 };
enum { TP_EPI_BIAS = 1, TP_EPI_RELU = 2 };
/* Kernel kinds: IGEMM_TC = tcgen05 implicit GEMM fed by
 * TMA im2col (bf16, g = 1, C % 8 == 0); DIRECT = CUDA-core FFMA direct conv
 * (fp32, depthwise); IGEMM_TC_GATHER = tcgen05 implicit GEMM whose A/B tiles
 * are gathered into shared memory by CUDA-core warps over the flattened
 * (r, s, c) axis (bf16, g = 1, C % 8 != 0: the C = 3 stems). */
enum { TP_KIND_IGEMM_TC = 0, TP_KIND_DIRECT = 1, TP_KIND_IGEMM_TC_GATHER = 2, TP_KIND_IGEMM_TC_ROW = 3,
       TP_KIND_IGEMM_TC_MT = 4, TP_KIND_IGEMM_TF32X3 = 5, TP_KIND_IGEMM_TC_STEM = 6, TP_KIND_IGEMM_TC_STRIP = 7,
       TP_KIND_IGEMM_TC_ROWW = 8 };
/* IGEMM_TC_ROWW ("row-halo, resident weights"): appended after the IGEMM_TC_ROW
 * tuples of row-halo layers with C = 64.  The nine taps' BN x 64 weight tiles
 * are loaded once per CTA; the ring carries input strips only.  Knobs BM
 * {64, 128}, BN {32..256}, stages (strips in flight) {2, 4, 6, 8},
 * tiles_per_cta {2, 4, 8, 16}; bk = 64, threads = 256, split_k = 1; grid as
 * IGEMM_TC_ROW. */
/* IGEMM_TC_STRIP ("strip"): appended after the gathered (and stem) tuples of
 * gathered layers with C <= 8, stride_w in {1, 2}, R, S <= 8.  A pre-pass inside
 * the call pads x to NHWC with 8 channels and w to [K][R][S][8] (16-byte pixel
 * rows, in the workspace); a tile is BM pixels of one output row; per filter row
 * one TMA box per column phase brings the input strip (element stride s_w) and
 * one MMA covers two taps of a phase (no-swizzle K-major core matrices 16 B
 * apart along K).  Knobs BM {64, 128}, BN {32, 64, 128}, stages {2, 4, 6},
 * tiles_per_cta {1, 2, 4, 8, 16}; bk = 16, threads = 256, split_k = 1;
 * grid = (ceil(N P ceil(Q / BM) / tiles_per_cta), ceil(K / BN), 1). */
/* IGEMM_TC_MT ("multi-tile im2col"): appended last to the space of IGEMM_TC
 * layers with ceil(M/64)*ceil(K/32) >= 1024.  The IGEMM_TC k-blocks (one TMA
 * im2col box + one weight box per (channel block, tap), BK = 64) run in the
 * multi-tile pipeline of the row-halo kernel: tiles_per_cta in {2, 4, 8}
 * consecutive BM-pixel tiles per CTA, two TMEM accumulators, 256 threads,
 * split_k = 1; stages in {2, 3, 4}.  grid = (ceil(ceil(M/BM)/tpc), ceil(K/BN), 1). */
/* IGEMM_TC_ROW ("row-halo"): an extra schedule kind appended to the space of
 * IGEMM_TC layers with 3x3 filters, stride 1, pad 1, C % 64 == 0 and Q >= 56.
 * A tile is BM pixels of one output row; per (64-channel block, filter row)
 * one TMA loads the BM+2-pixel input strip once and the MMA reads the three
 * taps as the strip shifted by 0/1/2 pixels (the im2col A tile is never
 * re-fetched per tap).  Knobs BM, BN, stages, threads, tiles_per_cta (a CTA
 * runs that many consecutive tiles, alternating two TMEM accumulators so one
 * drains while the other fills; > 1 needs 256 threads); BK = 64, split_k = 1;
 * grid = (ceil(N*P*ceil(Q/BM) / tiles_per_cta), ceil(K/BN), 1). */

/* One conv2d operator ("tuning task", P:947 [src]).  P/Q follow reading C3:
 * P = floor((h + 2 pad_h - dil_h (r-1) - 1) / stride_h) + 1; P < 1 -> TP_EINVAL. */
typedef struct {
    int32_t n, c, h, w, k, r, s;
    int32_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w, groups;
    int32_t in_layout;   /* TP_LAYOUT_*                       */
    int32_t dtype;       /* input/weight dtype, TP_DTYPE_*     */
    int32_t out_dtype;   /* output dtype, TP_DTYPE_*           */
    int32_t epilogue;    /* bit0 bias, bit1 relu (TP_EPI_*)    */
} tp_conv_desc;

/* One configuration of the operator's schedule space (P:256 knobs; DESIGN.md
 * "Schedule space v0").  IGEMM_TC uses bm,bn,bk,stages,threads,split_k; DIRECT
 * uses threads,tile_q,vec_k,tile_p,smem_stage.  grid_* is the frozen launch
 * geometry (reading C15): filled by tp_space_get, reused by tp_cross_eval. */
typedef struct {
    int32_t kind;
    int32_t bm, bn, bk, stages, threads, split_k;
    int32_t tile_q, vec_k, tile_p, smem_stage;
    int32_t tiles_per_cta;                     /* IGEMM_TC_ROW: consecutive tiles per CTA (1..16); 0 otherwise */
    int64_t space_index;                       /* rank in the layer's valid space */
    int32_t grid_x, grid_y, grid_z, sm_tuned;  /* frozen geometry; sm_tuned = SMs at tune time */
} tp_schedule;

/* One profiled configuration ("measures the execution time"; the
 * thread/wave fields are the paper's thread-count mechanism). */
typedef struct {
    double median_us, min_us, mean_us, std_us;   /* per-launch latency over groups (C12) */
    int32_t n_per_group, groups;
    int32_t sm_requested, sm_granted, device, status;   /* status: tp_status of this candidate */
    int64_t space_index;
    int64_t ctas;
    int32_t threads_per_cta, waves, ctas_per_sm, kind;
    double max_abs_err, max_ref;                 /* correctness gate (a10)               */
} tp_measurement;

/* Timing protocol (reading C12). NULL -> defaults {3, 5, 10, 20.0, 1, 0, 2.0}. */
typedef struct {
    int32_t warmup;           /* untimed launches before timing                      */
    int32_t groups;           /* r: number of timed groups (median over groups)      */
    int32_t n_min;            /* minimum launches per group                          */
    double target_group_us;   /* n = max(n_min, ceil(target / t_est))                */
    int32_t use_graph;        /* capture each group's n launches as one CUDA graph    */
    int32_t flush_l2;         /* 1: write a > L2 buffer before every launch (cold L2) */
    double prune_ratio;       /* tuner only (reading C12b): a candidate whose gate-run time
                                 exceeds prune_ratio x the fastest gate-run time of the same
                                 tp_tune / tp_tune_subset call is "raced": one warm-up and ONE
                                 group of n = max(min(3, n_min), ceil(target / t_est))
                                 launches (its record says groups = 1); a raced candidate that
                                 beats every fully-timed one is re-timed with the full
                                 protocol.  0 = every candidate gets the full protocol.
                                 Default 2.0.                                                */
} tp_timing;

typedef struct tp_partition tp_partition;   /* opaque: green context + stream (or whole device) */

/* ---- library lifetime -------------------------------------------------- */
tp_status tp_init(int32_t device);          /* idempotent; primary context + driver entry points */
void tp_shutdown(void);                     /* destroys cached partitions, events, buffers       */
const char* tp_status_str(tp_status s);
const char* tp_last_error(void);            /* thread-local message of the last failure          */
int64_t tp_launch_count(void);              /* kernels launched by libtp so far (all threads)    */

/* ---- partitions: "GPU%" as an SM share ------------
 * tp_partition_get: cached per (device, fraction, flags) -- created once and
 * reused, the long-lived-server analog of P:844-846.  fraction in (0, 1];
 * 1.0 -> whole device (no green context, own non-blocking stream).
 * requested = floor(sm_count * fraction) (reading C14); the granted count is
 * what the driver returns (multiples of 8 unless flags has
 * TP_PART_FINE_GRAINED = CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING).
 * TP_ECAPACITY if the driver cannot grant at least `requested` SMs. */
enum { TP_PART_FINE_GRAINED = 1 };
tp_status tp_partition_get(int32_t device, double fraction, int32_t flags, tp_partition** part,
                           int32_t* sm_requested, int32_t* sm_granted);
/* k disjoint partitions of sms_each SMs from ONE split (config 4: concurrent
 * tuners).  parts[k], granted[k] filled.  Not cached: close each. */
tp_status tp_partition_split(int32_t device, int32_t k, int32_t sms_each, int32_t flags,
                             tp_partition** parts, int32_t* granted);
/* k UNPARTITIONED handles on the whole device (the default-MPS
 * analog -- concurrent tuners with no SM isolation): each has its own
 * non-blocking stream in the primary context and sm_granted = the device's SM
 * count; the SMs are shared by whatever runs concurrently.  parts[k] filled.
 * Not cached: close each with tp_partition_close. */
tp_status tp_partition_shared(int32_t device, int32_t k, tp_partition** parts);
tp_status tp_partition_info(tp_partition* part, int32_t* device, int32_t* sm_requested,
                            int32_t* sm_granted, void** cu_stream);
tp_status tp_partition_sync(tp_partition* part);
tp_status tp_partition_close(tp_partition* part);   /* only for tp_partition_split handles */
/* %smid probe: launches `ctas` CTAs in the partition, each writes its SM id
 * to smids[i] (device int32 buffer).  Used to verify partition membership. */
tp_status tp_partition_probe(tp_partition* part, int32_t ctas, int32_t* smids_dev);
/* STREAM-copy probe inside the partition: copies `bytes` from src to dst
 * (device buffers) `reps` times; returns the best achieved GB/s (read+write). */
tp_status tp_partition_copy_bw(tp_partition* part, const void* src, void* dst, size_t bytes,
                               int32_t reps, double* gbps);

/* Latency floor of the timing protocol inside the partition (SURVEY 8(d):
 * the binding roof of a microsecond kernel is max(compute, HBM, this floor)).
 * Times an EMPTY kernel of `ctas` x `threads` launched exactly like the conv
 * kernels (same stream, PDL attribute, graph-captured groups, timing == NULL
 * -> the C12 defaults) and returns the per-launch statistics in *out
 * (space_index = -1, kind = 0).  Synchronous. */
tp_status tp_partition_floor(tp_partition* part, int32_t ctas, int32_t threads, const tp_timing* timing,
                             tp_measurement* out);

/* ---- schedule space (host-only) ------------ */
tp_status tp_output_shape(const tp_conv_desc* d, int32_t* p, int32_t* q);
tp_status tp_layer_kind(const tp_conv_desc* d, int32_t* kind);
tp_status tp_space_size(const tp_conv_desc* d, int64_t* n_valid);
tp_status tp_space_get(const tp_conv_desc* d, int64_t idx, tp_schedule* out);
/* trials >= |space| -> 0..n-1 in order; else SplitMix64(seed) partial
 * Fisher-Yates (reading C17).  *n_out = min(trials, |space|) <= cap. */
tp_status tp_space_sample(const tp_conv_desc* d, int32_t trials, uint64_t seed,
                          int64_t* idx_out, int32_t cap, int32_t* n_out);
/* Check points of the consensus gate (a10, used by tp_tune* when n_check == 0):
 * min(n, N*K*P*Q) distinct flat NKPQ logical indices, drawn uniformly without
 * replacement (Floyd's algorithm over SplitMix64 seeded by the output size),
 * sorted ascending.  *n_out <= cap; TP_EINVAL if cap is too small. */
tp_status tp_gate_points(const tp_conv_desc* d, int32_t n, int64_t* idx_out, int32_t cap, int32_t* n_out);
/* argmin over status==TP_OK records by median_us, ties -> lowest space_index
 * (reading C13).  *best = index into records, or -1 if none is OK. */
tp_status tp_select_best(const tp_measurement* records, int32_t n, int32_t* best);

/* ---- running the operator --------------------------------------------- */
/* Bytes of device workspace a (desc, schedule) needs: split-K arrival counters
 * (reserved at offset 0 for every schedule of a tensor-core layer), split-K
 * partials, NCHW transpose buffers.  The workspace must be zero-filled
 * before its first use; libtp leaves it zeroed after each completed call. */
tp_status tp_workspace_size(const tp_conv_desc* d, const tp_schedule* s, size_t* bytes);
/* Max workspace over the layer's whole space (for tuning). */
tp_status tp_workspace_size_max(const tp_conv_desc* d, size_t* bytes);

/* Run conv2d(desc) with schedule `s` inside partition `part` (NULL = whole
 * device).  timing == NULL: one asynchronous launch on the partition stream
 * (tp_partition_sync to wait).  timing != NULL: the C12 protocol, result in
 * *out (synchronous).  s->grid_* != 0 are taken as frozen geometry (C15). */
tp_status tp_conv2d_run(const tp_conv_desc* d, const tp_schedule* s, tp_partition* part,
                        const void* x, const void* w, const void* bias, void* y,
                        void* ws, size_t ws_bytes, const tp_timing* timing, tp_measurement* out);

/* Tracing (SURVEY 5 "tracing / profiling"): run one IGEMM_TC launch with an
 * in-kernel timeline.  trace_host receives grid_x*grid_y*grid_z rows of 96
 * uint64: [0] entry, [1] prologue done, [2] epilogue start, [3] end (SM
 * clock64 cycles), [4..19] k-block arrival in the MMA thread, [20..35]
 * producer past its empty-slot wait, [36..51] MMA thread after commit (first
 * 16 k-blocks), [52] barriers initialised, [53] past griddepcontrol.wait, [54..57] after
 * each of the first 4 ring-fill loads issued, [58] TMEM allocated (warp 2), [60] split-K via
 * DSMEM cluster (1) or global workspace (0), [61] %cluster_nctarank, [62] %smid,
 * [63] %globaltimer at entry (ns), [64] split-K slices sent (st.async), [65] past the
 * cluster barrier, [66] all slices received, [67] reduction stored; gathered kind,
 * first 8 k-blocks: [68..75] chunks stored, [76..83] past the proxy fence, [84..91]
 * past the empty-slot wait.
 * cap >= k x grid CTAs (k <= 4): k back-to-back launches captured in one CUDA graph (the
 * timing protocol's launch mode), rows [l CTAs, (l+1) CTAs) for launch l; *rows = k x CTAs.
 * The later launches expose the PDL overlap as the tuner measures it. */
tp_status tp_conv2d_trace(const tp_conv_desc* d, const tp_schedule* s, tp_partition* part, const void* x,
                          const void* w, const void* bias, void* y, void* ws, size_t ws_bytes,
                          uint64_t* trace_host, int32_t cap, int32_t* rows);

/* Tune: select candidates (a3), profile each inside `part` (a11) behind the
 * correctness gate (a10), record (a12), return the argmin.
 *   check_idx/check_ref/n_check : flat output indices (NKPQ logical) and
 *     reference values (e.g. the fp64 oracle's); a candidate fails the gate if
 *     max|y - ref| > tol * max|ref|.  n_check == 0 -> consensus gate: the first
 *     OK candidate's values at the 4096 tp_gate_points become the reference.
 *   tol <= 0 -> 2e-2 for bf16 inputs, 1e-5 for fp32 (north_star).
 *   records (cap records_cap) receive one tp_measurement per candidate in
 *   selection order; *n_records = number measured.
 * Candidates whose launch fails get status TP_ECUDA and are excluded. */
tp_status tp_tune(const tp_conv_desc* d, tp_partition* part, int32_t trials, uint64_t seed,
                  const void* x, const void* w, const void* bias, void* y, void* ws, size_t ws_bytes,
                  const int64_t* check_idx, const double* check_ref, int32_t n_check, double tol,
                  const tp_timing* timing, tp_schedule* best, tp_measurement* best_m,
                  tp_measurement* records, int32_t records_cap, int32_t* n_records);
/* Same loop over an explicit candidate list (the sharder's unit of work,
 * rank r measures idx = r mod G). */
tp_status tp_tune_subset(const tp_conv_desc* d, tp_partition* part, const int64_t* cand_idx,
                         int32_t n_cand, const void* x, const void* w, const void* bias, void* y,
                         void* ws, size_t ws_bytes, const int64_t* check_idx, const double* check_ref,
                         int32_t n_check, double tol, const tp_timing* timing,
                         tp_measurement* records, int32_t records_cap, int32_t* n_records);

/* Model-guided selection for budgets below |space| (the
 * paper's tuner ranks configurations with a learned cost model).
 * Host-only.  Given the schedules measured so far (space indices and median
 * latencies in us; latency <= 0 or non-finite = failed), returns up to
 * `batch` unmeasured indices in next_idx[] (*n_next of them): with no
 * measurements (or fewer than 4 successful ones) the next entries of the
 * SplitMix64 sample of reading C17; otherwise the (1 - explore) * batch
 * schedules with the lowest latency predicted by a ridge regression of
 * log(latency) on standardised schedule features
 * (tile knobs, CTAs, k-blocks per CTA, waves at sm_granted, padding waste,
 * kind), plus random unmeasured ones for the rest.  Deterministic.
 * TP_EINVAL on bad arguments or an index outside the space. */
tp_status tp_search_next(const tp_conv_desc* d, int32_t sm_granted, const int64_t* measured_idx,
                         const double* measured_us, int32_t n_measured, int32_t batch, double explore,
                         uint64_t seed, int64_t* next_idx, int32_t* n_next);
/* tp_tune with model-guided selection: batches of `batch` candidates chosen by
 * tp_search_next (explore fraction `explore`), each profiled like
 * tp_tune_subset, until min(trials, |space|) are measured; records in
 * measurement order; best / best_m / y as tp_tune. */
tp_status tp_tune_guided(const tp_conv_desc* d, tp_partition* part, int32_t trials, int32_t batch, double explore,
                         uint64_t seed, const void* x, const void* w, const void* bias, void* y, void* ws,
                         size_t ws_bytes, const int64_t* check_idx, const double* check_ref, int32_t n_check,
                         double tol, const tp_timing* timing, tp_schedule* best, tp_measurement* best_m,
                         tp_measurement* records, int32_t records_cap, int32_t* n_records);

/* Early stopping ("halts tuning if a newer
 * configuration generated by the explorer is worse than previously profiled
 * configurations", "stops tuning, when the new configurations ... do not
 * show latency improvement"; reading C19: TVM's rule, a patience count).
 * us[0..n): measured medians in measurement order, < 0 = a candidate that
 * failed (never an improvement).  Returns 1 when the last `early_stop`
 * candidates did not lower the best latency measured before them (strictly),
 * 0 otherwise; early_stop <= 0: never stops.  Host-only. */
int32_t tp_search_should_stop(const double* us, int32_t n, int32_t early_stop);

/* tp_tune_guided that checks tp_search_should_stop(records so far,
 * early_stop) after every batch and stops there (early_stop <= 0: exactly
 * tp_tune_guided). */
tp_status tp_tune_guided_es(const tp_conv_desc* d, tp_partition* part, int32_t trials, int32_t batch, double explore,
                            uint64_t seed, int32_t early_stop, const void* x, const void* w, const void* bias, void* y,
                            void* ws, size_t ws_bytes, const int64_t* check_idx, const double* check_ref,
                            int32_t n_check, double tol, const tp_timing* timing, tp_schedule* best,
                            tp_measurement* best_m, tp_measurement* records, int32_t records_cap, int32_t* n_records);

/* Cross-evaluation: run schedule tuned at p (frozen geometry, reading C15)
 * inside partition `part_q` with the timing protocol (a13). */
tp_status tp_cross_eval(const tp_conv_desc* d, const tp_schedule* tuned_at_p, tp_partition* part_q,
                        const void* x, const void* w, const void* bias, void* y, void* ws,
                        size_t ws_bytes, const tp_timing* timing, tp_measurement* out);

/* Model-level run (reading C21): layers 0..n-1 run in order
 * inside `part` -- each launch waits for its predecessor's completion
 * (programmatic dependent launch), so layer i+1 may read layer i's y
 * (x[i+1] == y[i]) -- `reps` times back to back, captured as ONE CUDA graph.
 * Per-layer arrays of length n: descs, scheds (any schedule of each layer's
 * space), device pointers x, w, bias (may be NULL), y, ws and ws_bytes as for
 * tp_conv2d_run.  timing == NULL and out == NULL: one asynchronous replay.
 * Otherwise warmup replays, then `groups` timed replays; out->median_us =
 * per-sequence latency (group time / reps), n_per_group = reps.  Errors: as
 * tp_conv2d_run for any layer. */
tp_status tp_chain_run(int32_t n_layers, const tp_conv_desc* descs, const tp_schedule* scheds, tp_partition* part,
                       const void* const* x, const void* const* w, const void* const* bias, void* const* y,
                       void* const* ws, const size_t* ws_bytes, int32_t reps, const tp_timing* timing,
                       tp_measurement* out);

/* ---- the same calls with GPU% given as a fraction (SURVEY 8(b) spelling) --
 * sm_fraction in (0, 1] selects the cached partition of (device of the last
 * tp_init, fraction, TP_PART_FINE_GRAINED) -- exactly the handle
 * tp_partition_get returns -- and forwards to tp_conv2d_run / tp_tune /
 * tp_cross_eval; errors as those calls plus TP_EINVAL (fraction out of range)
 * and TP_ECAPACITY (partition cannot be granted).  tp_partition_open is
 * tp_partition_get without the requested count; tp_partition_stream returns the
 * partition's CUstream (wrap it with torch.cuda.ExternalStream). */
tp_status tp_partition_open(int32_t device, double sm_fraction, int32_t flags, tp_partition** part,
                            int32_t* sm_granted);
tp_status tp_partition_stream(tp_partition* part, void** cu_stream);
tp_status tp_conv2d_run_at(const tp_conv_desc* d, const tp_schedule* s, double sm_fraction,
                           const void* x, const void* w, const void* bias, void* y,
                           void* ws, size_t ws_bytes, const tp_timing* timing, tp_measurement* out);
tp_status tp_tune_at(const tp_conv_desc* d, double sm_fraction, int32_t trials, uint64_t seed,
                     const void* x, const void* w, const void* bias, void* y, void* ws, size_t ws_bytes,
                     const int64_t* check_idx, const double* check_ref, int32_t n_check, double tol,
                     const tp_timing* timing, tp_schedule* best, tp_measurement* best_m,
                     tp_measurement* records, int32_t records_cap, int32_t* n_records);
tp_status tp_cross_eval_at(const tp_conv_desc* d, const tp_schedule* tuned_at_p, double q,
                           const void* x, const void* w, const void* bias, void* y, void* ws,
                           size_t ws_bytes, const tp_timing* timing, tp_measurement* out);

/* ---- operand preparation (a5; outside the timed region) ----------------
 * fp32 logical NCHW x -> layout/dtype of desc (NHWC or NCHW, bf16 RNE or fp32).
 * fp32 logical KCRS w -> KRSC in desc.dtype.  Asynchronous on part's stream. */
tp_status tp_pack_input(const tp_conv_desc* d, tp_partition* part, const float* x_nchw_f32, void* x_out);
tp_status tp_pack_weights(const tp_conv_desc* d, tp_partition* part, const float* w_kcrs_f32, void* w_out);
/* Gather y at flat NKPQ logical indices into fp64 host values (a10). */
tp_status tp_gather_output(const tp_conv_desc* d, tp_partition* part, const void* y,
                           const int64_t* idx_host, int32_t n, double* vals_host);

#ifdef __cplusplus
}
#endif
#endif /* TP_H_ */
