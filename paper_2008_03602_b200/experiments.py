"""The paper's experiments on the hot path, driven through the C-ABI (tp.py).

* ``tune_layers``      -- tune every layer of a catalog inside one partition
                          (a3-a12; "tune a DNN model at a GPU%").
* ``cross_eval``       -- tuned-at-p x run-at-q latency matrix per layer and
                          for the model (a13; T1-T3; frozen schedule
                          geometry, reading C15).
* ``concurrent_tune``  -- k tuners on k disjoint green-context partitions,
                          one host thread each (a14; "multiple TCIs/TSIs on
                          one GPU with distinct GPU%"),
                          with solo vs co-running latency of the winners
                          (isolation, reading C22).
* ``roofline``         -- the three fractions of SURVEY 8(d) for one layer at
                          its SM share: tensor, ALU (FP32 FFMA) and HBM
                          (against the copy bandwidth measured inside the same
                          partition), plus the measured launch floor.

Everything here is orchestration: every step of the path runs in libtp's
kernels.  Correctness gating: pass ``checks`` -- per layer (check_idx,
check_ref), the stored fp64 oracle points of ``refs.load`` -- and every
candidate is gated against the oracle; without them libtp's
consensus gate applies (the first OK candidate's values at tp_gate_points).
"""
from __future__ import annotations

import json
import os
import threading
import time

from . import datagen, tp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SM_COUNT = 148
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}


def peaks() -> dict:
    """Roofline denominators: MEASURED_PEAKS.json (driver-written) else the
    B200_PROFILING.md fallback; FP32 FFMA peak = SMs x 128 lanes x 2 x clock."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out = {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
               "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        out = dict(FALLBACK, source="fallback (B200_PROFILING.md)")
    out["fp32_tflops"] = SM_COUNT * 128 * 2 * out["sm_max_mhz"] * 1e6 / 1e12
    return out


def layer_work(d: dict) -> tuple[float, float]:
    """(FLOPs, compulsory bytes) of one invocation: F = 2 N K P Q Cg R S;
    B = x + w + y in the layer dtypes + fp32 bias."""
    P, Q = tp.output_shape(d)
    eb = 2 if d["dtype"] == tp.BF16 else 4
    ob = 2 if d.get("out_dtype", d["dtype"]) == tp.BF16 else 4
    cg = d["c"] // d.get("groups", 1)
    f = 2.0 * d["n"] * d["k"] * P * Q * cg * d["r"] * d["s"]
    b = d["n"] * d["c"] * d["h"] * d["w"] * eb + d["k"] * cg * d["r"] * d["s"] * eb + d["n"] * d["k"] * P * Q * ob \
        + 4 * d["k"]
    return f, float(b)


def roofline(d: dict, t_us: float, sm_granted: int, part_bw_gbs: float, floor_us: float, pk: dict,
             kind: int) -> dict:
    """Fractions of SURVEY 8(d) for one layer at its SM share.  The binding
    roof is the largest of the compute time (tensor for the tc path, FFMA for
    the direct path), the HBM time at the partition's measured bandwidth and
    the measured launch floor."""
    f, b = layer_work(d)
    share = sm_granted / SM_COUNT
    tensor_peak = pk["bf16_tflops"] * 1e12 * share
    alu_peak = pk["fp32_tflops"] * 1e12 * share
    t = t_us * 1e-6
    # 3xTF32: dense tf32 runs at half the bf16 rate and every product costs 3 MMAs.
    compute_peak = alu_peak if kind == tp.KIND_DIRECT else (tensor_peak / 6.0 if kind == tp.KIND_IGEMM_TF32X3
                                                             else tensor_peak)
    roofs = {"compute_us": f / compute_peak * 1e6, "hbm_us": b / (part_bw_gbs * 1e9) * 1e6, "floor_us": floor_us}
    bound = max(roofs, key=roofs.get)
    return {"flops": f, "bytes": b, "tensor_frac": f / (t * tensor_peak), "alu_frac": f / (t * alu_peak),
            "hbm_frac": b / (t * part_bw_gbs * 1e9), "roof_us": roofs, "binding": bound.replace("_us", ""),
            "frac_of_binding_roof": roofs[bound] / t_us}


def make_buffers(layers: list[dict], part=None, config: int = 2, device: int = 0) -> list:
    out = []
    for i, d in enumerate(layers):
        x, w, b = datagen.make_inputs(d, datagen.data_seed(config, i))
        out.append(tp.LayerBuffers(d, x, w, b, part=part, device=device))
    return out


def _check(checks, i):
    return (None, None) if checks is None else checks[i]


def tune_layers(layers, bufs, part, trials=1000, seed=42, timing_cfg=None, checks=None) -> list[dict]:
    """Tune each layer inside `part`; returns per-layer dicts with the best
    schedule, its measurement and the tuning throughput."""
    res = []
    for i, (d, buf) in enumerate(zip(layers, bufs)):
        t0 = time.perf_counter()
        ci, cr = _check(checks, i)
        best, m, recs = tp.tune(buf, part, trials, seed, check_idx=ci, check_ref=cr, timing_cfg=timing_cfg)
        el = time.perf_counter() - t0
        res.append({"layer": d["name"], "mult": d.get("mult", 1), "best": best, "best_m": m,
                    "candidates": len(recs), "ok": sum(1 for r in recs if r["status"] == 0),
                    "raced": sum(1 for r in recs if r["status"] == 0 and r["groups"] == 1), "wall_s": el,
                    "oracle_gate": checks is not None})
    return res


# the "Untuned" column of the paper's T1-T3
# restated inside this framework -- a fixed, fraction-independent default
# schedule, the one a user would pick without tuning: the valid schedule of the
# layer's base kind closest (sum of |log2| distances, ties to the lowest index)
# to a mid-range target tuple.
DEFAULT_TC = {"bm": 128, "bn": 128, "bk": 64, "stages": 4, "threads": 128, "split_k": 1}
DEFAULT_DIRECT = {"threads": 256, "tile_q": 2, "vec_k": 4, "tile_p": 2, "smem_stage": 1}


def default_schedule(d: dict) -> dict:
    """Fixed untuned schedule of layer d (host-only; see DEFAULT_TC / DEFAULT_DIRECT)."""
    import math
    kind = tp.layer_kind(d)
    target = DEFAULT_DIRECT if kind == tp.KIND_DIRECT else DEFAULT_TC
    best, best_key = None, None
    for i in range(tp.space_size(d)):
        s = tp.space_get(d, i)
        if s["kind"] != kind:
            continue
        dist = sum(abs(math.log2(max(s[k], 0.5) / max(v, 0.5))) for k, v in target.items())
        key = (dist, s["space_index"])
        if best_key is None or key < best_key:
            best, best_key = s, key
    return best


def aggregate_5k(model_sum_us: dict, fractions) -> dict:
    """P:399 / P:472 (T4): 1000 batch-1 images inferred at each run fraction q
    with the model tuned at p; total in ms = sum_q 1000 * model[p][q] us / 1000."""
    tot = {str(p): sum(model_sum_us[str(p)][str(q)] for q in fractions) for p in fractions}
    return {"images_per_fraction": 1000, "total_ms_by_tuned_at": tot,
            "sweet_spot_tuned_at": min(fractions, key=lambda p: (tot[str(p)], p))}


def partition_context(part) -> dict:
    """Granted SMs, measured copy bandwidth and launch floor of a partition."""
    bw = part.copy_bw(1 << 30, 5)
    fl = part.floor(1, 128)["median_us"]
    return {"fraction": part.fraction, "sm_requested": part.sm_requested, "sm_granted": part.sm_granted,
            "copy_bw_gbs": bw, "floor_us": fl}


def pd_check(per_layer: list[dict], fractions, k_cv: float = 3.0) -> dict:
    """P-D: with exhaustive tuning the diagonal is its column's
    minimum up to noise: M[q][q] <= M[p][q] (1 + eps), eps = k_cv x the larger
    coefficient of variation (std / mean over the timed groups) of the two
    cells.  Also the plain 10% rule of round 1."""
    viol, viol10, cells = [], [], 0
    for row in per_layer:
        m, cv = row["matrix_us"], row["matrix_cv"]
        for q in fractions:
            dq = m[str(q)][str(q)]
            for p in fractions:
                if p == q:
                    continue
                cells += 1
                eps = k_cv * max(cv[str(q)][str(q)], cv[str(p)][str(q)])
                if dq > m[str(p)][str(q)] * (1.0 + eps):
                    viol.append({"layer": row["layer"], "tuned_at": p, "run_at": q, "diag_us": dq,
                                 "cell_us": m[str(p)][str(q)], "eps": eps})
            if dq > min(m[str(p)][str(q)] for p in fractions) * 1.10:
                viol10.append({"layer": row["layer"], "q": q})
    return {"rule": f"M[q][q] <= M[p][q] (1 + {k_cv} CV)", "cells": cells, "violations": viol,
            "pass": not viol, "violations_gt10pct": viol10}


def cross_eval(layers, fractions=(0.10, 0.25, 0.50, 1.0), trials=1000, config=3, timing_cfg=None,
               log=print, checks=None, bufs=None) -> dict:
    """a13: tune every layer at each fraction p, then run each frozen best(p)
    at every fraction q.  Returns per-layer matrices M[p][q] (median us), the
    model sums Sum_l mult_l * M_l[p][q] (reading C21), the diagonal check
    (P-D) and per-cell rooflines of the diagonal."""
    pk = peaks()
    parts = {f: tp.Partition.get(f) for f in fractions}
    ctx = {f: partition_context(parts[f]) for f in fractions}
    bufs = bufs if bufs is not None else make_buffers(layers, None, config)
    tuned = {}
    tune_stats = {}
    for p in fractions:
        t0 = time.perf_counter()
        tuned[p] = tune_layers(layers, bufs, parts[p], trials, datagen.sampler_seed(fractions.index(p)), timing_cfg,
                               checks)
        el = time.perf_counter() - t0
        n = sum(r["candidates"] for r in tuned[p])
        tune_stats[p] = {"candidates": n, "ok": sum(r["ok"] for r in tuned[p]), "wall_s": el,
                         "candidates_per_s": n / el, "raced": sum(r["raced"] for r in tuned[p]),
                         "oracle_gate": checks is not None}
        log(f"tuned at {p}: {n} candidates in {el:.1f}s")
    per_layer = []
    model = {p: {q: 0.0 for q in fractions} for p in fractions}
    for li, d in enumerate(layers):
        mat, cvm = {}, {}
        for p in fractions:
            row, cvr = {}, {}
            for q in fractions:
                m = tp.cross_eval(bufs[li], tuned[p][li]["best"], parts[q], timing_cfg)
                row[q] = m["median_us"]
                cvr[q] = m["std_us"] / m["mean_us"] if m["mean_us"] > 0 else 0.0
                model[p][q] += d.get("mult", 1) * m["median_us"]
            mat[p] = row
            cvm[p] = cvr
        diag = {}
        for q in fractions:
            bm = tuned[q][li]["best_m"]
            diag[q] = roofline(d, mat[q][q], ctx[q]["sm_granted"], ctx[q]["copy_bw_gbs"], ctx[q]["floor_us"], pk,
                               bm["kind"])
        per_layer.append({"layer": d["name"], "mult": d.get("mult", 1),
                          "matrix_us": {str(p): {str(q): mat[p][q] for q in fractions} for p in fractions},
                          "matrix_cv": {str(p): {str(q): cvm[p][q] for q in fractions} for p in fractions},
                          "best_schedule": {str(p): {k: tuned[p][li]["best"][k] for k in
                                                     ("space_index", "kind", "bm", "bn", "bk", "stages", "threads",
                                                      "split_k", "tile_q", "vec_k", "tile_p", "smem_stage", "grid_x",
                                                      "grid_y", "grid_z")} for p in fractions},
                          "diag_roofline": {str(q): diag[q] for q in fractions}})
    # f2: the untuned default schedule at every run fraction (frozen nothing:
    # the default's geometry is derived at each q).
    model_default = {q: 0.0 for q in fractions}
    for li, d in enumerate(layers):
        ds = default_schedule(d)
        row = {}
        for q in fractions:
            row[str(q)] = tp.conv2d_run(bufs[li], ds, parts[q], timing_cfg or tp.timing())["median_us"]
            model_default[q] += d.get("mult", 1) * row[str(q)]
        per_layer[li]["default_us"] = row
        per_layer[li]["default_schedule"] = {k: ds[k] for k in ("space_index", "kind", "bm", "bn", "bk", "stages",
                                                                "threads", "split_k", "tile_q", "vec_k", "tile_p",
                                                                "smem_stage")}
    # P-D: with exhaustive tuning the diagonal is the column minimum up to noise.
    pd = pd_check(per_layer, fractions)
    return {"fractions": list(fractions), "partitions": {str(f): ctx[f] for f in fractions}, "peaks": pk,
            "tune": {str(p): tune_stats[p] for p in fractions},
            "model_sum_us": {str(p): {str(q): model[p][q] for q in fractions} for p in fractions},
            "model_sum_default_us": {str(q): model_default[q] for q in fractions},
            "aggregate_5k": dict(aggregate_5k({str(p): {str(q): model[p][q] for q in fractions} for p in fractions},
                                              fractions),
                                 untuned_total_ms=sum(model_default[q] for q in fractions)),
            "pd_check": pd, "diagonal_violations_gt10pct": pd["violations_gt10pct"], "layers": per_layer}


def _lpt(layers, k):
    """Longest-processing-time-first assignment of layers to k tuners by FLOPs."""
    order = sorted(range(len(layers)), key=lambda i: -layer_work(layers[i])[0])
    load = [0.0] * k
    assign = [[] for _ in range(k)]
    for i in order:
        j = min(range(k), key=lambda t: load[t])
        assign[j].append(i)
        load[j] += layer_work(layers[i])[0]
    return assign


def concurrent_tune(layers, k=4, sms_each=37, trials=1000, config=4, timing_cfg=None, flags=tp.PART_FINE_GRAINED,
                    log=print, checks=None) -> dict:
    """a14: k disjoint partitions of sms_each SMs (one split), one host thread
    per partition tuning its LPT share of the layers concurrently.  Then the
    winners are timed solo (one partition busy) and co-running (all k busy)."""
    pk = peaks()
    # The driver grants SMs in TPC pairs even when co-scheduling is ignored, so
    # k x sms_each may not fit exactly (4 x 37 = 148 does not): step down.
    parts, asked = None, sms_each
    while parts is None:
        try:
            parts = tp.Partition.split(k, asked, flags=flags)
        except tp.TPError as e:
            if e.status != tp.ECAPACITY or asked <= 8:
                raise
            asked -= 1
    ctx = [partition_context(p) for p in parts]
    assign = _lpt(layers, k)
    bufs = {}
    for j, idxs in enumerate(assign):
        for i in idxs:
            d = layers[i]
            x, w, b = datagen.make_inputs(d, datagen.data_seed(config, i))
            bufs[i] = tp.LayerBuffers(d, x, w, b, part=parts[j])
    results = [None] * k
    errors = []

    def worker(j):
        try:
            out = []
            t0 = time.perf_counter()
            for i in assign[j]:
                ci, cr = _check(checks, i)
                best, m, recs = tp.tune(bufs[i], parts[j], trials, datagen.sampler_seed(1), check_idx=ci, check_ref=cr,
                                        timing_cfg=timing_cfg)
                out.append({"layer": layers[i]["name"], "idx": i, "best": best, "best_m": m, "candidates": len(recs),
                            "ok": sum(1 for r in recs if r["status"] == 0)})
            results[j] = {"wall_s": time.perf_counter() - t0, "layers": out}
        except Exception as e:   # surfaced below
            errors.append(repr(e))

    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(j,)) for j in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    if errors:
        raise RuntimeError("; ".join(errors))
    n = sum(r["candidates"] for res in results for r in res["layers"])
    log(f"{k} concurrent tuners: {n} candidates in {wall:.1f}s")

    # isolation: winners solo vs co-running
    def time_all(j, out):
        for r in results[j]["layers"]:
            m = tp.conv2d_run(bufs[r["idx"]], r["best"], parts[j], timing_cfg or tp.timing())
            out[r["layer"]] = m["median_us"]

    solo = {}
    for j in range(k):
        time_all(j, solo)
    co = {}
    th = [threading.Thread(target=time_all, args=(j, co)) for j in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    layers_out = []
    for j in range(k):
        for r in results[j]["layers"]:
            d = layers[r["idx"]]
            layers_out.append({"layer": r["layer"], "tuner": j, "sm_granted": ctx[j]["sm_granted"],
                               "best_us": r["best_m"]["median_us"], "solo_us": solo[r["layer"]],
                               "corun_us": co[r["layer"]], "candidates": r["candidates"], "ok": r["ok"],
                               "schedule": {kk: r["best"][kk] for kk in ("space_index", "kind", "bm", "bn", "bk",
                                                                         "stages", "threads", "split_k")},
                               "roofline": roofline(d, solo[r["layer"]], ctx[j]["sm_granted"],
                                                    ctx[j]["copy_bw_gbs"], ctx[j]["floor_us"], pk,
                                                    r["best_m"]["kind"])})
    for p in parts:
        p.close()
    return {"k": k, "sms_each_requested": sms_each, "sms_each_split": asked, "partitions": ctx, "peaks": pk,
            "oracle_gate": checks is not None, "wall_s": wall, "candidates": n,
            "candidates_per_s": n / wall, "per_tuner_wall_s": [results[j]["wall_s"] for j in range(k)],
            "assignment": [[layers[i]["name"] for i in a] for a in assign], "layers": layers_out}


# ---------------------------------------------------------------------------------------------
# interference.  The paper keeps concurrent tuners apart with a
# fixed GPU% per server because "temporally sharing GPU for multiple tuning
# process will result in wrong latency being reported during profiling ...
# uncontrolled spatial sharing using default MPS does not provide hardware
# isolation" (appendix P:1103-1113 [src]).  Three ways to run k
# tuners on one GPU, each tuning its LPT share of the layers:
#   isolated    -- k disjoint green contexts (SM isolation; L2/HBM still shared)
#   shared      -- k streams on the whole device, no partition (default-MPS analog)
#   time_sliced -- k processes, one CUDA context each, no MPS (the driver time-slices)
# Each mode's winners are then re-timed alone on the target they were tuned for
# (a partition of the same size for `isolated`, the whole idle device otherwise):
# `report_err` = reported / solo latency - 1 (what the tuner believed vs what
# the schedule does alone), `choice_loss` = solo latency of the mode's winner /
# solo latency of the winner of a tuner that ran alone - 1.


def _make_share_buffers(layer_ids, layers, part, config):
    out = {}
    for i in layer_ids:
        d = layers[i]
        x, w, b = datagen.make_inputs(d, datagen.data_seed(config, i))
        out[i] = tp.LayerBuffers(d, x, w, b, part=part)
    return out


def _tune_share(layer_ids, layers, part, trials, config, seed, bufs=None):
    # Buffers are created before any concurrent tuner starts: a torch allocation
    # in one thread while another thread's stream is capturing a CUDA graph
    # fails with cudaErrorStreamCaptureUnsupported.
    bufs = bufs if bufs is not None else _make_share_buffers(layer_ids, layers, part, config)
    out = {}
    for i in layer_ids:
        buf = bufs[i]
        best, m, recs = tp.tune(buf, part, trials, seed)
        out[i] = {"space_index": int(best["space_index"]), "reported_us": float(m["median_us"]),
                  "candidates": len(recs)}
    return out


def _time_sliced_worker(args):
    layer_ids, cat, trials, config, seed, device = args
    from . import workloads as wl
    tp.init(device)
    layers = wl.catalog(cat)
    return _tune_share(layer_ids, layers, tp.Partition.get(1.0, device=device), trials, config, seed)


def interference(cat: str, k: int = 4, sms_each: int = 36, trials: int = 1000, config: int = 6,
                 modes=("isolated", "shared", "time_sliced"), device: int = 0, log=print) -> dict:
    from . import workloads as wl
    layers = wl.catalog(cat)
    assign = _lpt(layers, k)
    seed = datagen.sampler_seed(0)
    timing = tp.timing()

    def solo_time(part, i, idx):
        d = layers[i]
        x, w, b = datagen.make_inputs(d, datagen.data_seed(config, i))
        buf = tp.LayerBuffers(d, x, w, b, part=part)
        return tp.conv2d_run(buf, tp.space_get(d, idx), part, timing)["median_us"]

    res = {"catalog": cat, "k": k, "assignment": [[layers[i]["name"] for i in a] for a in assign], "modes": {}}
    # Ground truth: one tuner alone on each target (a sms_each partition; the whole device).
    iso_parts = tp.Partition.split(k, sms_each, device=device)
    whole = tp.Partition.get(1.0, device=device)
    alone = {"partition": _tune_share(range(len(layers)), layers, iso_parts[0], trials, config, seed),
             "whole": _tune_share(range(len(layers)), layers, whole, trials, config, seed)}
    for mode in modes:
        t0 = time.perf_counter()
        results = [None] * k
        if mode == "time_sliced":
            import multiprocessing as mp
            with mp.get_context("spawn").Pool(k) as pool:
                results = pool.map(_time_sliced_worker, [(a, cat, trials, config, seed, device) for a in assign])
        else:
            parts = iso_parts if mode == "isolated" else tp.Partition.shared(k, device=device)
            errs = []
            share_bufs = [_make_share_buffers(assign[j], layers, parts[j], config) for j in range(k)]
            import torch
            torch.cuda.synchronize()

            def worker(j):
                try:
                    results[j] = _tune_share(assign[j], layers, parts[j], trials, config, seed, share_bufs[j])
                except Exception as e:   # surfaced below
                    errs.append(repr(e))

            th = [threading.Thread(target=worker, args=(j,)) for j in range(k)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            if mode == "shared":
                for p in parts:
                    p.close()
            if errs:
                raise RuntimeError("; ".join(errs))
        wall = time.perf_counter() - t0
        target = iso_parts[0] if mode == "isolated" else whole
        ref = alone["partition"] if mode == "isolated" else alone["whole"]
        rows = []
        for j in range(k):
            for i, r in results[j].items():
                solo = solo_time(target, i, r["space_index"])
                ref_solo = solo_time(target, i, ref[i]["space_index"])
                rows.append({"layer": layers[i]["name"], "mult": layers[i].get("mult", 1), "tuner": j,
                             "space_index": r["space_index"], "reported_us": r["reported_us"], "solo_us": solo,
                             "alone_winner_solo_us": ref_solo, "report_err": r["reported_us"] / solo - 1.0,
                             "choice_loss": solo / ref_solo - 1.0})
        n = sum(r["candidates"] for res_j in results for r in res_j.values())
        msum = sum(r["mult"] * r["solo_us"] for r in rows)
        msum_ref = sum(r["mult"] * r["alone_winner_solo_us"] for r in rows)
        res["modes"][mode] = {
            "wall_s": wall, "candidates": n, "candidates_per_s": n / wall,
            "target": f"{sms_each}-SM partition" if mode == "isolated" else "whole device",
            "mean_abs_report_err": sum(abs(r["report_err"]) for r in rows) / len(rows),
            "max_abs_report_err": max(abs(r["report_err"]) for r in rows),
            "changed_winners": sum(1 for r in rows if r["choice_loss"] > 0.02),
            "model_sum_solo_us": msum, "model_sum_alone_tuned_us": msum_ref,
            "model_choice_loss": msum / msum_ref - 1.0, "layers": rows}
        log(f"{mode}: {n} candidates in {wall:.1f}s, mean |report err| "
            f"{res['modes'][mode]['mean_abs_report_err']:.3f}, model choice loss {msum / msum_ref - 1.0:.3f}")
    for p in iso_parts:
        p.close()
    return res
