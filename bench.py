#!/usr/bin/env python
"""bench.py -- tuning throughput + tuned conv2d latency on B200 (BASELINE.json metric).

One step = one pass of the whole hot path over the workload:
for every unique conv layer of ResNet-50 v1.5 batch 1 bf16 (BASELINE config 2),
select its full v0 schedule space (1000 trials per operator, covers
every space), profile each candidate inside the partition (correctness gate +
CUDA-event timing protocol, C12) and record it; rank 0 merges the per-layer
argmin.  `value` is candidates/s for the whole job (all ranks).  With --gpus N
the job holds N independent tuning jobs (one per GPU's worth of work, weak
scaling) whose candidates are dealt round-robin over the ranks (the sharder,
SURVEY 8(e)); the only exchange is a gloo gather of records.

Extra keys: latency_us (model sum of tuned per-layer latency), roofline of the
dominant kernel (igemm_tc), cpu_baseline (the fp64 oracle on host cores),
e2e (same metric with host buffers and H2D/D2H copies inside the timed
region), clocks, gpu_launches, parity (winners vs oracle, sampled points).

--impl reference times the fp64 CPU oracle (the tier's reference arm) on the
same workload and unit.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "conv2d latency (µs) at 25/50/100% SMs; tuning candidates/sec per box"
UNIT = "candidates/s"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--fraction", type=float, default=1.0)
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the 10/25/50%%, cross-eval, VGG, MBv2, cfg1 runs")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run this many steps only, no extras")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return dict(FALLBACK_PEAKS, bf16_tflops_sustained=1400.0,
                    source="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        if os.environ.get("TP_BENCH_NO_CLOCKS"):   # experiments only: no sampler (never for a reported line)
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ algorithmic work per layer
def layer_work(d: dict, P: int, Q: int) -> tuple[float, float]:
    """(FLOPs, compulsory bytes) of one layer invocation: F = 2 N K P Q Cg R S;
    B = x + w + y (+ fp32 bias) in the layer dtype."""
    eb = 2 if d["dtype"] == 0 else 4
    ob = 2 if d["out_dtype"] == 0 else 4
    cg = d["c"] // d["groups"]
    flops = 2.0 * d["n"] * d["k"] * P * Q * cg * d["r"] * d["s"]
    byts = (d["n"] * d["c"] * d["h"] * d["w"] * eb + d["k"] * cg * d["r"] * d["s"] * eb + d["n"] * d["k"] * P * Q * ob
            + d["k"] * 4)
    return flops, float(byts)


# ------------------------------------------------------------------ reference arm / CPU baseline (oracle)
def host_cores() -> int:
    """Host cores available to this process (torchrun sets OMP_NUM_THREADS=1,
    so the oracle is given the thread count explicitly)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_pass(layers, inputs, threads=0):
    """One evaluation of every unique layer with the fp64 oracle (C, OpenMP)."""
    from oracle import conv as oc
    for d, (x, w, b) in zip(layers, inputs):
        oc.conv2d_c(d, x, w, b, relu=True, threads=threads)


def cpu_inputs(layers, config=2):
    import torch

    from paper_2008_03602_b200 import datagen
    out = []
    for i, d in enumerate(layers):
        x, w, b = datagen.make_inputs(d, datagen.data_seed(config, i))
        if d["dtype"] == 0:
            x = torch.tensor(x).bfloat16().double().numpy()
            w = torch.tensor(w).bfloat16().double().numpy()
        out.append((x, w, b))
    return out


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(layers, config=2, min_s=10.0, max_s=30.0) -> dict:
    """The fp64 oracle on the host cores (SURVEY 8(d) "oracle timed beside the
    GPU run"): all-core passes over the unique layers for ~10-30 s, per-layer
    latency and GFLOP/s from the first pass, and one single-thread pass over the
    smallest layers for the single-core rate."""
    from oracle import conv as oc
    inputs = cpu_inputs(layers, config)
    cores = host_cores()
    per_layer = []
    t0 = time.perf_counter()
    passes = 0
    while True:
        for d, (x, w, b) in zip(layers, inputs):
            t1 = time.perf_counter()
            oc.conv2d_c(d, x, w, b, relu=True, threads=cores)
            if passes == 0:
                P, Q = oc.out_dim(d["h"], d["r"], d["stride_h"], d["pad_h"], 1), oc.out_dim(d["w"], d["s"],
                                                                                           d["stride_w"],
                                                                                           d["pad_w"], 1)
                ms = (time.perf_counter() - t1) * 1e3
                per_layer.append({"layer": d["name"], "ms": round(ms, 2),
                                  "gflops": round(layer_work(d, P, Q)[0] / (ms * 1e-3) / 1e9, 3)})
        passes += 1
        el = time.perf_counter() - t0
        if el >= min_s or el + el / passes > max_s:
            break
    evals = passes * len(layers)
    # single thread, on the cheapest layers (about a quarter of the FLOPs)
    order = sorted(range(len(layers)), key=lambda i: per_layer[i]["ms"])[: max(1, len(layers) // 4)]
    t1 = time.perf_counter()
    for i in order:
        x, w, b = inputs[i]
        oc.conv2d_c(layers[i], x, w, b, relu=True, threads=1)
    st = time.perf_counter() - t1
    return {"value": evals / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{passes} pass(es) over the {len(layers)} unique layers, one fp64 oracle evaluation per "
                      f"candidate (a CPU 'candidate' = one run of the layer), {el:.1f}s on {cores} threads",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "single_thread": {"value": len(order) / st, "unit": UNIT, "layers": len(order), "s": round(st, 2)},
            "per_layer": per_layer}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2008_03602_b200 import workloads as wl
    layers = wl.catalog(args.workload)
    inputs = cpu_inputs(layers, REF_CONFIG.get(args.workload, 2))
    cores = host_cores()
    # Each step is a bounded sample: one oracle evaluation of a rotating subset of layers (~5 s).
    probe0 = time.perf_counter()
    oracle_pass(layers[:1], inputs[:1], threads=cores)
    t_one = max(1e-3, time.perf_counter() - probe0)
    per_step = max(1, min(len(layers), int(5.0 / t_one)))
    order = list(range(len(layers)))

    def step(k):
        sel = [order[(k * per_step + j) % len(order)] for j in range(per_step)]
        oracle_pass([layers[i] for i in sel], [inputs[i] for i in sel], threads=cores)
        return len(sel)

    for k in range(args.warmup):
        step(k)
    t0 = time.perf_counter()
    n = 0
    for k in range(args.steps):
        n += step(args.warmup + k)
    el = time.perf_counter() - t0
    val = n / el
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1000 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload} unique conv layers, fp64 oracle evaluations",
                       "layers_per_step": per_step},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} layer evaluation(s) per step, rotating over the "
                                       f"{len(layers)} unique layers"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
REF_CONFIG = {"cfg1": 1, "resnet50": 2, "vgg19_b16": 4, "mobilenetv2": 5}
KERNEL_OF_KIND = {0: "igemm_tc_kernel", 1: "direct_conv_kernel", 2: "igemm_tc_kernel<gather>",
                  3: "igemm_row_kernel", 4: "igemm_mt_kernel", 5: "igemm_tf32_kernel", 6: "igemm_stem_kernel"}


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """--gpus N without a torchrun environment: re-launch this script as N
    ranks (one process per GPU, rendezvous on 127.0.0.1) and return rank 0's
    exit status; the ranks bind cuda:LOCAL_RANK."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def traffic_capture(winners: dict) -> dict | None:
    """Per-launch DRAM traffic of the tuned winners from the newest committed
    ncu capture (profiles/r*_ncu_dram_r50.json), with how many of the current
    winners it covers (the same space index)."""
    import glob
    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_dram_r50.json")))
    if not caps:
        return None
    try:
        d = json.load(open(caps[-1]))
    except Exception:
        return None
    layers = d.get("layers", [])
    same = sum(1 for r in layers if winners.get(r.get("layer")) == r.get("space_index"))
    return {"file": os.path.relpath(caps[-1], ROOT), "mean_dram_bytes_per_launch": d.get("mean_dram_bytes_per_launch"),
            "dram_over_algorithmic": d.get("dram_over_algorithmic"), "winners_covered": same,
            "winners_total": len(winners)}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))

    import torch
    import torch.distributed as dist

    from paper_2008_03602_b200 import datagen, refs, shard, tp, workloads as wl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if os.environ.get("TP_BENCH_DEVICE") is not None:   # path test: several ranks on one GPU
        local = int(os.environ["TP_BENCH_DEVICE"])
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPU(s) visible")
    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    tp.init(local)
    part = tp.Partition.get(args.fraction, device=local)

    layers = wl.catalog(args.workload)
    config = REF_CONFIG[args.workload]
    checks = refs.load(args.workload, config, layers)        # stored fp64 oracle points (refs/README.md)
    jobs = world                                   # weak scaling: one tuning job per GPU's worth
    bufs = {}                                      # (job, layer) -> LayerBuffers
    units = {}                                     # (job, layer) -> the unit's full candidate list
    n_units = 0
    for j in range(jobs):
        for li, d in enumerate(layers):
            x, w, b = datagen.make_inputs(d, datagen.data_seed(config, li))
            bufs[(j, li)] = tp.LayerBuffers(d, x, w, b, part=part, device=local)
            units[(j, li)] = tp.space_sample(d, args.trials, datagen.sampler_seed(0))
            n_units += len(units[(j, li)])
    cands = {key: shard.shard(u, rank, world) for key, u in units.items()}
    tcfg = tp.timing()                             # C12 defaults: W=3, r=5, n>=10, >=20us groups
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def measure(key, idx, timing_cfg=tcfg):
        ci, cr = checks[key[1]]
        return tp.tune_subset(bufs[key], part, idx, check_idx=ci, check_ref=cr, timing_cfg=timing_cfg)

    def step(timing_cfg=tcfg):
        return shard.run_sharded(units, lambda key, idx: measure(key, idx, timing_cfg), rank, world)

    def flush_l2(i):
        flush_buf.fill_(i & 0xFF)                  # > L2 (126 MB) between timed iterations
        torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    steps = args.profile_steps or args.steps
    warm = 0 if args.profile_steps else args.warmup
    for i in range(warm):
        step()
        flush_l2(i)

    stream = torch.cuda.ExternalStream(part.stream(), device=f"cuda:{local}")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = tp.launch_count()
    ev0.record(stream)
    last = None
    for i in range(steps):
        last = step()
        if i + 1 < steps:
            flush_l2(i + 100)
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = tp.launch_count() - l0
    clk = clocks.stop()
    barrier()
    el_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([el_ms], dtype=torch.float64)
    lc = torch.tensor([launches], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(lc, op=dist.ReduceOp.SUM)
    el_ms = float(t.item())
    value = n_units * steps / (el_ms / 1000.0)

    gathered = shard.gather_to_rank0(last)
    if args.profile_steps:
        if rank == 0:
            print(json.dumps({"profile_run": True, "value": value, "steps": steps}), flush=True)
        return

    # ---------------- e2e: same metric through the public API with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        host = {}
        h2d = d2h = 0
        for key, bf in bufs.items():
            hx = torch.empty(bf.x.numel(), dtype=torch.uint8, pin_memory=True)
            hw = torch.empty(bf.w.numel(), dtype=torch.uint8, pin_memory=True)
            hb = torch.empty(bf.b.numel(), dtype=torch.float32, pin_memory=True)
            hy = torch.empty(bf.y.numel(), dtype=torch.uint8, pin_memory=True)
            hx.copy_(bf.x); hw.copy_(bf.w); hb.copy_(bf.b)
            host[key] = (hx, hw, hb, hy)
            if cands[key]:
                h2d += hx.numel() + hw.numel() + hb.numel() * 4
                d2h += hy.numel()
        torch.cuda.synchronize()

        def e2e_step():
            for key in sorted(cands):
                if not cands[key]:
                    continue
                bf = bufs[key]
                hx, hw, hb, hy = host[key]
                bf.x.copy_(hx, non_blocking=True); bf.w.copy_(hw, non_blocking=True)
                bf.b.copy_(hb, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                measure(key, cands[key])
                hy.copy_(bf.y)                     # D2H read of the step's result

        e2e_step()
        barrier()
        torch.cuda.synchronize()
        e0 = time.perf_counter()
        ev0.record(stream)
        for i in range(steps):
            e2e_step()
        ev1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": n_units * steps / (float(e_ms.item()) / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "wall_s": time.perf_counter() - e0}

    if rank != 0:
        if world > 1:
            dist.barrier()
        return

    # ---------------- rank 0: merge, finalists, latency, roofline ----------------
    recs = shard.unpack(gathered)
    best = shard.merge_best(recs)
    n_ok = sum(1 for r in recs if r["status"] == 0)
    busy = shard.gpu_busy_us(recs) / 1000.0 / max(world, 1)      # ms per rank, last step
    # 8(e) merge: the top-3 of every (job, layer) are re-timed on this one device.
    merged = {key: b for key, b in best.items()}
    moves = []
    for key, fin in shard.finalists(recs, 3).items():
        d = layers[key[1]]
        rt = [dict(r, tuner_us=r["median_us"],
                   median_us=tp.conv2d_run(bufs[key], tp.space_get(d, r["space_index"]), part, tcfg)["median_us"])
              for r in fin]
        best[key] = min(rt, key=lambda r: (r["median_us"], r["space_index"]))
        if best[key]["space_index"] != merged[key]["space_index"]:
            old = [r for r in rt if r["space_index"] == merged[key]["space_index"]][0]
            moves.append({"job": key[0], "layer": d["name"], "tuner_winner": old["space_index"],
                          "tuner_winner_tuner_us": round(old["tuner_us"], 3),
                          "tuner_winner_retimed_us": round(old["median_us"], 3),
                          "new_winner": best[key]["space_index"],
                          "new_winner_tuner_us": round(best[key]["tuner_us"], 3),
                          "new_winner_retimed_us": round(best[key]["median_us"], 3),
                          "gain": round(old["median_us"] / best[key]["median_us"] - 1.0, 4)})
    lat_sum = 0.0
    flops_tc = bytes_tc = t_tc = 0.0
    t_direct = 0.0
    per_layer = []
    kernels: dict[str, int] = {}
    pk = peaks()
    floor_us = part.floor(1, 128)["median_us"]   # measured launch floor of the protocol
    roof_tc = 0.0                                # sum over tc layers of max(tensor, HBM, floor) time
    winners = {}
    for li, d in enumerate(layers):
        b = best.get((0, li))
        if b is None:
            continue
        P, Q = tp.output_shape(d)
        f, by = layer_work(d, P, Q)
        lat_sum += d["mult"] * b["median_us"]
        kind = tp.space_get(d, b["space_index"])["kind"]
        winners[d["name"]] = b["space_index"]
        roof_l = max(f / (pk["bf16_tflops"] * 1e6), by / (pk["hbm_gbs"] * 1e3), floor_us)
        if kind != tp.KIND_DIRECT:
            flops_tc += f
            bytes_tc += by
            t_tc += b["median_us"]
            roof_tc += roof_l
            kernels[KERNEL_OF_KIND[kind]] = kernels.get(KERNEL_OF_KIND[kind], 0) + 1
        else:
            t_direct += b["median_us"]
        per_layer.append({"layer": d["name"], "best_us": round(b["median_us"], 3), "space_index": b["space_index"],
                          "kind": kind, "ctas": b["ctas"], "waves": b["waves"],
                          "binding_roof_us": round(roof_l, 3), "binding_roof_frac": round(roof_l / b["median_us"], 3)})
    n_tc = sum(kernels.values())
    ach_gbs = bytes_tc / (t_tc * 1e-6) / 1e9 if t_tc else 0.0
    ach_tfs = flops_tc / (t_tc * 1e-6) / 1e12 if t_tc else 0.0
    hbm_bound = bytes_tc / pk["hbm_gbs"] > flops_tc / (pk["bf16_tflops"] * 1e3)
    cap = traffic_capture(winners)
    traffic = cap["mean_dram_bytes_per_launch"] if cap else None
    if hbm_bound:
        roof = {"bound": "hbm", "achieved": round(ach_gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach_gbs / pk["hbm_gbs"], 4), "traffic": traffic}
    else:
        roof = {"bound": "tensor", "achieved": round(ach_tfs, 2), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": round(ach_tfs / pk["bf16_tflops"], 4), "traffic": traffic}
    roof.update({"kernel": " + ".join(f"{k} x{v}" for k, v in sorted(kernels.items(), key=lambda kv: -kv[1])),
                 "peak_source": pk["source"],
                 "per_launch": f"one tuned conv layer; algorithmic bytes = x + w + y + bias (bf16), FLOPs = 2 N K P Q "
                               f"C R S; achieved = sum over the {n_tc} tensor-core layers / sum of their re-timed "
                               f"median latencies (CUDA events on the partition stream, warm L2)",
                 "tensor_frac": round(ach_tfs / pk["bf16_tflops"], 4), "hbm_frac": round(ach_gbs / pk["hbm_gbs"], 4),
                 "time_share_of_tuned_model": round(t_tc / max(t_tc + t_direct, 1e-9), 3),
                 "launch_floor_us": round(floor_us, 3),
                 "binding_roof_frac": round(roof_tc / max(t_tc, 1e-9), 4),
                 "binding_roof_note": "sum over the tensor-core layers of max(FLOPs / tensor peak, bytes / HBM "
                                      "peak, measured empty-kernel launch floor) / sum of their tuned latencies",
                 "traffic_capture": cap})

    # ---------------- measured model latency: the 53 layers as one graph (reading C21, f2) ----------------
    model_chain = None
    if args.workload == "resnet50":
        names = {d["name"]: li for li, d in enumerate(layers)}
        seq = [names[n] for n in wl.resnet50_sequence()]
        if all((0, li) in best for li in seq):
            mc = tp.chain_run([bufs[(0, li)] for li in seq],
                              [tp.space_get(layers[li], best[(0, li)]["space_index"]) for li in seq], part, reps=4,
                              timing_cfg=tp.timing())
            model_chain = {"layers": len(seq), "median_us": round(mc["median_us"], 2),
                           "min_us": round(mc["min_us"], 2), "sum_of_layer_latencies_us": round(lat_sum, 2),
                           "note": "tp_chain_run: the 53 ResNet-50 convs in execution order (each its own operands) "
                                   "captured as one CUDA graph with PDL between launches, 4 passes per timed group"}

    # ---------------- extras (N = 1): the rest of the metric on this box, clocks sampled ----------------
    extras = None
    if world == 1 and not args.no_extras and args.workload == "resnet50":
        extras = run_extras(args, tp, refs, shard, datagen, wl, part, bufs, units, checks, measure, n_units, pk, local)

    parity = None
    cpu = None
    if not args.no_cpu:
        try:
            from oracle import conv as oc
            inputs = cpu_inputs(layers, config)
            worst = 0.0
            for li, d in enumerate(layers):
                b = best.get((0, li))
                if b is None:
                    continue
                bf = bufs[(0, li)]
                tp.conv2d_run(bf, tp.space_get(d, b["space_index"]), part)
                part.sync()
                P, Q = tp.output_shape(d)
                idx = datagen.sample_points(d["n"] * d["k"] * P * Q, 4096, 5011 + li)   # not the gate's points
                x, w, bb = inputs[li]
                ref = oc.conv2d_points_c(d, x, w, bb, True, idx)
                got = bf.gather(idx, part)
                worst = max(worst, float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30)))
            parity = {"layers": len(best), "points_per_layer": 4096, "max_rel_err": worst,
                      "tol": 2e-2, "pass": worst <= 2e-2,
                      "note": "re-timed winners vs the fp64 oracle at 4096 points per layer drawn apart from the "
                              "gate's points"}
            if world == 1:
                cpu = cpu_baseline(layers, config)
        except Exception as e:   # the baseline is reported, never the product path
            cpu = {"error": str(e)}

    line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(el_ms / steps, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.workload} batch {layers[0]['n']} "
                                   f"{'bf16' if layers[0]['dtype'] == 0 else 'fp32'}: all {len(layers)} unique conv "
                                   f"layers, exhaustive v0 space tuned at {int(args.fraction * 100)}% SMs "
                                   f"({part.sm_granted} granted), {jobs} tuning job(s) sharded round-robin",
                       "candidates_per_step": n_units, "sm_fraction": args.fraction, "sm_granted": part.sm_granted,
                       "l2": "flushed (512 MiB write) between timed steps; candidates timed warm (TVM-like)",
                       "gate": "fp64 oracle points (refs/, 4096 per layer) at 2e-2 / 1e-5",
                       "parallelism": f"candidate-shard x{world}"},
            "latency_us": {"model_sum_tuned": round(lat_sum, 2), "at_fraction": args.fraction,
                           "model_chain": model_chain, "per_layer": per_layer},
            "candidates_ok": n_ok, "candidates_total": len(recs),
            "raced_frac": round(shard.raced_frac(recs), 4),
            "gpu_busy_frac": round(busy / (el_ms / steps), 3),
            "finalists": {"per_layer": 3, "retimed_on": "rank 0 device", "winner_changed": len(moves),
                          "max_gain": max((m["gain"] for m in moves), default=0.0),
                          "mean_gain": round(sum(m["gain"] for m in moves) / max(1, len(moves)), 4),
                          "changes": moves},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": int(lc.item()),
            "parity": parity}
    if extras is not None:
        line.update(extras)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()


def run_extras(args, tp, refs, shard, datagen, wl, part, bufs, units, checks, measure, n_units, pk, local) -> dict:
    """The rest of BASELINE.json's metric on the same box, after the timed
    region, with its own clock sampling: value_uniform (one step without C12b
    racing), the 10/25/50/100% exhaustive tunes and the 4x4 frozen cross-eval
    matrix (config 3), VGG-19 b16 with 4 concurrent 25% tuners (config 4),
    MobileNetV2 at 50% (config 5) and cfg1 (fp32, config 1).  Every tune is
    gated on the stored oracle points."""
    import torch

    from paper_2008_03602_b200 import experiments as ex
    out = {}
    clk = ClockSampler(local)
    clk.start()
    t_all = time.perf_counter()

    # (1) the headline unit without racing ((W + n r) launches + gate for every candidate)
    stream = torch.cuda.ExternalStream(part.stream(), device=f"cuda:{local}")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    uni = tp.timing(prune_ratio=0.0)
    torch.cuda.synchronize()
    e0.record(stream)
    recs_u = shard.unpack(shard.run_sharded(units, lambda key, idx: measure(key, idx, uni), 0, 1))
    e1.record(stream)
    torch.cuda.synchronize()
    ms_u = e0.elapsed_time(e1)
    out["value_uniform"] = {"value": round(n_units / (ms_u / 1000.0), 2), "unit": UNIT, "steps": 1,
                            "candidates_ok": sum(1 for r in recs_u if r["status"] == 0),
                            "raced_frac": shard.raced_frac(recs_u),
                            "note": "one step with prune_ratio = 0: every candidate gets 3 warm-ups and 5 groups of "
                                    "n >= 10 launches"}

    # (2) config 3: tuned at p, run at q (frozen geometry), fractions 10/25/50/100%
    layers = wl.catalog("resnet50")
    fr = (0.10, 0.25, 0.50, 1.0)
    cx = ex.cross_eval(layers, fr, trials=args.trials, config=2, checks=checks,
                       bufs=[bufs[(0, li)] for li in range(len(layers))], log=lambda *a: None)
    lbf = {}
    for q in fr:
        rows = []
        for row in cx["layers"]:
            rl = row["diag_roofline"][str(q)]
            rows.append({"layer": row["layer"], "space_index": row["best_schedule"][str(q)]["space_index"],
                         "kind": row["best_schedule"][str(q)]["kind"],
                         "best_us": round(row["matrix_us"][str(q)][str(q)], 3),
                         "binding": rl["binding"], "binding_roof_us": round(rl["roof_us"][rl["binding"] + "_us"], 3),
                         "binding_roof_frac": round(rl["frac_of_binding_roof"], 3),
                         "tensor_frac": round(rl["tensor_frac"], 4), "hbm_frac": round(rl["hbm_frac"], 4)})
        st = cx["tune"][str(q)]
        lbf[str(q)] = {"sm_granted": cx["partitions"][str(q)]["sm_granted"],
                       "model_sum_us": round(cx["model_sum_us"][str(q)][str(q)], 2),
                       "candidates": st["candidates"], "candidates_ok": st["ok"],
                       "candidates_per_s": round(st["candidates_per_s"], 1), "raced": st["raced"],
                       "binding_roof_frac": round(sum(r["binding_roof_us"] for r in rows)
                                                  / sum(r["best_us"] for r in rows), 4),
                       "per_layer": rows}
    out["latency_us_by_fraction"] = lbf
    out["crosseval_r50"] = {"fractions": list(fr),
                            "model_sum_us": {p: {q: round(v, 2) for q, v in r.items()}
                                             for p, r in cx["model_sum_us"].items()},
                            "model_sum_default_us": {q: round(v, 2) for q, v in cx["model_sum_default_us"].items()},
                            "aggregate_5k": cx["aggregate_5k"], "pd_check": cx["pd_check"],
                            "per_layer_us": {row["layer"]: {p: {q: round(v, 3) for q, v in r.items()}
                                                            for p, r in row["matrix_us"].items()}
                                             for row in cx["layers"]}}

    # (3) config 4: VGG-19 b16, 4 concurrent tuners on disjoint 25% green contexts
    vl = wl.catalog("vgg19_b16")
    cc = ex.concurrent_tune(vl, k=4, sms_each=37, trials=args.trials, config=4,
                            checks=refs.load("vgg19_b16", 4, vl), log=lambda *a: None)
    out["vgg19_concurrent"] = {
        "k": cc["k"], "sms_each": [p["sm_granted"] for p in cc["partitions"]],
        "candidates": cc["candidates"], "candidates_per_s": round(cc["candidates_per_s"], 1),
        "wall_s": round(cc["wall_s"], 2), "assignment": cc["assignment"],
        "layers": [{"layer": r["layer"], "tuner": r["tuner"], "sm_granted": r["sm_granted"],
                    "kind": r["schedule"]["kind"], "candidates_ok": r["ok"], "candidates": r["candidates"],
                    "best_us": round(r["best_us"], 2), "solo_us": round(r["solo_us"], 2),
                    "corun_us": round(r["corun_us"], 2),
                    "tensor_frac_of_share": round(r["roofline"]["tensor_frac"], 3),
                    "binding": r["roofline"]["binding"],
                    "binding_roof_frac": round(r["roofline"]["frac_of_binding_roof"], 3)} for r in cc["layers"]],
        "note": "tensor_frac_of_share = FLOPs / (solo latency x measured bf16 peak x granted/148)"}
    del cc
    torch.cuda.empty_cache()

    # (4) config 5: MobileNetV2 at 50%; (5) config 1: fp32 at 100%
    for key, cat, cfg, frac in (("mbv2_50", "mobilenetv2", 5, 0.5), ("cfg1_100", "cfg1", 1, 1.0)):
        cl = wl.catalog(cat)
        p = tp.Partition.get(frac, device=local)
        cb = ex.make_buffers(cl, p, cfg, device=local)
        t0 = time.perf_counter()
        res = ex.tune_layers(cl, cb, p, args.trials, datagen.sampler_seed(0), None, refs.load(cat, cfg, cl))
        el = time.perf_counter() - t0
        n = sum(r["candidates"] for r in res)
        ctx = ex.partition_context(p)
        out[key] = {"sm_granted": p.sm_granted, "candidates": n, "candidates_ok": sum(r["ok"] for r in res),
                    "candidates_per_s": round(n / el, 1),
                    "model_sum_us": round(sum(r["mult"] * r["best_m"]["median_us"] for r in res), 2),
                    "per_layer": [{"layer": r["layer"], "best_us": round(r["best_m"]["median_us"], 3),
                                   "kind": r["best"]["kind"],
                                   **{k2: round(v, 4) for k2, v in ex.roofline(
                                       d, r["best_m"]["median_us"], p.sm_granted, ctx["copy_bw_gbs"], ctx["floor_us"],
                                       ex.peaks(), r["best"]["kind"]).items()
                                      if k2 in ("tensor_frac", "alu_frac", "hbm_frac", "frac_of_binding_roof")}}
                                  for d, r in zip(cl, res)]}
        del cb
    out["extras_clocks"] = clk.stop()
    out["extras_wall_s"] = round(time.perf_counter() - t_all, 1)
    return out


if __name__ == "__main__":
    main()
