"""Run the paper's experiments on the GPU and write JSON reports.

  python tools/report.py crosseval  [--workload resnet50] [--fractions 0.1,0.25,0.5,1.0] out.json
  python tools/report.py concurrent [--workload vgg19_b16] [--k 4] [--sms 37] out.json
  python tools/report.py tune       [--workload mobilenetv2] [--fraction 0.5] out.json
  python tools/report.py interference [--workload resnet50] [--k 4] [--sms 36] out.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_03602_b200 import experiments as ex, tp, workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["crosseval", "concurrent", "tune", "interference"])
    ap.add_argument("out")
    ap.add_argument("--workload", default=None)
    ap.add_argument("--fractions", default="0.1,0.25,0.5,1.0")
    ap.add_argument("--fraction", type=float, default=0.5)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--sms", type=int, default=37)
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--layers", default=None, help="comma-separated subset of layer names")
    a = ap.parse_args()
    tp.init(0)
    wlname = a.workload or {"crosseval": "resnet50", "concurrent": "vgg19_b16", "tune": "mobilenetv2",
                            "interference": "resnet50"}[a.mode]
    layers = wl.catalog(wlname)
    if a.layers:
        keep = set(a.layers.split(","))
        layers = [d for d in layers if d["name"] in keep]
    t0 = time.time()
    if a.mode == "interference":
        res = ex.interference(a.workload or "resnet50", a.k, a.sms if a.sms != 37 else 36, a.trials)
        res["workload"] = a.workload or "resnet50"
        res["elapsed_s"] = time.time() - t0
        json.dump(res, open(a.out, "w"), indent=1)
        return
    if a.mode == "crosseval":
        res = ex.cross_eval(layers, tuple(float(f) for f in a.fractions.split(",")), a.trials)
    elif a.mode == "concurrent":
        res = ex.concurrent_tune(layers, a.k, a.sms, a.trials)
    else:
        part = tp.Partition.get(a.fraction)
        ctx = ex.partition_context(part)
        bufs = ex.make_buffers(layers, part, 5)
        t1 = time.perf_counter()
        tuned = ex.tune_layers(layers, bufs, part, a.trials)
        el = time.perf_counter() - t1
        pk = ex.peaks()
        rows = []
        for d, r in zip(layers, tuned):
            rows.append({"layer": d["name"], "mult": d["mult"], "best_us": r["best_m"]["median_us"],
                         "space_index": r["best"]["space_index"],
                         "sched": {k: r["best"][k] for k in ("bm", "bn", "bk", "stages", "threads", "split_k")},
                         "kind": r["best_m"]["kind"], "candidates": r["candidates"],
                         "roofline": ex.roofline(d, r["best_m"]["median_us"], ctx["sm_granted"], ctx["copy_bw_gbs"],
                                                 ctx["floor_us"], pk, r["best_m"]["kind"])})
        n = sum(r["candidates"] for r in tuned)
        res = {"partition": ctx, "peaks": pk, "candidates": n, "ok": sum(r["ok"] for r in tuned), "wall_s": el,
               "candidates_per_s": n / el,
               "model_sum_us": sum(d["mult"] * r["best_m"]["median_us"] for d, r in zip(layers, tuned)),
               "layers": rows}
    res["workload"] = wlname
    res["elapsed_s"] = time.time() - t0
    json.dump(res, open(a.out, "w"), indent=1, default=str)
    print(json.dumps({k: v for k, v in res.items() if k not in ("layers",)}, default=str)[:3000])


if __name__ == "__main__":
    main()
