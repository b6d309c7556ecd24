"""Summarise tools/ncu_winners.py captures (one CSV per fraction) into
profiles/r02_ncu_fractions_r50.json: per layer and SM fraction, the winner's
cold-cache duration, tensor-pipe activity over the partition's SMs, DRAM bytes
and GB/s, beside its algorithmic bytes and FLOPs.
  python tools/ncu_winners_summary.py out.json gpurun_out/r2_win_{f}.json gpurun_out/r2_ncuw_{f}.csv ..."""
import collections
import csv
import json
import sys

sys.path.insert(0, ".")
from paper_2008_03602_b200 import experiments as ex, workloads as wl  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "msecond": 1e3,
         "nsecond": 1e-3, "ms": 1e3, "%": 1, "cycle": 1, "": 1}
out_path, pairs = sys.argv[1], sys.argv[2:]
layers = wl.catalog("resnet50")
res = []
for wpath, cpath in zip(pairs[::2], pairs[1::2]):
    win = json.load(open(wpath))
    rows = list(csv.reader(open(cpath)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        e = per.setdefault(r[ii], {"kernel": r[ki].split("(")[0]})
        e[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    launches = list(per.values())
    pos = 0
    for d, w in zip(layers, win["layers"]):
        kpc = 2 if w["kind"] == 7 else 1
        mine = launches[pos + kpc:pos + 2 * kpc]     # the second call (the first may include setup)
        pos += 2 * kpc
        t = sum(k.get("gpu__time_duration.sum", 0) for k in mine)
        dram = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in mine)
        conv = mine[-1]
        f, b = ex.layer_work(d)
        res.append({"layer": d["name"], "fraction": win["fraction"], "sm_granted": win["sm_granted"],
                    "space_index": w["space_index"], "kind": w["kind"], "kernel": conv["kernel"],
                    "grid": conv.get("launch__grid_size"), "duration_us_cold": round(t, 3),
                    "tuned_us_warm": round(w["median_us"], 3),
                    "tensor_pipe_pct_of_partition": round(conv.get(
                        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0), 2),
                    "dram_bytes": dram, "algorithmic_bytes": b, "dram_over_algorithmic": round(dram / b, 3),
                    "dram_gbs": round(dram / (t * 1e-6) / 1e9, 1) if t else None,
                    "tensor_tflops_cold": round(f / (t * 1e-6) / 1e12, 2) if t else None})
    assert pos == len(launches), (cpath, pos, len(launches))
json.dump({"what": "ncu --metrics (cold caches, --clock-control none) of every ResNet-50 b1 winner at each SM "
                   "fraction, tuned oracle-gated in the same partition (tools/ncu_winners.py); "
                   "tensor_pipe_pct_of_partition = sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed "
                   "over the green context's SMs (nominal tensor peak)", "runs": res}, open(out_path, "w"), indent=1)
for f in sorted({r["fraction"] for r in res}):
    rr = [r for r in res if r["fraction"] == f]
    print(f, "layers", len(rr), "tensor% median", sorted(r["tensor_pipe_pct_of_partition"] for r in rr)[len(rr) // 2],
          "max", max(r["tensor_pipe_pct_of_partition"] for r in rr), "dram/alg mean",
          round(sum(r["dram_over_algorithmic"] for r in rr) / len(rr), 2),
          "GB/s median", sorted(r["dram_gbs"] for r in rr)[len(rr) // 2])
