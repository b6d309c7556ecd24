"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv> <out.json>
  python tools/ncu_summary.py full <prof.ncu-rep> <out.json>
  python tools/ncu_summary.py dram <dram.csv> <out.json> [catalog]   (one launch per layer, catalog order)
  python tools/ncu_summary.py fractions <out.json> <ncuf_*.csv ...>   (tuned winner per SM fraction)
"""
import collections
import csv
import io
import json
import subprocess
import sys

FULL_KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
             "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
             "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
             "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
             "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
             "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
             "lts__t_bytes.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "msecond": 1e3,
         "nsecond": 1e-3, "ms": 1e3}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size")
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows[hi + 1:]:
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-3)
        name = r[ki].split("(")[0]
        key = f"{name} grid={r[gi]}"
        a = agg.setdefault(key, {"kernel": name, "grid": r[gi], "launches": 0, "total_us": 0.0})
        a["launches"] += 1
        a["total_us"] += us
        total += us
    res = []
    for a in agg.values():
        a["mean_us"] = round(a["total_us"] / a["launches"], 3)
        a["share"] = round(a["total_us"] / total, 4)
        a["total_us"] = round(a["total_us"], 3)
        res.append(a)
    res.sort(key=lambda a: -a["total_us"])
    by_kernel = collections.defaultdict(float)
    for a in res:
        by_kernel[a["kernel"].split("<")[0]] += a["total_us"]
    json.dump({"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, "
                                       "serialised per-launch times; compare shares, not absolutes",
               "total_us": round(total, 3),
               "share_by_kernel": {k: round(v / total, 4) for k, v in sorted(by_kernel.items(), key=lambda t: -t[1])},
               "launch_groups": res}, open(out, "w"), indent=1)


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else ""}
        for k in FULL_KEYS:
            if k in h:
                i = h.index(k)
                try:
                    val = float(v[i].replace(",", ""))
                except ValueError:
                    val = v[i]
                d[k] = val
                d[k + ".unit"] = u[i]
        # normalised per-launch DRAM traffic in bytes
        rb = d.get("dram__bytes_read.sum", 0) * SCALE.get(d.get("dram__bytes_read.sum.unit", "byte"), 1)
        wb = d.get("dram__bytes_write.sum", 0) * SCALE.get(d.get("dram__bytes_write.sum.unit", "byte"), 1)
        d["dram_bytes_per_launch"] = rb + wb
        res.append(d)
    json.dump({"source": path, "kernels": res}, open(out, "w"), indent=1)


def dram(path, out, catalog="resnet50", winners=None):
    """Per-launch DRAM traffic (ncu replays with cold caches: the compulsory
    bytes each tuned layer really moves) next to its algorithmic bytes.
    winners: the bench JSON line (or {layer: space_index}) the capture ran,
    recorded per layer so bench.py can tell which winners it covers."""
    sys.path.insert(0, ".")
    from paper_2008_03602_b200 import experiments as ex, workloads as wl
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ii, mi, vi, ui, ki = (h.index(k) for k in ("ID", "Metric Name", "Metric Value", "Metric Unit", "Kernel Name"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        e = per.setdefault(r[ii], {"kernel": r[ki].split("(")[0]})
        e[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    layers = wl.catalog(catalog)
    win = {}
    if winners:
        src = json.load(open(winners))
        win = {r["layer"]: r["space_index"] for r in src["latency_us"]["per_layer"]} if "latency_us" in src else src
    res = []
    for d, e in zip(layers, per.values()):
        alg = ex.layer_work(d)[1]
        traffic = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
        res.append({"layer": d["name"], "space_index": win.get(d["name"]), "kernel": e["kernel"],
                    "dram_bytes": traffic, "algorithmic_bytes": alg,
                    "ratio": traffic / alg, "cold_us": e.get("gpu__time_duration.sum")})
    n = len(res)
    json.dump({"source": path, "note": "ncu default cache control (caches flushed before each replay): DRAM bytes are "
                                       "the cold-cache traffic of one launch of each tuned layer",
               "launches": n, "mean_dram_bytes_per_launch": sum(r["dram_bytes"] for r in res) / max(n, 1),
               "mean_algorithmic_bytes_per_launch": sum(r["algorithmic_bytes"] for r in res) / max(n, 1),
               "dram_over_algorithmic": sum(r["dram_bytes"] for r in res) / max(1.0, sum(r["algorithmic_bytes"]
                                                                                         for r in res)),
               "layers": res}, open(out, "w"), indent=1)


def fractions(out, *paths):
    """Tensor-pipe and DRAM evidence of the tuned winner at each SM fraction.
    Under a green context ncu's per-SM averages cover the context's SMs only
    (a 38-SM VGG run reads 64% tensor-pipe active; a 148-SM normalisation
    would exceed 100% for the 14-SM runs), so the value is reported as is --
    a percentage of the nominal tensor peak of the partition's SMs."""
    granted = {"0.1": 14, "0.25": 38, "0.5": 74, "1.0": 148}
    res = []
    for path in paths:
        name = path.split("ncuf_")[1].rsplit(".csv", 1)[0]
        layer, frac = name.rsplit("_", 1)
        rows = list(csv.reader(open(path)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        mi, vi, ui, ki = (h.index(k) for k in ("Metric Name", "Metric Value", "Metric Unit", "Kernel Name"))
        m, kern = {}, ""
        for r in rows[hi + 1:]:
            m[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
            kern = r[ki].split("(")[0]
        g = granted.get(frac, 148)
        t_us = m.get("gpu__time_duration.sum", 0.0)
        dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        tp_dev = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        res.append({"layer": layer, "fraction": float(frac), "sm_granted": g, "kernel": kern,
                    "grid": m.get("launch__grid_size"), "duration_us_cold": t_us,
                    "tensor_pipe_pct_of_partition": tp_dev,
                    "dram_bytes": dram, "dram_gbs": dram / (t_us * 1e-6) / 1e9 if t_us else None})
    res.sort(key=lambda r: (r["layer"], r["fraction"]))
    json.dump({"note": "ncu --metrics, --clock-control none, caches flushed per replay (cold); "
                       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed averages over the "
                       "green context's SMs (nominal tensor peak)", "runs": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "fractions":
        fractions(sys.argv[2], *sys.argv[3:])
    else:
        fn = {"launches": launches, "full": full, "dram": dram}[sys.argv[1]]
        fn(*sys.argv[2:])
