"""Tune the ResNet-50 b1 layers at one SM fraction (oracle-gated) and write the
winners, or (--run) launch each winner twice inside that fraction's partition --
the short command ncu profiles for per-fraction tensor-pipe / DRAM evidence.
  python tools/ncu_winners.py tune <fraction> <out.json>
  FRAC=<fraction> python tools/ncu_winners.py run <winners.json>"""
import json
import os
import sys

sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, refs, tp, workloads as wl  # noqa: E402

tp.init(0)
layers = wl.catalog("resnet50")
if sys.argv[1] == "tune":
    frac = float(sys.argv[2])
    part = tp.Partition.get(frac)
    checks = refs.load("resnet50", 2, layers)
    out = {"fraction": frac, "sm_granted": part.sm_granted, "layers": []}
    for li, d in enumerate(layers):
        x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
        buf = tp.LayerBuffers(d, x, w, b, part=part)
        best, m, recs = tp.tune(buf, part, 1000, datagen.sampler_seed(0), check_idx=checks[li][0],
                                check_ref=checks[li][1])
        out["layers"].append({"layer": d["name"], "space_index": best["space_index"], "kind": best["kind"],
                              "median_us": m["median_us"], "sm_tuned": best["sm_tuned"]})
    json.dump(out, open(sys.argv[3], "w"), indent=1)
else:
    src = json.load(open(sys.argv[2]))
    part = tp.Partition.get(float(os.environ.get("FRAC", src["fraction"])))
    for li, (d, r) in enumerate(zip(layers, src["layers"])):
        x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
        buf = tp.LayerBuffers(d, x, w, b, part=part)
        s = dict(tp.space_get(d, r["space_index"]), sm_tuned=r["sm_tuned"])
        for _ in range(2):
            tp.conv2d_run(buf, s, part)
        part.sync()
    print("ran", len(layers))
