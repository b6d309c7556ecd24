"""Exhaustive tuning records (median us per space index) of every layer of a
catalog at one SM fraction -- ground truth for the offline search evaluation.
usage: dump_exhaustive.py catalog fraction out.json"""
import json
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat, frac, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
part = tp.Partition.get(frac)
res = {"catalog": cat, "fraction": frac, "sm_granted": part.sm_granted, "layers": {}}
for li, d in enumerate(wl.catalog(cat)):
    x, w, b = datagen.make_inputs(d, datagen.data_seed(3, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    recs = tp.tune_subset(buf, part, list(range(tp.space_size(d))), timing_cfg=tp.timing(prune_ratio=0.0))
    res["layers"][d["name"]] = [r["median_us"] if r["status"] == 0 else -1.0 for r in recs]
    print(d["name"], len(recs), round(min(r["median_us"] for r in recs if r["status"] == 0), 3), flush=True)
json.dump(res, open(out, "w"))
