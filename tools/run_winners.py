"""Launch each tuned winner of a bench JSON line once, in catalog order, inside
the tuning fraction's partition -- the short command the DRAM-traffic ncu
capture profiles (tools/ncu_summary.py dram).
usage: python tools/run_winners.py <bench.json> [catalog] [config]"""
import json
import os
import sys

sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl  # noqa: E402

tp.init(0)
line = [ln for ln in open(sys.argv[1]).read().splitlines() if ln.strip().startswith("{")][-1]
src = json.loads(line)
cat = sys.argv[2] if len(sys.argv) > 2 else "resnet50"
config = int(sys.argv[3]) if len(sys.argv) > 3 else 2
win = {r["layer"]: r["space_index"] for r in src["latency_us"]["per_layer"]}
part = tp.Partition.get(float(os.environ.get("FRAC", src["latency_us"].get("at_fraction", 1.0))))
for li, d in enumerate(wl.catalog(cat)):
    x, w, b = datagen.make_inputs(d, datagen.data_seed(config, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    tp.conv2d_run(buf, dict(tp.space_get(d, win[d["name"]]), sm_tuned=part.sm_granted), part,
                  tp.timing(warmup=0, groups=1, n_min=1, target_group_us=0.0, use_graph=0))
    part.sync()
print("ran", len(win))
