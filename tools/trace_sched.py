"""Trace one schedule of one layer: python tools/trace_sched.py catalog layer bm bn bk stages threads split [frac]"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog(sys.argv[1])
li = [d['name'] for d in cat].index(sys.argv[2])
d = cat[li]
ov = dict(zip(("bm", "bn", "bk", "stages", "threads", "split_k"), map(int, sys.argv[3:9])))
part = tp.Partition.get(float(sys.argv[9]) if len(sys.argv) > 9 else 1.0)
x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
buf = tp.LayerBuffers(d, x, w, b, part=part)
import os
if os.environ.get("KIND"):
    ov["kind"] = int(os.environ["KIND"])
s = next(tp.space_get(d, i) for i in range(tp.space_size(d)) if all(tp.space_get(d, i)[k] == v for k, v in ov.items()))
m = tp.conv2d_run(buf, s, part, tp.timing())
tr = tp.conv2d_trace(buf, s, part).astype(np.int64)
g = (tr[:, 63] - tr[:, 63].min()) / 1000.0
life = (tr[:, 3] - tr[:, 0])
print(d['name'], ov, f"loop {m['median_us']:.2f}us ctas {len(tr)} ctas/sm {m['ctas_per_sm']}")
print("  median cycles: prologue", int(np.median(tr[:, 1] - tr[:, 0])), "main", int(np.median(tr[:, 2] - tr[:, 1])),
      "epi", int(np.median(tr[:, 3] - tr[:, 2])), "life", int(np.median(life)))
print("  kb arrivals (MMA)", [int(np.median(tr[:, 4 + i] - tr[:, 0])) for i in range(16) if (tr[:, 4 + i] > 0).all()])
print("  producer kb done", [int(np.median(tr[:, 20 + i] - tr[:, 0])) for i in range(16) if (tr[:, 20 + i] > 0).all()])
print("  start times us: span", round(float(g.max()), 2), "per-SM CTAs:", np.bincount(tr[:, 62].astype(int)).max(),
      "concurrency est", round(float(np.sum(life) / 1.9e3 / max(g.max(), 1e-9)), 1))
if (tr[:, 84] > 0).any():
    print("  gather: past empty-wait", [int(np.median(tr[:, 84 + i] - tr[:, 0])) for i in range(8) if (tr[:, 84 + i] > 0).all()])
    print("  gather: chunks stored  ", [int(np.median(tr[:, 68 + i] - tr[:, 0])) for i in range(8) if (tr[:, 68 + i] > 0).all()])
    print("  gather: past fence     ", [int(np.median(tr[:, 76 + i] - tr[:, 0])) for i in range(8) if (tr[:, 76 + i] > 0).all()])
