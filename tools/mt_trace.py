"""Per-tile timeline of a multi-tile schedule (row-halo, multi-tile im2col, strip):
tile i's loads issued (producer; stem kind: patch landed, then im2col tile built), MMAs issued (MMA warp), accumulator ready and
drained (epilogue issuer warp), for the first 8 tiles of each CTA, in cycles from CTA entry.
usage: python tools/mt_trace.py catalog layer space_index [fraction]"""
import os
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
from paper_2008_03602_b200 import datagen, tp, workloads as wl  # noqa: E402
tp.init(0)
cat = wl.catalog(sys.argv[1])
li = [d["name"] for d in cat].index(sys.argv[2])
d = cat[li]
part = tp.Partition.get(float(sys.argv[4]) if len(sys.argv) > 4 else 1.0)
x, w, b = datagen.make_inputs(d, datagen.data_seed(4, li))
buf = tp.LayerBuffers(d, x, w, b, part=part)
s = dict(tp.space_get(d, int(sys.argv[3])), sm_tuned=part.sm_granted)
m = tp.conv2d_run(buf, s, part, tp.timing())
# the last of 4 launches captured in one graph (the timing loop's mode: warm
# caches, weights issued before the PDL wait); MT_LAUNCHES=1 for a lone launch
nl = int(os.environ.get("MT_LAUNCHES", "4"))
tr = tp.conv2d_trace(buf, s, part, launches=nl).astype(np.int64)
tr = tr[(len(tr) // nl) * (nl - 1):]
tr = tr[tr[:, 3] > 0]
rel = lambda c: tr[:, c] - tr[:, 0]  # noqa: E731
print(d["name"], {k: s[k] for k in ("kind", "bm", "bn", "stages", "tiles_per_cta")}, f"loop {m['median_us']:.1f}us",
      "ctas run", len(tr), "threads", m["threads_per_cta"])
print("median cycles from entry: prologue", int(np.median(rel(1))), "end", int(np.median(rel(3))),
      *(("weights staged", int(np.median(rel(2)))) if (tr[:, 2] > 0).all() else ()),
      *(("| stem: first patches issued", int(np.median(rel(52)))) if (tr[:, 52] > 0).all() else ()),
      *(("weights landed", int(np.median(rel(53)))) if (tr[:, 53] > 0).all() else ()),
      *(("| stem: after trigger", int(np.median(rel(54))), "before staging", int(np.median(rel(55))),
         "patch 0", int(np.median(rel(56))), "patch 1", int(np.median(rel(57))))
        if (tr[:, 57] > 0).all() else ()))
for name, base in (("loads issued", 4), ("stem: a free", 44), ("tile built", 36), ("MMAs issued", 12), ("acc ready", 28), ("drained", 20)):
    print(f"  {name:13s}", [int(np.median(rel(base + i))) for i in range(8) if (tr[:, base + i] > 0).all()])
d_tile = np.diff(np.stack([rel(20 + i) for i in range(8) if (tr[:, 20 + i] > 0).all()], 1), axis=1)
print("  drain period per tile (median over CTAs)", [int(v) for v in np.median(d_tile, 0)])
