"""Where does a b1 launch's time go?  Two back-to-back launches of each layer's
tuned winner (from a bench/report JSON), traced in-kernel (tp_conv2d_trace):
the second launch's CTA entry, PDL-wait release, first k-block ready at the
MMA, epilogue start and end, relative to the first launch's last CTA end (ns).

  python tools/gap_trace.py profiles/r01_bench.json [layer,layer,...] [fraction]
"""
import json
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_2008_03602_b200 import datagen, tp, workloads as wl  # noqa: E402

tp.init(0)
src = json.load(open(sys.argv[1]))
rows = src["latency_us"]["per_layer"] if "latency_us" in src else src["layers"]
best = {r["layer"]: r["space_index"] for r in rows}
names = sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] else list(best)
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
part = tp.Partition.get(frac)
cat = {d["name"]: (i, d) for i, d in enumerate(wl.catalog("resnet50"))}
GHZ = float(__import__("os").environ.get("SM_GHZ", "1.965"))
for name in names:
    li, d = cat[name]
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    s = tp.space_get(d, best[name])
    if s["kind"] == tp.KIND_DIRECT:
        continue
    m = tp.conv2d_run(buf, s, part, tp.timing())
    tr = tp.conv2d_trace(buf, s, part, launches=2).astype(np.int64)
    n = len(tr) // 2
    ent = tr[:, 63]                                   # globaltimer ns at entry
    cyc = lambda col: ent + (tr[:, col] - tr[:, 0]) / GHZ   # noqa: E731
    end = cyc(3)
    t1 = end[:n].max()                                # first launch: last CTA end
    L2 = slice(n, 2 * n)
    f = lambda v: f"{np.min(v) - t1:7.0f}/{np.median(v) - t1:7.0f}/{np.max(v) - t1:7.0f}"  # noqa: E731
    print(f"{name:14s} k{s['kind']} {s['bm']}x{s['bn']}x{s['bk']} st{s['stages']} sk{s['split_k']} "
          f"ctas {n} loop {m['median_us']:.2f}us | L1 span {t1 - ent[:n].min():.0f} ns", flush=True)
    print(f"   L2 (min/med/max ns after L1 end) entry {f(ent[L2])} wait-pass {f(cyc(53)[L2])} "
          f"kb0-ready {f(cyc(4)[L2])} epi {f(cyc(2)[L2])} end {f(end[L2])}", flush=True)
    c = tr[L2]
    med = lambda a, b: int(np.median(c[:, a] - c[:, b]))  # noqa: E731
    kbs = [int(np.median(c[:, 4 + i] - c[:, 53])) for i in range(16) if (c[:, 4 + i] > 0).all()]
    print(f"   L2 cycles: wait->issued {[med(54 + i, 53) for i in range(4) if (c[:, 54 + i] > 0).all()]} "
          f"wait->kb ready {kbs} wait->epi {med(2, 53)} epi {med(3, 2)}", flush=True)
    print(f"   L2 cycles from entry: bar-init {med(52, 0)} tmem-alloc {med(58, 0)} wait-pass {med(53, 0)} "
          f"sync {med(1, 0)} kb0 {med(4, 0)} epi {med(2, 0)} end {med(3, 0)}", flush=True)
