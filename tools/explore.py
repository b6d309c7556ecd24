"""GPU exploration: exhaustive tune of selected layers, dump every record with
its schedule, summarise by knob, trace the best split-1 / split>1 schedules,
and time the empty-kernel floor.  Usage: python tools/explore.py cat name,name,... [out.json]"""
import collections, json, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl

tp.init(0)
part = tp.Partition.get(float(__import__('os').environ.get('FRAC', '1.0')))
out = {"floor": {}}
for c, t in ((1, 32), (1, 128), (148, 128), (148, 256), (296, 128)):
    m = part.floor(c, t)
    out["floor"][f"{c}x{t}"] = m["median_us"]
print("floor us:", out["floor"], flush=True)
cat = wl.catalog(sys.argv[1])
names = sys.argv[2].split(',') if len(sys.argv) > 2 and sys.argv[2] != 'all' else [d['name'] for d in cat]
KN = ("bm", "bn", "bk", "stages", "threads", "split_k", "tile_q", "vec_k", "tile_p", "smem_stage")
for li, d in enumerate(cat):
    if d['name'] not in names:
        continue
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    best, bm, recs = tp.tune(buf, part, 100000, 42)
    rows = []
    for r in recs:
        s = tp.space_get(d, r["space_index"])
        rows.append(dict({k: s[k] for k in KN}, us=r["median_us"], ctas=r["ctas"], st=r["status"]))
    out[d['name']] = rows
    ok = [r for r in rows if r["st"] == 0]
    ok.sort(key=lambda r: r["us"])
    print(f"== {d['name']} space={len(rows)} best={ok[0]['us']:.2f}us", flush=True)
    for r in ok[:6]:
        print("   ", r)
    knobs = ("bm", "bn", "bk", "stages", "threads", "split_k") if d.get('kind_hint', tp.layer_kind(d)) == 0 else \
        ("threads", "tile_q", "vec_k", "tile_p", "smem_stage")
    for k in knobs:
        g = collections.defaultdict(list)
        for r in ok:
            g[r[k]].append(r["us"])
        print(f"   best by {k}:", {v: round(min(u), 2) for v, u in sorted(g.items())})
    if tp.layer_kind(d) == 0:
        for pick in (lambda r: r["split_k"] == 1, lambda r: r["split_k"] > 1):
            cand = [r for r in ok if pick(r)]
            if not cand:
                continue
            r = cand[0]
            s = next(tp.space_get(d, i) for i in range(tp.space_size(d))
                     if all(tp.space_get(d, i)[k] == r[k] for k in ("bm", "bn", "bk", "stages", "threads", "split_k")))
            tr = tp.conv2d_trace(buf, s, part).astype(np.int64)
            pro = tr[:, 1] - tr[:, 0]; main = tr[:, 2] - tr[:, 1]; epi = tr[:, 3] - tr[:, 2]
            kb = [int(np.median(tr[:, 4 + i] - tr[:, 0])) for i in range(16) if (tr[:, 4 + i] > 0).all()]
            gstart = (tr[:, 63] - tr[:, 63].min()) / 1000.0
            print(f"   trace split={r['split_k']} {r['us']:.2f}us: prologue {int(np.median(pro))} main {int(np.median(main))}"
                  f" epi {int(np.median(epi))} total {int(np.median(tr[:, 3] - tr[:, 0]))} cyc; kb arrivals {kb};"
                  f" start skew max {gstart.max():.2f}us", flush=True)
if len(sys.argv) > 3:
    json.dump(out, open(sys.argv[3], 'w'))
