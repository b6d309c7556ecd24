"""Two back-to-back launches of one schedule, traced: does launch 2 start before launch 1 ends (PDL)?"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
for name in sys.argv[1].split(','):
    cat = wl.catalog('resnet50')
    li = [d['name'] for d in cat].index(name)
    d = cat[li]
    x, w, b = datagen.make_inputs(d, 1)
    buf = tp.LayerBuffers(d, x, w, b)
    # the bench winner for the layer
    import json
    best = {r["layer"]: r["space_index"] for r in json.load(open("profiles/r01_bench.json"))["latency_us"]["per_layer"]}
    s = tp.space_get(d, best[name])
    m = tp.conv2d_run(buf, s, None, tp.timing())
    tr = tp.conv2d_trace(buf, s, None, launches=2).astype(np.int64)
    n = len(tr) // 2
    g = tr[:, 63]                                  # globaltimer ns at entry
    life = (tr[:, 3] - tr[:, 0]) / 1.92            # ns (cycles at ~1.92 GHz)
    end = g + life
    t0 = g[:n].min()
    print(name, {k: s[k] for k in ('bm', 'bn', 'bk', 'stages', 'split_k')}, f"loop {m['median_us']:.2f}us",
          f"| L1 entry [{(g[:n].min()-t0)/1e3:.2f},{(g[:n].max()-t0)/1e3:.2f}] end max {(end[:n].max()-t0)/1e3:.2f}",
          f"| L2 entry [{(g[n:].min()-t0)/1e3:.2f},{(g[n:].max()-t0)/1e3:.2f}] past-wait med {(np.median(g[n:] + (tr[n:,53]-tr[n:,0])/1.92)-t0)/1e3:.2f}"
          f" end max {(end[n:].max()-t0)/1e3:.2f} us", flush=True)
