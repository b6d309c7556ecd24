"""Print the in-kernel timeline (tp_conv2d_trace) of a few schedules of a layer."""
import json, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog('resnet50')
names = sys.argv[1].split(',')
extra = [json.loads(a) for a in sys.argv[2:]]   # schedule overrides, e.g. '{"bm":128,"bn":64,...}'
best = json.load(open('tools/r50_best_r01.json'))
for li, d in enumerate(cat):
    if d['name'] not in names: continue
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
    buf = tp.LayerBuffers(d, x, w, b)
    scheds = [tp.space_get(d, best[d['name']])]
    n = tp.space_size(d)
    for ov in extra:
        for i in range(n):
            s = tp.space_get(d, i)
            if all(s[k] == v for k, v in ov.items()):
                scheds.append(s); break
    for s in scheds:
        for _ in range(3): tp.conv2d_run(buf, s)
        buf.poison()
        tr = tp.conv2d_trace(buf, s).astype(np.int64)
        m = tp.conv2d_run(buf, s, None, tp.timing())
        pro = tr[:, 1] - tr[:, 0]; main = tr[:, 2] - tr[:, 1]; epi = tr[:, 3] - tr[:, 2]
        kb = [tr[:, 4 + i] - tr[:, 0] for i in range(8) if (tr[:, 4 + i] > 0).all()]
        prod = [tr[:, 20 + i] - tr[:, 0] for i in range(8) if (tr[:, 20 + i] > 0).all()]
        com = [tr[:, 36 + i] - tr[:, 0] for i in range(8) if (tr[:, 36 + i] > 0).all()]
        gstart = (tr[:, 63] - tr[:, 63].min()) / 1000.0
        key = {k: s[k] for k in ('bm', 'bn', 'bk', 'stages', 'threads', 'split_k', 'grid_x', 'grid_y', 'grid_z')}
        print(d['name'], key, f"loop {m['median_us']:.2f}us")
        print("   cycles median: prologue", int(np.median(pro)), "mainloop", int(np.median(main)), "epilogue",
              int(np.median(epi)), "total", int(np.median(tr[:, 3] - tr[:, 0])))
        print("   kb arrival (cyc from entry, median):", [int(np.median(k)) for k in kb])
        print("   producer past empty-wait:", [int(np.median(k)) for k in prod])
        print("   mma after commit:", [int(np.median(k)) for k in com])
        print("   CTA start skew us: max", round(float(gstart.max()), 2), "p50", round(float(np.median(gstart)), 2))
