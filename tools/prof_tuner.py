import sys, time
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
for li in (2, 16, 19):
    d = wl.catalog('resnet50')[li]
    x, w, b = datagen.make_inputs(d, 1)
    buf = tp.LayerBuffers(d, x, w, b)
    t0 = time.perf_counter()
    recs = tp.tune_subset(buf, None, list(range(tp.space_size(d))), timing_cfg=tp.timing())
    print(d['name'], len(recs), f"{(time.perf_counter()-t0)*1e3:.1f} ms", flush=True)
