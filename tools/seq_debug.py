import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
FAST = dict(warmup=1, groups=3, n_min=3, target_group_us=5.0)
def buf_for(li):
    d = wl.catalog("resnet50")[li]
    x, w, b = datagen.make_inputs(d, 3)
    return d, tp.LayerBuffers(d, x, w, b)
mode = sys.argv[1]
if "p" in mode:
    d, buf = buf_for(10)
    p25 = tp.Partition.get(0.25)
    tp.tune(buf, p25, trials=64, seed=43, timing_cfg=tp.timing(**FAST))
    print("p25 tune ok")
if "x" in mode:
    d, buf = buf_for(10)
    p25, p100 = tp.Partition.get(0.25), tp.Partition.get(1.0)
    b25, m25, r = tp.tune(buf, p25, trials=64, seed=43, timing_cfg=tp.timing(**FAST))
    tp.cross_eval(buf, b25, p100, tp.timing(**FAST))
    print("cross ok", b25["split_k"])
d, buf = buf_for(2)
best, m, recs = tp.tune(buf, None, trials=10**6, seed=42, timing_cfg=tp.timing(**FAST))
bad = [r["space_index"] for r in recs if r["status"] != 0]
print(mode, "bad", len(bad), bad[:5], tp._lib.tp_last_error())
