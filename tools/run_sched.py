"""Launch one schedule of one layer a few times (short command for ncu):
python tools/run_sched.py catalog layer bm bn bk stages threads split [reps]"""
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog(sys.argv[1])
li = [d['name'] for d in cat].index(sys.argv[2])
d = cat[li]
ov = dict(zip(("bm", "bn", "bk", "stages", "threads", "split_k"), map(int, sys.argv[3:9])))
reps = int(sys.argv[9]) if len(sys.argv) > 9 else 3
x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
buf = tp.LayerBuffers(d, x, w, b)
s = next(tp.space_get(d, i) for i in range(tp.space_size(d)) if all(tp.space_get(d, i)[k] == v for k, v in ov.items()))
for _ in range(reps):
    tp.conv2d_run(buf, s)
tp.Partition.get(1.0).sync()
print("done", d['name'], ov)
