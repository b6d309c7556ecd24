"""Launch one schedule (by space index) of one layer a few times inside the
FRAC partition -- a short command for ncu.  usage: run_idx.py catalog layer idx [reps]"""
import os
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog(sys.argv[1])
li = [d['name'] for d in cat].index(sys.argv[2])
d = cat[li]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
part = tp.Partition.get(float(os.environ.get("FRAC", "1.0")))
x, w, b = datagen.make_inputs(d, datagen.data_seed(3, li))
buf = tp.LayerBuffers(d, x, w, b, part=part)
s = tp.space_get(d, int(sys.argv[3]))
for _ in range(reps):
    tp.conv2d_run(buf, s, part)
part.sync()
print("ok", d["name"], s["space_index"], part.sm_granted)
