"""Launch one schedule of one layer a few times (short command for ncu):
python tools/run_sched.py catalog layer bm bn bk stages threads split [reps]
(direct kind: catalog layer D threads tile_q vec_k tile_p smem_stage [reps]);
FRAC=<p> runs it inside a green-context partition of that SM share."""
import os
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog(sys.argv[1])
li = [d['name'] for d in cat].index(sys.argv[2])
d = cat[li]
if sys.argv[3] == "D":
    ov = dict(zip(("threads", "tile_q", "vec_k", "tile_p", "smem_stage"), map(int, sys.argv[4:9])))
else:
    ov = dict(zip(("bm", "bn", "bk", "stages", "threads", "split_k"), map(int, sys.argv[3:9])))
reps = int(sys.argv[9]) if len(sys.argv) > 9 else 3
part = tp.Partition.get(float(os.environ.get("FRAC", "1.0")))
x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
buf = tp.LayerBuffers(d, x, w, b, part=part)
if os.environ.get("KIND"):
    ov["kind"] = int(os.environ["KIND"])
if os.environ.get("TPC"):
    ov["tiles_per_cta"] = int(os.environ["TPC"])
s = next(tp.space_get(d, i) for i in range(tp.space_size(d)) if all(tp.space_get(d, i)[k] == v for k, v in ov.items()))
for _ in range(reps):
    tp.conv2d_run(buf, s, part)
part.sync()
print("done", d['name'], ov)
