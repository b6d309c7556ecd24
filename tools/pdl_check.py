"""Loop latency of a few schedules of one layer (run under different env settings)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog('resnet50')
name = sys.argv[1] if len(sys.argv) > 1 else 'r50.l3.b1.c1'
d = cat[[x['name'] for x in cat].index(name)]
x, w, b = datagen.make_inputs(d, 5)
buf = tp.LayerBuffers(d, x, w, b)
part = tp.Partition.get(1.0)
fl = part.floor(1, 128)['median_us']
out = [f"{name} PDL={os.environ.get('TP_PDL','1')} NOCL={os.environ.get('TP_NO_CLUSTER','0')} floor={fl:.2f}"]
for sk in (1, 2, 4, 8):
    cands = [i for i in range(tp.space_size(d)) if tp.space_get(d, i)['split_k'] == sk and tp.space_get(d, i)['bn'] == 32
             and tp.space_get(d, i)['threads'] == 256 and tp.space_get(d, i)['stages'] == 4]
    best = None
    for i in cands:
        s = tp.space_get(d, i)
        m = tp.conv2d_run(buf, s, part, tp.timing())
        g = tp.conv2d_run(buf, s, part, tp.timing(use_graph=0))
        if best is None or m['median_us'] < best[0]:
            best = (m['median_us'], g['median_us'], s['bm'], s['bk'])
    if best:
        out.append(f"sk{sk}: graph {best[0]:.2f} nograph {best[1]:.2f} (bm{best[2]} bk{best[3]})")
print(" | ".join(out), flush=True)
