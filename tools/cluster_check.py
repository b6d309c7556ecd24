"""Check which split-K reduction a schedule uses (trace slots 60/61) and its timing."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog('resnet50')
li = [d['name'] for d in cat].index('r50.l3.b1.c1')
d = cat[li]
x, w, b = datagen.make_inputs(d, 5)
buf = tp.LayerBuffers(d, x, w, b)
for sk in (1, 2, 4, 8):
    s = next(tp.space_get(d, i) for i in range(tp.space_size(d))
             if tp.space_get(d, i)['split_k'] == sk and tp.space_get(d, i)['bm'] == 64 and tp.space_get(d, i)['bn'] == 32
             and tp.space_get(d, i)['bk'] == 128 and tp.space_get(d, i)['stages'] == 4 and tp.space_get(d, i)['threads'] == 256)
    tr = tp.conv2d_trace(buf, s).astype(np.int64)
    m = tp.conv2d_run(buf, s, None, tp.timing())
    print(sk, "cluster_red", set(tr[:, 60].tolist()), "nctarank", set(tr[:, 61].tolist()), "us", round(m['median_us'], 2),
          "epi", int(np.median(tr[:, 3] - tr[:, 2])), "main", int(np.median(tr[:, 2] - tr[:, 1])), flush=True)
    if sk > 1:
        sub = [int(np.median(tr[:, j] - tr[:, 2])) for j in (65, 64, 66, 67, 3)]
        print("   epi sub-points from tmem_full (cluster wait, sent, received, stored, end):", sub,
              "entry skew cyc", int(np.max(tr[:, 0]) - np.min(tr[:, 0])), flush=True)
