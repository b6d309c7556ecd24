"""Trace one schedule of a layer (k-block arrival spacing).  TP_DEBUG_TC=1/2
skips the A/B TMA loads (experiments only).  Usage: tma_probe.py name bm bn bk stages threads split"""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
name = sys.argv[1]
ov = dict(zip(("bm", "bn", "bk", "stages", "threads", "split_k"), map(int, sys.argv[2:8])))
for li, d in enumerate(wl.catalog('resnet50')):
    if d['name'] != name:
        continue
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
    buf = tp.LayerBuffers(d, x, w, b)
    s = next(tp.space_get(d, i) for i in range(tp.space_size(d)) if all(tp.space_get(d, i)[k] == v for k, v in ov.items()))
    for _ in range(3):
        tp.conv2d_run(buf, s)
    rows = []
    for rep in range(3):
        tr = tp.conv2d_trace(buf, s).astype(np.int64)
        rows.append(tr)
    tr = rows[-1]
    m = tp.conv2d_run(buf, s, None, tp.timing())
    kb = [int(np.median(tr[:, 4 + i] - tr[:, 0])) for i in range(16) if (tr[:, 4 + i] > 0).all()]
    ex = [int(np.median(tr[:, 52 + i] - tr[:, 0])) for i in range(8)]
    print(f"{name} dbg={os.environ.get('TP_DEBUG_TC','0')} {ov} loop={m['median_us']:.2f}us prologue={int(np.median(tr[:,1]-tr[:,0]))}"
          f" main={int(np.median(tr[:,2]-tr[:,1]))} epi={int(np.median(tr[:,3]-tr[:,2]))} kb={kb} extra={ex}", flush=True)
