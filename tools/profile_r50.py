"""Run each ResNet-50 layer's tuned-best schedule (tools/r50_best_*.json) a few
times -- a short, deterministic command for ncu launch lists / full captures."""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_2008_03602_b200 import datagen, tp, workloads as wl
best = json.load(open(sys.argv[1] if len(sys.argv) > 1 else 'tools/r50_best_r01.json'))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
only = sys.argv[3].split(',') if len(sys.argv) > 3 else None
tp.init(0)
part = tp.Partition.get(1.0)
for li, d in enumerate(wl.catalog('resnet50')):
    if only and d['name'] not in only: continue
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    s = tp.space_get(d, best[d['name']])
    for _ in range(reps):
        tp.conv2d_run(buf, s, part)
    part.sync()
    m = tp.conv2d_run(buf, s, part, tp.timing())
    print(d['name'], best[d['name']], round(m['median_us'], 3), flush=True)
