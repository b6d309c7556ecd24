"""Compare green-context partitions with and without SM co-scheduling (fine-grained split):
granted SMs, whether (1,1,k) clusters can launch, and the tuned latency of a few layers."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
cat = wl.catalog('resnet50')
names = ['r50.l3.b1.c2', 'r50.l4.b1.c2', 'r50.l4.b0.c2', 'r50.l2.b1.c2']
for frac in (0.1, 0.25, 0.5):
    for flags in (1, 0):
        part = tp.Partition.get(frac, flags=flags)
        out = []
        for name in names:
            li = [d['name'] for d in cat].index(name)
            d = cat[li]
            x, w, b = datagen.make_inputs(d, 1)
            buf = tp.LayerBuffers(d, x, w, b, part=part)
            best, m, recs = tp.tune(buf, part, 10 ** 6, 42)
            s = [r for r in recs if r['status'] == 0]
            sk = {}
            for r in s:
                k = tp.space_get(d, r['space_index'])['split_k']
                sk[k] = min(sk.get(k, 1e9), r['median_us'])
            tr = tp.conv2d_trace(buf, dict(tp.space_get(d, min((r for r in s if tp.space_get(d, r['space_index'])['split_k'] > 1), key=lambda r: r['median_us'])['space_index'])), part)
            out.append(f"{name}: best {m['median_us']:.2f} (sk{best['split_k']}) cluster={int(tr[0, 60])} by_sk={ {k: round(v, 1) for k, v in sorted(sk.items())} }")
        print(f"frac {frac} flags {flags} granted {part.sm_granted}: " + " | ".join(out), flush=True)
