"""Run each ResNet-50 layer's tuned-best schedule a few times, without the
timing protocol -- a short, deterministic command for ncu launch lists and
full captures.  usage: profile_r50.py best.json [reps] [layer,layer,...]
(best.json: {layer name: space_index}, or a bench.py JSON line)."""
import json
import sys


def _load_json(path):
    """A JSON file, or the last JSON line of a bench.py stdout capture."""
    text = open(path).read()
    try:
        return json.loads(text)
    except ValueError:
        return json.loads([ln for ln in text.splitlines() if ln.strip().startswith('{')][-1])


sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl
src = _load_json(sys.argv[1])
if "latency_us" in src:
    src = {r["layer"]: r["space_index"] for r in src["latency_us"]["per_layer"]}
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
only = sys.argv[3].split(',') if len(sys.argv) > 3 else None
tp.init(0)
part = tp.Partition.get(1.0)
for li, d in enumerate(wl.catalog('resnet50')):
    if only and d['name'] not in only:
        continue
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    s = tp.space_get(d, src[d['name']])
    for _ in range(reps):
        tp.conv2d_run(buf, s, part)
    part.sync()
print("ok", flush=True)
