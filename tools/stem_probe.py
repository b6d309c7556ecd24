"""Best stem-kind vs best other schedule of the three C = 3 stems (tune_subset over each kind).
usage: python tools/stem_probe.py"""
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl  # noqa: E402
tp.init(0)
for cat, li, frac in (("resnet50", 0, 1.0), ("resnet50", 0, 0.25), ("vgg19_b16", 0, 0.25), ("mobilenetv2", 0, 0.5)):
    d = wl.catalog(cat)[li]
    part = tp.Partition.get(frac)
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    n = tp.space_size(d)
    scheds = [tp.space_get(d, i) for i in range(n)]
    recs = tp.tune_subset(buf, part, list(range(n)), timing_cfg=tp.timing())
    best = {}
    for s, r in zip(scheds, recs):
        if r["status"] == 0 and (s["kind"] not in best or r["median_us"] < best[s["kind"]][0]):
            best[s["kind"]] = (r["median_us"], {k: s[k] for k in ("bm", "bn", "bk", "stages", "threads", "split_k",
                                                                  "tiles_per_cta")})
    print(d["name"], frac, {k: (round(v[0], 2), v[1]) for k, v in best.items()}, flush=True)
