"""Exhaustive tune of VGG-19 b16 (config 4 data, oracle-gated) inside ONE 25% partition:
best per kind per layer and the tensor fraction of the partition's share.
usage: python tools/vgg_probe.py [fraction] [layer,...]"""
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, experiments as ex, refs, tp, workloads as wl  # noqa: E402
tp.init(0)
frac = float(sys.argv[1]) if len(sys.argv) > 1 else 0.25
layers = wl.catalog("vgg19_b16")
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
checks = refs.load("vgg19_b16", 4, layers)
part = tp.Partition.get(frac)
pk = ex.peaks()
for li, d in enumerate(layers):
    if only and d["name"] not in only:
        continue
    x, w, b = datagen.make_inputs(d, datagen.data_seed(4, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    n = tp.space_size(d)
    scheds = [tp.space_get(d, i) for i in range(n)]
    recs = tp.tune_subset(buf, part, list(range(n)), check_idx=checks[li][0], check_ref=checks[li][1])
    best = {}
    for s, r in zip(scheds, recs):
        if r["status"] == 0 and (s["kind"] not in best or r["median_us"] < best[s["kind"]][0]):
            best[s["kind"]] = (r["median_us"], s["space_index"], s["bm"], s["bn"], s["stages"], s["tiles_per_cta"])
    f = ex.layer_work(d)[0]
    share = pk["bf16_tflops"] * 1e12 * part.sm_granted / 148
    print(d["name"], part.sm_granted, "ok", sum(r["status"] == 0 for r in recs), "/", n,
          {k: (round(v[0], 1), round(f / (v[0] * 1e-6) / share, 3), v[1:]) for k, v in sorted(best.items())}, flush=True)
del buf
