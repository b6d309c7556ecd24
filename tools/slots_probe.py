"""Per-schedule medians of the multi-tile kinds (row-halo, multi-tile im2col,
stem) on VGG-19 b16 layers in a 25% partition, for the A/B of the balanced
tile spans (TcArgs::slots; run once with TP_NO_SLOTS=1 and once without).
usage: python tools/slots_probe.py out.json [layer indices, default 0,1,2]"""
import json
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl  # noqa: E402
tp.init(0)
out = sys.argv[1]
lis = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2").split(",")]
part = tp.Partition.get(0.25)
res = []
for li in lis:
    d = wl.catalog("vgg19_b16")[li]
    x, w, b = datagen.make_inputs(d, datagen.data_seed(4, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    idx = [i for i in range(tp.space_size(d))
           if tp.space_get(d, i)["kind"] in (tp.KIND_IGEMM_TC_ROW, tp.KIND_IGEMM_TC_MT, tp.KIND_IGEMM_TC_STEM)
           and tp.space_get(d, i)["tiles_per_cta"] > 1]
    recs = tp.tune_subset(buf, part, idx, timing_cfg=tp.timing())
    for i, r in zip(idx, recs):
        s = tp.space_get(d, i)
        res.append({"layer": d["name"], "idx": i, "kind": s["kind"], "bm": s["bm"], "bn": s["bn"],
                    "stages": s["stages"], "tpc": s["tiles_per_cta"], "grid_x": s["grid_x"],
                    "us": r["median_us"], "ctas_per_sm": r["ctas_per_sm"], "status": r["status"],
                    "sm": part.sm_granted})
    best = min((r for r in res if r["layer"] == d["name"] and r["status"] == 0), key=lambda r: r["us"], default=None)
    print(d["name"], best, flush=True)
    del buf
json.dump(res, open(out, "w"))
