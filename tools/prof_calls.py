"""Python-side cost around each tune_subset call of one bench step (TP_PROFILE=1 for the C++ phases).
usage: TP_PROFILE=1 python tools/prof_calls.py"""
import sys
import time
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, shard, tp, workloads as wl  # noqa: E402
tp.init(0)
part = tp.Partition.get(1.0)
layers = wl.catalog("resnet50")
bufs = [tp.LayerBuffers(d, *datagen.make_inputs(d, datagen.data_seed(2, i)), part=part) for i, d in enumerate(layers)]
cands = [tp.space_sample(d, 1000, datagen.sampler_seed(0)) for d in layers]
tm = tp.timing()
for rep in range(2):
    t_call = t_pack = 0.0
    t0 = time.perf_counter()
    for i, d in enumerate(layers):
        a = time.perf_counter()
        recs = tp.tune_subset(bufs[i], part, cands[i], timing_cfg=tm)
        b = time.perf_counter()
        shard.pack(recs, 0, i, 0)
        t_call += b - a
        t_pack += time.perf_counter() - b
        sys.stderr.write(f"[py] {d['name']} call {1e3 * (b - a):.1f} ms\n")
    print(f"step {rep}: {time.perf_counter() - t0:.2f} s, tune_subset {t_call:.2f} s, pack {t_pack:.3f} s", flush=True)
