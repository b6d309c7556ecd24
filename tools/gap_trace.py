"""Where does a b1 launch's time go?  Four back-to-back launches of each
layer's tuned winner (from a bench/report JSON), captured in one CUDA graph
(the timing protocol's launch mode) and traced in-kernel (tp_conv2d_trace).
For launches 2..3 (steady state) it prints, relative to the previous launch's
last CTA end (ns, median over CTAs): CTA entry, PDL-wait release, first
k-block ready at the MMA, epilogue start and end; and the per-CTA cycle
breakdown of the last launch.

  python tools/gap_trace.py profiles/r02_bench_first.json [layer,layer,...] [fraction] [catalog]
"""
import json
import sys


def _load_json(path):
    """A JSON file, or the last JSON line of a bench.py stdout capture."""
    text = open(path).read()
    try:
        return json.loads(text)
    except ValueError:
        return json.loads([ln for ln in text.splitlines() if ln.strip().startswith('{')][-1])
import os
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_2008_03602_b200 import datagen, tp, workloads as wl  # noqa: E402

tp.init(0)
src = _load_json(sys.argv[1])
rows = src["latency_us"]["per_layer"] if "latency_us" in src else src["layers"]
best = {r["layer"]: r["space_index"] for r in rows}
names = sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] else list(best)
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
catname = sys.argv[4] if len(sys.argv) > 4 else "resnet50"
config = {"resnet50": 2, "vgg19_b16": 4, "mobilenetv2": 5}[catname]
part = tp.Partition.get(frac)
cat = {d["name"]: (i, d) for i, d in enumerate(wl.catalog(catname))}
GHZ = float(os.environ.get("SM_GHZ", "1.965"))
summary = []
for name in names:
    li, d = cat[name]
    x, w, b = datagen.make_inputs(d, datagen.data_seed(config, li))
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    s = tp.space_get(d, best[name])
    if s["kind"] not in (tp.KIND_IGEMM_TC, tp.KIND_IGEMM_TC_GATHER):
        continue
    m = tp.conv2d_run(buf, s, part, tp.timing())
    tr = tp.conv2d_trace(buf, s, part, launches=4).astype(np.int64)
    n = len(tr) // 4
    ent = tr[:, 63]                                   # globaltimer ns at entry
    cyc = lambda col: ent + (tr[:, col] - tr[:, 0]) / GHZ   # noqa: E731
    end = cyc(3)
    ends = [end[l * n:(l + 1) * n].max() for l in range(4)]
    print(f"{name:14s} k{s['kind']} {s['bm']}x{s['bn']}x{s['bk']} st{s['stages']} sk{s['split_k']} ctas {n} "
          f"loop {m['median_us']:.2f}us | graph period L1->L2 {ends[2] - ends[1]:.0f} ns, L2->L3 {ends[3] - ends[2]:.0f} ns",
          flush=True)
    for l in (2, 3):
        sl = slice(l * n, (l + 1) * n)
        t1 = ends[l - 1]
        med = lambda v: f"{np.median(v) - t1:6.0f}"  # noqa: E731
        print(f"   L{l} after L{l-1} end (ns, median): entry {med(ent[sl])} wait-pass {med(cyc(53)[sl])} "
              f"kb0 {med(cyc(4)[sl])} epi {med(cyc(2)[sl])} end {med(end[sl])} (last end {ends[l] - t1:.0f})",
              flush=True)
    c = tr[3 * n:]
    mc = lambda a, b: int(np.median(c[:, a] - c[:, b]))  # noqa: E731
    kbs = [int(np.median(c[:, 4 + i] - c[:, 53])) for i in range(16) if (c[:, 4 + i] > 0).all()]
    print(f"   L3 cycles from entry: bar-init {mc(52, 0)} tmem-alloc {mc(58, 0)} sync {mc(1, 0)} wait-pass {mc(53, 0)} | "
          f"wait->kb ready {kbs[:10]} wait->epi {mc(2, 53)} epi {mc(3, 2)}", flush=True)
    if (c[:, 68] > 0).all():
        print(f"   L3 epilogue cycles (thread 0) from tmem_full: first tcgen05.ld done {mc(68, 2)} stores issued "
              f"{mc(69, 2)} pre-sync {mc(70, 2)} end {mc(3, 2)}; split-K: sent {mc(64, 2) if (c[:, 64] > 0).all() else '-'} "
              f"received {mc(66, 2) if (c[:, 66] > 0).all() else '-'}", flush=True)
    sm = c[:, 62]
    cnt = np.bincount(sm.astype(int), minlength=148)
    shared = cnt[sm.astype(int)] > 1
    endc = end[3 * n:] - ends[2]
    print(f"   L3 placement: SMs used {int((cnt > 0).sum())}, max CTAs/SM {int(cnt.max())}, CTAs sharing an SM "
          f"{int(shared.sum())}/{n}; end ns (median) shared {np.median(endc[shared]) if shared.any() else 0:.0f} "
          f"alone {np.median(endc[~shared]) if (~shared).any() else 0:.0f}; slowest 5 CTAs end "
          f"{[int(v) for v in np.sort(endc)[-5:]]}", flush=True)
    summary.append({"layer": name, "loop_us": m["median_us"], "period_ns": float(ends[3] - ends[2]),
                    "end_to_wait_ns": float(np.median(cyc(53)[3 * n:]) - ends[2]),
                    "wait_to_kb0_cyc": kbs[0] if kbs else None, "wait_to_epi_cyc": mc(2, 53), "epi_cyc": mc(3, 2)})
print(json.dumps(summary))
