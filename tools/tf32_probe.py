"""Time selected 3xTF32 schedules of cfg1 (experiments: TP_DEBUG_TC bit2 = no hi/lo split work,
bit3 = one MMA per k-step).  usage: python tools/tf32_probe.py"""
import sys
sys.path.insert(0, '.')
from paper_2008_03602_b200 import datagen, tp, workloads as wl  # noqa: E402
tp.init(0)
d = wl.catalog("cfg1")[0]
x, w, b = datagen.make_inputs(d, 1)
buf = tp.LayerBuffers(d, x, w, b)
want = [(64, 32, 4, 1), (128, 64, 3, 1), (64, 32, 4, 2), (128, 64, 4, 4)]
for i in range(tp.space_size(d)):
    s = tp.space_get(d, i)
    if s["kind"] == tp.KIND_IGEMM_TF32X3 and (s["bm"], s["bn"], s["stages"], s["split_k"]) in want:
        m = tp.conv2d_run(buf, s, None, tp.timing())
        print(f"bm{s['bm']} bn{s['bn']} st{s['stages']} sk{s['split_k']}: {m['median_us']:.2f} us", flush=True)
