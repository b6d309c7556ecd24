"""Debug helper: run every schedule of a layer, report mismatches vs the oracle."""
import sys, collections
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import conv as oc
from paper_2008_03602_b200 import datagen, tp, workloads as wl

tp.init(0)
cat, li = sys.argv[1], int(sys.argv[2])
integer = len(sys.argv) > 3 and sys.argv[3] == "int"
d = wl.catalog(cat)[li]
if integer:
    d = dict(d, out_dtype=tp.FP32, epilogue=1)
x, w, b = datagen.make_inputs(d, 3, integer=integer)
xr = torch.tensor(x).bfloat16().double().numpy() if d["dtype"] == tp.BF16 else x
wr = torch.tensor(w).bfloat16().double().numpy() if d["dtype"] == tp.BF16 else w
ref = oc.conv2d_c(d, xr, wr, b, relu=bool(d["epilogue"] & 2))
buf = tp.LayerBuffers(d, x, w, b)
n = tp.space_size(d)
bad = collections.Counter(); badlist = []
for i in range(n):
    s = tp.space_get(d, i)
    buf.poison()
    tp.conv2d_run(buf, s)
    torch.cuda.synchronize()
    y = buf.output()
    err = np.max(np.abs(y - ref)) / np.max(np.abs(ref))
    if not (err <= (0 if integer else 2e-2)):
        key = tuple(s[k] for k in ("bm", "bn", "bk", "stages", "threads", "split_k"))
        badlist.append(key)
        if len(badlist) <= 6:
            nanmask = ~np.isfinite(y)
            # y is NKPQ; locate bad pixels
            bad_px = np.argwhere(np.any(~np.isclose(y, ref, rtol=0.05, atol=0.05) | nanmask, axis=1))
            print("BAD", key, "err", err, "nan", int(nanmask.sum()), "of", y.size, "bad px", len(bad_px),
                  "first", bad_px[:4].tolist(), "last", bad_px[-2:].tolist())
print(d["name"], "space", n, "bad", len(badlist))
for k in range(6):
    c = collections.Counter(b[k] for b in badlist)
    print(["bm", "bn", "bk", "stages", "threads", "split_k"][k], dict(c))
