"""Repeat the sampled schedules of test_layer_random_parity many times to catch races."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle import conv as oc, space as sp
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
names = sys.argv[1].split(",")
reps = int(sys.argv[2])
for d in wl.catalog("resnet50"):
    if d["name"] not in names: continue
    x, w, b = datagen.make_inputs(d, datagen.data_seed(9, 0))
    xr = torch.tensor(x).bfloat16().double().numpy(); wr = torch.tensor(w).bfloat16().double().numpy()
    ref = oc.conv2d_c(d, xr, wr, b, relu=True)
    buf = tp.LayerBuffers(d, x, w, b)
    for i in sp.sample(tp.space_size(d), 6, 1):
        s = tp.space_get(d, i)
        nbad = 0
        for r in range(reps):
            buf.poison()
            tp.conv2d_run(buf, s)
            torch.cuda.synchronize()
            y = buf.output()
            err = np.max(np.abs(y - ref)) / np.max(np.abs(ref))
            if not err <= 2e-2:
                nbad += 1
                if nbad <= 2:
                    nanpx = np.argwhere(~np.isfinite(y))
                    print("  bad rep", r, "err", err, "nan count", len(nanpx), "first", nanpx[:3].tolist(), flush=True)
        print(d["name"], i, {k: s[k] for k in ("bm","bn","bk","stages","threads","split_k","grid_x","grid_y","grid_z")}, "bad", nbad, "/", reps, flush=True)
