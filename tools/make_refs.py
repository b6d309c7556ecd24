"""Write the fp64 oracle reference points used by the in-loop correctness gate
("compare with oracle reference points").

Calls only ``oracle/`` (and the seeded input generators of ``datagen``, which
hold none of the method's arithmetic).  For every layer of each benchmarked
(catalog, config) it draws the layer's inputs with the config's data seed
(DESIGN.md section 13), rounds x and w to bf16 (RNE, reading C7) for bf16
layers, picks 4096 output points with ``datagen.sample_points(total, 4096,
11 + layer)`` and stores the oracle's fp64 values at them:

    refs/<catalog>_cfg<config>.npz   ref_<layer> (float64 [<= 4096]), meta (json)

bench.py and the experiments read these files (they never execute the
oracle); the indices are regenerated from the same seed and checked against
the stored count and checksum.

    python tools/make_refs.py            # all sets
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import conv as oc  # noqa: E402
from paper_2008_03602_b200 import datagen, workloads as wl  # noqa: E402

SETS = (("cfg1", 1), ("resnet50", 2), ("vgg19_b16", 4), ("mobilenetv2", 5))
POINTS = 4096


def point_seed(layer: int) -> int:
    return 11 + layer


def bf16_round(a: np.ndarray) -> np.ndarray:
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).bfloat16().double().numpy()


def make_set(cat: str, config: int) -> str:
    layers = wl.catalog(cat)
    arrays = {}
    meta = {"catalog": cat, "config": config, "points": POINTS, "point_seed": "11 + layer",
            "data_seed": f"datagen.data_seed({config}, layer)", "layers": []}
    for li, d in enumerate(layers):
        x, w, b = datagen.make_inputs(d, datagen.data_seed(config, li))
        if d["dtype"] == wl.BF16:
            x, w = bf16_round(x), bf16_round(w)
        P = oc.out_dim(d["h"], d["r"], d["stride_h"], d["pad_h"], 1)
        Q = oc.out_dim(d["w"], d["s"], d["stride_w"], d["pad_w"], 1)
        total = d["n"] * d["k"] * P * Q
        idx = datagen.sample_points(total, POINTS, point_seed(li))
        ref = oc.conv2d_points_c(d, x, w, b if d["epilogue"] & 1 else None, bool(d["epilogue"] & 2), idx)
        arrays[f"ref_{li}"] = ref
        meta["layers"].append({"name": d["name"], "total": total, "n_points": int(idx.shape[0]),
                               "idx_sum": int(idx.sum()), "epilogue": d["epilogue"]})
    path = os.path.join(ROOT, "refs", f"{cat}_cfg{config}.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **arrays)
    return path


if __name__ == "__main__":
    for cat, cfg in SETS:
        t0 = time.perf_counter()
        print(make_set(cat, cfg), f"{time.perf_counter() - t0:.1f}s", flush=True)
