"""The stored gate references (refs/, written by tools/make_refs.py from the
oracle) agree bit for bit with the oracle recomputed here, and the loader
regenerates the same indices."""
import numpy as np
import pytest

from oracle import conv as oc
from paper_2008_03602_b200 import datagen, refs, workloads as wl

SETS = (("cfg1", 1), ("resnet50", 2), ("vgg19_b16", 4), ("mobilenetv2", 5))


def _bf16(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).bfloat16().double().numpy()


@pytest.mark.parametrize("cat,cfg", SETS)
def test_refs_match_oracle(cat, cfg):
    layers = wl.catalog(cat)
    got = refs.load(cat, cfg, layers)
    assert len(got) == len(layers)
    # recompute the cheapest and the last layer through the oracle
    for li in sorted({0, len(layers) - 1}):
        d = layers[li]
        x, w, b = datagen.make_inputs(d, datagen.data_seed(cfg, li))
        if d["dtype"] == wl.BF16:
            x, w = _bf16(x), _bf16(w)
        idx, ref = got[li]
        P = oc.out_dim(d["h"], d["r"], d["stride_h"], d["pad_h"], 1)
        Q = oc.out_dim(d["w"], d["s"], d["stride_w"], d["pad_w"], 1)
        assert np.array_equal(idx, datagen.sample_points(d["n"] * d["k"] * P * Q, 4096, refs.point_seed(li)))
        exp = oc.conv2d_points_c(d, x, w, b, True, idx)
        assert np.array_equal(ref, exp)
