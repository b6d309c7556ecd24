"""The C-ABI library loads without a GPU, exports every symbol include/tp.h
declares, and its host-only entry points validate descriptors (no compute)."""
import ctypes

import pytest

from paper_2008_03602_b200 import tp, workloads as wl


def test_exports_every_declared_symbol():
    syms = tp.exported_symbols()
    assert len(syms) >= 25
    lib = ctypes.CDLL(tp.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_status_strings():
    for s in range(7):
        assert tp._lib.tp_status_str(s)
    assert tp._lib.tp_status_str(5) == b"mismatch"


@pytest.mark.parametrize("bad", [dict(c=0), dict(groups=3), dict(stride_h=0), dict(pad_w=-1), dict(r=300),
                                 dict(dtype=7), dict(epilogue=8)])
def test_invalid_descriptors_rejected(bad):
    d = dict(wl.catalog("resnet50")[2], **bad)
    with pytest.raises(tp.TPError) as e:
        tp.space_size(d)
    assert e.value.status == tp.EINVAL


def test_unsupported_on_gpu_path():
    d = dict(wl.catalog("resnet50")[2], dil_h=2, dil_w=2)
    with pytest.raises(tp.TPError) as e:
        tp.space_size(d)
    assert e.value.status == tp.EUNSUPPORTED
    d = dict(wl.catalog("resnet50")[2], groups=2)
    with pytest.raises(tp.TPError) as e:
        tp.space_size(d)
    assert e.value.status == tp.EUNSUPPORTED


def test_space_get_out_of_range():
    d = wl.catalog("resnet50")[2]
    with pytest.raises(tp.TPError) as e:
        tp.space_get(d, tp.space_size(d))
    assert e.value.status == tp.EINVALID_CONFIG


def test_workspace_sizes():
    d = wl.catalog("resnet50")[18]     # l4.b0.c2: split-K candidates need partials
    s1 = next(s for s in (tp.space_get(d, i) for i in range(tp.space_size(d))) if s["split_k"] == 1)
    s8 = next(s for s in (tp.space_get(d, i) for i in range(tp.space_size(d))) if s["split_k"] == 8)
    # every schedule of a tensor-core layer reserves the split-K arrival counters at offset 0
    # (one int per 64 x 32 tile) so no other workspace region can overlap them
    counters = -(-(-(-49 // 64) * -(-512 // 32) * 4) // 256) * 256
    assert tp.workspace_size(d, s1) == counters
    tiles = -(-49 // s8["bm"]) * -(-512 // s8["bn"])
    assert tp.workspace_size(d, s8) >= 8 * tiles * s8["bm"] * s8["bn"] * 4
    assert tp.workspace_size(d) >= tp.workspace_size(d, s8)
    dn = dict(d, in_layout=tp.NCHW)
    assert tp.workspace_size(dn, s1) >= d["n"] * d["c"] * d["h"] * d["w"] * 2 + 49 * 512 * 2


def test_launch_count_starts_at_zero_without_gpu():
    assert tp.launch_count() >= 0
