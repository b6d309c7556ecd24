"""Host-side logic of the experiment drivers (paper_2008_03602_b200/experiments.py):
LPT assignment of layers to concurrent tuners and the roofline arithmetic of
SURVEY 8(d).  CPU only."""
import pytest

from paper_2008_03602_b200 import experiments as ex
from paper_2008_03602_b200 import workloads as wl


def test_layer_work_matches_survey_appendix():
    # R50 l1.b0.c2 = 0.2312 GFLOP, 0.877 MB; VGG conv2_1 b16 = 29.595 GFLOP.
    d = wl.catalog("resnet50")[2]
    f, b = ex.layer_work(d)
    assert abs(f / 1e9 - 0.2312) < 5e-4 and abs(b / 1e6 - 0.877) < 5e-3
    f, _ = ex.layer_work(wl.catalog("vgg19_b16")[2])
    assert abs(f / 1e9 - 29.595) < 5e-3


def test_lpt_balances_and_covers():
    layers = wl.catalog("vgg19_b16")
    for k in (1, 2, 4):
        a = ex._lpt(layers, k)
        assert sorted(i for part in a for i in part) == list(range(len(layers)))
        loads = [sum(ex.layer_work(layers[i])[0] for i in part) for part in a]
        biggest = max(ex.layer_work(d)[0] for d in layers)
        assert max(loads) - min(loads) <= biggest + 1e-6      # LPT bound


def test_roofline_fractions_and_binding():
    pk = {"hbm_gbs": 6000.0, "bf16_tflops": 1480.0, "fp32_tflops": 74.0, "sm_max_mhz": 1965.0}
    d = wl.catalog("vgg19_b16")[8]
    f, b = ex.layer_work(d)
    # at 37 of 148 SMs the tensor share is 370 TFLOP/s; time the layer at exactly that roof
    t_us = f / 370e12 * 1e6
    r = ex.roofline(d, t_us, 37, 1500.0, 0.8, pk, 0)
    assert r["tensor_frac"] == pytest.approx(1.0) and r["binding"] == "compute"
    assert r["frac_of_binding_roof"] == pytest.approx(1.0)
    # a tiny layer is floor-bound
    dd = wl.catalog("resnet50")[1]
    r2 = ex.roofline(dd, 3.0, 148, 6000.0, 0.8, pk, 0)
    assert r2["binding"] == "floor" and r2["frac_of_binding_roof"] == pytest.approx(0.8 / 3.0)
    # the direct kind is measured against the FFMA roof
    r3 = ex.roofline(dd, 3.0, 148, 6000.0, 0.8, pk, 1)
    assert r3["roof_us"]["compute_us"] == pytest.approx(ex.layer_work(dd)[0] / 74e12 * 1e6)
