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
    # the 3xTF32 kind: tf32 at half the bf16 rate, three MMAs per product
    r4 = ex.roofline(dd, 3.0, 148, 6000.0, 0.8, pk, 5)
    assert r4["roof_us"]["compute_us"] == pytest.approx(ex.layer_work(dd)[0] / (1480e12 / 6) * 1e6)


@pytest.mark.parametrize("name", ["cfg1", "resnet50", "vgg19_b16", "mobilenetv2"])
def test_default_schedule_is_valid_base_kind(name):
    """f2 untuned column: one fixed schedule per layer, in the layer's space, of
    its base kind, and the closest one to the documented target tuple."""
    from paper_2008_03602_b200 import tp
    for d in wl.catalog(name):
        s = ex.default_schedule(d)
        assert s is not None and s["kind"] == tp.layer_kind(d)
        assert tp.space_get(d, s["space_index"]) == s
        P, Q = tp.output_shape(d)
        if s["kind"] == tp.KIND_IGEMM_TC and d["c"] >= 64 and d["k"] >= 128 and d["n"] * P * Q >= 128:
            # the target tuple itself is valid for these layers
            assert (s["bm"], s["bn"], s["bk"], s["stages"], s["split_k"]) == (128, 128, 64, 4, 1)


def test_aggregate_5k_sweet_spot():
    fr = (0.1, 0.25, 0.5, 1.0)
    m = {str(p): {str(q): 100.0 * (1 + abs(p - q)) / q for q in fr} for p in fr}
    a = ex.aggregate_5k(m, fr)
    assert a["total_ms_by_tuned_at"]["0.25"] == pytest.approx(sum(m["0.25"][str(q)] for q in fr))
    assert a["sweet_spot_tuned_at"] == min(fr, key=lambda p: sum(m[str(p)][str(q)] for q in fr))


def test_pd_check_flags_a_diagonal_above_its_column():
    fr = (0.1, 1.0)

    def row(m, cv=0.01):
        return {"layer": "x", "matrix_us": {str(p): {str(q): m[(p, q)] for q in fr} for p in fr},
                "matrix_cv": {str(p): {str(q): cv for q in fr} for p in fr}}
    ok = row({(0.1, 0.1): 10.0, (1.0, 0.1): 10.2, (0.1, 1.0): 5.0, (1.0, 1.0): 4.0})
    r = ex.pd_check([ok], fr)
    assert r["pass"] and r["cells"] == 2
    # diagonal 10.0 vs off-diagonal 9.5 at q = 0.1: 10.0 > 9.5 (1 + 3 x 0.01) -> violation
    bad = row({(0.1, 0.1): 10.0, (1.0, 0.1): 9.5, (0.1, 1.0): 5.0, (1.0, 1.0): 4.0})
    r = ex.pd_check([bad], fr)
    assert not r["pass"] and r["violations"][0]["tuned_at"] == 1.0 and r["violations"][0]["run_at"] == 0.1
    # the same gap is noise when the cells' CV is 2%: eps = 0.06 and 10.0 <= 9.5 x 1.06
    assert ex.pd_check([row({(0.1, 0.1): 10.0, (1.0, 0.1): 9.5, (0.1, 1.0): 5.0, (1.0, 1.0): 4.0}, 0.02)],
                       fr)["pass"]


def test_resnet50_sequence_matches_multiplicities():
    import collections
    seq = wl.resnet50_sequence()
    cnt = collections.Counter(seq)
    assert len(seq) == 53 and seq[0] == "r50.conv1"
    assert all(cnt[d["name"]] == d["mult"] for d in wl.catalog("resnet50"))
    # each stage's first block ends with its downsample projection (torchvision order)
    assert seq[1:5] == ["r50.l1.b0.c1", "r50.l1.b0.c2", "r50.l1.b0.c3", "r50.l1.b0.c3"]
    assert seq[seq.index("r50.l4.b0.c1") + 3] == "r50.l4.b0.ds"
