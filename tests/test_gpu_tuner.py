"""GPU: partitions (green contexts), the tuning loop, the correctness gate and
cross-evaluation."""
import numpy as np
import pytest
import torch

from oracle import conv as oc
from oracle import space as sp
from paper_2008_03602_b200 import datagen, tp, workloads as wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _init():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a GPU")
    tp.init(0)
    yield


FAST = dict(warmup=1, groups=3, n_min=3, target_group_us=5.0)


def test_whole_device_probe_uses_all_sms():
    part = tp.Partition.get(1.0)
    assert part.sm_granted == torch.cuda.get_device_properties(0).multi_processor_count
    ids = part.probe_smids(4 * part.sm_granted)
    assert ids.min() >= 0 and len(set(ids.tolist())) == part.sm_granted


@pytest.mark.parametrize("frac", [0.10, 0.25, 0.50])
def test_partition_membership(frac):
    part = tp.Partition.get(frac)
    assert part.sm_requested == sp.requested_sms(frac)
    assert part.sm_granted >= part.sm_requested
    ids = part.probe_smids(8 * part.sm_granted)
    used = set(ids.tolist())
    assert min(used) >= 0
    assert len(used) <= part.sm_granted, (len(used), part.sm_granted)
    # the same partition object is cached (long-lived)
    assert tp.Partition.get(frac).handle == part.handle


def test_split_partitions_disjoint():
    parts = tp.Partition.split(4, 32)
    try:
        sets = [set(p.probe_smids(8 * p.sm_granted).tolist()) for p in parts]
        for i in range(4):
            assert len(sets[i]) <= parts[i].sm_granted
            for j in range(i + 1, 4):
                assert not (sets[i] & sets[j])
    finally:
        for p in parts:
            p.close()


def _layer_with_ref(d, seed=3):
    x, w, b = datagen.make_inputs(d, seed)
    xr = torch.tensor(x).bfloat16().double().numpy() if d["dtype"] == tp.BF16 else x
    wr = torch.tensor(w).bfloat16().double().numpy() if d["dtype"] == tp.BF16 else w
    ref = oc.conv2d_c(d, xr, wr, b, relu=True)
    return tp.LayerBuffers(d, x, w, b), ref


def test_tune_exhaustive_small_layer_selects_argmin():
    d = wl.catalog("resnet50")[19]          # l4.b0.c3 49x2048x512
    buf, ref = _layer_with_ref(d)
    idx = datagen.sample_points(ref.size, 1024, 1)
    n = tp.space_size(d)
    best, best_m, recs = tp.tune(buf, None, trials=10 ** 6, seed=42, check_idx=idx, check_ref=ref.reshape(-1)[idx],
                                 timing_cfg=tp.timing(**FAST))
    assert len(recs) == n
    assert [r["space_index"] for r in recs] == list(range(n))
    assert all(r["status"] == 0 for r in recs), [r for r in recs if r["status"]][:3]
    k = sp.argmin(recs)
    assert recs[k]["space_index"] == best["space_index"] == best_m["space_index"]
    assert best["grid_x"] > 0 and best["sm_tuned"] == best_m["sm_granted"]
    # y holds the winner's output
    assert np.max(np.abs(buf.output() - ref)) / np.max(np.abs(ref)) <= 2e-2


def test_tune_sampled_matches_mirror_order():
    d = wl.catalog("resnet50")[2]
    buf, ref = _layer_with_ref(d)
    _, _, recs = tp.tune(buf, None, trials=20, seed=7, timing_cfg=tp.timing(**FAST))
    assert [r["space_index"] for r in recs] == sp.sample(tp.space_size(d), 20, 7)


def test_gate_rejects_wrong_reference():
    d = wl.catalog("resnet50")[3]
    buf, ref = _layer_with_ref(d)
    idx = datagen.sample_points(ref.size, 256, 2)
    bad = ref.reshape(-1)[idx] + 1.0
    recs = tp.tune_subset(buf, None, [0, 1, 2], check_idx=idx, check_ref=bad, timing_cfg=tp.timing(**FAST))
    assert all(r["status"] == tp.EMISMATCH for r in recs)


def test_tune_in_partition_and_cross_eval():
    d = wl.catalog("resnet50")[10]
    buf, ref = _layer_with_ref(d)
    p25, p100 = tp.Partition.get(0.25), tp.Partition.get(1.0)
    best25, m25, recs = tp.tune(buf, p25, trials=64, seed=43, timing_cfg=tp.timing(**FAST))
    assert m25["sm_granted"] == p25.sm_granted and best25["sm_tuned"] == p25.sm_granted
    x100 = tp.cross_eval(buf, best25, p100, tp.timing(**FAST))
    assert x100["status"] == 0 and x100["sm_granted"] == p100.sm_granted
    assert x100["ctas"] == m25["ctas"]          # frozen geometry (C15)
    assert np.max(np.abs(buf.output() - ref)) / np.max(np.abs(ref)) <= 2e-2


def test_direct_tune_fp32_cfg1_parity():
    d = wl.catalog("cfg1")[0]
    buf, ref = _layer_with_ref(d)
    idx = datagen.sample_points(ref.size, 4096, 4)
    best, m, recs = tp.tune(buf, None, trials=48, seed=1, check_idx=idx, check_ref=ref.reshape(-1)[idx],
                            timing_cfg=tp.timing(**FAST))
    assert all(r["status"] == 0 for r in recs)
    assert np.max(np.abs(buf.output() - ref)) / np.max(np.abs(ref)) <= 1e-5


def test_cold_l2_timing_runs():
    d = wl.catalog("resnet50")[2]
    buf, _ = _layer_with_ref(d)
    s = tp.space_get(d, 0)
    hot = tp.conv2d_run(buf, s, None, tp.timing(**FAST))
    cold = tp.conv2d_run(buf, s, None, tp.timing(warmup=1, groups=3, n_min=3, flush_l2=1))
    assert hot["median_us"] > 0 and cold["median_us"] > 0


def test_launch_counter_advances():
    d = wl.catalog("resnet50")[2]
    buf, _ = _layer_with_ref(d)
    c0 = tp.launch_count()
    tp.conv2d_run(buf, tp.space_get(d, 0))
    torch.cuda.synchronize()
    assert tp.launch_count() == c0 + 1


def test_prune_ratio_times_slow_candidates_with_one_group():
    """Reading C12b: with prune_ratio > 0 the clearly-slow candidates get one
    timed group; the winner always gets the full protocol; 0 disables it."""
    d = wl.catalog("resnet50")[2]
    buf, _ = _layer_with_ref(d)
    best, m, recs = tp.tune(buf, None, trials=10 ** 6, seed=42, timing_cfg=tp.timing(**dict(FAST, prune_ratio=2.0)))
    groups = FAST.get("groups", 5)
    bad = [(r["space_index"], r["status"], r["groups"]) for r in recs if r["status"] != 0]
    assert not bad, (bad[:10], tp._lib.tp_last_error())
    assert any(r["groups"] == 1 for r in recs) and all(r["groups"] in (1, groups) for r in recs)
    assert m["groups"] == groups
    _, _, recs0 = tp.tune(buf, None, trials=50, seed=42, timing_cfg=tp.timing(**dict(FAST, prune_ratio=0.0)))
    assert all(r["groups"] == groups for r in recs0)


def test_tune_guided_measures_distinct_candidates_and_returns_argmin():
    d = wl.catalog("resnet50")[16]
    buf, ref = _layer_with_ref(d)
    best, m, recs = tp.tune_guided(buf, None, trials=48, batch=16, explore=0.25, seed=5,
                                   timing_cfg=tp.timing(**FAST))
    idx = [r["space_index"] for r in recs]
    assert len(recs) == 48 and len(set(idx)) == 48
    assert idx[:16] == sp.sample(tp.space_size(d), 16, 5)          # batch 0 = C17 sample prefix
    assert all(r["status"] == 0 for r in recs)
    assert recs[sp.argmin(recs)]["space_index"] == best["space_index"] == m["space_index"]
    assert np.max(np.abs(buf.output() - ref)) / np.max(np.abs(ref)) <= 2e-2


def test_graph_update_times_the_right_schedule(monkeypatch):
    """The tuner reuses a window slot's executable graph through
    cudaGraphExecUpdate (new function / grid / attributes in the same chain
    topology).  If an update silently kept the old parameters, every candidate
    would time the same kernel: the per-candidate medians must match those of
    freshly instantiated graphs (TP_GRAPH_UPDATE=0) candidate by candidate."""
    d = wl.catalog("resnet50")[22]                        # l4.b1.c2: split-K clusters and plain grids
    x, w, b = datagen.make_inputs(d, 3)
    buf = tp.LayerBuffers(d, x, w, b)
    idx = list(range(0, tp.space_size(d), 7))[:96]
    tm = tp.timing()
    monkeypatch.setenv("TP_GRAPH_UPDATE", "1")
    upd = tp.tune_subset(buf, None, idx, timing_cfg=tm)
    monkeypatch.setenv("TP_GRAPH_UPDATE", "0")
    ins = tp.tune_subset(buf, None, idx, timing_cfg=tm)
    a = np.array([r["median_us"] for r in upd])
    c = np.array([r["median_us"] for r in ins])
    ok = np.array([r["status"] == 0 and q["status"] == 0 for r, q in zip(upd, ins)])
    assert ok.all()
    ratio = a / c
    assert a.max() / a.min() > 2.0                         # the candidates really differ
    dev = np.abs(ratio - 1)
    assert np.median(dev) < 0.05 and np.percentile(dev, 95) < 0.15 and dev.max() < 0.35, ratio
    # the winner is the same schedule or one within noise of it
    wu, wi = int(np.argmin(a)), int(np.argmin(c))
    assert wu == wi or abs(c[wu] / c[wi] - 1) < 0.05
