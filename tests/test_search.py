"""Model-guided candidate selection (tp_search_next, host-only).

Pins: batch 0 is the C17 SplitMix64 sample prefix; batches never repeat a
measured index; the call is deterministic; and on a synthetic latency
surface with a known optimum (a smooth function of the schedule's tile shape
plus a wave-quantisation term) the guided search reaches the optimum within
a budget where random sampling does not."""
import math

import pytest

from oracle import space as sp
from paper_2008_03602_b200 import tp, workloads as wl

D = wl.catalog("resnet50")[16]          # l3.b1.c2: 920 TMA-kind schedules


def synthetic_us(s, sm=148):
    """A smooth surrogate latency: optimum at BM=64, BN=32, BK=128, split_k=4."""
    ctas = s["grid_x"] * s["grid_y"] * s["grid_z"]
    waves = math.ceil(ctas / sm)
    return (2.0 + 0.6 * abs(math.log2(s["bm"]) - 6) + 0.5 * abs(math.log2(s["bn"]) - 5)
            + 0.4 * abs(math.log2(s["bk"]) - 7) + 0.3 * abs(math.log2(s["split_k"]) - 2)
            + 0.05 * s["stages"] + 0.2 * (s["threads"] == 128) + 0.8 * (waves - 1))


def test_batch0_is_c17_sample_prefix_and_deterministic():
    n = tp.space_size(D)
    first = tp.search_next(D, 148, [], [], 16, 0.25, 7)
    assert first == sp.sample(n, 16, 7)
    assert first == tp.search_next(D, 148, [], [], 16, 0.25, 7)


def test_batches_are_new_distinct_and_deterministic():
    space = sp.enumerate_space(D)
    idx, us = [], []
    for _ in range(6):
        nxt = tp.search_next(D, 148, idx, us, 16, 0.25, 3)
        assert len(nxt) == 16 and len(set(nxt)) == 16 and not set(nxt) & set(idx)
        assert nxt == tp.search_next(D, 148, idx, us, 16, 0.25, 3)
        idx += nxt
        us += [synthetic_us(space[i]) for i in nxt]
    # failed measurements (<= 0) count as measured but are not fitted
    nxt = tp.search_next(D, 148, idx, [-1.0] + us[1:], 8, 0.0, 3)
    assert not set(nxt) & set(idx)


def test_guided_beats_random_on_synthetic_surface():
    space = sp.enumerate_space(D)
    lat = [synthetic_us(s) for s in space]
    opt = min(lat)
    budget, batch = 96, 16
    idx, us = [], []
    while len(idx) < budget:
        nxt = tp.search_next(D, 148, idx, us, batch, 0.25, 11)
        idx += nxt
        us += [lat[i] for i in nxt]
    guided = min(us)
    rand = [min(lat[i] for i in sp.sample(len(space), budget, seed)) for seed in range(20)]
    assert guided <= opt * 1.02
    assert guided <= sorted(rand)[len(rand) // 2]      # at least as good as the median random run


def test_exhaustive_budget_returns_everything():
    d = wl.catalog("resnet50")[19]
    n = tp.space_size(d)
    idx = []
    while True:
        nxt = tp.search_next(d, 148, idx, [1.0 + (i % 7) for i in idx], 64, 0.5, 1)
        if not nxt:
            break
        idx += nxt
    assert sorted(idx) == list(range(n))


def test_bad_arguments():
    with pytest.raises(tp.TPError):
        tp.search_next(D, 148, [10 ** 6], [1.0], 4)
    with pytest.raises(tp.TPError):
        tp.search_next(D, 148, [], [], 0)


def test_early_stop_rule_hand_cases():
    """Reading C19 (TVM stops when new configurations show no
    latency improvement): stop once the last `early_stop` measured candidates
    did not strictly lower the best latency measured before them."""
    f = tp.search_should_stop
    assert not f([], 3)
    assert not f([5.0, 4.0, 3.0], 3)                 # every candidate improves
    assert not f([5.0, 4.0, 6.0, 7.0], 3)            # two after the last improvement
    assert f([5.0, 4.0, 6.0, 7.0, 4.5], 3)           # three after it
    assert not f([5.0, 4.0, 6.0, 4.0], 3)            # a tie is no improvement, but only two so far
    assert f([5.0, 4.0, 6.0, 4.0, 4.0], 3)
    assert f([5.0, 4.0, 6.0, 4.0, 4.0, 3.9], 3) is False   # the newest one improves
    assert f([-1.0, -1.0, -1.0], 3)                  # failed candidates never improve
    assert not f([-1.0, -1.0, 2.0], 3)               # the first valid one is an improvement
    assert not f([9.0] * 10, 0)                      # early_stop <= 0: never
    assert f([1.0] + [2.0] * 5, 5) and not f([1.0] + [2.0] * 4, 5)
