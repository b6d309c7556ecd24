"""GPU parity and path tests added in round 2 (VERDICT r01 "Next round" 3, 8):

* epilogue codes 0 (none) and 2 (ReLU only) in the integer sweeps (SURVEY 8(d):
  parity with and without the epilogue);
* VGG-19 b16 at full size: schedules of every kind of every layer, and the
  exhaustive-tune winners, against 4096 stored oracle points;
* all 30 MobileNetV2 layers on random data;
* concurrent tuners (a14): k host threads x tp_tune on disjoint green contexts,
  gated on oracle points, winners checked against the full oracle output;
* the fraction-taking entry points of SURVEY 8(b);
* f2 (model-level cross-eval) and f3 (interference) drivers;
* bench.py --gpus 2 and the resumable sharded tuning job (two ranks on one GPU,
  TP_BENCH_DEVICE: the ranks' kernels never wait on each other);
* guard bands around y and the workspace: no out-of-bounds writes by any
  schedule of any kind (compute-sanitizer is closed on this GPU pool).
"""
import json
import os
import subprocess
import sys
import threading

import numpy as np
import pytest
import torch

from oracle import conv as oc
from oracle import space as sp
from paper_2008_03602_b200 import datagen, refs, shard, tp, workloads as wl

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _init():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a GPU")
    tp.init(0)
    yield


def bf16_round(a):
    return torch.tensor(np.asarray(a, dtype=np.float32)).bfloat16().double().numpy()


def oracle_ref(d, x, w, b):
    if d["dtype"] == tp.BF16:
        x, w = bf16_round(x), bf16_round(w)
    return oc.conv2d_c(d, x, w, b if d["epilogue"] & 1 else None, relu=bool(d["epilogue"] & 2))


def rel_err(y, ref):
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))


def mk(n, c, h, w, k, r, s, st=1, pad=0, g=1, dtype=tp.BF16, out=None, epi=3):
    return dict(n=n, c=c, h=h, w=w, k=k, r=r, s=s, stride_h=st, stride_w=st, pad_h=pad, pad_w=pad, dil_h=1, dil_w=1,
                groups=g, in_layout=tp.NHWC, dtype=dtype, out_dtype=dtype if out is None else out, epilogue=epi)


def kinds_of(d):
    out = {}
    for i in range(tp.space_size(d)):
        s = tp.space_get(d, i)
        out.setdefault(s["kind"], []).append(s)
    return out


# ------------------------------------------------------------------ epilogue 0 / 2, every schedule (O11)
EPI_SHAPES = [mk(1, 64, 10, 9, 64, 3, 3, 1, 1, out=tp.FP32),          # TMA im2col kind + split-K clusters
              mk(1, 64, 6, 60, 40, 3, 3, 1, 1, out=tp.FP32),          # + row-halo kind
              mk(1, 3, 23, 140, 64, 7, 7, 2, 3, out=tp.FP32),         # gathered + stem kinds
              mk(1, 64, 128, 128, 128, 3, 3, 1, 1, out=tp.FP32),      # + multi-tile kind
              mk(1, 36, 9, 9, 40, 3, 3, 1, 1, dtype=tp.FP32),         # direct + 3xTF32 kinds
              mk(1, 16, 9, 9, 16, 3, 3, 2, 1, g=16, dtype=tp.FP32)]   # depthwise direct


@pytest.mark.parametrize("epi", [0, 2])
@pytest.mark.parametrize("d", EPI_SHAPES, ids=lambda d: f"{d['c']}x{d['h']}x{d['w']}_k{d['k']}_g{d['groups']}")
def test_every_schedule_bit_exact_epilogue_variants(d, epi):
    """Epilogue code 0 (no bias, no ReLU: negative outputs must survive) and 2
    (ReLU without bias): every schedule of every kind equals the oracle bit
    for bit on integer data."""
    d = dict(d, epilogue=epi)
    x, w, b = datagen.make_inputs(d, 41 + epi, integer=True)
    ref = oracle_ref(d, x, w, b)
    if epi == 0:
        assert ref.min() < 0
    buf = tp.LayerBuffers(d, x, w, b)
    step = 1 if tp.space_size(d) <= 1200 else 3     # the 128x128 layer: every third schedule (~500)
    bad, n = [], 0
    for i in range(0, tp.space_size(d), step):
        s = tp.space_get(d, i)
        n += 1
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        if not np.array_equal(buf.output(), ref):
            bad.append((i, s["kind"], s["bm"], s["bn"], s["split_k"], s["tiles_per_cta"]))
    assert not bad, f"{len(bad)}/{n} schedules differ, first: {bad[:5]}"


# ------------------------------------------------------------------ VGG-19 b16 at full size, every kind
def _vgg_exhaustive_winners():
    p = os.path.join(ROOT, "profiles", "r01_exhaustive_vgg19_25.json")
    out = {}
    if os.path.exists(p):
        d = json.load(open(p))
        for name, med in d["layers"].items():
            med = np.asarray(med, dtype=np.float64)
            if np.isfinite(med).any():
                out[name] = (len(med), int(np.nanargmin(np.where(med > 0, med, np.nan))))
    return out


VGG = wl.catalog("vgg19_b16")


@pytest.mark.parametrize("li", range(len(VGG)), ids=[d["name"] for d in VGG])
def test_vgg_full_size_every_kind_vs_oracle(li):
    """Full BASELINE size (batch 16): for every kind in the layer's space, four
    seeded schedules (first, last and two sampled) plus the winner of the
    recorded exhaustive tune at 25%, run in a 25% partition with the geometry
    frozen at its granted SMs, against the 4096 stored oracle points."""
    d = VGG[li]
    part = tp.Partition.get(0.25)
    x, w, b = datagen.make_inputs(d, datagen.data_seed(4, li))
    idx, ref = refs.load("vgg19_b16", 4, VGG)[li]
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    chosen = []
    for kind, scheds in kinds_of(d).items():
        pick = {0, len(scheds) - 1} | {int(j) for j in sp.sample(len(scheds), 2, 100 + li + kind)}
        chosen += [scheds[j] for j in sorted(pick)]
    win = _vgg_exhaustive_winners().get(d["name"])
    if win is not None and win[0] == tp.space_size(d):
        chosen.append(tp.space_get(d, win[1]))
    # the round-2 code paths at full size: the resident-weight row kind with two
    # MMA-issuing warps (N = 64, ring >= 2 tiles of k-blocks) and both stem paths
    # (ring for >= 4 tiles per CTA, im2col tile below)
    for kind, pred in ((tp.KIND_IGEMM_TC_ROWW, lambda s: s["bn"] == 64 and s["stages"] >= 6),
                       (tp.KIND_IGEMM_TC_STEM, lambda s: s["tiles_per_cta"] >= 4),
                       (tp.KIND_IGEMM_TC_STEM, lambda s: s["tiles_per_cta"] <= 2)):
        extra = [s for s in kinds_of(d).get(kind, []) if pred(s)]
        if extra:
            chosen.append(extra[len(extra) // 2])
    bad = []
    for s in chosen:
        s = dict(s, sm_tuned=part.sm_granted)
        buf.y.fill_(0xFF)
        torch.cuda.synchronize()
        tp.conv2d_run(buf, s, part)
        part.sync()
        err = rel_err(buf.gather(idx, part), ref)
        if not err <= 2e-2:
            bad.append((s["space_index"], s["kind"], s["bm"], s["bn"], s["tiles_per_cta"], err))
    assert len({s["kind"] for s in chosen}) == len(kinds_of(d))
    assert not bad, f"{len(bad)}/{len(chosen)} schedules off, first: {bad[:5]}"


# ------------------------------------------------------------------ all 30 MobileNetV2 layers, random data
MB = wl.catalog("mobilenetv2")


@pytest.mark.parametrize("li", range(len(MB)), ids=[d["name"] for d in MB])
def test_mobilenetv2_layer_random_parity(li):
    d = MB[li]
    x, w, b = datagen.make_inputs(d, datagen.data_seed(5, li))
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    chosen = []
    for kind, scheds in kinds_of(d).items():
        chosen += [scheds[j] for j in sp.sample(len(scheds), 4, 7 + li)]
    for s in chosen:
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        err = rel_err(buf.output(), ref)
        assert err <= 2e-2, (s["space_index"], s["kind"], err)


# ------------------------------------------------------------------ a14: concurrent tuners, oracle-gated
def test_concurrent_tuners_oracle_gate_and_winners():
    """4 disjoint green contexts (one split), one host thread each running
    tp_tune on its own two ResNet-50 layers with oracle check points: every
    record passes the oracle gate, and each winner's full output (left in y by
    tp_tune) matches the full fp64 oracle output."""
    layers = wl.catalog("resnet50")
    share = [[1, 12], [2, 16], [5, 19], [10, 22]]
    parts = tp.Partition.split(4, 32)
    try:
        work = {}
        for j, ids in enumerate(share):
            for li in ids:
                d = layers[li]
                x, w, b = datagen.make_inputs(d, datagen.data_seed(2, li))
                ref = oracle_ref(d, x, w, b)
                idx = datagen.sample_points(ref.size, 4096, 61 + li)
                work[li] = (tp.LayerBuffers(d, x, w, b, part=parts[j]), ref, idx)
        torch.cuda.synchronize()
        results, errors = {}, []

        def worker(j):
            try:
                for li in share[j]:
                    buf, ref, idx = work[li]
                    best, m, recs = tp.tune(buf, parts[j], 96, datagen.sampler_seed(1), check_idx=idx,
                                            check_ref=ref.reshape(-1)[idx])
                    results[li] = (best, m, recs, buf.output())
            except Exception as e:   # surfaced below
                errors.append(repr(e))

        th = [threading.Thread(target=worker, args=(j,)) for j in range(4)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
        for j, ids in enumerate(share):
            for li in ids:
                best, m, recs, y = results[li]
                assert all(r["status"] == 0 for r in recs), [r for r in recs if r["status"]][:3]
                assert best["sm_tuned"] == parts[j].sm_granted
                assert rel_err(y, work[li][1]) <= 2e-2, (layers[li]["name"], best)
    finally:
        for p in parts:
            p.close()


# ------------------------------------------------------------------ SURVEY 8(b) fraction-taking entry points
def test_fraction_entry_points_match_partition_calls():
    d = wl.catalog("resnet50")[2]
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, 2))
    idx, ref = refs.load("resnet50", 2, wl.catalog("resnet50"))[2]
    buf = tp.LayerBuffers(d, x, w, b)
    best, m, recs = tp.tune_at(buf, 0.25, 32, 42, check_idx=idx, check_ref=ref)
    part = tp.Partition.get(0.25)
    assert m["sm_granted"] == part.sm_granted and best["sm_tuned"] == part.sm_granted
    assert all(r["status"] == 0 for r in recs) and len(recs) == 32
    assert rel_err(buf.gather(idx), ref) <= 2e-2
    r = tp.conv2d_run_at(buf, best, 0.5)
    c = tp.cross_eval_at(buf, best, 0.5)
    assert r["status"] == 0 and c["status"] == 0 and r["sm_granted"] == c["sm_granted"] == tp.Partition.get(0.5).sm_granted
    assert c["ctas"] == m["ctas"]          # frozen geometry (reading C15)


# ------------------------------------------------------------------ f2 / f3 drivers
def test_model_cross_eval_driver_f2():
    from paper_2008_03602_b200 import experiments as ex
    layers = wl.catalog("resnet50")[1:4]
    fr = (0.25, 1.0)
    checks = refs.load("resnet50", 2, wl.catalog("resnet50"))[1:4]
    bufs = [tp.LayerBuffers(d, *datagen.make_inputs(d, datagen.data_seed(2, li + 1))) for li, d in enumerate(layers)]
    res = ex.cross_eval(layers, fr, trials=24, config=2, checks=checks, bufs=bufs, log=lambda *a: None)
    assert set(res["model_sum_us"]) == {"0.25", "1.0"}
    for row in res["layers"]:
        for p in ("0.25", "1.0"):
            assert all(v > 0 for v in row["matrix_us"][p].values())
        assert set(row["default_us"]) == {"0.25", "1.0"}
    assert res["tune"]["0.25"]["ok"] == res["tune"]["0.25"]["candidates"] == 3 * 24
    assert res["pd_check"]["cells"] == 3 * 2
    agg = res["aggregate_5k"]
    assert agg["sweet_spot_tuned_at"] in fr and agg["untuned_total_ms"] > 0


def test_interference_driver_f3():
    from paper_2008_03602_b200 import experiments as ex
    res = ex.interference("cfg1", k=2, sms_each=36, trials=24, log=lambda *a: None)
    assert set(res["modes"]) == {"isolated", "shared", "time_sliced"}
    for mode, r in res["modes"].items():
        assert r["candidates"] == 24 and r["candidates_per_s"] > 0
        assert all(row["solo_us"] > 0 for row in r["layers"])


# ------------------------------------------------------------------ multi-rank paths (two ranks, one GPU)
def _run(cmd, env_extra, timeout=900):
    env = dict(os.environ, TP_BENCH_DEVICE="0", **env_extra)
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_bench_gpus2_launches_two_ranks():
    """bench.py --gpus 2 with no torchrun environment re-launches itself as two
    ranks; the job's candidates are the two weak-scaling jobs' lists, all
    measured (each rank its round-robin share) and all oracle-gated OK."""
    out = _run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0", "--no-cpu", "--no-e2e",
                "--workload", "mobilenetv2", "--fraction", "0.5"], {})
    line = out[-1]
    n = sum(tp.space_size(d) for d in MB)
    assert line["n_gpus"] == 2 and line["config"]["candidates_per_step"] == 2 * n
    assert line["candidates_total"] == 2 * n and line["candidates_ok"] == 2 * n
    assert line["config"]["sm_granted"] == tp.Partition.get(0.5).sm_granted


def test_tune_job_two_ranks_union_merge_and_resume(tmp_path):
    """The sharded tuning job: the two ranks' logged candidates are exactly the
    single list of every layer; rank 0's merged argmin equals the argmin over
    the union of the logs; a --resume run re-measures nothing."""
    log = str(tmp_path / "log")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + os.getpid() % 1000),
           "-m", "paper_2008_03602_b200.tune_job", "--workload", "cfg1", "--fraction", "0.5", "--log-dir", log]
    first = _run(cmd, {})[-1]
    cat = wl.catalog("cfg1")
    logged = shard.RecordLog.load(log)
    full = {(0, li, i) for li, d in enumerate(cat) for i in tp.space_sample(d, 1000, 42)}
    assert shard.measured_set(logged) == full and len(logged) == len(full)
    assert {r["rank"] for r in logged} == {0, 1}
    merged = shard.merge_best(logged)
    assert [w["merged_argmin"] for w in first["winners"]] == [merged[(0, li)]["space_index"] for li in range(len(cat))]
    again = _run(cmd + ["--resume"], {})[-1]
    assert again["resumed"] == len(full) and again["measured_by_rank0"] == 0 and again["records"] == len(full)
    assert len(shard.RecordLog.load(log)) == len(full)


# ------------------------------------------------------------------ out-of-bounds writes: guard bands
# compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset), so
# out-of-bounds writes are caught with our own guard bands: y and the workspace sit inside larger
# allocations whose margins hold a canary pattern, and every schedule of every kind (ragged
# shapes) must leave the canaries intact and match the oracle.
GUARD = 1 << 16


def _guarded(t):
    """A view of a larger canary-filled allocation with t's size (16-byte aligned)."""
    big = torch.full((t.numel() + 2 * GUARD,), 0xA5, dtype=torch.uint8, device=t.device)
    return big, big[GUARD:GUARD + t.numel()]


GUARD_SHAPES = [mk(1, 64, 10, 9, 40, 3, 3, 1, 1, out=tp.FP32, epi=1),       # TMA kind, split-K, ragged N
                mk(1, 64, 6, 60, 40, 3, 3, 1, 1, out=tp.FP32, epi=1),       # row-halo
                mk(1, 3, 23, 140, 64, 7, 7, 2, 3, out=tp.FP32, epi=1),      # gathered + stem
                mk(1, 64, 100, 100, 72, 3, 3, 1, 1, out=tp.FP32, epi=1),    # multi-tile, ragged tiles
                mk(1, 36, 9, 9, 40, 3, 3, 1, 1, dtype=tp.FP32, epi=1),      # direct + 3xTF32
                mk(1, 24, 7, 7, 24, 3, 3, 2, 1, g=24, dtype=tp.FP32, epi=1)]


@pytest.mark.parametrize("d", GUARD_SHAPES, ids=lambda d: f"guard_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_g{d['groups']}")
def test_no_out_of_bounds_writes_every_schedule(d):
    x, w, b = datagen.make_inputs(d, 43, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    ybig, buf.y = _guarded(buf.y)
    wbig, ws = _guarded(buf.ws)
    ws.zero_()
    buf.ws = ws
    torch.cuda.synchronize()
    bad, n = [], tp.space_size(d)
    step = 1 if n <= 1200 else 3
    for i in range(0, n, step):
        s = tp.space_get(d, i)
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        if not np.array_equal(buf.output(), ref):
            bad.append(("value", i, s["kind"]))
        for big in (ybig, wbig):
            if not (bool((big[:GUARD] == 0xA5).all()) and bool((big[-GUARD:] == 0xA5).all())):
                bad.append(("guard", i, s["kind"]))
                big[:GUARD] = 0xA5
                big[-GUARD:] = 0xA5
    assert not bad, f"{len(bad)} failures, first: {bad[:5]}"


# ------------------------------------------------------------------ model-level run (tp_chain_run)
def _chain_pair(c=8, hw=20, k1=8, k2=16):
    a = mk(1, c, hw, hw, k1, 3, 3, 1, 1, epi=2)                       # bf16 out: the next layer's input
    b = mk(1, k1, hw, hw, k2, 1, 1, 1, 0, out=tp.FP32, epi=0)         # reads a's y
    return a, b


@pytest.mark.parametrize("reps", [1, 6])
def test_chain_run_next_layer_reads_previous_output(reps):
    """tp_chain_run with x[B] == y[A]: B's output equals the oracle of B(A(x))
    bit for bit for every pairing of A's and B's TMA-kind schedules sampled
    here (integer data, |values| exact in bf16).  y[A] and y[B] are poisoned
    (NaN) before each chain, so B reading before A's writes land would show."""
    da, db = _chain_pair()
    xa, wa, ba = datagen.make_inputs(da, 51, integer=True)
    xa = np.clip(xa, -1, 1)
    wa = np.clip(wa, -1, 1)
    ya = oc.conv2d_c(da, xa, wa, None, relu=True)                      # |ya| <= 72: exact in bf16
    _, wb, bb = datagen.make_inputs(db, 52, integer=True)
    ref = oc.conv2d_c(db, ya, wb, None, relu=False)
    bufa = tp.LayerBuffers(da, xa, wa, ba)
    bufb = tp.LayerBuffers(db, np.zeros((1, 8, 20, 20), np.float32), wb, bb)
    bufb.x = bufa.y                                                   # chained operand
    sa = [s for s in kinds_of(da).get(tp.KIND_IGEMM_TC, [])]
    sb = [s for s in kinds_of(db).get(tp.KIND_IGEMM_TC, [])]
    pairs = [(sa[i], sb[j]) for i, j in zip(sp.sample(len(sa), 6, 3), sp.sample(len(sb), 6, 4))]
    bad = []
    for s1, s2 in pairs:
        bufa.y.fill_(0xFF)
        bufb.y.fill_(0xFF)
        torch.cuda.synchronize()
        tp.chain_run([bufa, bufb], [s1, s2], reps=reps)
        torch.cuda.synchronize()
        if not np.array_equal(bufb.output(), ref):
            bad.append((s1["space_index"], s2["space_index"]))
    assert not bad, bad
    # timed chains leave the workspace counters zeroed and the result intact
    m = tp.chain_run([bufa, bufb], list(pairs[0]), reps=reps, timing_cfg=tp.timing())
    torch.cuda.synchronize()
    assert m["status"] == 0 and m["median_us"] > 0 and np.array_equal(bufb.output(), ref)


def test_chain_run_mixed_kinds_and_timed_layer_counter_zeroed():
    """A chain mixing kinds (TMA im2col, row-halo, direct depthwise) keeps the
    producer -> consumer order; a timed tp_conv2d_run leaves the workspace
    zeroed."""
    c = 64
    d1 = mk(1, c, 8, 60, c, 3, 3, 1, 1, epi=2)                         # row-halo + TMA kinds
    d2 = mk(1, c, 8, 60, c, 3, 3, 1, 1, g=c, epi=2)                    # depthwise direct (bf16)
    d3 = mk(1, c, 8, 60, 32, 1, 1, 1, 0, out=tp.FP32, epi=0)           # TMA kind
    x1, w1, b1 = datagen.make_inputs(d1, 61, integer=True)
    x1, w1 = np.clip(x1, -1, 1), np.clip(w1, -1, 1) * (np.arange(c) < 4)[None, :, None, None]   # |y1| <= 36
    _, w2, _ = datagen.make_inputs(d2, 62, integer=True)
    w2 = np.clip(w2, -1, 1)                                            # |y2| <= 9 * 36 = 324 -> not exact in bf16
    w2 = w2 * (np.arange(9).reshape(1, 1, 3, 3) == 4)                  # centre tap only: |y2| <= 36
    _, w3, _ = datagen.make_inputs(d3, 63, integer=True)
    y1 = oc.conv2d_c(d1, x1, w1, None, relu=True)
    y2 = oc.conv2d_c(d2, y1, w2, None, relu=True)
    ref = oc.conv2d_c(d3, y2, w3, None, relu=False)
    zx = np.zeros((1, c, 8, 60), np.float32)
    b1_, b2_, b3_ = tp.LayerBuffers(d1, x1, w1), tp.LayerBuffers(d2, zx, w2), tp.LayerBuffers(d3, zx, w3)
    b2_.x, b3_.x = b1_.y, b2_.y
    k1, k3 = kinds_of(d1), kinds_of(d3)
    firsts = [k1[tp.KIND_IGEMM_TC][0], k1[tp.KIND_IGEMM_TC_ROW][0]]
    s2 = kinds_of(d2)[tp.KIND_DIRECT][0]
    for s1 in firsts:
        for s3 in (k3[tp.KIND_IGEMM_TC][0], k3[tp.KIND_IGEMM_TC][-1]):
            for bb in (b1_, b2_, b3_):
                bb.y.fill_(0xFF)
            torch.cuda.synchronize()
            tp.chain_run([b1_, b2_, b3_], [s1, s2, s3], reps=3)
            torch.cuda.synchronize()
            assert np.array_equal(b3_.output(), ref), (s1["kind"], s3["space_index"])
    m = tp.conv2d_run(b3_, k3[tp.KIND_IGEMM_TC][0], timing_cfg=tp.timing())
    torch.cuda.synchronize()
    assert m["status"] == 0 and int(b3_.ws.view(torch.int32).abs().sum()) == 0


# ------------------------------------------------------------------ strip kind (C <= 8 stems, padded strips)
STRIP_TINY = [mk(2, 3, 10, 70, 64, 3, 3, 1, 1, out=tp.FP32, epi=1),      # VGG conv1_1-like, 2 images
              mk(1, 3, 23, 140, 64, 7, 7, 2, 3, out=tp.FP32, epi=1),     # R50 conv1-like (7x7 s2 p3)
              mk(1, 3, 9, 132, 32, 3, 3, 2, 1, out=tp.FP32, epi=1),      # MobileNetV2 conv0-like (3x3 s2)
              mk(1, 5, 6, 80, 40, 3, 3, 1, 1, out=tp.FP32, epi=1),       # C = 5, ragged N tile
              mk(1, 3, 12, 20, 16, 3, 3, 1, 1, out=tp.FP32, epi=3),      # Q = 20 < BM, K = 16 < BN
              mk(2, 4, 11, 37, 24, 5, 5, 2, 2, out=tp.FP32, epi=1),      # 5x5 s2 p2, odd W
              mk(1, 6, 7, 30, 8, 3, 3, 1, 0, out=tp.FP32, epi=1),        # C = 6, pad 0, K = 8
              mk(1, 3, 16, 64, 64, 3, 3, 1, 1, epi=3)]                   # bf16 output


def _strip_scheds(d):
    out = [s for s in (tp.space_get(d, i) for i in range(tp.space_size(d))) if s["kind"] == tp.KIND_IGEMM_TC_STRIP]
    assert out, "layer has no strip schedules"
    return out


@pytest.mark.parametrize("d", STRIP_TINY, ids=lambda d: f"strip_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_r{d['r']}s{d['stride_h']}_o{d['out_dtype']}")
def test_strip_every_schedule_bit_exact_integer(d):
    """O11 for the strip kind: every schedule (ragged last tile of each row,
    zero-padded borders, both column phases of stride 2, odd tap counts paired
    with the zero taps, several images, every tiles_per_cta) equals the oracle
    bit for bit (within one bf16 rounding for bf16 output)."""
    x, w, b = datagen.make_inputs(d, 71, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    bad = []
    for s in _strip_scheds(d):
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        y = buf.output()
        ok = np.array_equal(y, ref) if d["out_dtype"] == tp.FP32 else rel_err(y, ref) <= 2 ** -8
        if not ok:
            bad.append((s["space_index"], s["bm"], s["bn"], s["stages"], s["tiles_per_cta"]))
    assert not bad, f"{len(bad)} strip schedules differ, first: {bad[:5]}"


@pytest.mark.parametrize("sm_tuned", [1, 3, 7])
def test_strip_balanced_spans_and_timed_bit_exact(sm_tuned):
    """Multi-tile strip schedules frozen at a few SMs (ragged balanced spans),
    timed (the last timed launch leaves y), in a 25% partition."""
    d = STRIP_TINY[1]
    part = tp.Partition.get(0.25)
    x, w, b = datagen.make_inputs(d, 73, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    bad = []
    for s in _strip_scheds(d):
        if s["tiles_per_cta"] < 2:
            continue
        s = dict(s, sm_tuned=sm_tuned)
        buf.poison()
        m = tp.conv2d_run(buf, s, part, tp.timing(warmup=1, groups=1, n_min=2, target_group_us=1.0))
        part.sync()
        if m["status"] != 0 or not np.array_equal(buf.output(), ref):
            bad.append((s["space_index"], s["tiles_per_cta"]))
    assert not bad, bad


@pytest.mark.parametrize("cat,li,cfg", [("resnet50", 0, 2), ("mobilenetv2", 0, 5), ("vgg19_b16", 0, 4)],
                         ids=["r50_conv1", "mbv2_conv0", "vgg_conv1_1"])
def test_strip_full_size_vs_oracle(cat, li, cfg):
    layers = wl.catalog(cat)
    d = layers[li]
    x, w, b = datagen.make_inputs(d, datagen.data_seed(cfg, li))
    idx, ref = refs.load(cat, cfg, layers)[li]
    buf = tp.LayerBuffers(d, x, w, b)
    for s in _strip_scheds(d):
        buf.y.fill_(0xFF)
        torch.cuda.synchronize()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        assert rel_err(buf.gather(idx), ref) <= 2e-2, s


# ------------------------------------------------------------------ row-halo with resident weights (kind 8)
ROWW_TINY = [mk(2, 64, 5, 130, 48, 3, 3, 1, 1, out=tp.FP32, epi=1),    # BM 128 fits (Q = 130), 20 tiles
             mk(1, 64, 5, 100, 40, 3, 3, 1, 1, out=tp.FP32, epi=1),    # one q-block per row: 5 tiles (odd)
             mk(1, 64, 6, 60, 64, 3, 3, 1, 1, epi=3)]                  # bf16 output, BM 64 only


@pytest.mark.parametrize("d", ROWW_TINY, ids=lambda d: f"roww_{d['n']}x{d['h']}x{d['w']}_k{d['k']}_o{d['out_dtype']}")
def test_roww_every_schedule_bit_exact_integer(d):
    """Every resident-weight row-halo schedule (and, with TP_ROWW2=1 in the
    environment, its CTA-pair cta_group::2 form for BM = 128) equals the oracle
    (bit for bit with fp32 output, within one bf16 rounding otherwise), also
    with the geometry frozen at a few SMs and in a 25% partition."""
    x, w, b = datagen.make_inputs(d, 81, integer=True)
    ref = oracle_ref(d, x, w, b)
    part = tp.Partition.get(0.25)
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    scheds = kinds_of(d).get(tp.KIND_IGEMM_TC_ROWW, [])
    assert scheds
    bad = []
    for s in scheds:
        for sm_tuned in (0, 3):
            buf.poison()
            tp.conv2d_run(buf, dict(s, sm_tuned=sm_tuned), part)
            part.sync()
            y = buf.output()
            ok = np.array_equal(y, ref) if d["out_dtype"] == tp.FP32 else rel_err(y, ref) <= 2 ** -8
            if not ok:
                bad.append((s["space_index"], s["bm"], s["bn"], s["stages"], s["tiles_per_cta"], sm_tuned))
    assert not bad, f"{len(bad)} schedules differ, first: {bad[:5]}"


def test_roww_cta_pair_variant_bit_exact():
    """The CTA-pair (cta_group::2, 256-row MMA) form of the resident-weight
    row-halo kind is an experiment switched on by TP_ROWW2=1 (read once per
    process): run the resident-weight bit-exact test in a child process with it."""
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_r2.py", "-q", "-x", "-p", "no:cacheprovider",
                        "-k", "test_roww_every_schedule_bit_exact_integer"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, TP_ROWW2="1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "3 passed" in r.stdout


@pytest.mark.parametrize("mode", ["0", "2"], ids=["im2col_only", "ring_only"])
def test_stem_both_paths_every_schedule(mode):
    """The stem kind builds its A operand two ways -- an im2col tile per tile, or
    (spans of >= 4 tiles) a ring of widened input rows read in place by the MMAs.
    TP_STEM_WIDE (read once per process) forces one path for every schedule: rerun
    the every-schedule bit-exact and full-size stem tests in a child process."""
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-x", "-p", "no:cacheprovider",
                        "-k", "stem_every_schedule or stem_full_size or stem_vgg"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900, env=dict(os.environ, TP_STEM_WIDE=mode))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


def test_tune_guided_early_stop_stops_at_the_first_batch_boundary_where_the_rule_holds():
    """f1 early stopping (reading C19, P:284 / P:388): tp_tune_guided_es checks
    tp_search_should_stop after every batch.  The records it returns must end at
    the first batch boundary where the rule holds (or at the budget), the
    winner is the fastest gated record, and it matches the oracle."""
    d = mk(1, 64, 28, 28, 64, 3, 3, 1, 1, out=tp.FP32, epi=3)   # fp32 output: exact on integer data
    x, w, b = datagen.make_inputs(d, 41, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    batch, es, trials = 8, 12, 200
    best, best_m, recs = tp.tune_guided(buf, None, trials, batch=batch, explore=0.25, seed=5, early_stop=es,
                                        timing_cfg=tp.timing(warmup=1, groups=2, n_min=3, target_group_us=5.0))
    us = [r["median_us"] if r["status"] == 0 else -1.0 for r in recs]
    n = len(us)
    budget = min(trials, tp.space_size(d))
    assert n <= budget and n > 0
    for k in range(batch, n, batch):
        assert not tp.search_should_stop(us[:k], es), k
    assert n == budget or tp.search_should_stop(us, es)
    ok = [r for r in recs if r["status"] == 0]
    assert best_m["median_us"] == min(r["median_us"] for r in ok)
    tp.conv2d_run(buf, best)
    torch.cuda.synchronize()
    assert np.array_equal(buf.output(), ref)
