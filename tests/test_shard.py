"""Sharder host logic on CPU with a world_size-2 gloo group."""
import os
import random

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import space as sp
from paper_2008_03602_b200 import shard


def _fake_records(n, seed):
    rng = random.Random(seed)
    return [dict(space_index=i, status=rng.choice([0, 0, 0, 5]), median_us=rng.choice([1.0, 1.5, 2.0, 2.5]),
                 min_us=0.9, mean_us=1.0, std_us=0.1, sm_granted=148, ctas=10, threads_per_cta=128, waves=1,
                 n_per_group=10, groups=rng.choice([1, 5]))
            for i in range(n)]


def test_shards_disjoint_and_cover():
    cand = sp.sample(920, 1000, 42)
    for world in (1, 2, 3, 8):
        parts = [shard.shard(cand, r, world) for r in range(world)]
        flat = sorted(c for p in parts for c in p)
        assert flat == sorted(cand)
        assert sum(len(p) for p in parts) == len(set(flat))
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_merge_equals_single_list_argmin():
    recs = _fake_records(300, 1)
    single = sp.argmin(recs)
    for world in (2, 4, 8):
        blocks = [shard.pack(shard.shard(recs, r, world), 0, 7, r) for r in range(world)]
        merged = shard.merge_best(shard.unpack(np.concatenate(blocks)))
        assert merged[(0, 7)]["space_index"] == recs[single]["space_index"]


def test_pack_roundtrip_exact():
    recs = _fake_records(50, 2)
    back = shard.unpack(shard.pack(recs, 3, 4, 1))
    for a, b in zip(recs, back):
        assert a["median_us"] == b["median_us"] and a["space_index"] == b["space_index"]
        assert b["job"] == 3 and b["layer"] == 4 and b["rank"] == 1


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    recs = _fake_records(101, 9)
    mine = shard.shard(recs, rank, world)
    got = shard.gather_to_rank0(shard.pack(mine, 0, 0, rank))
    if rank == 0:
        merged = shard.merge_best(shard.unpack(got))
        q.put((got.shape[0], merged[(0, 0)]["space_index"], recs[sp.argmin(recs)]["space_index"]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randint(0, 2000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    n, merged_idx, single_idx = q.get(timeout=5)
    assert n == 101
    assert merged_idx == single_idx


def test_finalists_top3_sorted_and_ok_only():
    recs = [dict(r, job=0, layer=r["space_index"] % 2) for r in _fake_records(200, 3)]
    fin = shard.finalists(recs, 3)
    for key, top in fin.items():
        assert len(top) == 3 and all(r["status"] == 0 for r in top)
        ok = sorted((r for r in recs if (r["job"], r["layer"]) == key and r["status"] == 0),
                    key=lambda r: (r["median_us"], r["space_index"]))
        assert [r["space_index"] for r in top] == [r["space_index"] for r in ok[:3]]
        assert top[0]["space_index"] == shard.merge_best(recs)[key]["space_index"]


def test_gpu_busy_counts_gate_warmup_and_groups():
    recs = [dict(status=0, median_us=2.0, n_per_group=10, groups=5), dict(status=0, median_us=4.0, n_per_group=10,
                                                                           groups=1),
            dict(status=5, median_us=1.0, n_per_group=0, groups=0)]
    # full protocol: (gate 1 + 3 warm-ups + 5 x 10) * 2; raced (C12b, one group): (1 + 1 warm-up + 10) * 4
    assert shard.gpu_busy_us(recs) == 54 * 2.0 + 12 * 4.0
    assert shard.raced_frac(recs) == 0.5


def _fake_measure(calls):
    def measure(key, idx):
        calls.append((key, list(idx)))
        rng = random.Random(hash(key) & 0xFFFF)
        base = {i: rng.choice([1.0, 1.5, 2.0]) for i in range(1000)}
        return [dict(space_index=int(i), status=0, median_us=base[int(i)] + 0.001 * i, min_us=0.9, mean_us=1.0,
                     std_us=0.1, sm_granted=148, ctas=10, threads_per_cta=128, waves=1, n_per_group=10, groups=5)
                for i in idx]
    return measure


def test_record_log_resume(tmp_path):
    units = {(0, 0): sp.sample(300, 1000, 1), (0, 1): sp.sample(200, 50, 2), (1, 0): sp.sample(120, 1000, 3)}
    # reference: one uninterrupted single-rank pass
    full = shard.unpack(shard.run_sharded(units, _fake_measure([]), 0, 1))
    # an interrupted pass: rank 0 of 2 logs unit (0, 0) and dies with a torn last line
    log = shard.RecordLog(str(tmp_path), 0)
    calls = []
    shard.run_sharded({(0, 0): units[(0, 0)]}, _fake_measure(calls), 0, 2, log=log)
    with open(log.path, "a") as f:
        f.write('{"job": 0, "layer": 1, "space_ind')
    logged = shard.RecordLog.load(str(tmp_path))
    assert len(logged) == len(shard.shard(units[(0, 0)], 0, 2))
    # restart (both ranks): rank 0 re-measures nothing of unit (0, 0); the union covers every candidate once
    calls = []
    blocks = [shard.run_sharded(units, _fake_measure(calls), r, 2, log=shard.RecordLog(str(tmp_path), r),
                                resumed=logged) for r in range(2)]
    remeasured = {(k, i) for k, idx in calls for i in idx}
    assert not any(k == (0, 0) and i in set(shard.shard(units[(0, 0)], 0, 2)) for k, i in remeasured)
    merged = shard.unpack(np.concatenate(blocks))
    assert sorted((r["job"], r["layer"], r["space_index"]) for r in merged) == \
        sorted((r["job"], r["layer"], r["space_index"]) for r in full)
    a, b = shard.merge_best(merged), shard.merge_best(full)
    assert {k: v["space_index"] for k, v in a.items()} == {k: v["space_index"] for k, v in b.items()}
    # the log now holds every record exactly once (the torn line is ignored)
    assert len(shard.measured_set(shard.RecordLog.load(str(tmp_path)))) == len(full)
