"""Candidate sharder across the GPUs of one box (the paper's TCI
sharding, and TSI load balancing).

Every (job, layer, candidate) measurement is independent, so units are dealt
round-robin: rank r measures candidate idx with idx % world == r.  The only
exchange is one host-side gather of fixed-size records to rank 0 over a gloo
process group (no NCCL, nothing crosses NVLink).  Rank 0 merges with the same
argmin rule as a single device (min median, ties -> lowest space_index), so
the merged choice equals the single-list choice ("combine the tuning results",
P:841).
"""
from __future__ import annotations

import glob
import json
import os

import numpy as np

# Fixed-size record exchanged between ranks (float64 row).
REC_FIELDS = ("job", "layer", "space_index", "status", "median_us", "min_us", "mean_us", "std_us", "sm_granted",
              "ctas", "threads_per_cta", "waves", "rank", "n_per_group", "groups")


def shard(cand: list[int] | np.ndarray, rank: int, world: int) -> list[int]:
    """Round-robin deal of one candidate list (keeps selection order)."""
    return [c for i, c in enumerate(cand) if i % world == rank]


def pack(records: list[dict], job: int, layer: int, rank: int) -> np.ndarray:
    out = np.zeros((len(records), len(REC_FIELDS)), dtype=np.float64)
    for i, r in enumerate(records):
        row = dict(r, job=job, layer=layer, rank=rank)
        out[i] = [float(row[f]) for f in REC_FIELDS]
    return out


def unpack(arr: np.ndarray) -> list[dict]:
    recs = []
    for row in np.asarray(arr).reshape(-1, len(REC_FIELDS)):
        d = dict(zip(REC_FIELDS, row.tolist()))
        for f in ("job", "layer", "space_index", "status", "sm_granted", "ctas", "threads_per_cta", "waves", "rank",
                  "n_per_group", "groups"):
            d[f] = int(d[f])
        recs.append(d)
    return recs


def gather_to_rank0(local: np.ndarray, group=None) -> np.ndarray | None:
    """Gather variable-length float64 record blocks to rank 0 over gloo."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(s.item() for s in sizes))
    buf = torch.zeros((mx, len(REC_FIELDS)), dtype=torch.float64)
    buf[: local.shape[0]] = torch.from_numpy(local)
    rank = dist.get_rank(group)
    outs = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, outs, dst=0, group=group)
    if rank != 0:
        return None
    return np.concatenate([o[: int(s.item())].numpy() for o, s in zip(outs, sizes)], axis=0)


def merge_best(records: list[dict]) -> dict[tuple[int, int], dict]:
    """Best OK record per (job, layer): min median_us, ties -> lowest space_index."""
    best: dict[tuple[int, int], dict] = {}
    for r in records:
        if r["status"] != 0:
            continue
        key = (r["job"], r["layer"])
        b = best.get(key)
        if b is None or r["median_us"] < b["median_us"] or (r["median_us"] == b["median_us"]
                                                            and r["space_index"] < b["space_index"]):
            best[key] = r
    return best


def finalists(records: list[dict], k: int = 3) -> dict[tuple[int, int], list[dict]]:
    """Top-k OK records per (job, layer) by (median_us, space_index) -- the
    candidates rank 0 re-times on one device after the gather (SURVEY 8(e):
    clock/thermal differences between GPUs must not pick the winner)."""
    by: dict[tuple[int, int], list[dict]] = {}
    for r in records:
        if r["status"] == 0:
            by.setdefault((r["job"], r["layer"]), []).append(r)
    return {key: sorted(v, key=lambda r: (r["median_us"], r["space_index"]))[:k] for key, v in by.items()}


def is_raced(r: dict, full_groups: int = 5) -> bool:
    """Reading C12b: a raced candidate's record has a single timed group."""
    return r["status"] == 0 and full_groups > 1 and r["groups"] == 1


def raced_frac(records: list[dict], full_groups: int = 5) -> float:
    ok = [r for r in records if r["status"] == 0]
    return sum(1 for r in ok if is_raced(r, full_groups)) / max(1, len(ok))


def gpu_busy_us(records: list[dict], warmup: int = 3, full_groups: int = 5) -> float:
    """Kernel time a tuning pass spent on the GPU for these records: per
    candidate, the gate launch + its warm-ups (1 for a raced candidate, reading
    C12b; `warmup` otherwise) + groups x n timed launches, each at the
    candidate's median latency (SURVEY 8(d) "GPU-busy fraction")."""
    return sum((1 + (1 if is_raced(r, full_groups) else warmup) + r["groups"] * r["n_per_group"]) * r["median_us"]
               for r in records if r["status"] == 0)


# ---------------------------------------------------------------------------------------------
# Record log and resume (the orchestrator analog, PAPER.md P:921-925 [src]: a tuning job that
# dies part-way must not redo the measurements it already made).  Every rank appends its
# records, one JSON object per line, to <dir>/rank<r>.jsonl as each (job, layer) unit
# finishes; a restarted job reads every rank's log, skips the (job, layer, space_index)
# triples already measured and merges the logged records with the new ones.
class RecordLog:
    def __init__(self, directory: str, rank: int):
        os.makedirs(directory, exist_ok=True)
        self.path = os.path.join(directory, f"rank{rank}.jsonl")
        # A rank that died mid-write leaves a torn last line: cut it, so the next
        # append starts on a fresh line.
        if os.path.exists(self.path):
            with open(self.path, "rb+") as f:
                data = f.read()
                if data and not data.endswith(b"\n"):
                    f.truncate(data.rfind(b"\n") + 1)

    def append(self, records: list[dict], job: int, layer: int, rank: int) -> None:
        with open(self.path, "a") as f:
            for r in records:
                row = {k: r[k] for k in REC_FIELDS if k in r}
                row.update(job=job, layer=layer, rank=rank)
                f.write(json.dumps(row) + "\n")
            f.flush()
            os.fsync(f.fileno())

    @staticmethod
    def load(directory: str) -> list[dict]:
        """All complete lines of every rank's log (a torn last line is dropped)."""
        out = []
        for path in sorted(glob.glob(os.path.join(directory, "rank*.jsonl"))):
            with open(path) as f:
                for ln in f:
                    try:
                        row = json.loads(ln)
                    except json.JSONDecodeError:
                        continue
                    if all(k in row for k in REC_FIELDS):
                        out.append(row)
        return out


def measured_set(records: list[dict]) -> set[tuple[int, int, int]]:
    return {(int(r["job"]), int(r["layer"]), int(r["space_index"])) for r in records}


def run_sharded(units: dict, measure, rank: int, world: int, log: RecordLog | None = None,
                resumed: list[dict] | None = None) -> np.ndarray:
    """Measure this rank's share of every unit and return its packed records.

    units: {(job, layer): [space_index, ...]} in selection order (the full list,
    identical on every rank); measure(key, idx_list) -> list of record dicts.
    Rank r takes the round-robin share of each list (shard), minus what
    `resumed` (records read back from a RecordLog) already holds; the resumed
    records that belong to this rank's share are returned with the new ones."""
    done = measured_set(resumed or [])
    blocks = []
    for key in sorted(units):
        mine = shard(units[key], rank, world)
        mine_set = {int(c) for c in mine}
        todo = [c for c in mine if (key[0], key[1], int(c)) not in done]
        old = [r for r in (resumed or []) if (int(r["job"]), int(r["layer"])) == key
               and int(r["space_index"]) in mine_set]
        if old:
            blocks.append(pack(old, key[0], key[1], rank))
        if todo:
            recs = measure(key, todo)
            if log is not None:
                log.append(recs, key[0], key[1], rank)
            blocks.append(pack(recs, key[0], key[1], rank))
    return np.concatenate(blocks) if blocks else np.zeros((0, len(REC_FIELDS)))
