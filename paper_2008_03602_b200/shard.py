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


def gpu_busy_us(records: list[dict], warmup: int = 3) -> float:
    """Kernel time a tuning pass spent on the GPU for these records: per
    candidate, the gate launch + warm-ups + groups x n timed launches, each
    at the candidate's median latency (SURVEY 8(d) "GPU-busy fraction")."""
    return sum((1 + warmup + r["groups"] * r["n_per_group"]) * r["median_us"] for r in records if r["status"] == 0)
