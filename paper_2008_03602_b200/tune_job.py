"""A resumable, sharded tuning job over the GPUs of one box (the
paper's TCI sharding, and its orchestrator's restart of
failed work, P:921-925 [src]).

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        -m paper_2008_03602_b200.tune_job --workload resnet50 --fraction 0.25 --log-dir runs/r50_25 [--resume]

Every rank binds cuda:LOCAL_RANK, tunes the round-robin share of every
layer's candidate list inside its own partition (gate: the stored oracle
points of refs/), and appends its records to <log-dir>/rank<r>.jsonl as each
layer finishes.  With --resume, measurements already in the logs are skipped.
Rank 0 gathers the records over gloo, merges the per-layer argmin (ties to the
lowest space index), re-times the top-3 finalists of every layer on its own
device and prints one JSON line with the winners.
"""
from __future__ import annotations

import argparse
import json
import os


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--fraction", type=float, default=1.0)
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--log-dir", required=True)
    ap.add_argument("--resume", action="store_true")
    args = ap.parse_args(argv)

    import torch
    import torch.distributed as dist

    from . import datagen, refs, shard, tp, workloads as wl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("TP_BENCH_DEVICE") is not None:   # path tests: several ranks on one GPU
        local = int(os.environ["TP_BENCH_DEVICE"])
    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    tp.init(local)
    part = tp.Partition.get(args.fraction, device=local)
    config = {"cfg1": 1, "resnet50": 2, "vgg19_b16": 4, "mobilenetv2": 5}[args.workload]
    layers = wl.catalog(args.workload)
    checks = refs.load(args.workload, config, layers)
    bufs, units = {}, {}
    for li, d in enumerate(layers):
        x, w, b = datagen.make_inputs(d, datagen.data_seed(config, li))
        bufs[(0, li)] = tp.LayerBuffers(d, x, w, b, part=part, device=local)
        units[(0, li)] = tp.space_sample(d, args.trials, args.seed)
    resumed = shard.RecordLog.load(args.log_dir) if args.resume else []
    log = shard.RecordLog(args.log_dir, rank)

    def measure(key, idx):
        ci, cr = checks[key[1]]
        return tp.tune_subset(bufs[key], part, idx, check_idx=ci, check_ref=cr)

    local_recs = shard.run_sharded(units, measure, rank, world, log=log, resumed=resumed)
    n_new = local_recs.shape[0] - sum(1 for r in resumed if r["rank"] == rank)
    got = shard.gather_to_rank0(local_recs)
    if rank == 0:
        recs = shard.unpack(got)
        best = shard.merge_best(recs)
        out = []
        for key, fin in sorted(shard.finalists(recs, 3).items()):
            d = layers[key[1]]
            rt = [dict(r, median_us=tp.conv2d_run(bufs[key], tp.space_get(d, r["space_index"]), part,
                                                 tp.timing())["median_us"]) for r in fin]
            w = min(rt, key=lambda r: (r["median_us"], r["space_index"]))
            out.append({"layer": d["name"], "space_index": w["space_index"], "median_us": w["median_us"],
                        "merged_argmin": best[key]["space_index"]})
        print(json.dumps({"workload": args.workload, "fraction": args.fraction, "sm_granted": part.sm_granted,
                          "ranks": world, "records": len(recs), "resumed": len(resumed),
                          "measured_by_rank0": int(n_new),
                          "model_sum_us": sum(layers[i]["mult"] * o["median_us"] for i, o in enumerate(out)),
                          "winners": out}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
