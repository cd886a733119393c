"""One rank of a k-GPU scaling run (benchmark.run_scaling): loads the binary
cache, keeps its chunk-sliced shard of the rows (ShardPlan), mines with the
per-stop NCCL sum-allreduce, times each repetition as the max over ranks and
has rank 0 write {time_s, digest} as JSON."""

from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from .benchmark import frequent_digest
from .bitmap import BitDatabase
from .config import MiningParams
from .datasets import load_bitdb
from .miner import run_engine
from .sharding import ShardPlan


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--cache", required=True)
    ap.add_argument("--minsup", type=float, required=True)
    ap.add_argument("--interval", type=int, required=True)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    db = load_bitdb(a.cache)
    params = MiningParams.create(db.n, a.minsup, interval=a.interval)
    plan = ShardPlan.for_params(params, world, rank)
    rows = db.rows
    mine = np.concatenate([rows[b:b + ln] for b, ln in plan.ranges() if ln > 0]) if plan.local_rows() else rows[:0]
    local_db = BitDatabase.from_device_rows(torch.from_numpy(np.array(mine)).cuda(), db.m) if mine.shape[0] else None
    tids = local_db.device_tids() if local_db is not None else torch.zeros(1, dtype=torch.int32, device="cuda")
    best, digest = float("inf"), None
    for _ in range(a.reps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run_engine(tids, plan.local_rows(), db.m, params, plan=plan, group=dist.group.WORLD)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        best = min(best, float(t.item()))
        digest = frequent_digest(res.frequent)
    if rank == 0:
        with open(a.out, "w") as fh:
            json.dump({"time_s": best, "digest": digest}, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
