"""Per-stop cost of the cross-rank reduction on one GPU (a 1-rank NCCL
group): cfg4 mined by the native loop with no communicator, with the fused
peer-memory reduction (DIC_FUSED_REDUCE=1, default) and with ncclAllReduce
(DIC_FUSED_REDUCE=0).  With one rank nothing crosses NVLink, so the
differences are the fixed per-stop costs a sharded run pays on top of its
count work: barriers + reduction launch vs. two NCCL launches sized by the
slot capacity.  Prints one JSON line."""

from __future__ import annotations

import json
import os
import socket
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1812_10959_b200 as dic  # noqa: E402
from paper_1812_10959_b200.miner import StopTrace, run_engine  # noqa: E402
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr  # noqa: E402


def main() -> None:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    cfg = CONFIGS[4]
    ip, ix = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
    tids = db.device_tids()
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    plan = dic.ShardPlan.for_params(params, 1, 0)
    out = {}
    ref = None
    for name, env, kw in [("no_comm", None, {}),
                          ("fused", "1", {"plan": plan, "group": dist.group.WORLD, "collective": "native"}),
                          ("nccl_allreduce", "0", {"plan": plan, "group": dist.group.WORLD, "collective": "native"})]:
        if env is not None:
            os.environ["DIC_FUSED_REDUCE"] = env
        times = []
        for _ in range(6):
            torch.cuda.synchronize()
            tr = StopTrace()
            t = time.perf_counter()
            res = run_engine(tids, cfg.n, cfg.m, params, trace=tr, **kw)
            torch.cuda.synchronize()
            times.append((time.perf_counter() - t) * 1e3)
        got = [(f.mask, f.support) for f in res.frequent]
        ref = ref or got
        assert got == ref
        out[name] = {"ms_min": min(times[1:]), "ms_median": sorted(times[1:])[2],
                     "collective": (tr.native or {}).get("collective"), "stops": len(tr.stops),
                     "phases_ms": {k: round(v, 3) for k, v in tr.phases.items()}}
    stops = out["no_comm"]["stops"]
    for k in ("fused", "nccl_allreduce"):
        out[k]["us_per_stop_over_no_comm"] = (out[k]["ms_min"] - out["no_comm"]["ms_min"]) * 1e3 / stops
    print(json.dumps({"workload": cfg.name, "world": 1, **out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
