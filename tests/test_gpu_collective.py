"""The sharded driver's collective path on one GPU: a 1-rank NCCL process
group, the Python pipelined loop with the per-stop all_reduce of the count
deltas and of the dense pair triangle (the same calls an 8-GPU run makes),
against the oracle.  (Ranks that wait on one another must not share a GPU,
so world sizes > 1 are covered on CPU by tests/test_multirank.py.)"""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist

import paper_1812_10959_b200 as dic
from oracle import oracle as O
from paper_1812_10959_b200.miner import run_engine
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr, scaled

pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("idx,n,interval", [(4, 60_000, 6_000), (3, 30_000, 3_000), (1, 10_000, 1_000)])
def test_collective_loop_matches_oracle(nccl_group, idx, n, interval):
    cfg = scaled(CONFIGS[idx], n, interval=interval)
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    plan = dic.ShardPlan.for_params(params, 1, 0)
    res = run_engine(db.device_tids(), cfg.n, cfg.m, params, plan=plan, group=nccl_group, collective=True)
    want = O.mine(db.rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=8)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    s = res.stats
    assert (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts) == (
        want.db_passes, want.peak_dashed, want.candidates_generated, want.candidates_pruned, want.interval_counts)
    # and the native single-GPU loop agrees with it
    res2 = run_engine(db.device_tids(), cfg.n, cfg.m, params)
    assert [(f.mask, f.support) for f in res2.frequent] == [(f.mask, f.support) for f in res.frequent]


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("idx,n,interval", [(4, 60_000, 6_000), (3, 30_000, 3_000), (2, 20_000, 2_000)])
def test_native_nccl_loop_matches_oracle(nccl_group, monkeypatch, idx, n, interval, fused):
    """The library's own NCCL communicator (dic_nccl_comm_init) on 1 rank:
    item counts allreduced, and per stop the deltas and the dense pair
    triangle reduced inside dic_engine_run, the loop fully native — either
    by the fused peer-memory kernel over NCCL symmetric windows (fused=1,
    the default) or by ncclAllReduce (DIC_FUSED_REDUCE=0)."""
    from paper_1812_10959_b200.miner import StopTrace

    monkeypatch.setenv("DIC_FUSED_REDUCE", fused)
    cfg = scaled(CONFIGS[idx], n, interval=interval)
    indptr, indices = generate_csr(cfg)
    db = dic.BitDatabase.from_csr(indptr, indices, cfg.m)
    params = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
    plan = dic.ShardPlan.for_params(params, 1, 0)
    trace = StopTrace()
    res = run_engine(db.device_tids(), cfg.n, cfg.m, params, plan=plan, group=nccl_group, collective="native",
                     trace=trace)
    assert trace.native["collective"] == ("fused" if fused == "1" else "nccl")
    want = O.mine(db.rows, cfg.m, cfg.minsup, interval=cfg.interval, threads=8)
    assert [(f.mask, f.size, f.support) for f in res.frequent] == want.frequent
    s = res.stats
    assert (s.db_passes, s.peak_dashed, s.candidates_generated, s.candidates_pruned, s.interval_counts) == (
        want.db_passes, want.peak_dashed, want.candidates_generated, want.candidates_pruned, want.interval_counts)
