import sys, time
sys.path.insert(0, '.')
import torch
import paper_1812_10959_b200 as dic
from paper_1812_10959_b200.miner import StopTrace, run_engine
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr
cfg = CONFIGS[1]
ip, ix = generate_csr(cfg)
db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
tids = db.device_tids()
p = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
for i in range(6):
    tr = StopTrace()
    torch.cuda.synchronize(); t = time.perf_counter()
    res = run_engine(tids, cfg.n, cfg.m, p, trace=tr)
    dt = (time.perf_counter() - t) * 1e3
    if i >= 3:
        print(round(dt, 3), {k: round(v, 3) for k, v in tr.phases.items()}, tr.native)
