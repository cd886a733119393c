import sys, os
sys.path.insert(0, "/root/repo")
import paper_1812_10959_b200 as dic
from paper_1812_10959_b200.miner import StopTrace, run_engine
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr
cfg = CONFIGS[4]
ip, ix = generate_csr(cfg)
db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
p = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
for B in ("8", "4", "2", "6"):
    os.environ["DIC_BATCH_STOPS"] = B
    tr = StopTrace()
    res = run_engine(db.device_tids(), cfg.n, cfg.m, p, trace=tr)
    print(B, len(res.frequent), tr.native)
