import sys; sys.path.insert(0, "/root/repo")
import paper_1812_10959_b200 as dic
from paper_1812_10959_b200.miner import DeviceEngine, StopTrace, run_engine
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr
cfg = CONFIGS[4]
ip, ix = generate_csr(cfg)
db = dic.BitDatabase.from_csr(ip, ix, cfg.m)
p = dic.MiningParams.create(cfg.n, cfg.minsup, interval=cfg.interval)
tr = StopTrace()
res = run_engine(db.device_tids(), cfg.n, cfg.m, p, trace=tr, engine_factory=DeviceEngine)
st = tr.stops
for key in ("promoted", "inserted", "pruned", "finalized", "dashed_at_start"):
    v = [s[key] for s in st]
    print(key, [round(sum(v[i:i+25]) / len(v[i:i+25])) for i in range(0, len(v), 25)])
