"""e2e encode leg alone: pinned uint16/int32 host CSR of cfg4 -> BitDatabase.from_csr
at several slab counts (H2D of slab i+1 overlaps the encode of slab i)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1812_10959_b200 as dic
from paper_1812_10959_b200.workloads import CONFIGS, generate_csr
cfg = CONFIGS[4]
ip, ix = generate_csr(cfg)
hp = torch.from_numpy(ip.astype(np.int32)).pin_memory()
hx = torch.from_numpy(ix.astype(np.uint16)).pin_memory()
for slabs in (4, 8, 16, 32):
    best = 1e30
    for _ in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        db = dic.BitDatabase.from_csr(hp, hx, cfg.m, slabs=slabs)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
        del db
    mb = (hp.numel() * 4 + hx.numel() * 2) / 1e6
    print(f"slabs {slabs}: {best * 1e3:.2f} ms  ({mb / best / 1e3:.1f} GB/s of {mb:.0f} MB)")
