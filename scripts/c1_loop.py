import faulthandler, sys, os, time
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_03709_b200 import BlockHashSet, workloads
dev = torch.device("cuda", 0)
keys, absent = workloads.config1_keys()
import numpy as np
dk = torch.from_numpy(keys).to(dev); dp = torch.from_numpy(np.concatenate([keys, absent])).to(dev)
s = BlockHashSet(1 << 17, 1 << 17, device=dev)
for it in range(300):
    c, _ = s.insert_keys(dk); f, _ = s.find_keys(dp); e, _ = s.erase_keys(dk)
    torch.cuda.synchronize()
    cs, es = int(c.sum()), int(e.sum())
    if it % 20 == 0 or cs != 80000 or es != 80000:
        a = s.audit() if hasattr(s, "audit") else None
        print(it, cs, int(f.sum()), es, a, flush=True)
    if cs != 80000 or es != 80000: break
print("done")
