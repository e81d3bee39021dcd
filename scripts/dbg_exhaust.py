import sys, faulthandler, torch
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, '.')
from paper_1805_03709_b200 import BlockHashSet, CapacityExhausted
keys = [(i, 0, 0) for i in range(40)]
s = BlockHashSet(4, 16)
print("free", s.free_count(), flush=True)
created, index = s.insert_keys(keys)
torch.cuda.synchronize()
print("created", created.cpu().tolist(), flush=True)
print("index", index.cpu().tolist(), flush=True)
print("audit", s.audit(), "free", s.free_count(), flush=True)
try:
    s.check_capacity()
except CapacityExhausted as e:
    print("capacity", e, flush=True)
f = int(torch.nonzero(index < 0)[0, 0]); print("f", f, flush=True)
later = created.clone(); later[: f + 1] = 0
undo = torch.tensor(keys, dtype=torch.int32)[later.cpu().bool()]
print("undo", undo.shape, flush=True)
er, ei = s.erase_keys(undo)
torch.cuda.synchronize()
print("erased", er.cpu().tolist(), ei.cpu().tolist(), flush=True)
print("audit", s.audit(), "free", s.free_count(), flush=True)
c1, i1 = s.insert_keys(keys[f:f+1]); torch.cuda.synchronize(); print("single", c1.tolist(), i1.tolist(), flush=True)
