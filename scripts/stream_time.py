"""Phase timing of the config-4 tick (experiments)."""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_03709_b200 import BlockHashSet, StreamSet, _lib, fan_out, remove_everywhere, workloads
dev = torch.device("cuda", 0)
keys = torch.from_numpy(workloads.room_block_keys()).to(dev)
M = keys.shape[0]
C = 16
clients = [StreamSet(1 << 21, 1 << 21, device=dev, fifo_capacity=1 << 22) for _ in range(C)]
scratch = BlockHashSet(1 << 14, 1 << 14, device=dev)
fan_out(clients, keys)
aff = torch.empty((4096, 3), dtype=torch.int32, device=dev)
n_aff = torch.empty(1, dtype=torch.int64, device=dev)
lib = _lib.load()
gen = torch.Generator(device=dev); gen.manual_seed(1)
T = {}
def tm(name, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
for t in range(int(os.environ.get("TICKS", 20))):
    upd = keys[torch.randint(0, M, (512,), generator=gen, device=dev)]
    def dd():
        st = torch.cuda.current_stream(dev)
        _lib.check(lib.vs_affected_dedup(scratch.handle, _lib.ptr(upd), 512, _lib.ptr(aff), _lib.ptr(n_aff), ctypes.c_void_p(st.cuda_stream)))
        return int(n_aff.item())
    A = tm("dedup", dd)
    tm("fan_out", lambda: fan_out(clients, aff[:A]))
    tm("extract16", lambda: [c._set.extract_keys(512) for c in clients])
    tm("extract1", lambda: clients[0]._set.extract_keys(512))
    tm("snapshot1", lambda: clients[0]._set.snapshot_tensor())
tm("clear", lambda: clients[3].clear())
tm("fill1", lambda: fan_out([clients[3]], keys))
tm("reset", lambda: remove_everywhere(clients, keys[:256]))
print({k: round(v * 1e3 / (20 if k not in ("clear", "fill1", "reset") else 1), 3) for k, v in T.items()}, "ms")
