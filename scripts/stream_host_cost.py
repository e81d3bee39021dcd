"""Host-side cost per call of the config-4 tick's pieces (experiments): the
GPU work is made trivial (tiny sets, one key) so the loop measures the
Python + ctypes + launch overhead of each call."""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1805_03709_b200 import BlockHashSet, StreamSet, _lib, extract_random_many, fan_out
dev = torch.device("cuda", 0)
C = 16
clients = [StreamSet(1 << 10, 1 << 10, device=dev, fifo_capacity=1 << 22) for _ in range(C)]
scratch = BlockHashSet(1 << 14, 1 << 14, device=dev)
keys = torch.randint(0, 1000, (4096, 3), dtype=torch.int32, device=dev)
aff = torch.empty((4096, 3), dtype=torch.int32, device=dev)
n_aff = torch.ones(1, dtype=torch.int64, device=dev)
gen = torch.Generator(device=dev); gen.manual_seed(1)
lib = _lib.load()
acc = torch.zeros(1, dtype=torch.int64, device=dev)

def t(name, fn, n=400):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:28s} {1e6 * (t1 - t0) / n:8.1f} us host/call")

t("randint+index", lambda: keys[torch.randint(0, 4096, (512,), generator=gen, device=dev)])
st = torch.cuda.current_stream(dev)
t("affected_dedup", lambda: lib.vs_affected_dedup(scratch.handle, _lib.ptr(keys), 1, _lib.ptr(aff), _lib.ptr(n_aff), ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
t("fan_out(16, n_dev)", lambda: fan_out(clients, keys[:1], sync=False, n_dev=n_aff), n=200)
t("add_", lambda: acc.add_(n_aff))
t("extract_random_many(16)", lambda: extract_random_many(clients, 512))
t("n.sum()+add_", lambda: acc.add_(n_aff.sum()))
t("current_stream", lambda: torch.cuda.current_stream(dev))
t("empty", lambda: torch.empty(16, dtype=torch.int64, device=dev))
