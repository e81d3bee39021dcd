import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1805_03709_b200 import BlockHashSet, BlockHashMap
s = BlockHashSet(1 << 12, 1 << 12)
for k in range(100): s.insert((k, 0, 0))
t0 = time.perf_counter()
for k in range(2000): s.insert((k, 1, 0))
t1 = time.perf_counter()
for k in range(2000): (k, 1, 0) in s
t2 = time.perf_counter()
for k in range(2000): s.remove((k, 1, 0))
t3 = time.perf_counter()
print(f"per-key us: insert {(t1-t0)/2000*1e6:.1f} find {(t2-t1)/2000*1e6:.1f} remove {(t3-t2)/2000*1e6:.1f}")
