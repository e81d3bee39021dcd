"""Host-side profile of the config-4 tick loop (experiments): cProfile over bench.run_stream."""
import cProfile, os, pstats, sys, types
sys.path.insert(0, os.getcwd())
import torch
import bench
dev = torch.device("cuda", 0)
args = types.SimpleNamespace(stream_ticks=int(os.environ.get("TICKS", 200)))
r = bench.run_stream(args, dev)
print("plain:", round(r["ms_per_tick"], 4), "ms/tick", round(r["wall_s"] * 1e3 / r["ticks"], 4), "ms wall/tick")
pr = cProfile.Profile()
pr.enable()
r = bench.run_stream(args, dev)
pr.disable()
print("profiled:", round(r["ms_per_tick"], 4), "ms/tick")
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
