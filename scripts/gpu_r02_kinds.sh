# per-op-kind cost of k_apply on the config-2 table (scripts/hash_mix_time.py), three repeats
mkdir -p gpurun_out
for r in 1 2 3; do echo "== round $r"; timeout 600 python scripts/hash_mix_time.py; done > gpurun_out/kinds.txt 2>&1
echo rc=$?; cat gpurun_out/kinds.txt
