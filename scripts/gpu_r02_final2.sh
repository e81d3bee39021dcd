# round-2 re-verification after the late drop-in / shard / growth changes: full GPU suite, smoke,
# full bench (wall-clocked), reference arm, shard ncu (128-key partition), sanitizer over every kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? wall=$(( $(date +%s) - t0 ))s
tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:"k_wpart_count|k_wpart_base|k_wpart_push|k_shard_apply|k_shard_return" -s 15 -c 5 -o gpurun_out/r02_shard $R python scripts/shard_time.py 3 125000000 24 > gpurun_out/nf5.log 2>&1; echo shard=$?
bash scripts/sanitize.sh
