# round 2: new bench sections (config 1, config-5 slice), SOL vs table size, per-key path latency
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --no-mc-parity --no-rc > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo bench=$?
tail -3 gpurun_out/bench_a.err
timeout 600 python bench.py --config5-slice 8 --steps 20 --no-mc --no-stream --no-server --no-rc --no-config1 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5=$?
tail -3 gpurun_out/bench_c5.err
timeout 600 python scripts/sol_sizes.py > gpurun_out/sol_sizes.txt 2>&1; echo sol=$?
timeout 300 python scripts/single_time.py > gpurun_out/single_time.txt 2>&1; echo single=$?
cat gpurun_out/single_time.txt gpurun_out/sol_sizes.txt
