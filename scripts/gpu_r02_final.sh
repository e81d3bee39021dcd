# round-2 closing evidence: full GPU suite, smoke, full bench, launch list, ncu of the kernels changed late in the round
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-mc-parity --mc-steps 2 --stream-ticks 20 --rc-frames 3 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
N="ncu --set full --clock-control none --import-source on"
R="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc-parity --stream-ticks 40 --rc-frames 3 --mc-steps 1"
timeout 600 $N -k regex:k_mc_encode -s 2 -c 1 -o gpurun_out/r02_mc $R --no-stream --no-server --no-rc --no-config1 > gpurun_out/nf1.log 2>&1; echo mc=$?
timeout 600 $N -k regex:k_apply -s 3 -c 1 -o gpurun_out/r02_apply $R --no-mc --no-stream --no-server --no-rc --no-config1 > gpurun_out/nf2.log 2>&1; echo apply=$?
timeout 600 $N -k regex:k_stream_tick -s 30 -c 1 -o gpurun_out/r02_tick $R --no-mc --no-server --no-rc --no-config1 > gpurun_out/nf3.log 2>&1; echo tick=$?
timeout 600 $N -k regex:"k_put_rows|k_mc_encode|k_multi_fan_small" -s 60 -c 3 -o gpurun_out/r02_server $R --no-mc --no-stream --no-rc --no-config1 > gpurun_out/nf4.log 2>&1; echo server=$?
timeout 900 $N -k regex:"k_wpart_count|k_wpart_push|k_shard_apply|k_shard_return" -s 12 -c 4 -o gpurun_out/r02_shard python scripts/shard_time.py 3 125000000 24 > gpurun_out/nf5.log 2>&1; echo shard=$?
