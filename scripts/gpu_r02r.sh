# round-2 refresh after the tick / server-tick / per-key changes: full GPU suite, full bench, launch list, ncu of the new kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -2 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-mc-parity --mc-steps 2 --stream-ticks 20 --rc-frames 3 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
N="ncu --set full --clock-control none --import-source on"
R="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc-parity --stream-ticks 40 --rc-frames 3 --mc-steps 1"
timeout 600 $N -k regex:k_stream_tick -s 30 -c 1 -o gpurun_out/r02_tick $R --no-mc --no-server --no-rc --no-config1 > gpurun_out/ncu_t.log 2>&1; echo tick=$?
timeout 600 $N -k regex:"k_multi_fan_small|k_put_rows|k_mc_encode|k_dedup_small" -s 60 -c 4 -o gpurun_out/r02_server $R --no-mc --no-stream --no-rc --no-config1 > gpurun_out/ncu_s.log 2>&1; echo server=$?
timeout 600 $N -k regex:k_post -s 3 -c 1 -o gpurun_out/r02_post python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-mc --no-stream --no-server --no-rc --no-config1 > gpurun_out/ncu_p.log 2>&1; echo post=$?
