mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_tick -s 30 -c 1 -o gpurun_out/r02_tick \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc --no-server --no-rc --no-config1 --stream-ticks 40 > gpurun_out/ncu_tick.log 2>&1; echo ncu=$?
