# one GPU call: tests, bench, launch list, full ncu captures of the two dominant kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -3 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --mc-steps 2 --stream-ticks 20 \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 3 -c 1 \
  -o gpurun_out/prof_apply python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc \
  > gpurun_out/ncu_apply.log 2>&1; echo ncu_apply=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mc_encode -s 2 -c 1 \
  -o gpurun_out/prof_mc python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --mc-steps 1 \
  > gpurun_out/ncu_mc.log 2>&1; echo ncu_mc=$?
fi
