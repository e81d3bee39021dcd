# round-2 closing evidence after the post-pass change: full GPU suite, smoke, full bench,
# reference arm, launch list, ncu --set full of k_post and k_apply
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? wall=$(( $(date +%s) - t0 ))s
tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-mc-parity --mc-steps 2 --stream-ticks 20 --rc-frames 3 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
N="ncu --set full --clock-control none --import-source on"
R="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc-parity --stream-ticks 20 --rc-frames 3 --mc-steps 1"
H="--no-mc --no-stream --no-server --no-rc --no-config1"
timeout 600 $N -k regex:k_apply -s 3 -c 1 -o gpurun_out/r02_apply $R $H > gpurun_out/ncu1.log 2>&1; echo apply=$?
timeout 600 $N -k regex:k_post -s 8 -c 1 -o gpurun_out/r02_post $R $H > gpurun_out/ncu2.log 2>&1; echo post=$?
ls gpurun_out/*.ncu-rep
