# full bench line + reference arm (numbers for the docs)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? wall=$(( $(date +%s) - t0 ))s
tail -2 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
