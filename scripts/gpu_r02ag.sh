mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_shard_gpu.py tests/test_shard_cpu.py -q -x -rf > gpurun_out/pytest_shard.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_shard.log
for lib in build/ab/lib_noreg.so default; do
  if [ $lib = default ]; then E=""; else E="VSB_LIB=$lib"; fi
  echo "== $lib"; env $E timeout 900 python scripts/shard_time.py 20 125000000 24 2>&1 | grep peer:
  env $E timeout 600 python scripts/shard_time.py 30 2>&1 | grep peer:
done
