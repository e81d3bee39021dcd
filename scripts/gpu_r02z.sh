mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hash_gpu.py tests/test_stream_gpu.py tests/test_shard_gpu.py -q -x -rf > gpurun_out/pytest_h.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_h.log
timeout 900 python scripts/ab.py --rounds 2 --section hash build/ab/lib_head.so default 2>&1 | tee gpurun_out/ab_home.txt
A="python bench.py --no-cpu --no-mc --no-stream --no-rc --no-e2e --no-server --steps 3 --live 2000000 --batch-log2 18"
for lib in build/ab/lib_head.so default; do
  if [ $lib = default ]; then E=""; else E="VSB_LIB=$lib"; fi
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_recycle|k_erase_win|k_post|k_insert" --csv --log-file gpurun_out/home_$(basename $lib).csv $A > /dev/null 2>&1
  echo "== $lib"; python scripts/launch_summary.py gpurun_out/home_$(basename $lib).csv | tee -a gpurun_out/ab_home.txt
done
timeout 900 python scripts/ab.py --rounds 2 --section config1 build/ab/lib_head.so default 2>&1 | tee -a gpurun_out/ab_home.txt
