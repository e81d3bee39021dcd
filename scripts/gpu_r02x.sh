mkdir -p gpurun_out
A="python bench.py --no-cpu --no-mc --no-stream --no-rc --no-e2e --no-server --steps 3 --live 2000000 --batch-log2 18"
for lib in build/ab/lib_head.so default; do
  if [ $lib = default ]; then E=""; else E="VSB_LIB=$lib"; fi
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_recycle|k_erase_win|k_erase_claim" --csv --log-file gpurun_out/rec_$(basename $lib).csv $A > gpurun_out/rec_$(basename $lib).log 2>&1; tail -3 gpurun_out/rec_$(basename $lib).log
  echo "== $lib"; python scripts/launch_summary.py gpurun_out/rec_$(basename $lib).csv
done
