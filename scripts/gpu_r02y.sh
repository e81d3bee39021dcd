mkdir -p gpurun_out
timeout 900 python scripts/ab.py --rounds 2 --section hash default build/ab/lib_st512.so build/ab/lib_st1024.so build/ab/lib_st2048.so 2>&1 | tee gpurun_out/ab_stripes.txt
A="python bench.py --no-cpu --no-mc --no-stream --no-rc --no-e2e --no-server --steps 3 --live 2000000 --batch-log2 18"
for lib in default build/ab/lib_st512.so build/ab/lib_st1024.so build/ab/lib_st2048.so; do
  if [ $lib = default ]; then E=""; else E="VSB_LIB=$lib"; fi
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_recycle|k_erase_win|k_post|k_insert" --csv --log-file gpurun_out/st_$(basename $lib).csv $A > /dev/null 2>&1
  echo "== $lib"; python scripts/launch_summary.py gpurun_out/st_$(basename $lib).csv | tee -a gpurun_out/ab_stripes.txt
done
