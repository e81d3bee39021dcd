mkdir -p gpurun_out
for lib in default build/ab/lib_win21.so build/ab/lib_win23.so build/ab/lib_win25.so; do
  if [ $lib = default ]; then E=""; else E="VSB_LIB=$lib"; fi
  echo "== $lib"; env $E timeout 300 python scripts/sol_sizes.py 2>&1 | grep -E "MiB" | tail -5
done
