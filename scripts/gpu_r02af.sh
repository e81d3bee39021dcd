mkdir -p gpurun_out
for lib in build/ab/lib_noreg.so build/ab/lib_reg2.so build/ab/lib_reg4.so build/ab/lib_reg8.so default; do
  if [ $lib = default ]; then E=""; else E="VSB_LIB=$lib"; fi
  echo "== $lib"; env $E timeout 900 python scripts/shard_time.py 20 125000000 24 2>&1 | grep peer: 
done
