# A/B the in-tree MC encoder against build/ab/lib_head.so on the same box (experiments)
for i in 1 2; do
  echo "head $(VSB_LIB=build/ab/lib_head.so timeout 300 python scripts/mc_time.py)"
  echo "new  $(timeout 300 python scripts/mc_time.py)"
done
