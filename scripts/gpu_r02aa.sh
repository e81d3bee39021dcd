mkdir -p gpurun_out
timeout 900 python scripts/ab.py --rounds 2 --section hash build/ab/lib_head.so default build/ab/lib_home1024.so build/ab/lib_home4096.so 2>&1 | tee gpurun_out/ab_home2.txt
timeout 900 python scripts/ab.py --rounds 2 --section config1 build/ab/lib_head.so default build/ab/lib_home1024.so 2>&1 | tee -a gpurun_out/ab_home2.txt
timeout 900 python scripts/ab.py --rounds 1 --section stream default build/ab/lib_home1024.so 2>&1 | cut -c1-200 | tee -a gpurun_out/ab_home2.txt
