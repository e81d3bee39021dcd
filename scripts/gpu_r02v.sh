# line layout at higher ops-in-flight per thread vs the kept flat design (config 2 and the config-5 slice)
mkdir -p gpurun_out
timeout 1500 python scripts/ab.py --rounds 2 --section hash default build/ab/lib_flat_ops2.so build/ab/lib_lines_ops1.so build/ab/lib_lines_ops2.so build/ab/lib_lines_ops4.so 2>&1 | tee gpurun_out/ab_lines_ops.txt
timeout 1500 python scripts/ab.py --rounds 1 --section hash --extra "--config5-slice 8 --steps 10" default build/ab/lib_lines_ops2.so build/ab/lib_lines_ops4.so 2>&1 | tee gpurun_out/ab_lines_ops_c5.txt
