mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mc_gpu.py tests/test_edge_gpu.py -q -x -rf > gpurun_out/pytest_mc.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_mc.log
timeout 1500 python scripts/ab.py --rounds 3 --section mc build/ab/lib_nolut.so default 2>&1 | cut -c1-200 | tee gpurun_out/ab_lut.txt
