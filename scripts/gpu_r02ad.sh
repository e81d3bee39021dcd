mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hash_gpu.py -q -x -rf > gpurun_out/pytest_h.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_h.log
timeout 1500 python scripts/ab.py --rounds 2 --section hash --extra "--config5-slice 8 --steps 20" build/ab/lib_noorder.so default 2>&1 | tee gpurun_out/ab_order.txt
timeout 900 python scripts/ab.py --rounds 1 --section hash build/ab/lib_noorder.so default 2>&1 | tee -a gpurun_out/ab_order.txt
