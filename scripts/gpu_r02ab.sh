mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hash_gpu.py -q -x -rf > gpurun_out/pytest_h.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_h.log
timeout 900 python scripts/ab.py --rounds 3 --section hash build/ab/lib_head.so default 2>&1 | tee gpurun_out/ab_postcta.txt
