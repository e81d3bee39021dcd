mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hash_gpu.py tests/test_stream_gpu.py -q -x -rf > gpurun_out/pytest_h.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_h.log
timeout 900 python scripts/ab.py --rounds 2 --section config1 build/ab/lib_head.so default 2>&1 | tee gpurun_out/ab_push.txt
timeout 900 python scripts/ab.py --rounds 2 --section hash build/ab/lib_head.so default 2>&1 | tee -a gpurun_out/ab_push.txt
timeout 900 python scripts/ab.py --rounds 1 --section stream build/ab/lib_head.so default 2>&1 | cut -c1-250 | tee -a gpurun_out/ab_push.txt
