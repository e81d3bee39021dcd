mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_shim_gpu.py tests/test_hash_gpu.py tests/test_stream_gpu.py tests/test_fusion_gpu.py -q -x -rf > gpurun_out/pytest_shim.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_shim.log
timeout 300 python scripts/single_time.py | tee gpurun_out/single_time.txt
