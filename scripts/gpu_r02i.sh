mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py -q -x -rf > gpurun_out/pytest_stream.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_stream.log
