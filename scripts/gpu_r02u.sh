mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_shim_gpu.py -q -x -rf > gpurun_out/pytest_stream.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_stream.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-mc --no-rc --no-e2e --no-config1 --no-stream --steps 5 > gpurun_out/srv.json 2> gpurun_out/srv.err; echo srv=$?
python -c "
import json; d=json.loads(open('gpurun_out/srv.json').read().splitlines()[-1])['server']; print({k: d.get(k) for k in ('value','ms_per_tick','host_ms_per_tick','ok','gpu_launches','error')})"
done
