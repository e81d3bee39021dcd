# server tick host-path A/B: HEAD (srvhead lib + HEAD python is not separable: python fast path + C scratch together) 
mkdir -p gpurun_out
timeout 600 python scripts/server_py_cost.py 2>&1 | tail -1
timeout 600 python scripts/server_host_cost.py 2>&1 | grep "host per tick"
timeout 900 python scripts/ab.py --rounds 3 --section server default build/ab/lib_srvhead.so 2>&1 | tail -6
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_shim_gpu.py -q -m gpu -rf 2>&1 | tail -2
