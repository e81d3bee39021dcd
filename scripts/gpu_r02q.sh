# MC x-runs with run-strided sweeps: tests + A/B (default = runs of 8, 3 stages)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mc_gpu.py tests/test_edge_gpu.py -q -x -rf > gpurun_out/pytest_mc.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_mc.log
timeout 2000 python scripts/ab.py --rounds 2 --section mc build/ab/lib_mcold.so default build/ab/lib_run4.so build/ab/lib_run16.so build/ab/lib_run8s2.so 2>&1 | tee gpurun_out/ab_mc2.txt
