# MC x-runs: MC GPU tests, A/B of the config-3 section (default = x-runs + 3 stages)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mc_gpu.py tests/test_edge_gpu.py -q -x -rf > gpurun_out/pytest_mc.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_mc.log
timeout 1500 python scripts/ab.py --rounds 2 --section mc default build/ab/lib_mcold.so build/ab/lib_xrun2.so 2>&1 | tee gpurun_out/ab_mc.txt
timeout 600 python bench.py --steps 3 --no-cpu --no-e2e --no-stream --no-server --no-rc --no-config1 > gpurun_out/mc_full.json 2>gpurun_out/mc_full.err; echo mcfull=$?
python -c "
import json; d=json.loads(open('gpurun_out/mc_full.json').read().splitlines()[-1])['mc']; print({k: d.get(k) for k in ('value','ms_per_step','ok','parity')}, d['roofline']['frac'], d['compact']['ms_per_step'], d['compact']['ok'])"
