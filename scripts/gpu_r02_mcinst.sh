# MC instruction diet A/B: HEAD (tickets) vs carried sweep index vs + range-check predicates; digests + MC tests
mkdir -p gpurun_out
for L in build/ab/lib_tkhead.so build/ab/lib_carry.so ""; do VSB_LIB=$L timeout 300 python scripts/mc_drift.py 2>&1 | tail -1; done | tee gpurun_out/mc_inst.txt
timeout 900 python scripts/ab.py --rounds 3 --section mc default build/ab/lib_tkhead.so build/ab/lib_carry.so 2>&1 | tail -9 | tee -a gpurun_out/mc_inst.txt
timeout 900 python -m pytest tests/test_mc_gpu.py tests/test_fusion_gpu.py -q -m gpu -rf 2>&1 | tail -2
