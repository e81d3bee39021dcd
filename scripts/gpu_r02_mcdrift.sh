# MC work distribution: CTA drift (static vs chunk tickets), digests must match, A/B, GPU tests
mkdir -p gpurun_out
for L in "" build/ab/lib_static.so build/ab/lib_drift_static.so build/ab/lib_drift_tk.so; do
  VSB_LIB=$L timeout 300 python scripts/mc_drift.py 2>&1 | tail -1
done | tee gpurun_out/mc_drift.txt
for sec in mc server config1; do
  timeout 900 python scripts/ab.py --rounds 2 --section $sec default build/ab/lib_static.so 2>&1 | tail -4
done | tee gpurun_out/ab_mc_ticket.txt
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
