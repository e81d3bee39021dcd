# RC integrate ticketed work A/B + fusion tests + ncu of the ticketed MC encode
mkdir -p gpurun_out
timeout 900 python scripts/ab.py --rounds 3 --section rc default build/ab/lib_rcstatic.so 2>&1 | tail -6 | tee gpurun_out/ab_rc_ticket.txt
timeout 900 python -m pytest tests/test_fusion_gpu.py tests/test_mc_gpu.py -q -m gpu -rf 2>&1 | tail -2
N="ncu --set full --clock-control none --import-source on"
R="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc-parity --stream-ticks 40 --rc-frames 3 --mc-steps 1"
timeout 600 $N -k regex:k_mc_encode -s 2 -c 1 -o gpurun_out/r02_mc $R --no-stream --no-server --no-rc --no-config1 > gpurun_out/nf1.log 2>&1; echo mc=$?
timeout 600 $N -k regex:"k_rc_cull|k_rc_integrate" -s 6 -c 2 -o gpurun_out/r02_rc $R --no-mc --no-stream --no-server --no-config1 > gpurun_out/nf6.log 2>&1; echo rc=$?
