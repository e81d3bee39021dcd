# round 2 evidence: A/B of the evict_first excess hops, the full bench, the
# launch list of a reduced bench, and ncu --set full captures of every kernel family
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python scripts/ab.py --rounds 2 --section hash default build/ab/lib_evf.so 2>&1 | tee gpurun_out/ab_evf.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -2 gpurun_out/bench.err
N="ncu --set full --clock-control none --import-source on"
R="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc-parity --stream-ticks 20 --rc-frames 3 --mc-steps 1"
H="--no-mc --no-stream --no-server --no-rc --no-config1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-mc-parity --mc-steps 2 --stream-ticks 20 --rc-frames 3 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 600 $N -k regex:k_apply -s 3 -c 1 -o gpurun_out/r02_apply $R $H > gpurun_out/ncu1.log 2>&1; echo apply=$?
timeout 600 $N -k regex:k_post -s 8 -c 1 -o gpurun_out/r02_post $R $H > gpurun_out/ncu2.log 2>&1; echo post=$?
timeout 600 $N -k regex:k_mc_encode -s 2 -c 1 -o gpurun_out/r02_mc $R --no-stream --no-server --no-rc --no-config1 > gpurun_out/ncu3.log 2>&1; echo mc=$?
timeout 600 $N -k regex:"k_mc_faces|k_mc_compact" -c 2 -o gpurun_out/r02_mcaux $R --no-stream --no-server --no-rc --no-config1 > gpurun_out/ncu4.log 2>&1; echo mcaux=$?
timeout 600 $N -k regex:"k_dedup_small|k_multi_fan_small|k_multi_extract" -s 30 -c 3 -o gpurun_out/r02_stream $R --no-mc --no-server --no-rc --no-config1 > gpurun_out/ncu5.log 2>&1; echo stream=$?
timeout 600 $N -k regex:"k_put_rows|k_mc_encode" -s 40 -c 2 -o gpurun_out/r02_server $R --no-mc --no-stream --no-rc --no-config1 > gpurun_out/ncu6.log 2>&1; echo server=$?
timeout 600 $N -k regex:"k_rc_integrate|k_rc_cull_table" -s 4 -c 2 -o gpurun_out/r02_rc $R --no-mc --no-stream --no-server --no-config1 > gpurun_out/ncu7.log 2>&1; echo rc=$?
timeout 600 $N -k regex:"k_wpart_push|k_shard_apply|k_shard_return" -s 9 -c 3 -o gpurun_out/r02_shard python scripts/shard_time.py 3 > gpurun_out/ncu8.log 2>&1; echo shard=$?
ls gpurun_out/*.ncu-rep
