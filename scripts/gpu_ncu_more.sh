# ncu --set full captures of the other kernel families (one launch each):
# stream fan-out insert, RC integrate, MC compaction, the peer-shard kernels.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --live 1000000 --batch-log2 16"
timeout 600 $N -k regex:k_multi_insert -s 20 -c 1 -o gpurun_out/prof_stream $B --no-mc --no-rc --stream-ticks 30 > gpurun_out/ncu_stream.log 2>&1; echo ncu_stream=$?
timeout 600 $N -k regex:k_rc_integrate -s 10 -c 1 -o gpurun_out/prof_rc $B --no-mc --no-stream --rc-frames 12 > gpurun_out/ncu_rc.log 2>&1; echo ncu_rc=$?
timeout 600 $N -k regex:"k_wpart_push|k_shard_apply|k_shard_return" -s 9 -c 3 -o gpurun_out/prof_shard python scripts/shard_time.py 3 > gpurun_out/ncu_shard.log 2>&1; echo ncu_shard=$?
