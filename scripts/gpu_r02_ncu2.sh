# the remaining kernel families under ncu --set full (one launch each)
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
H="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-mc-parity --mc-steps 1 --stream-ticks 20 --rc-frames 3"
timeout 600 $N -k regex:"k_insert" -s 1 -c 1 -o gpurun_out/r02_insert $H --no-mc --no-stream --no-server --no-rc --no-config1 > gpurun_out/n1.log 2>&1; echo insert=$?
timeout 600 $N -k regex:"k_find|k_erase_claim|k_erase_win|k_recycle" -s 12 -c 4 -o gpurun_out/r02_c1ops $H --no-mc --no-stream --no-server --no-rc > gpurun_out/n2.log 2>&1; echo c1ops=$?
timeout 600 $N -k regex:"k_mc_compact|k_tile_sums|k_scan_tiles|k_tile_scan" -c 4 -o gpurun_out/r02_compact $H --no-stream --no-server --no-rc --no-config1 > gpurun_out/n3.log 2>&1; echo compact=$?
timeout 600 $N -k regex:"k_multi_insert|k_multi_fixup|k_fifo_append" -c 3 -o gpurun_out/r02_fill $H --no-mc --no-server --no-rc --no-config1 > gpurun_out/n4.log 2>&1; echo fill=$?
timeout 600 $N -k regex:"k_chunk_count|k_chunk_write" -s 2 -c 2 -o gpurun_out/r02_snapshot $H --no-mc --no-server --no-rc --no-config1 > gpurun_out/n5.log 2>&1; echo snap=$?
ls gpurun_out/r02_insert* gpurun_out/r02_c1ops* gpurun_out/r02_compact* gpurun_out/r02_fill* gpurun_out/r02_snapshot*
