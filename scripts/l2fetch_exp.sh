for g in default 0 32 64 128; do
  echo "== VSB_L2_FETCH=$g"
  if [ $g = default ]; then python scripts/sol_probe.py 2>&1 | tail -6; else VSB_L2_FETCH=$g python scripts/sol_probe.py 2>&1 | tail -6; fi
done
VSB_L2_FETCH=32 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:"k_apply|k_probe_sol" -c 6 --clock-control none --csv --log-file gpurun_out/sol_metrics32.csv python scripts/sol_probe.py > /dev/null 2>&1
