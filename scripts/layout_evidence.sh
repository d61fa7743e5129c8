#!/bin/bash
# Layout evidence: bench lines and one ncu capture of the persistent kernel per
# (config, layout): DRAM bytes and L2 read sectors for the schedule-order vs PQ plans.
mkdir -p gpurun_out
for c in cfg3 cfg2 cfg5; do
  for l in schedule pq; do
    timeout -s KILL 300 python bench.py --config $c --layout $l --cpu-seconds 0.5 --e2e-steps 1 > gpurun_out/lay_${c}_${l}.json 2>/dev/null
    timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors.sum,smsp__inst_executed_op_ldgsts.sum,smsp__inst_executed_op_global_ld.sum \
      --clock-control none -k regex:ed_persistent -s 3 -c 1 --csv python bench.py --config $c --layout $l --steps 1 --warmup 3 --e2e-steps 1 --cpu-seconds 0.5 > gpurun_out/lay_ncu_${c}_${l}.csv 2>/dev/null
    echo "$c $l rc=$?"
  done
done
