#!/bin/bash
# repeat bench runs of one config with each library: scripts/repeat_cfg.sh CFG N lib...
C=$1; N=$2; shift 2
for L in "$@"; do
  ok=0; bad=0
  for i in $(seq $N); do
    ED_BATCH_LIB=$PWD/$L timeout -s KILL 120 python bench.py --config $C --cpu-seconds 0.2 --e2e-steps 1 --steps 5 --warmup 3 > gpurun_out/rep.json 2>gpurun_out/rep_$i.err && ok=$((ok+1)) || { bad=$((bad+1)); grep -m2 -i "error\|watchdog\|fail" gpurun_out/rep_$i.err; }
  done
  echo "$C $L ok=$ok bad=$bad"
done
