#!/bin/bash
# A/B: scripts/ab3.sh "configs" "label@ENV=..@lib ..." -- each variant run twice, alternating
mkdir -p gpurun_out
for C in $1; do
for rep in 1 2; do
for V in $2; do
  L=${V%%@*}; R=${V#*@}; E=${R%%@*}; LIB=${R#*@}
  env $E ED_BATCH_LIB=$PWD/$LIB timeout -s KILL 300 python bench.py --config $C --cpu-seconds 0.3 --e2e-steps 1 > gpurun_out/ab.json 2>gpurun_out/ab.err || { echo "FAIL $C $L"; tail -3 gpurun_out/ab.err; continue; }
  python - "$C $L" <<'PY'
import json, sys
d=json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:24s} {d['ms_per_step']*1e3:7.1f} us", [round(s["t_meas_us"],1) for s in d["per_step_roofline"]["steps"]][:16])
PY
done; done; done
