#!/bin/bash
# A/B bench lines: each argument is a quoted set of bench.py flags; prints value, us/pass, per-step us
mkdir -p gpurun_out
for a in "$@"; do
  timeout -s KILL 300 python bench.py --cpu-seconds 0.5 --e2e-steps 1 $a > gpurun_out/ab.json 2>gpurun_out/ab.err || { echo "FAIL $a"; tail -3 gpurun_out/ab.err; continue; }
  python - "$a" <<'PY'
import json, sys
d=json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:40s} {d['value']:10.0f} inst/s {d['ms_per_step']*1e3:7.1f} us frac {d['roofline']['frac']:.3f}", [round(s["t_meas_us"],1) for s in d["per_step_roofline"]["steps"]])
PY
done
