#!/bin/bash
# A/B over variant libraries: scripts/ab_libs.sh "bench flags" lib1 lib2 ...
mkdir -p gpurun_out
FLAGS=$1; shift
for L in "$@"; do
  ED_BATCH_LIB=$PWD/$L timeout -s KILL 300 python bench.py --cpu-seconds 0.5 --e2e-steps 1 $FLAGS > gpurun_out/ab.json 2>gpurun_out/ab.err || { echo "FAIL $L"; tail -3 gpurun_out/ab.err; continue; }
  python - "$L $FLAGS" <<'PY'
import json, sys
d=json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:50s} {d['value']:10.0f} inst/s {d['ms_per_step']*1e3:7.1f} us", [round(s["t_meas_us"],1) for s in d["per_step_roofline"]["steps"]])
PY
done
