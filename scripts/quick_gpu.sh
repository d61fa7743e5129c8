#!/bin/bash
# quick GPU iteration: gpu tests, trace, bench (cfg given by $CFG, default cfg3)
mkdir -p gpurun_out
CFG=${CFG:-cfg3}
timeout -s KILL 400 python -m pytest tests -x -q -m gpu > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
timeout -s KILL 300 python bench.py --config $CFG --cpu-seconds 1 --e2e-steps 2 ${BENCH_ARGS} > gpurun_out/b.json 2>gpurun_out/b.err; echo "bench rc=$?"; tail -2 gpurun_out/b.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], [(s["m"], s["t_meas_us"]) for s in d["per_step_roofline"]["steps"]])
PY
