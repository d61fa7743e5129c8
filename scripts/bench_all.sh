#!/bin/bash
# secondary bench lines: every config, both layouts (development / DESIGN.md numbers)
mkdir -p gpurun_out
TAG=${TAG:-r01}
for c in cfg3 cfg3_gru cfg3_2type cfg2 cfg5 cfg5_h512 cfg5_gru cfg4_treefc cfg4_mvrnn cfg1; do
  for l in ${LAYOUTS:-schedule pq}; do
    timeout -s KILL 300 python bench.py --config $c --layout $l --cpu-seconds 3 --e2e-steps 3 > gpurun_out/bench_${c}_${l}_$TAG.json 2>gpurun_out/bench_${c}_${l}_$TAG.err
    python - "$c" "$l" "gpurun_out/bench_${c}_${l}_$TAG.json" <<'PY'
import json, sys
c, l, f = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ps = d["per_step_roofline"]
    print(f"{c:12s} {l:9s} {d['value']:12.0f} inst/s  {d['ms_per_step']*1e3:8.1f} us  roofline {d['roofline']['frac']:.3f}  per-step {ps['frac']:.3f}  contig? e2e {d['e2e']['value']:.0f}")
except Exception as e:
    print(c, l, "FAILED", e)
PY
  done
done
timeout -s KILL 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference_$TAG.json 2>&1; tail -c 600 gpurun_out/bench_reference_$TAG.json
