mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests -x -q -m gpu > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt.log
for C in cfg3 cfg2 cfg5; do
for S in 0 1; do
ED_SPLIT=$S timeout -s KILL 300 python bench.py --config $C --cpu-seconds 0.5 --e2e-steps 1 > gpurun_out/b_$S.json 2>gpurun_out/b.err || { echo FAIL $C $S; tail -3 gpurun_out/b.err; continue; }
python - $C $S <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/b_{sys.argv[1]}_{sys.argv[2]}.json".replace("_"+sys.argv[1]+"_","_")).read().strip().splitlines()[-1]) if False else json.loads(open("gpurun_out/b_%s.json"%sys.argv[2] if False else "gpurun_out/b_"+sys.argv[2]+".json").read().strip().splitlines()[-1])
print(sys.argv[1:], round(d["value"]), round(d["ms_per_step"]*1e3,1), [round(s["t_meas_us"],1) for s in d["per_step_roofline"]["steps"]][:20])
PY
done; done
