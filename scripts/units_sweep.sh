for ov in "" "1:64" "1:48" "1:32" "2:32" "2:16" "1:32,2:32" "1:64,2:32"; do
  ED_UNITS="$ov" timeout -s KILL 300 python bench.py --config cfg3 --cpu-seconds 0.5 --e2e-steps 1 > gpurun_out/u.json 2>/dev/null
  python - "$ov" <<'PY'
import json, sys
d=json.loads(open("gpurun_out/u.json").read().strip().splitlines()[-1])
print(f"ED_UNITS={sys.argv[1]:12s} {d['ms_per_step']*1e3:7.1f} us", [round(s["t_meas_us"],1) for s in d["per_step_roofline"]["steps"]][:6])
PY
done
