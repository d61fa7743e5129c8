mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_bench_configs.py -x -q > gpurun_out/pt_bench_cfgs.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_bench_cfgs.log
for c in cfg5 cfg5_h512 cfg5_gru; do
timeout -s KILL 300 python bench.py --config $c --cpu-seconds 1 --e2e-steps 2 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; echo "bench $c rc=$?"; tail -2 gpurun_out/b_$c.err
python -c "
import json
d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d['ms_per_step'], d['config']['batches'], d['roofline']['frac'], d['per_step_roofline']['t_floor_us'])
"
done
