#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture. Outputs -> gpurun_out/
set -x
TAG=${TAG:-r01}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke_$TAG.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" = "1" ]; then
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/bench_ncu_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:ed_persistent -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --e2e-steps 1 --cpu-seconds 1 > gpurun_out/prof_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
