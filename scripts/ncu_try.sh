for C in 1 0; do
ED_CLUSTER_COOP=$C timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_coop$C.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --cpu-seconds 0.3 > gpurun_out/bn$C.log 2>&1; echo "coop=$C rc=$?"; grep -c persistent gpurun_out/launches_coop$C.csv; grep ERROR gpurun_out/launches_coop$C.csv | head -3
done
