mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v3.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_l.log 2>&1; echo list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_pool_ring|k_rowscan" -c 3 -o gpurun_out/r1_full_v3 -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full3.log 2>&1; echo full rc=$?
