mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/prof_plain.json 2>&1; echo plain rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_pool_fwd|k_rowscan|k_sort_down" -c 4 -o gpurun_out/r1_full -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out/
