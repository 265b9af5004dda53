mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pool_ring" -c 1 -o gpurun_out/r1_ring -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_ring.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_ring.log
