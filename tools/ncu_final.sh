# one ncu --set full capture of the two dominant kernels at the final commit (GPU box)
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/prof_plain.json 2>&1; echo plain rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_pool_ring" -s 2 -c 2 -o gpurun_out/r1_final_full -f python bench.py --profile --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_final.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_final.log
