# usage (GPU box): tools/ncu_r2.sh <tag> -- launch list of one bench step + ncu --set full of the top kernels
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 2 --warmup 1 --no-cpu > gpurun_out/prof_plain_$1.json 2>&1; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_$1.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_$1.log 2>&1; echo launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_$1.csv > gpurun_out/launches_$1.txt 2>&1; head -40 gpurun_out/launches_$1.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_pool_ring|k_rowscan|k_onesweep|k_copy|k_occ|k_grad_u_flat|k_expand" -c 12 -o gpurun_out/ncu_$1 -f python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/ncu_$1.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_$1.log
python tools/ncu_summary.py gpurun_out/ncu_$1.ncu-rep > gpurun_out/ncu_$1_summary.txt 2>&1; head -5 gpurun_out/ncu_$1_summary.txt
