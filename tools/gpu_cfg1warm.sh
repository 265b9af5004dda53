mkdir -p gpurun_out
RECD_LIB=paper_2211_05239_b200/librecd.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_cfg1warm.csv python bench.py --config cfg1 --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_cfg1warm.log 2>&1; echo rc=$?
python profiles/launches_summary.py gpurun_out/launches_cfg1warm.csv
