# usage: tools/launches.sh <tag> [variant]  (GPU box): ncu launch list (times only) of one bench step
mkdir -p gpurun_out
lib=paper_2211_05239_b200/librecd.so; [ -n "$2" ] && lib=build/variants/librecd_$2.so
RECD_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_$1.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_$1.log 2>&1; echo launches $1 rc=$?
python profiles/launches_summary.py gpurun_out/launches_$1.csv
