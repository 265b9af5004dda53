# usage: tools/ncu_kernel.sh <kernel-regex> <tag> [variant]  (GPU box): ncu --set full of one launch
mkdir -p gpurun_out
lib=paper_2211_05239_b200/librecd.so; [ -n "$3" ] && lib=build/variants/librecd_$3.so
RECD_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${SKIP:-1} -c ${COUNT:-1} -o gpurun_out/ncu_$2 -f python bench.py --profile --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_$2.log 2>&1; echo ncu $2 rc=$?
