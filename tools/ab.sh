# usage: tools/ab.sh "<pytest -k expr or empty>" v1 v2 ...  (GPU box) -- tests on the in-tree lib, then bench per variant
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/ab_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/ab_pytest.log; fi
shift
for v in "$@"; do
  if [ "$v" = "cur" ]; then lib=paper_2211_05239_b200/librecd.so; else lib=build/variants/librecd_$v.so; fi
  RECD_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e $BENCH_ARGS > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  echo "$v rc=$?"
  python -c "
import json,sys
d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, {k:round(v['ms'],3) for k,v in d['kernels'].items()})
"
done
