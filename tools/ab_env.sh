# usage (GPU box): tools/ab_env.sh "ENV=val ..." tag  -- one bench line with extra env vars
mkdir -p gpurun_out
env $1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e $BENCH_ARGS > gpurun_out/env_$2.json 2> gpurun_out/env_$2.err
echo "$2 rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/env_$2.json').read().strip().splitlines()[-1])
print('$2', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, {k:round(v['ms'],3) for k,v in d['kernels'].items()})
"
