# last verification at the final commit: GPU suite, smoke, default bench, cfg1, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_last.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_last.log
timeout 600 python bench.py > gpurun_out/bench_last.json 2> gpurun_out/bench_last.err; echo bench rc=$?
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_last20.json 2> gpurun_out/bench_last20.err; echo bench20 rc=$?
timeout 300 python bench.py --config cfg1 --steps 200 --warmup 20 > gpurun_out/cfg1_last.json 2> gpurun_out/cfg1_last.err; echo cfg1 rc=$?
python -c "
import json
for n in ('bench_last','bench_last20','cfg1_last'):
    d=json.loads(open('gpurun_out/'+n+'.json').read().strip().splitlines()[-1])
    print(n, round(d['ms_per_step'],3), round(d['value']/1e6,3), 'M/s roof', round(d['roofline']['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'e2e', (d.get('e2e') or {}).get('value'), d.get('clocks'))
"
bash tools/launches.sh last
