# final 1-GPU evidence at HEAD: GPU suite, smoke, bench (default) + reference arm, launch lists (cfg2 cold,
# cfg1 warm), ncu --set full of the top kernels -> traffic
mkdir -p gpurun_out
T=${1:-r2f}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_$T.log
timeout 600 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench rc=$?
timeout 300 python bench.py --config cfg1 --steps 200 --warmup 20 > gpurun_out/cfg1_$T.json 2> gpurun_out/cfg1_$T.err; echo cfg1 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_$T.json 2> gpurun_out/ref_$T.err; echo ref rc=$?
python -c "
import json
for n in ('bench','cfg1','ref'):
    d=json.loads(open('gpurun_out/'+n+'_$T.json').read().strip().splitlines()[-1])
    print(n, round(d['ms_per_step'],3) if 'ms_per_step' in d else '', round(d['value']/1e6,3), 'M/s', 'roof', (d.get('roofline') or {}).get('frac'), 'step', (d.get('step_roofline') or {}).get('frac'), 'e2e', (d.get('e2e') or {}).get('value'), d.get('clocks'))
"
bash tools/launches.sh $T
RECD_LIB=paper_2211_05239_b200/librecd.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_${T}_cfg1warm.csv python bench.py --config cfg1 --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_${T}_cfg1warm.log 2>&1; echo cfg1 warm launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_${T}_cfg1warm.csv
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_pool_ring|k_rowscan|k_onesweep|k_copy|k_occ|k_grad_u_flat" -c 12 -o gpurun_out/ncu_$T -f python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/ncu_$T.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py gpurun_out/ncu_$T.ncu-rep > gpurun_out/ncu_${T}_summary.txt 2>&1; head -30 gpurun_out/ncu_${T}_summary.txt
