# e2e raw-share sweep (row-coded wire) on one B200: prints e2e ms/step per share
mkdir -p gpurun_out
for sh in ${SHARES:-0.15 0.2 0.25 0.3 0.38}; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-raw-share $sh > gpurun_out/e2e_$sh.json 2> gpurun_out/e2e_$sh.err
  python -c "
import json
d=json.loads(open('gpurun_out/e2e_$sh.json').read().strip().splitlines()[-1])
e=d['e2e']; print('share $sh', round(d['ms_per_step'],3), 'e2e ms', round(e['ms_per_step'],3), round(e['value']/1e6,2), 'M/s h2d MB', round(e['h2d_bytes_per_step']/1e6,1))
"
done
