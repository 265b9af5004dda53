# round-2 HEAD verification on one B200: GPU tests, smoke, bench cfg2 + cfg1, reference arm, launch lists
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/v_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_n1.json 2> gpurun_out/v_n1.err; echo bench rc=$?
tail -c 1500 gpurun_out/v_n1.json
timeout 300 python bench.py --config cfg1 --steps 200 --warmup 20 > gpurun_out/v_cfg1.json 2> gpurun_out/v_cfg1.err; echo cfg1 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err; echo ref rc=$?
tail -c 600 gpurun_out/v_ref.json
bash tools/launches.sh v_cfg2
RECD_LIB=paper_2211_05239_b200/librecd.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --csv --log-file gpurun_out/launches_v_cfg1.csv python bench.py --config cfg1 --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/launches_v_cfg1.log 2>&1; echo cfg1 launches rc=$?
python profiles/launches_summary.py gpurun_out/launches_v_cfg1.csv
