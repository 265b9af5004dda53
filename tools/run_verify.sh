# full verification on one B200: GPU tests, smoke, bench (both arms), ncu launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/n1.json 2> gpurun_out/n1.err; echo bench rc=$?
tail -c 3000 gpurun_out/n1.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref rc=$?
tail -c 800 gpurun_out/ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
