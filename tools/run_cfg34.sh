mkdir -p gpurun_out
timeout 600 python tools/bench_encoder.py > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo cfg4 rc=$?; cat gpurun_out/cfg4.json; tail -3 gpurun_out/cfg4.err
bash tools/sweep_cfg3.sh
