mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_encoder.py -x -q > gpurun_out/enc.log 2>&1; echo enc rc=$?
tail -40 gpurun_out/enc.log
