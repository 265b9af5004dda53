# usage (GPU box, >= 2 GPUs): NVLink bytes of the N=2 peer step from NVML counters
mkdir -p gpurun_out
for st in 20 220; do
  python tools/nvml_probe.py > gpurun_out/nvml_before_$st.json 2>&1
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 python bench.py --gpus 2 --steps $st --warmup 5 --no-e2e > gpurun_out/nvl_bench_$st.json 2> gpurun_out/nvl_bench_$st.err
  echo "n2 steps=$st rc=$?"
  python tools/nvml_probe.py > gpurun_out/nvml_after_$st.json 2>&1
  cat gpurun_out/nvml_before_$st.json gpurun_out/nvml_after_$st.json
done
