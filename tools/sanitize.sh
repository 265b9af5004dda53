# usage (GPU box): tools/sanitize.sh <tag> -- compute-sanitizer memcheck / racecheck / synccheck
# over the single-GPU kernel tests (small shapes) and smoke()
mkdir -p gpurun_out
T="tests/test_gpu_sort.py tests/test_gpu_dedup.py tests/test_gpu_pool.py tests/test_gpu_bwd.py tests/test_gpu_step.py tests/test_gpu_jagged.py tests/test_gpu_graph_batches.py tests/test_gpu_runs.py tests/test_gpu_partial.py tests/test_gpu_transforms.py tests/test_gpu_wire.py"
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest $T -m gpu -x -q -k "not fullsize" > gpurun_out/san_$1_$tool.log 2>&1
  echo $tool rc=$?
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_$1_$tool.log | tail -3
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$1_smoke.log 2>&1; echo smoke memcheck rc=$?
tail -3 gpurun_out/san_$1_smoke.log
