timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_all.log
for rep in 1 2; do bash tools/ab_env.sh "RECD_FUSED_EXPAND=0" unfused; bash tools/ab_env.sh "" fused; done
