# GPU box: correctness of grouped grad_u/scatter + A/B of RECD_SC_GROUP
for g in 0 3; do
  RECD_SC_GROUP=$g timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_step.py -x -q > gpurun_out/pytest_scg$g.log 2>&1
  echo "pytest group=$g rc=$?"; tail -2 gpurun_out/pytest_scg$g.log
done
for rep in 1 2; do
  for g in 0 2 4 7 13; do bash tools/ab_env.sh "RECD_SC_GROUP=$g" g$g; done
done
