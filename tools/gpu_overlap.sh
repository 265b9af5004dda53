# GPU box: A/B of lookup CTA cap and side-stream priority (sort overlap)
for rep in 1 2; do
  bash tools/ab_env.sh "RECD_POOL_CTAS=16" base
  bash tools/ab_env.sh "RECD_SIDE_PRIORITY=-1" sp
  bash tools/ab_env.sh "RECD_POOL_CTAS=2" pc2
  bash tools/ab_env.sh "RECD_POOL_CTAS=2 RECD_SIDE_PRIORITY=-1" pc2sp
  bash tools/ab_env.sh "RECD_POOL_CTAS=3" pc3
  bash tools/ab_env.sh "RECD_POOL_CTAS=2 RECD_OS_CTAS=1 RECD_SIDE_PRIORITY=-1" pc2os1sp
  bash tools/ab_env.sh "RECD_POOL_CTAS=1 RECD_SIDE_PRIORITY=-1" pc1sp
done
