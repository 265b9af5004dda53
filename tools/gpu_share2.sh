# lookup CTAs per SM beside the (faster) occurrence sort: default (2 = resident - 1) vs 3 vs 1; sort CTAs 2 / 3
mkdir -p gpurun_out
for rep in 1 2; do
  bash tools/ab_env.sh "RECD_POOL_CTAS=2" pc2
  bash tools/ab_env.sh "RECD_POOL_CTAS=3" pc3
  bash tools/ab_env.sh "RECD_POOL_CTAS=1" pc1
  bash tools/ab_env.sh "RECD_OS_CTAS=2" os2
done
