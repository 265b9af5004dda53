# row-scan occupancy with the stepped coalesced scan: 4 (cur) / 5 / 6 CTAs per SM
mkdir -p gpurun_out
for rep in 1 2 3; do bash tools/ab.sh "" cur rsm5 rsm6; done
