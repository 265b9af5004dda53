SKIP=0 COUNT=1 bash tools/ncu_kernel.sh k_rowscan rs3
SKIP=2 COUNT=1 bash tools/ncu_kernel.sh k_onesweep os4
SKIP=0 COUNT=1 bash tools/ncu_kernel.sh k_scatter sc5
