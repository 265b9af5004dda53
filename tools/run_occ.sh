timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 bash tools/ab.sh "" cur
CUDA_VISIBLE_DEVICES=0 bash tools/launches.sh occ2 2>&1 | grep -i "k_occ\|k_copy\|in step"
