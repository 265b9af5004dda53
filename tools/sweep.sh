#!/bin/bash
# usage: tools/sweep.sh v1 v2 ...   (runs on the GPU box; writes gpurun_out/var_<v>.json)
for v in "$@"; do
  RECD_LIB=build/variants/librecd_$v.so python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/var_$v.json 2>&1
  echo "$v rc=$?"
done
