# usage (GPU box): tools/ncu_scatter_dram.sh v1 v2 ... -- DRAM bytes + time of one k_scatter launch per variant
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "cur" ]; then lib=paper_2211_05239_b200/librecd.so; else lib=build/variants/librecd_$v.so; fi
  RECD_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:"k_scatter" -c 1 --csv --log-file gpurun_out/scd_$v.csv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graph > gpurun_out/scd_$v.log 2>&1
  echo "$v rc=$?"; grep -o '"[a-z_]*__[a-z_.]*","[a-z]*","[0-9.,]*"' gpurun_out/scd_$v.csv
done
