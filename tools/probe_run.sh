mkdir -p gpurun_out
timeout 300 ./tools/gather_probe2 > gpurun_out/probe2.txt 2>&1; echo probe rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,dram__bytes_read.sum --csv -s 32 -c 12 ./tools/gather_probe2 > gpurun_out/probe2_ncu.csv 2>&1; echo ncu rc=$?
bash tools/ab.sh "bwd or pool or smoke or sharded" cur
