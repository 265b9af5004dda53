timeout 300 ./tools/gather_probe2 > gpurun_out/probe3.txt 2>&1; echo probe rc=$?; grep rmw gpurun_out/probe3.txt
bash tools/ab.sh "bwd or step" cur l2keep full l2full
