mkdir -p gpurun_out
timeout 600 python tools/sort_probe.py
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_onesweep" --csv --log-file gpurun_out/sortprobe.csv python tools/sort_probe.py > gpurun_out/sortprobe_ncu.log 2>&1; echo ncu rc=$?
grep -h "gpu__time" gpurun_out/sortprobe.csv | awk -F'","' '{print $15}' | tr -d '"' | tr '\n' ' ' | fold -w 200
