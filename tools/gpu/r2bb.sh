timeout 600 python tools/time_kernels.py water12m > gpurun_out/r2bb_kernels.jsonl 2>&1
python tools/prof_force.py water12m 3 > gpurun_out/r2bb_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bb_launches.csv python tools/prof_force.py water12m 3 > gpurun_out/r2bb_ncu.log 2>&1
