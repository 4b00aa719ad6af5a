python tools/search_breakdown.py stmv 20 266657 >> gpurun_out/r2bc_breakdown.jsonl 2>>gpurun_out/r2bc.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bc_launches.csv python tools/search_breakdown.py stmv 2 266657 > gpurun_out/r2bc_ncu.log 2>&1
