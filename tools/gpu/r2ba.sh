for c in rnase24k water3k stmv; do python tools/search_breakdown.py $c 20 >> gpurun_out/r2ba_breakdown.jsonl 2>>gpurun_out/r2ba.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ba_launches.csv python tools/search_breakdown.py rnase24k 2 > gpurun_out/r2ba_ncu.log 2>&1
