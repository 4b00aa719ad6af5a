timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2bd_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2bd_parity.log
for c in "rnase24k 20" "water3k 20" "stmv 20 266657" "stmv 10" "mem82k 20" "water12m 3"; do python tools/search_breakdown.py $c >> gpurun_out/r2bd_breakdown.jsonl 2>>gpurun_out/r2bd.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bd_launches.csv python tools/search_breakdown.py stmv 2 266657 > gpurun_out/r2bd_ncu.log 2>&1
