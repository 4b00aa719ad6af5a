timeout 600 python tools/search_stall.py water12m 30 > gpurun_out/r2l_stall.jsonl 2>&1
timeout 600 python tools/search_stall.py stmv 60 >> gpurun_out/r2l_stall.jsonl 2>&1
