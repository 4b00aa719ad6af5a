ncu --set full --import-source on --clock-control none -k regex:k_search -s 2 -c 1 -o gpurun_out/r2bf_search python tools/search_breakdown.py stmv 1 266657 > gpurun_out/r2bf_ncu.log 2>&1
