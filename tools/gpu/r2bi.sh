ncu --set full --import-source on --clock-control none -k regex:k_prune_packed -s 2 -c 1 -o gpurun_out/r2bi_prune python tools/search_breakdown.py water12m 1 1500000 > gpurun_out/r2bi_ncu.log 2>&1
