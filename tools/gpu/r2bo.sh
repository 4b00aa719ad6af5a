timeout 2400 python tools/results_table.py --steps 100 > gpurun_out/r2bo_results.md 2> gpurun_out/r2bo_results.err
