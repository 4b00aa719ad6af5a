timeout 1800 python tools/results_table.py --steps 100 > gpurun_out/r2v_results.md 2> gpurun_out/r2v_results.err
cp gpurun_out/results_rows.json gpurun_out/r2v_results_rows.json 2>/dev/null
