timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2ay_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ay_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ay_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2ay_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2ay_bench.json 2>/dev/null
timeout 1800 python tools/results_table.py --steps 100 > gpurun_out/r2ay_results.md 2> gpurun_out/r2ay_results.err
