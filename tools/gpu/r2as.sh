timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2as_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2as_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2as_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2as_smoke.log
timeout 600 python tools/time_kernels.py water12m stmv > gpurun_out/r2as_kernels.jsonl 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2as_bench.json 2>/dev/null
python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r2as_bench100.json 2>/dev/null
