timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2ba_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ba_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ba_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2ba_smoke.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ba_bench.json 2>/dev/null
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ba_bench2.json 2>/dev/null
