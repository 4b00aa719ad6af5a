timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2az_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2az_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2az_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2az_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2az_bench.json 2>gpurun_out/r2az_bench.err
timeout 600 python -m paper_2405_01420_b200.costs_adapter gpurun_out/b200_costs_r02.cfg > gpurun_out/r2az_costs.log 2>&1
