timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2ab_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ab_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2ab_smoke.log
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2ab_ref.json 2> gpurun_out/r2ab_ref.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2ab_bench.json 2> gpurun_out/r2ab_bench.err
