timeout 900 python -m pytest tests -q -x -m gpu --deselect tests/test_dd_gpu.py > gpurun_out/r2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_tests.log
timeout 900 python -m pytest tests/test_dd_gpu.py -q -x -m gpu -k oversub > gpurun_out/r2o_dd.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_dd.log
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r2o_n1.json 2>/dev/null
python bench.py --steps 20 --warmup 5 > gpurun_out/r2o_n1_k20.json 2>/dev/null
for c in mem82k rnase24k water3k stmv; do python bench.py --config $c --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r2o_$c.json 2>/dev/null; done
