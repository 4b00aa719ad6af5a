timeout 600 python -m pytest tests/test_known_answers.py -q -m gpu > gpurun_out/r2c_ka.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_ka.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/r2c_bench100.json 2>> gpurun_out/r2c_bench.err
timeout 600 python bench.py --config stmv --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_stmv.json 2>> gpurun_out/r2c_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c_ref.json 2>> gpurun_out/r2c_bench.err
