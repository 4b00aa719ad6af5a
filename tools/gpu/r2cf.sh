timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pair_search_gpu.py -q -x > gpurun_out/r2cf_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2cf_parity.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2cf_n1.json 2>gpurun_out/r2cf_n1.err
