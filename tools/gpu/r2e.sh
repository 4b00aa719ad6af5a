timeout 900 python -m pytest tests -x -q -m gpu --deselect tests/test_dd_gpu.py > gpurun_out/r2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests.log
timeout 600 python tools/time_kernels.py water12m stmv rnase24k > gpurun_out/r2e_kernels.jsonl 2>&1
