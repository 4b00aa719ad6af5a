timeout 900 python -m pytest tests -q -x -m gpu --deselect tests/test_dd_gpu.py > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
timeout 600 python tools/time_kernels.py water12m stmv water3k > gpurun_out/r2g_kernels.jsonl 2>&1
