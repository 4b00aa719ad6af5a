timeout 1500 python -m pytest tests/test_dd_gpu.py -q -m gpu > gpurun_out/r2ai_dd.log 2>&1; echo "rc=$?" >> gpurun_out/r2ai_dd.log
