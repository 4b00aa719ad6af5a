timeout 900 python -m pytest tests/test_dd_gpu.py -q -m gpu -k regrow > gpurun_out/r2ac.log 2>&1; echo "rc=$?" >> gpurun_out/r2ac.log
