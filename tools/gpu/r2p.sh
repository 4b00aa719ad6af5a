timeout 1200 python -m pytest tests/test_dd_gpu.py -q -x -m gpu -k oversub > gpurun_out/r2p_dd.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_dd.log
