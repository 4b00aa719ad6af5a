timeout 600 python -m pytest tests/test_peer_gpu.py -q -m gpu > gpurun_out/r2aj.log 2>&1; echo "rc=$?" >> gpurun_out/r2aj.log
timeout 900 python -m pytest tests/test_dd_gpu.py -q -m gpu -k "oversub or regrow" >> gpurun_out/r2aj.log 2>&1; echo "rc=$?" >> gpurun_out/r2aj.log
