nvidia-smi --query-gpu=name,compute_mode,clocks.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests/test_dd_gpu.py -x -q -m gpu -k oversub --durations=0 > gpurun_out/r2a_dd_oversub.log 2>&1
echo "dd rc=$?" >> gpurun_out/r2a_dd_oversub.log
timeout 900 python -m pytest tests -x -q -m gpu --deselect tests/test_dd_gpu.py --durations=15 > gpurun_out/r2a_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2a_gpu_tests.log
tail -3 gpurun_out/r2a_dd_oversub.log gpurun_out/r2a_gpu_tests.log
