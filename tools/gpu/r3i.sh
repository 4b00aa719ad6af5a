mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prune_kernels_identical" 2>&1 | grep -E "Error|error|FAIL" | head -20 > gpurun_out/r3i_tests.log
NBX_LIB=scratch/variants/libnbx_base.so python tools/time_kernels.py rnase24k >> gpurun_out/r3i_tests.log 2>&1
