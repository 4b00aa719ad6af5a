export NBX_LIB=$PWD/scratch/checked/libnbx.so
python -c "from paper_2405_01420_b200 import nbx; print(nbx.lib().nbx_version())" > gpurun_out/r2bw_checked_dd2.log 2>&1
timeout 1800 python -m pytest tests/test_dd_gpu.py tests/test_peer_gpu.py tests/test_checked_build.py -q -m gpu -rs >> gpurun_out/r2bw_checked_dd2.log 2>&1; echo "rc=$?" >> gpurun_out/r2bw_checked_dd2.log
