# 2-GPU: real NCCL / NVLink DD parity at full STMV size
nvidia-smi topo -m > gpurun_out/r2b_topo.txt 2>&1
timeout 1500 python -m pytest tests/test_dd_gpu.py -q -m gpu -k "not oversub" --durations=0 -rs > gpurun_out/r2b_dd2.log 2>&1
echo "dd rc=$?" >> gpurun_out/r2b_dd2.log
