NBX_REPART=device timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29611 tools/dd_repart_timing.py stmv > gpurun_out/r2bk_stmv_n4.log 2>&1
timeout 1500 python -m pytest tests/test_dd_gpu.py -q -x -k "stmv_full and 4" > gpurun_out/r2bk_dd4.log 2>&1; echo "rc=$?" >> gpurun_out/r2bk_dd4.log
