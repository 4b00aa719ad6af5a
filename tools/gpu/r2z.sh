NBX_REPART=device python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 tools/dd_repart_timing.py water12m > gpurun_out/r2z_repart_dev.log 2>&1
NBX_REPART=device python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572 tools/dd_repart_timing.py stmv > gpurun_out/r2z_repart_dev_stmv.log 2>&1
