python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29644 tools/dbg_regrow_worker.py none squeeze > gpurun_out/r2ah.log 2>&1
