python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 tools/dd_repart_timing.py water12m > gpurun_out/r2j_repart.log 2>&1
