python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port 29622 tests/dd_gpu_worker.py water12m full /tmp/r2q_dd8.npz p2p oversub > gpurun_out/r2q.log 2>&1
echo rc=$? >> gpurun_out/r2q.log
python tools/dd_diag.py /tmp/r2q_dd8.npz water12m f4 > gpurun_out/r2q_diag.txt 2>&1
python tools/dd_diag.py /tmp/r2q_dd8.npz water12m f3 >> gpurun_out/r2q_diag.txt 2>&1
