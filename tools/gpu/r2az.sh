timeout 1500 python -m pytest tests/test_dd_gpu.py tests/test_peer_gpu.py -q -m gpu -rs > gpurun_out/r2az_dd4.log 2>&1; echo "rc=$?" >> gpurun_out/r2az_dd4.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2az_n4.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2az_n2.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 4 --steps 100 --warmup 10 --config stmv --no-e2e > gpurun_out/r2az_n4_stmv.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 2 --steps 100 --warmup 10 --config stmv --no-e2e > gpurun_out/r2az_n2_stmv.json 2>/dev/null
python bench.py --steps 100 --warmup 10 --config stmv --no-cpu-baseline --no-e2e > gpurun_out/r2az_n1_stmv.json 2>/dev/null
python bench.py --steps 20 --warmup 5 > gpurun_out/r2az_n1.json 2>/dev/null
