timeout 1500 python -m pytest tests/test_dd_gpu.py -q -m gpu -rs > gpurun_out/r2ak_dd4.log 2>&1; echo "rc=$?" >> gpurun_out/r2ak_dd4.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2ak_n4.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2ak_n2.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29583 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2ak_ref4.json 2>/dev/null
