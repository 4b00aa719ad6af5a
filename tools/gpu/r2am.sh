for i in 1 2; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2959$i bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2am_n4_$i.json 2>/dev/null
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29593 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2am_ref4.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2am_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2am_parity.log
