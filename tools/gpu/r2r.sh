timeout 1500 python -m pytest tests/test_dd_gpu.py -q -m gpu -k "not oversub" -rs > gpurun_out/r2r_dd4.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_dd4.log
for cfg in water12m stmv; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e --config $cfg > gpurun_out/r2r_n4_$cfg.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --config $cfg > gpurun_out/r2r_n2_$cfg.json 2>/dev/null
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2r_n4_default.json 2>/dev/null
