for cfg in water12m stmv; do
python bench.py --steps 100 --warmup 10 --no-e2e --config $cfg > gpurun_out/r2bm_n1_$cfg.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --config $cfg > gpurun_out/r2bm_n2_$cfg.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e --config $cfg > gpurun_out/r2bm_n4_$cfg.json 2>/dev/null
done
