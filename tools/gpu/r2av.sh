python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2av_n4.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2av_n2.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus 4 --steps 100 --warmup 10 --config stmv --no-e2e > gpurun_out/r2av_n4_stmv.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29604 bench.py --gpus 2 --steps 100 --warmup 10 --config stmv --no-e2e > gpurun_out/r2av_n2_stmv.json 2>/dev/null
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2av_n1.json 2>/dev/null
python bench.py --steps 100 --warmup 10 --config stmv --no-cpu-baseline --no-e2e > gpurun_out/r2av_n1_stmv.json 2>/dev/null
