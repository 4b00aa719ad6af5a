N=$1
nvidia-smi --query-gpu=index,name,clocks.sm --format=csv > gpurun_out/r2i_smi_n$N.txt
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2i_bench_n${N}_12m.json 2> gpurun_out/r2i_bench_n${N}_12m.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $N --steps 100 --warmup 10 --config stmv --no-e2e > gpurun_out/r2i_bench_n${N}_stmv.json 2> gpurun_out/r2i_bench_n${N}_stmv.err
python bench.py --steps 100 --warmup 10 --config stmv --no-e2e --no-cpu-baseline > gpurun_out/r2i_bench_n1_stmv.json 2> gpurun_out/r2i_bench_n1_stmv.err
