# end of round 2: final-HEAD validation on a 4-GPU box (GPU suite incl. real multi-GPU DD, smoke,
# default benches N = 1/2/4 and the reference arm, STMV N = 1/2/4, launch list of the N = 1 bench)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/r3z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3z_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3z_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r3z_n1.json 2> gpurun_out/r3z_n1.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r3z_ref.json 2> gpurun_out/r3z_ref.err
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r3z_n1_k100.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r3z_n2.json 2>gpurun_out/r3z_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r3z_n4.json 2>gpurun_out/r3z_n4.err
python bench.py --config stmv --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r3z_stmv_n1.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29573 bench.py --gpus 2 --steps 100 --warmup 10 --no-e2e --config stmv > gpurun_out/r3z_stmv_n2.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29574 bench.py --gpus 4 --steps 100 --warmup 10 --no-e2e --config stmv > gpurun_out/r3z_stmv_n4.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3z_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3z_ncu.log 2>&1
