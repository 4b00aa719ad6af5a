timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/r2cd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2cd_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cd_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2cd_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2cd_n1.json 2>gpurun_out/r2cd_n1.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2cd_ref_n1.json 2>gpurun_out/r2cd_ref_n1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2cd_n2.json 2>gpurun_out/r2cd_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2cd_n4.json 2>gpurun_out/r2cd_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29573 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/r2cd_ref_n4.json 2>gpurun_out/r2cd_ref_n4.err
