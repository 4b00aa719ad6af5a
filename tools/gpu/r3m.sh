# final HEAD on a 2-GPU box: whole GPU suite (real 2-GPU DD + oversubscribed), smoke, default benches N = 1 / 2, reference arm, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/r3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3m_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r3m_n1.json 2> gpurun_out/r3m_n1.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r3m_ref.json 2> gpurun_out/r3m_ref.err
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r3m_n1_k100.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r3m_n2.json 2>gpurun_out/r3m_n2.err
python bench.py --config stmv --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r3m_stmv_n1.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3m_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3m_ncu.log 2>&1
