python bench.py --steps 100 --warmup 5 > gpurun_out/r2bh_bench100.json 2>gpurun_out/r2bh_bench.err
python bench.py --steps 20 --warmup 5 > gpurun_out/r2bh_bench20.json 2>>gpurun_out/r2bh_bench.err
