python bench.py --steps 20 --warmup 5 > gpurun_out/r2ci_n1.json 2>gpurun_out/r2ci_n1.err
python bench.py --steps 100 --warmup 5 > gpurun_out/r2ci_n1_100.json 2>>gpurun_out/r2ci_n1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2ci_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/r2ci_ncu_bench.log 2>&1
