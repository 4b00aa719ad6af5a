ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2bs_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e > gpurun_out/r2bs_ncu_bench.log 2>&1
