python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2aa_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2aa_launches.csv python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2aa_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2aa_ncu.log
