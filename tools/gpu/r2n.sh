NBX_TRACE_ALLOCS=1 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r2n_n1.json 2> gpurun_out/r2n_n1.err
