timeout 300 python tools/search_timing.py water12m > gpurun_out/r2d_search.jsonl 2>&1
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench100a.json 2>&1
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench100b.json 2>&1
