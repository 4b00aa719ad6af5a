for c in rnase24k water3k mem82k; do python bench.py --config $c --steps 100 --warmup 10 --no-e2e > gpurun_out/r2cb_$c.json 2>/dev/null; done
