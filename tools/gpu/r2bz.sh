for c in rnase24k mem82k stmv:266657 water12m:300000; do python tools/force_variants.py run $c >> gpurun_out/r2bz.jsonl 2>>gpurun_out/r2bz.err; done
