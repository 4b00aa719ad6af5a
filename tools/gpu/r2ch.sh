for c in water12m stmv rnase24k mem82k; do python tools/force_variants.py run $c >> gpurun_out/r2ch.jsonl 2>>gpurun_out/r2ch.err; done
