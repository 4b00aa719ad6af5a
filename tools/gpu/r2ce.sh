for c in water12m stmv stmv:266657 rnase24k mem82k; do python tools/force_variants.py run $c >> gpurun_out/r2ce.jsonl 2>>gpurun_out/r2ce.err; done
