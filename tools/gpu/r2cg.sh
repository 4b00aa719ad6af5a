for c in water12m stmv stmv:266657 rnase24k; do python tools/force_variants.py run $c >> gpurun_out/r2cg.jsonl 2>>gpurun_out/r2cg.err; done
