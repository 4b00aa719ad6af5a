for c in stmv:266657 rnase24k stmv water12m; do python tools/force_variants.py run $c >> gpurun_out/r2be_variants.jsonl 2>>gpurun_out/r2be.err; done
