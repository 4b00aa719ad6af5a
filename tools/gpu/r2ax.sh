for c in water12m stmv rnase24k; do python tools/force_variants.py run $c base,s10,s12,vf3 >> gpurun_out/r2ax.jsonl 2>&1; done
