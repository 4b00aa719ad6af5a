for c in water12m stmv; do python tools/force_variants.py run $c base,pjs8,pjs8m6,pm6 >> gpurun_out/r2aw.jsonl 2>&1; done
