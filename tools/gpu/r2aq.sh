for c in water12m stmv; do python tools/force_variants.py run $c base,minb4,minb2 >> gpurun_out/r2aq.jsonl 2>&1; done
