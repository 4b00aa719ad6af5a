for c in water12m stmv mem82k; do python tools/force_variants.py run $c base,u1,pairs,pairs_u1 >> gpurun_out/r2ao.jsonl 2>&1; done
for c in water12m stmv; do python tools/force_variants.py run $c base,u1 >> gpurun_out/r2ao.jsonl 2>&1; done
