for c in water12m stmv; do python tools/force_variants.py run $c base,large5,large4u2,t128 >> gpurun_out/r2at.jsonl 2>&1; done
