for c in water12m stmv stmv_fsw grappa1.5m; do python tools/force_variants.py run $c base,minb4 >> gpurun_out/r2ar.jsonl 2>&1; done
for c in stmv water12m; do NBX_ENTRY_ORDER=0 python tools/force_variants.py run $c base,minb4 | sed 's/^/eo0 /' >> gpurun_out/r2ar.jsonl 2>&1; done
for c in stmv water12m; do NBX_ENTRY_ORDER=1 python tools/force_variants.py run $c base,minb4 | sed 's/^/eo1 /' >> gpurun_out/r2ar.jsonl 2>&1; done
