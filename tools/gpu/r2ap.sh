for c in water12m stmv; do python tools/force_variants.py run $c base,jred1,jred0,packf,leanlj,leancut,nolean >> gpurun_out/r2ap.jsonl 2>&1; done
