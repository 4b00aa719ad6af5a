for c in rnase24k water3k mem82k stmv:266657; do
  NBX_VARIANT_FLUSH=1 python tools/force_variants.py run $c >> gpurun_out/r2ca_flush.jsonl 2>>gpurun_out/r2ca.err
  python tools/force_variants.py run $c base,pf0 >> gpurun_out/r2ca_warm.jsonl 2>>gpurun_out/r2ca.err
done
