for c in rnase24k water3k mem82k; do
  for sp in 0 4 6 8 12 16 24 32; do echo "split=$sp" >> gpurun_out/r2bx.jsonl; NBX_FORCE_SPLIT=$sp python tools/force_variants.py run $c base >> gpurun_out/r2bx.jsonl 2>>gpurun_out/r2bx.err; done
done
