timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pair_search_gpu.py -q -x > gpurun_out/r2bp_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2bp_parity.log
for c in water3k rnase24k mem82k stmv:266657 stmv; do
  for ps in 0 1; do echo "split=$ps" >> gpurun_out/r2bp_variants.jsonl; NBX_PRUNE_SPLIT=$ps python tools/force_variants.py run $c base >> gpurun_out/r2bp_variants.jsonl 2>>gpurun_out/r2bp.err; done
done
