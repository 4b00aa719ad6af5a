timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2bg_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2bg_parity.log
for c in stmv:266657 rnase24k stmv water12m; do python tools/force_variants.py run $c >> gpurun_out/r2bg_variants.jsonl 2>>gpurun_out/r2bg.err; done
