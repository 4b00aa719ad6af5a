python tools/force_variants.py run stmv base,pairs,pairs_u1,u1,minb4,pairs_minb4 > gpurun_out/r2h_variants.jsonl 2>&1
python tools/force_variants.py run water12m base,pairs,minb4,pairs_minb4 >> gpurun_out/r2h_variants.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k entry_order > gpurun_out/r2h_f2.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_f2.log
NBX_ENTRY_ORDER=0 timeout 300 python tools/time_entry_order.py water3k rnase24k mem82k stmv water12m > gpurun_out/r2h_order.jsonl 2>&1
NBX_ENTRY_ORDER=1 timeout 300 python tools/time_entry_order.py water3k rnase24k mem82k stmv water12m >> gpurun_out/r2h_order.jsonl 2>&1
