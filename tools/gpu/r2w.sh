for eo in 0 1; do NBX_ENTRY_ORDER=$eo timeout 600 python tools/time_entry_order.py stmv_tab stmv_fsw grappa1.5m stmv >> gpurun_out/r2w_order.jsonl 2>&1; done
