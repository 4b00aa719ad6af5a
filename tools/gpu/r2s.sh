NBX_JSTAGE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/r2s_js_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_js_tests.log
for js in 0 1 0 1; do NBX_JSTAGE=$js timeout 300 python tools/time_entry_order.py stmv water12m rnase24k | sed "s/^/js=$js /" >> gpurun_out/r2s_js_time.txt 2>&1; done
