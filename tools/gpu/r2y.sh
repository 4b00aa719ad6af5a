for i in 1 2 3; do python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2y_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_smoke.log; done
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2y_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_tests.log
timeout 600 python tools/time_kernels.py water12m stmv > gpurun_out/r2y_kernels.jsonl 2>&1
