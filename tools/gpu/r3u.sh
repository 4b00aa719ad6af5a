# energy kernels with the raw-MUFU G(z) reciprocal by default: accuracy x2, energy-step tests, smoke x3, VF time
mkdir -p gpurun_out
for k in 1 2; do timeout 300 python tools/vf_accuracy.py gpu >> gpurun_out/r3u_acc.jsonl 2>> gpurun_out/r3u_err.log; done
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/r3u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3u_tests.log
for k in 1 2 3; do python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r3u_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3u_smoke.log; done
timeout 400 python tools/time_kernels.py water12m stmv > gpurun_out/r3u_tk.jsonl 2>> gpurun_out/r3u_err.log
