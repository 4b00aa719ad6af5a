# energy steps with fp64 force accumulation (single domain, <= 2M slots): accuracy, VF time, whole GPU suite, smoke
mkdir -p gpurun_out
timeout 300 python tools/vf_accuracy.py gpu > gpurun_out/r3r_acc.jsonl 2> gpurun_out/r3r_err.log
NBX_F64_FORCES=0 timeout 300 python tools/vf_accuracy.py gpu > gpurun_out/r3r_acc_f32.jsonl 2>> gpurun_out/r3r_err.log
for m in 1 0 1 0; do
  NBX_F64_FORCES=$m timeout 400 python tools/time_kernels.py stmv mem82k rnase24k water3k | sed "s/^{/{\"f64\": $m, /" >> gpurun_out/r3r_tk.jsonl 2>> gpurun_out/r3r_err.log
done
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/r3r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3r_tests.log
for k in 1 2 3 4 5; do python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r3r_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3r_smoke.log; done
