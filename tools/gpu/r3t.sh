# virial about the box centre: accuracy (water 3k virial margin), whole GPU suite, smoke x3
mkdir -p gpurun_out
for k in 1 2 3; do timeout 300 python tools/vf_accuracy.py gpu >> gpurun_out/r3t_acc.jsonl 2>> gpurun_out/r3t_err.log; done
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/r3t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3t_tests.log
for k in 1 2 3; do python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r3t_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3t_smoke.log; done
