NBX_PRUNE_KERNEL=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "prune or full_size or cadence or entry_order" > gpurun_out/r2u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_tests.log
for k in 2 3 2 3; do NBX_PRUNE_KERNEL=$k timeout 300 python tools/time_kernels.py water12m stmv rnase24k | sed "s/^/k=$k /" >> gpurun_out/r2u_time.txt 2>&1; done
