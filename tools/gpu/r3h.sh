# prune row sweep (NBX_PRUNE_REP): list parity tests, then prune timing vs the full-test kernel
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "prune or list or cadence or stmv or water12m" 2>&1 | tail -15 > gpurun_out/r3h_tests.log
for v in base rep0 rep1m5 base rep0; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 400 python tools/time_kernels.py water12m stmv mem82k rnase24k | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/r3h_tk.jsonl 2>> gpurun_out/r3h_err.log
done
