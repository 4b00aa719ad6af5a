# prune: swizzled staged rows (NBX_PRUNE_SWZ) on top of the row-major i staging; parity, timing, ncu
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "prune or list or cadence or stmv or water12m" 2>&1 | tail -3 > gpurun_out/r3o_tests.log
for v in base noswz base noswz; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 400 python tools/time_kernels.py water12m stmv mem82k rnase24k | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/r3o_tk.jsonl 2>> gpurun_out/r3o_err.log
done
ncu --set full --import-source on --clock-control none -k regex:k_prune_packed -s 1 -c 1 -o gpurun_out/r3o_prune_12m python tools/time_kernels.py water12m > gpurun_out/r3o_ncu.log 2>&1
