# energy-kernel variants: accuracy vs the oracle (tools/vf_accuracy.py) and VF timing
mkdir -p gpurun_out
for v in base vf0 r0 r2 r2l n2; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 300 python tools/vf_accuracy.py gpu >> gpurun_out/r3b_acc.jsonl 2>> gpurun_out/r3b_err.log
done
for v in base vf0 r0 r2 r2l n2; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 300 python tools/time_kernels.py water12m stmv | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/r3b_tk.jsonl 2>> gpurun_out/r3b_err.log
done
