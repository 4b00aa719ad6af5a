# energy kernels: G(z) with the raw MUFU reciprocal (NBX_VF_G=2) -- accuracy and time
mkdir -p gpurun_out
for v in g2 base; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 300 python tools/vf_accuracy.py gpu >> gpurun_out/r3q_acc.jsonl 2>> gpurun_out/r3q_err.log
done
for v in base g2 base g2; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 400 python tools/time_kernels.py water12m stmv | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/r3q_tk.jsonl 2>> gpurun_out/r3q_err.log
done
