# energy kernels: tile pairs (NBX_TILE_PAIRS_E) vs shipped
mkdir -p gpurun_out
for v in base tpe base tpe; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 400 python tools/time_kernels.py water12m stmv mem82k | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/r3f_tk.jsonl 2>> gpurun_out/r3f_err.log
done
NBX_LIB=scratch/variants/libnbx_tpe.so timeout 300 python tools/vf_accuracy.py gpu >> gpurun_out/r3f_acc.jsonl 2>> gpurun_out/r3f_err.log
