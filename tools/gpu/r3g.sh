# energy-kernel occupancy variants (CTA size / CTAs per SM)
mkdir -p gpurun_out
for v in base t160 t128 t192; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 400 python tools/time_kernels.py water12m stmv | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/r3g_tk.jsonl 2>> gpurun_out/r3g_err.log
done
