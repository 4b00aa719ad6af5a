# energy-kernel variants with the IEEE 1/r: accuracy vs the oracle
mkdir -p gpurun_out
for v in vf0 r0 r2 r2l; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 300 python tools/vf_accuracy.py gpu >> gpurun_out/r3c_acc.jsonl 2>> gpurun_out/r3c_err.log
done
