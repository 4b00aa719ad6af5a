# energy kernels, final form (G refined, 1/r and H IEEE, LJ x12): accuracy, timing, GPU suite, smoke
mkdir -p gpurun_out
for v in base e3; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 300 python tools/vf_accuracy.py gpu >> gpurun_out/r3d_acc.jsonl 2>> gpurun_out/r3d_err.log
done
for v in base vf0 e3; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 400 python tools/time_kernels.py water12m stmv mem82k rnase24k water3k | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/r3d_tk.jsonl 2>> gpurun_out/r3d_err.log
done
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r3d_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3d_smoke.log 2>&1
