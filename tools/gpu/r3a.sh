# round 2 (late): energy kernels on the fast path (NBX_VF_FAST=1) -- GPU suite, smoke, VF timing vs the IEEE path
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r3a_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.log 2>&1
for v in base vf0; do
  NBX_LIB=scratch/variants/libnbx_$v.so timeout 600 python tools/time_kernels.py water12m stmv mem82k > gpurun_out/r3a_tk_$v.jsonl 2>&1
done
