# final HEAD, one B200: whole GPU suite, smoke x3, default bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/r3s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3s_tests.log
for k in 1 2 3; do python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r3s_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3s_smoke.log; done
python bench.py > gpurun_out/r3s_n1_default.json 2> gpurun_out/r3s_n1.err
python bench.py --impl reference > gpurun_out/r3s_ref_default.json 2> gpurun_out/r3s_ref.err
