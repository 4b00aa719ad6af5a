timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2bl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2bl_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bl_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2bl_smoke.log
