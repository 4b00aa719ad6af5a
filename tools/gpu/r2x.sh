timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2x_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2x_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_smoke.log
