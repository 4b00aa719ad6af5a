export NBX_LIB=$PWD/scratch/checked/libnbx.so
python -c "from paper_2405_01420_b200 import nbx; print(nbx.lib().nbx_version())" > gpurun_out/r2bu_checked_tests.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rs >> gpurun_out/r2bu_checked_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2bu_checked_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bu_checked_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2bu_checked_smoke.log
python bench.py --steps 20 --warmup 3 --no-e2e > gpurun_out/r2bu_checked_bench.json 2>gpurun_out/r2bu_checked_bench.err; echo "rc=$?" >> gpurun_out/r2bu_checked_bench.err
unset NBX_LIB
timeout 600 python -m pytest tests/test_checked_build.py -q -rs > gpurun_out/r2bu_unchecked_skip.log 2>&1
