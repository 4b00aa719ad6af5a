# checked build (device-side range checks) of the final HEAD: GPU suite, smoke, a short bench
export NBX_LIB=$PWD/scratch/checked/libnbx.so
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -q -m gpu -rs > gpurun_out/r3p_checked_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3p_checked_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3p_checked_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3p_checked_smoke.log
python bench.py --steps 20 --warmup 3 --no-e2e > gpurun_out/r3p_checked_bench.json 2>gpurun_out/r3p_checked_bench.err; echo "rc=$?" >> gpurun_out/r3p_checked_bench.err
