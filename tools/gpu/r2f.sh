timeout 900 python -m pytest tests -q -m gpu --deselect tests/test_dd_gpu.py > gpurun_out/r2f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_tests.log
timeout 600 python tools/time_kernels.py water12m stmv > gpurun_out/r2f_kernels.jsonl 2>&1
# ncu: the prune kernel and the VF force kernel on STMV (plain run first, same command)
python tools/prof_force.py stmv 2 energy > gpurun_out/r2f_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_prune_packed|k_force" -c 4 -o gpurun_out/r2f_stmv python tools/prof_force.py stmv 2 energy > gpurun_out/r2f_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2f_ncu.log
