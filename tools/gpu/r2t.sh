python tools/prof_force.py stmv 2 > gpurun_out/r2t_plain.log 2>&1 && NBX_JSTAGE=1 python tools/prof_force.py stmv 2 >> gpurun_out/r2t_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_force" -s 1 -c 1 -o gpurun_out/r2t_stmv_base python tools/prof_force.py stmv 2 > gpurun_out/r2t_ncu.log 2>&1 && \
NBX_JSTAGE=1 ncu --set full --clock-control none --import-source on -k regex:"k_force" -s 1 -c 1 -o gpurun_out/r2t_stmv_js python tools/prof_force.py stmv 2 >> gpurun_out/r2t_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2t_ncu.log
