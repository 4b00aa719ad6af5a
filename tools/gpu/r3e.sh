# ncu --set full of the shipped energy kernel (STMV)
mkdir -p gpurun_out
python tools/vf_once.py stmv > gpurun_out/r3e_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_force -c 1 -o gpurun_out/r3e_vf_stmv python tools/vf_once.py stmv > gpurun_out/r3e_ncu.log 2>&1
