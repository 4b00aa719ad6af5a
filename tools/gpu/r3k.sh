# ncu --set full of the shipped prune (row sweep + 4-lane full test) on 12 M
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_prune_packed -s 1 -c 1 -o gpurun_out/r3k_prune_12m python tools/time_kernels.py water12m > gpurun_out/r3k_ncu.log 2>&1
