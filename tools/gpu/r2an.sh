python tools/prof_step.py water12m > gpurun_out/r2an_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_search|k_prune_packed|k_force|k_put_x|k_get_f|k_compact|k_slab" -c 20 -o gpurun_out/r2an_12m python tools/prof_step.py water12m > gpurun_out/r2an_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2an_ncu.log
