ncu --set full --import-source on --clock-control none -k regex:"k_force" -s 5 -c 1 -o gpurun_out/r2by_force_rnase python tools/force_variants.py one rnase24k base > gpurun_out/r2by_ncu.log 2>&1
