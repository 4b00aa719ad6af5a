python tools/nan_probe.py > gpurun_out/r2ae.log 2>&1
