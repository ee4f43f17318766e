timeout 900 python tools/surface_timing.py > gpurun_out/surface_timing.log 2>&1
