timeout 2700 python tools/press_run.py 106 94 > gpurun_out/press_run2.log 2>&1
