IBF_TRACE=1 timeout 1200 python tools/frame_breakdown.py 50 > gpurun_out/breakdown1.json 2> gpurun_out/trace1.err
timeout 1200 python tools/frame_breakdown.py 50 > gpurun_out/breakdown0.json 2> gpurun_out/trace0.err
