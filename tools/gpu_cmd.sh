mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt 2>&1
nproc > gpurun_out/r2/nproc.txt; lscpu | head -20 >> gpurun_out/r2/nproc.txt
timeout 300 python tools/squishy_run.py --frames 40 --n 8 --stem 8 --tip 4 --cell 0.01 --plate-speed 1.0 --certify > gpurun_out/r2/sq_small.log 2>&1
timeout 600 python tools/squishy_run.py --frames 30 --cell 0.01 --plate-speed 1.0 --certify --every 1 > gpurun_out/r2/sq_full_1cm.log 2>&1
timeout 600 python tools/squishy_run.py --frames 30 --cell 0.02 --plate-speed 2.0 --every 1 > gpurun_out/r2/sq_full_2cm.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/tests.log 2>&1
