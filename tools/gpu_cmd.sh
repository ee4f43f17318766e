timeout 1200 python bench.py > gpurun_out/bench_r1e.log 2>&1
