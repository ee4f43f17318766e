timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.log 2>&1
