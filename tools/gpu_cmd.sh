for c in 1 8; do timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 --concurrency $c > gpurun_out/bench_c5_$c.log 2>&1; done
