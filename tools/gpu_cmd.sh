for c in 1 8; do timeout 900 python bench.py --workload c5 --concurrency $c --steps 5 --warmup 3 > gpurun_out/c5_$c.json 2> gpurun_out/c5_$c.err; done
