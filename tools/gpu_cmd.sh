O=gpurun_out/r2bu; mkdir -p $O
timeout 600 python bench.py --workload c5 --steps 10 --warmup 2 --no-cpu-baseline --concurrency 8 > $O/c5_k8.json 2> $O/c5_k8.err
timeout 600 python bench.py --workload c5 --steps 10 --warmup 2 --no-cpu-baseline --concurrency 1 > $O/c5_k1.json 2> $O/c5_k1.err
