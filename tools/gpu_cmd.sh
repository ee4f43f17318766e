timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/single_tests.log 2>&1
timeout 600 python tools/c5_trace.py > gpurun_out/c5_trace.log 2>&1
for c in 1 8; do timeout 900 python bench.py --workload c5 --concurrency $c > gpurun_out/c5s_$c.json 2> gpurun_out/c5s_$c.err; done
