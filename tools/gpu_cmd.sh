for v in nosplit split; do IBF_LIB=tools/variants/libibf_$v.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/split_tests.log 2>&1
