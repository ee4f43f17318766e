O=gpurun_out/r2at; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -rA > $O/tests.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
IBF_LIB=tools/variants/libibf_nostop.so timeout 900 python bench.py --no-cpu-baseline > $O/bench_nostop.json 2> $O/bench_nostop.err
