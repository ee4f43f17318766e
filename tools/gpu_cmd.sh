O=gpurun_out/r2ak; mkdir -p $O
timeout 900 python bench.py --no-cpu-baseline > $O/bench_base.json 2> $O/bench_base.err
IBF_LIB=tools/variants/libibf_pmat.so timeout 900 python bench.py --no-cpu-baseline > $O/bench_pmat.json 2> $O/bench_pmat.err
timeout 900 python bench.py --no-cpu-baseline > $O/bench_base2.json 2> $O/bench_base2.err
