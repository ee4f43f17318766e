IBF_LIB=tools/variants/libibf_il.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/il_tests.log 2>&1
for v in noil il noil il; do echo "== $v"; IBF_LIB=tools/variants/libibf_$v.so timeout 300 python tools/bench_spmv.py; done > gpurun_out/il_micro.log 2>&1
for v in noil il noil il; do IBF_LIB=tools/variants/libibf_$v.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/bench_il_all.jsonl 2> gpurun_out/bench_$v.err; done
