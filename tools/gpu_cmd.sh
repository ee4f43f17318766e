IBF_LIB=tools/variants/libibf_even.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ev_tests.log 2>&1
for v in noeven even noeven even; do IBF_LIB=tools/variants/libibf_$v.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/bench_ev_all.jsonl 2> gpurun_out/bench_$v.err; done
