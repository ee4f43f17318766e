python tools/bench_spmv.py > gpurun_out/spmv_new.json 2> gpurun_out/spmv_new.err
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu3.log
timeout 1200 python bench.py > gpurun_out/bench_r1h.log 2>&1
