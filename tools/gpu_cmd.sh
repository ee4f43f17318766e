python tools/bench_spmv.py > gpurun_out/spmv_new.json 2> gpurun_out/spmv_new.err
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu3.log
