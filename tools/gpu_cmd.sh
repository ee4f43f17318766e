mkdir -p gpurun_out/r2g
timeout 1200 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -s -k "partitioned" > gpurun_out/r2g/tests_dist.log 2>&1
timeout 600 ncu --clock-control none -k regex:k_elem -c 1 --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv python tools/squishy_run.py --frames 1 > gpurun_out/r2g/ncu_elem_flops.csv 2>&1
IBF_BENCH_PROFILE_RANGE=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2g/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-certify > gpurun_out/r2g/bench_under_ncu.log 2>&1
gzip -f gpurun_out/r2g/launches_bench.csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2g/tests.log 2>&1
