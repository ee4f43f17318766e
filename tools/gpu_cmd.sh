timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/pcg_final python tools/bench_spmv.py > gpurun_out/ncu_final.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_spmv -c 1 -o gpurun_out/spmv_final python tools/bench_spmv.py >> gpurun_out/ncu_final.log 2>&1
