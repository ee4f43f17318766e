python tools/bench_spmv.py > gpurun_out/spmv_new.json 2> gpurun_out/spmv_new.err
timeout 1200 python bench.py > gpurun_out/bench_r1d.log 2>&1
cp profiles/c4_frame_counts.json gpurun_out/c4_frame_counts.json
