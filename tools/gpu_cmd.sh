timeout 1200 python bench.py > gpurun_out/bench_r1c.log 2>&1
cp profiles/c4_frame_counts.json gpurun_out/c4_frame_counts.json 2>/dev/null
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_r1c.log 2>&1
