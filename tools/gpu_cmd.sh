{ nproc; cat /proc/loadavg; lscpu | grep -i "model name\|MHz\|^CPU(s)\|NUMA"; cat /sys/fs/cgroup/cpu.max 2>/dev/null; } > gpurun_out/host_info.txt 2>&1
( for i in $(seq 1 40); do cat /proc/loadavg; top -bn1 | sed -n 7,14p; sleep 3; done ) > gpurun_out/host_load.txt 2>&1 &
LP=$!
for i in 1 2; do IBF_BENCH_CLOCKS=off timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_diag$i.json 2> gpurun_out/bench_diag$i.err; done
kill $LP
